# iteration run: GPU tests, bench, optional ncu captures (NCU=1)
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 200 --warmup 10 ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ -n "$NCU" ]; then
SMALL="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $SMALL > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_validate -s 8 -c 1 -o gpurun_out/prof_k_validate -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo ncu_k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k k_batch -s 3 -c 1 -o gpurun_out/prof_k_batch -f $SMALL > gpurun_out/ncu_full_batch.log 2>&1; echo ncu_k2=$?
fi
