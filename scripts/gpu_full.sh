# Full measurement pass on one B200 (run via gpurun): tests, bench (all legs),
# reference arm, the torchrun launch path, ncu launch list and full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi.csv 2>&1
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" >> gpurun_out/host.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bench_ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err; echo bench_torchrun=$?
SMALL="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
timeout 600 $SMALL > gpurun_out/bench_small.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_validate -s 8 -c 1 -o gpurun_out/prof_k_validate -f $SMALL > gpurun_out/ncu_full.log 2>&1; echo ncu_k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k k_batch -s 5 -c 1 -o gpurun_out/prof_k_batch -f python tools/k2bench.py c3 8 > gpurun_out/ncu_full_batch.log 2>&1; echo ncu_k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k k_batch_large -s 3 -c 1 -o gpurun_out/prof_k_batch_large -f python tools/k2bench.py c2 8 > gpurun_out/ncu_full_batch_large.log 2>&1; echo ncu_k2l=$?
