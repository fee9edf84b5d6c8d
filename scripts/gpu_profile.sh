# ncu evidence for profiles/ (run via gpurun, one GPU): the launch list of the
# default bench command, then one --set full capture each of K1 (the bench's
# kernel), K2 (C3 via tools/k2bench.py) and K2L (C2), with source lines.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/prof_bench.json 2> gpurun_out/prof_bench.err; echo bench=$?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py > gpurun_out/ncu_launch.log 2>&1; echo ncu_launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_validate -s 20 -c 1 -o gpurun_out/prof_k_validate -f python bench.py --steps 40 --warmup 3 --no-extras --no-cpu-baseline --e2e-steps 1 > gpurun_out/ncu_k1.log 2>&1; echo ncu_k1=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^k_batch$ -s 5 -c 1 -o gpurun_out/prof_k_batch -f python tools/k2bench.py c3 8 > gpurun_out/ncu_k2.log 2>&1; echo ncu_k2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_batch_large -s 3 -c 1 -o gpurun_out/prof_k_batch_large -f python tools/k2bench.py c2 8 > gpurun_out/ncu_k2l.log 2>&1; echo ncu_k2l=$?
ls -la gpurun_out/*.ncu-rep
