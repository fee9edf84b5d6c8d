# Round-2 iteration on one B200 (via gpurun): host facts, smoke, GPU tests,
# bench (N=1), the N=2 launch path with ranks sharing the GPU (gloo), the
# reference arm.  BENCH_ARGS / PYTEST_ARGS / SKIP_TESTS tune it.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
(nproc; free -g; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > gpurun_out/host.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
if [ -z "$SKIP_TESTS" ]; then
  T0=$(date +%s); timeout 2400 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
  echo pytest_wall_s=$(( $(date +%s) - T0 )); tail -5 gpurun_out/pytest_gpu.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
head -c 600 gpurun_out/bench.json; echo; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err; echo bench_n2_gloo=$?
head -c 400 gpurun_out/bench_n2_gloo.json; echo; tail -3 gpurun_out/bench_n2_gloo.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo bench_ref=$?
head -c 300 gpurun_out/bench_ref.json; echo
