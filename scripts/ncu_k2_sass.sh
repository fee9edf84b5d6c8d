# Per-opcode SASS mix of K2 variants on C3 (DEVELOPMENT): one --set full
# capture per library variant given as arguments.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in "$@"; do
  n=$(basename $(dirname $v))
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:^k_batch -s 3 -c 1 -o gpurun_out/k2_$n -f python tools/k2bench.py c3 4 $v > gpurun_out/k2_$n.log 2>&1; echo $n=$?
done
