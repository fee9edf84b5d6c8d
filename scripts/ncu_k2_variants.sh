cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,lts__t_sectors_srcunit_tex_op_write.sum
for v in paper_2010_03090_b200/libutf8v_cuda.so build/var_nolane/libutf8v_cuda.so build/var_noattr/libutf8v_cuda.so; do
  echo "== $v"
  timeout 600 ncu --metrics $M --clock-control none -k regex:^k_batch -s 3 -c 1 python tools/k2bench.py c3 4 $v 2>&1 | grep -E "k_batch|duration|inst_executed|dram__bytes|issue_active|lts__t" | head -12
done
