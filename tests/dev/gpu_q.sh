mkdir -p gpurun_out
for i in 1 2; do for v in ns cs; do
  if [ $v = ns ]; then export HP_DEV_LIB=paper_1404_5997_b200/lib/libns.so; else unset HP_DEV_LIB; fi
  LABEL=$v timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "==|fc_wgrad|fc_dgrad"
done; done
