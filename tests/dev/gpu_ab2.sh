# Dev A/B on one box: graph-replayed step times of lib/libold.so vs the current build
# (+ optional env variant $AB_ENV), alternated; then per-kernel ncu times of one eager
# step for both (tests/dev/ab_kernels.py).
mkdir -p gpurun_out
run() { echo -n "$1 "; timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "step" | head -1; }
for i in 1 2 3; do
  HP_DEV_LIB=paper_1404_5997_b200/lib/libold.so run old
  run new
  if [ -n "$AB_ENV" ]; then env $AB_ENV python tests/dev/gemm_times.py 2>&1 | grep -E "step" | head -1 | sed 's/^/variant /'; fi
done
for v in old new; do
  if [ $v = old ]; then export HP_DEV_LIB=paper_1404_5997_b200/lib/libold.so; else unset HP_DEV_LIB; fi
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/k_$v.csv python tests/dev/one_step.py 3 > /dev/null 2>&1
  echo "ncu $v rc=$?"
done
unset HP_DEV_LIB
python tests/dev/ab_kernels.py gpurun_out/k_old.csv gpurun_out/k_new.csv
if [ -n "$AB_TESTS" ]; then timeout 900 python -m pytest -x -q -m gpu $AB_TESTS 2>&1 | tail -3; fi
