# Dev A/B on one box: step time of lib/libold.so (HP_DEV_LIB) vs the current build,
# alternated, then the kernel-level and AlexNet parity tests on the current build.
mkdir -p gpurun_out
for i in 1 2 3; do for v in old new; do
  if [ $v = old ]; then export HP_DEV_LIB=paper_1404_5997_b200/lib/libold.so; else unset HP_DEV_LIB; fi
  echo -n "$v "; timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "step" | head -1
done; done
unset HP_DEV_LIB
timeout 900 python -m pytest -x -q -m gpu ${AB_TESTS:-tests/test_lrn_pool_gpu.py tests/test_alexnet_parity_gpu.py} 2>&1 | tail -3
