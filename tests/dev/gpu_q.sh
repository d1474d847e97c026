mkdir -p gpurun_out
for i in 1 2; do for d in build_old/tests/dev tests/dev; do
  HP_DEV_TIMELINE=gpurun_out/tl.csv LABEL=$d timeout 300 python $d/gemm_times.py 2>&1 | head -1
  python tests/dev/timeline.py gpurun_out/tl.csv 27 | grep -E "sgd_conv|rotate"
done; done
for i in 1 2 3; do for d in build_old/tests/dev tests/dev; do LABEL=$d timeout 300 python $d/gemm_times.py 2>&1 | head -1; done; done
timeout 900 python -m pytest tests/test_step_gpu.py -x -q -m gpu -k "alexnet or tiny_k1" > gpurun_out/pt.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pt.log
