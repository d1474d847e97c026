mkdir -p gpurun_out
for i in 1 2 3; do
  LABEL=plain timeout 300 python tests/dev/gemm_times.py | head -1
  HP_DEV_S2D_PIPE=1 LABEL=pipe timeout 300 python tests/dev/gemm_times.py | head -1
done
