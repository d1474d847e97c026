mkdir -p gpurun_out
for i in 1 2 3; do for d in build_r0/tests/dev tests/dev; do LABEL=$d timeout 300 python $d/gemm_times.py 2>&1 | head -1; done; done > gpurun_out/ab_r0.log
cat gpurun_out/ab_r0.log
for f in 0 32 64; do HP_DEV_GEMM_DBG=$f LABEL=dbg$f timeout 300 python tests/dev/gemm_times.py 2>&1 | grep -E "==|wgrad"; done > gpurun_out/skip.log
cat gpurun_out/skip.log
