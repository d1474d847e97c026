# ncu --set full of the step's memory-bound kernels (2nd eager step): LRN+pool fwd/bwd,
# s2d, colsum partials, and the FC wgrad + fused-SGD light GEMM.
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none -k regex:'lrn_pool|s2d_input|colsum_partial|gemm_kernel<128, 0, 1>' --launch-skip 11 --launch-count 11 -o gpurun_out/memk -f python tests/dev/one_step.py 2 > gpurun_out/ncu_memk.log 2>&1; echo "memk rc=$?"
ls -la gpurun_out/memk.ncu-rep
