# parity + LRN kernels check
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_alexnet_parity_gpu.py tests/test_lrn_pool_gpu.py tests/test_kernel_variants_gpu.py -q -s -rf --timeout 600 > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|decisions|momentum err|^\{|Error|assert" gpurun_out/pytest_parity.log | head -60
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --profile-out gpurun_out/prof.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench.log | cut -c1-400
