# Quick GPU pass: facade GPU test, tolerance report of the step tests, wgrad GEMM sweep.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_facade.py -q -m gpu > gpurun_out/facade.log 2>&1; echo "facade rc=$?"; tail -2 gpurun_out/facade.log
HP_TOL_REPORT=1 timeout 900 python -m pytest tests/test_step_gpu.py -q -s -m gpu > gpurun_out/tol.log 2>&1; echo "tol rc=$?"; tail -2 gpurun_out/tol.log
timeout 600 python tests/dev/wgrad_bench.py > gpurun_out/wgrad_bench.log 2>&1; echo "wgrad rc=$?"
