mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants_gpu.py tests/test_lrn_pool_gpu.py tests/test_alexnet_parity_gpu.py -q -rf --timeout 600 > gpurun_out/pytest_lrn.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_lrn.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
python tests/dev/traffic_summary.py gpurun_out/traffic.csv gpurun_out/traffic.json | head -24
