# Round-2 measurement pass: bench (+reference arm), plan dump, ncu launch list, per-launch
# DRAM traffic of one eager step, full ncu capture of every GEMM launch of a step (exported
# to CSV on the box; the .ncu-rep itself is too large to bring back).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
if [ "$1" = "tests" ]; then
timeout 1200 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
fi
HP_DEV_PLANS=1 timeout 300 python tests/dev/one_step.py 1 > gpurun_out/plans.log 2>&1; echo "plans rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --profile-out gpurun_out/prof.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
if [ "$1" != "nofull" ]; then
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'gemm|conv_shift' --launch-skip 23 --launch-count 23 -o /tmp/gemms_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/gemms_full.ncu-rep --page raw --csv > gpurun_out/gemms_full_raw.csv 2>/dev/null; echo "export rc=$?"
gzip -f gpurun_out/gemms_full_raw.csv
fi
du -sh gpurun_out
