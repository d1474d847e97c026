# Round-2 measurement pass: GPU tests, smoke, bench (+reference arm), plan dump, ncu launch
# list, per-launch DRAM traffic of one eager step, full ncu capture of every GEMM launch of a
# step and of the memory-bound kernels (exported to CSV on the box; the .ncu-rep files are
# too large to bring back), dev timeline of one graph-replayed step.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
if [ "$1" != "notests" ]; then
timeout 1500 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
fi
HP_DEV_PLANS=1 timeout 300 python tests/dev/one_step.py 1 2>&1 | grep plan | head -23 > gpurun_out/plans.log
for i in 1 2; do timeout 600 python bench.py --steps 20 --warmup 5 --profile-out gpurun_out/prof$i.json > gpurun_out/bench$i.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench$i.log | cut -c1-200; done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
HP_DEV_TIMELINE=gpurun_out/timeline.csv timeout 300 python tests/dev/gemm_times.py > gpurun_out/tl_times.log 2>&1
python tests/dev/timeline.py gpurun_out/timeline.csv 25 > gpurun_out/timeline_graph.txt 2>&1
python tests/dev/timeline.py gpurun_out/timeline.csv 27 > gpurun_out/timeline_serial.txt 2>&1
if [ "$1" != "nofull" ]; then
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:'gemm|conv_shift' --launch-skip 23 --launch-count 23 -o /tmp/gemms_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/gemms_full.ncu-rep --page raw --csv > gpurun_out/gemms_full_raw.csv 2>/dev/null; gzip -f gpurun_out/gemms_full_raw.csv
timeout 1200 ncu --set full --clock-control none -k regex:'lrn|pool|s2d|colsum|sgd|epi_apply|rotate' --launch-skip 20 --launch-count 20 -o /tmp/mem_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_mem.log 2>&1; echo "ncu mem rc=$?"
ncu -i /tmp/mem_full.ncu-rep --page raw --csv > gpurun_out/mem_full_raw.csv 2>/dev/null; gzip -f gpurun_out/mem_full_raw.csv
fi
du -sh gpurun_out
