# Round-level measurement: full GPU tests, smoke, bench (+reference arm), ncu launch list,
# per-launch DRAM traffic of one eager step, ncu --set full of the step's GEMMs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py --steps 20 --warmup 5 --profile-out gpurun_out/prof.json > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_ncu.log 2>&1; echo "ncu list rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'gemm|conv_shift' --launch-skip 23 --launch-count 5 -o gpurun_out/gemms_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
