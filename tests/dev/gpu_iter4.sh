# GPU iteration: full gpu tests, step timing, eager-step launch list (per-kernel times)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_iter.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_iter.log
timeout 300 python tests/dev/step_dev.py time > gpurun_out/step_time.log 2>&1; grep "step " gpurun_out/step_time.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_eager.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python tests/dev/launch_table.py gpurun_out/launches_eager.csv 2>&1 | head -40
