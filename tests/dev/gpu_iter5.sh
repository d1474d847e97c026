mkdir -p gpurun_out
timeout 120 python tests/dev/h2d_probe.py
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_eager.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
python tests/dev/launch_table.py gpurun_out/launches_eager.csv 2>&1 | grep -E "colsum|lrn|s2d|total"
