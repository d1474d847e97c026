# ncu: launch list of 2 eager steps + full capture of the step's 23 GEMM launches
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_eager.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_list.log 2>&1; echo "list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm --launch-skip 23 --launch-count 23 -o gpurun_out/gemms_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
tail -3 gpurun_out/ncu_full.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'lrn|pool|im2col|colsum|sgd|nchw' --launch-skip 12 --launch-count 12 -o gpurun_out/mem_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_mem.log 2>&1; echo "mem rc=$?"
ls -la gpurun_out
