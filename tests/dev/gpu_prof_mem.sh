# launch list + DRAM traffic of one eager step, and a full capture of the LRN/pool kernels
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/traffic.csv python tests/dev/one_step.py 2 > gpurun_out/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
python tests/dev/traffic_summary.py gpurun_out/traffic.csv gpurun_out/traffic.json | head -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'lrn_pool|bias_part|maxpool' --launch-skip 5 --launch-count 5 -o gpurun_out/lrn_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
