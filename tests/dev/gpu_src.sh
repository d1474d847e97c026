# Dev: ncu full capture with source of the first conv_shift launch (conv1 fprop) of an
# eager step; exports the details + source pages as CSV, plus the GEMM plan dump.
mkdir -p gpurun_out
HP_DEV_PLANS=1 timeout 300 python tests/dev/one_step.py 1 2>&1 | grep plan | head -30 > gpurun_out/plans.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${SRC_K:-conv_shift}" --launch-skip ${SRC_SKIP:-0} --launch-count 1 -o /tmp/src -f python tests/dev/one_step.py 1 > gpurun_out/ncu_src.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/src.ncu-rep --page details --csv > gpurun_out/src_details.csv 2>/dev/null
ncu -i /tmp/src.ncu-rep --page source --csv > gpurun_out/src_source.csv 2>/dev/null
ncu -i /tmp/src.ncu-rep --page raw --csv > gpurun_out/src_raw.csv 2>/dev/null
ls -la gpurun_out
