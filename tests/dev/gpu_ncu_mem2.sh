mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'lrn|s2d_input|colsum_partial' --launch-skip 6 --launch-count 6 -o gpurun_out/mem3 -f python tests/dev/one_step.py 2 > gpurun_out/ncu_mem3.log 2>&1; echo "mem rc=$?"
ls -la gpurun_out/mem3.ncu-rep
