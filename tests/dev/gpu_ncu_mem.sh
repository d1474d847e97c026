mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'lrn|im2col|epi_apply|rotate|colsum' --launch-skip 20 --launch-count 20 -o gpurun_out/mem2_full -f python tests/dev/one_step.py 2 > gpurun_out/ncu_mem2.log 2>&1; echo "mem rc=$?"
