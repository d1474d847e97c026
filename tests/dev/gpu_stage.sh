# Stage-depth variants: conv shapes + whole step per variant .so
mkdir -p gpurun_out
for v in "" _s24 _s36; do
  L=paper_1404_5997_b200/lib/libhpsim_b200$v.so
  HP_DEV_LIB=$PWD/$L timeout 300 python tests/dev/stage_probe.py >> gpurun_out/stage_probe.log 2>&1
  echo "== $v" >> gpurun_out/stage_step.log
  HP_DEV_LIB=$PWD/$L timeout 300 python tests/dev/step_dev.py time >> gpurun_out/stage_step.log 2>&1
done
cat gpurun_out/stage_probe.log; cat gpurun_out/stage_step.log | grep -v "^ "
