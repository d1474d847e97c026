mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do for w in tiny tiny_bf16 alexnet; do
  echo "=== $t $w"; timeout 900 compute-sanitizer --tool $t --print-limit 20 python tests/dev/sanitize_step.py $w 2>&1 | tail -6
done; done > gpurun_out/sanitizer.log 2>&1
echo done
