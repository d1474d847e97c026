# usage: gpu_ncu_k.sh <regex> <skip> <count> <name>
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$1" --launch-skip $2 --launch-count $3 -o gpurun_out/$4 -f python tests/dev/one_step.py 2 > gpurun_out/ncu_$4.log 2>&1; echo "ncu rc=$?"
