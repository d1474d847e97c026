mkdir -p gpurun_out
nvidia-smi --query-gpu=clocks.sm,clocks.mem,clocks.max.sm,power.draw,temperature.gpu --format=csv
timeout 900 python -m pytest tests/test_data_gen.py tests/test_cli.py tests/test_abi.py -x -q -m gpu > gpurun_out/dg.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dg.log
python - <<'PY'
import time, torch, sys
sys.path.insert(0, '.')
from paper_1404_5997_b200 import data as D
s = D.DatasetSpec(num_examples=1280, input_shape=(3, 224, 224), num_classes=1000, seed=1, separation=0.1)
x, t = D.generate(s, 0, 128)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for i in range(10): D.generate(s, 128 * (i % 10), 128)
e1.record(); torch.cuda.synchronize()
print(f"datagen AlexNet batch (128 x 3x224x224): {e0.elapsed_time(e1) / 10 * 1e3:.1f} us")
PY
LABEL=clk timeout 300 python tests/dev/gemm_times.py | head -1
nvidia-smi --query-gpu=clocks.sm,clocks.mem,clocks.max.sm,power.draw,temperature.gpu --format=csv
