import os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from relu_probe import run  # noqa
for ws, lr, steps in [(30.0, 1e-4, 2), (30.0, 1e-5, 2), (10.0, 1e-3, 2), (1.0, 0.05, 2), (1.0, 0.05, 3), (30.0, 1e-3, 2)]:
    run(2, "C", False, steps, False, ws=ws, lr=lr)
    run(2, "C", False, steps, False, ws=ws, lr=lr, relu_last=False)
