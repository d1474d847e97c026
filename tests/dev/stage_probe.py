"""Dev: AlexNet conv layer shapes through the flat-shift kernel (q-layout), for
comparing stage-depth variants (HP_DEV_LIB=<variant .so>)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1404_5997_b200._lib import lib, last_error, LIB_PATH


def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def run(rows, Cin, R, S, wq, F, useful):
    x = torch.randn(rows + 256, Cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(F, R * S * Cin, device="cuda") * 0.1).to(torch.bfloat16)
    y = torch.empty(rows, F, device="cuda")
    def f():
        assert lib.hp_kernel_conv_shift(x.data_ptr(), rows, Cin, R, S, wq, w.data_ptr(), F, y.data_ptr(), 0, None) == 0, last_error()
    t = timeit(f)
    return t, 2.0 * useful * F * R * S * Cin / t / 1e9


print(os.path.basename(LIB_PATH))
b = 128
shapes = {  # name: (H(out), pad, C, R, F)
    "conv2 fwd": (27, 2, 64, 5, 192), "conv2 dgrad": (27, 2, 192, 5, 64),
    "conv3 fwd": (13, 1, 192, 3, 384), "conv3 dgrad": (13, 1, 384, 3, 192),
    "conv4 fwd": (13, 1, 384, 3, 384), "conv5 fwd": (13, 1, 384, 3, 256), "conv5 dgrad": (13, 1, 256, 3, 384)}
tot = 0.0
for name, (H, p, Cin, R, F) in shapes.items():
    wq = H + p  # q-layout: one shared zero border per row and column
    t, tf = run(b * wq * wq, Cin, R, R, wq, F, b * H * H)
    tot += t
    print(f"{name:12s} {t*1e3:7.1f} us  {tf:6.0f} TF/s (useful)", flush=True)
print(f"total {tot*1e3:.1f} us")
