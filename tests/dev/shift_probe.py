"""Dev: does the flat-shift kernel slow down on row offsets that are not
multiples of 8 (unaligned swizzle phase)? Same GEMM size, taps at offsets
0..8 vs multiples of 8 (wq = 8), and 1x1 with 9x the channels."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1404_5997_b200._lib import lib, last_error

def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters

def run(rows, Cin, R, S, wq, F):
    x = torch.randn(rows, Cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(F, R * S * Cin, device="cuda") * 0.1).to(torch.bfloat16)
    y = torch.empty(rows, F, device="cuda")
    def f():
        assert lib.hp_kernel_conv_shift(x.data_ptr(), rows, Cin, R, S, wq, w.data_ptr(), F, y.data_ptr(), 0, None) == 0, last_error()
    t = timeit(f)
    return t, 2.0 * rows * F * R * S * Cin / t / 1e9

rows = 128 * 14 * 14
for flags in (1, 0):
    lib.hp_debug_gemm_flags(flags)
    for (Cin, R, S, wq) in [(384, 3, 3, 14), (384, 3, 3, 16), (384, 3, 3, 8), (3456, 1, 1, 14), (384, 1, 9, 1), (384, 9, 1, 8)]:
        for F in (192, 256):
            t, tf = run(rows, Cin, R, S, wq, F)
            offs = sorted({r * wq + s for r in range(R) for s in range(S)})
            aligned = sum(o % 8 == 0 for o in offs)
            print(f"flags={flags} C={Cin} R={R} S={S} wq={wq} F={F}: {t:.4f} ms {tf:6.0f} TF/s  taps aligned {aligned}/{len(offs)}", flush=True)
lib.hp_debug_gemm_flags(0)
