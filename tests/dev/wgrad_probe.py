"""Dev: conv wgrad GEMM (TMA im2col B, MN-major dY A) mainloop-only vs full."""
import os, sys
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

for flags in (0, 1):
    lib.hp_debug_gemm_flags(flags)
    for (B, C, H, F, R, pad) in [(128, 384, 13, 384, 3, 1), (128, 64, 27, 192, 5, 2), (128, 192, 13, 384, 3, 1)]:
        for cta2, bn in ((-1, 0), (1, 256), (0, 256), (1, 192)):
            lib.hp_debug_gemm_force(cta2, bn)
            x = torch.randn(B, H, H, C, device="cuda").to(torch.bfloat16)
            dy = torch.randn(B * H * H, F, device="cuda").to(torch.bfloat16)
            dw = torch.empty(F, R * R * C, device="cuda")
            ws = torch.empty(64 * F * R * R * C, device="cuda")
            def f():
                assert lib.hp_kernel_conv_wgrad(0, x.data_ptr(), B, H, H, C, dy.data_ptr(), F, R, R, 1, pad, dw.data_ptr(),
                                                ws.data_ptr(), ws.numel(), None) == 0, last_error()
            t = timeit(f)
            fl = 2.0 * B * H * H * F * R * R * C
            print(f"flags={flags} wgrad C={C} H={H} F={F} R={R} cta2={cta2} bn={bn}: {t:.4f} ms {fl/t/1e9:6.0f} TF/s", flush=True)
lib.hp_debug_gemm_force(-1, 0)
lib.hp_debug_gemm_flags(0)
