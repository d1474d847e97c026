"""Dev microbenchmark: FC-shaped GEMMs (weight streaming, n=128) across split-K
factors and tile configs; bf16, fp32 output; includes the split-K reduce."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1404_5997_b200._lib import HpGemmDesc, lib, last_error


def timeit(fn, iters=30):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def run(M, N, K, a_mn, b_mn, splits, bn, cta2):
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_mn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_mn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Cc = torch.empty(M, N, device="cuda")
    d = HpGemmDesc(); d.math = 0
    d.a, d.a_mn, d.lda = A.data_ptr(), a_mn, (M if a_mn else K)
    d.b, d.b_mn, d.ldb = B.data_ptr(), b_mn, (N if b_mn else K)
    d.M, d.N, d.K = M, N, K
    d.c, d.ldc, d.c_type, d.alpha = Cc.data_ptr(), N, 0, 1.0
    d.splits, d.bn, d.cta2 = splits, bn, cta2
    s = lib.hp_kernel_gemm_splits(C.byref(d))
    ws = torch.empty(max(1, s) * M * N, device="cuda")
    d.ws = ws.data_ptr()
    def f():
        assert lib.hp_kernel_gemm(C.byref(d), None) == 0, last_error()
    t = timeit(f)
    return t, s


shapes = {"fc6 fwd": (4096, 128, 9216, 0, 0), "fc7 fwd": (4096, 128, 4096, 0, 1), "fc8 fwd": (1000, 128, 4096, 0, 1),
          "fc7 dgrad": (4096, 128, 4096, 1, 1), "fc6 dgrad": (128, 9216, 4096, 1, 1)}
for name, (M, N, K, am, bm) in shapes.items():
    wbytes = M * K * 2 if name.endswith("fwd") or name == "fc7 dgrad" else N * K * 2
    res = []
    for cta2, bn in ((0, 128), (1, 128), (0, 64), (-1, 0)):
        for sp in (0, 1, 2, 3, 4, 6, 8, 12, 16):
            try:
                t, s = run(M, N, K, am, bm, sp, bn, cta2)
            except AssertionError as e:
                continue
            res.append((t, cta2, bn, sp, s))
    res.sort()
    auto = [r for r in res if r[3] == 0 and r[1] == -1]
    print(f"{name} {M}x{N}x{K}: weight stream bound {wbytes / 6.5e12 * 1e3:.4f} ms; auto {auto[0] if auto else None}")
    for r in res[:6]:
        print(f"   {r[0]:.4f} ms cta2={r[1]} bn={r[2]} splits(req={r[3]}, got={r[4]}) {2*M*N*K/r[0]/1e9:.0f} TF/s")
