"""Dev: tcgen05 GEMM throughput by operand major-ness (mainloop-only and full)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1404_5997_b200._lib import HpGemmDesc, lib, last_error
from gemm_probe2 import timeit

def run(M, N, K, am, bm, cta2, bn, flags):
    lib.hp_debug_gemm_flags(flags)
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if am else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if bm else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Cc = torch.empty(M, N, device="cuda")
    d = HpGemmDesc(); d.math = 0
    d.a, d.a_mn, d.lda = A.data_ptr(), am, (M if am else K)
    d.b, d.b_mn, d.ldb = B.data_ptr(), bm, (N if bm else K)
    d.M, d.N, d.K = M, N, K
    d.c, d.ldc, d.c_type, d.alpha = Cc.data_ptr(), N, 0, 1.0
    d.splits, d.bn, d.cta2 = 1, bn, cta2
    def f():
        assert lib.hp_kernel_gemm(C.byref(d), None) == 0, last_error()
    t = timeit(f)
    return t, 2.0 * M * N * K / t / 1e9

for (M, N, K) in [(8192, 8192, 8192), (384, 3456, 25088)]:
    for am, bm in ((0, 0), (1, 0), (0, 1), (1, 1)):
        for flags in (1,):
            t, tf = run(M, N, K, am, bm, 1, 256, flags)
            print(f"{str((M,N,K)):20s} a_mn={am} b_mn={bm} flags={flags}: {t:.4f} ms {tf:6.0f} TF/s", flush=True)
lib.hp_debug_gemm_flags(0)
