"""Dev microbenchmark: tcgen05 GEMM vs cuBLAS on plain and conv shapes."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1404_5997_b200._lib import HpGemmDesc, lib, last_error

def timeit(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters

def gemm_fn(M, N, K, a_mn=0, b_mn=0, bn=0, cta2=-1, splits=1):
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_mn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_mn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Cc = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    d = HpGemmDesc(); d.math = 0
    d.a, d.a_mn, d.lda = A.data_ptr(), a_mn, (M if a_mn else K)
    d.b, d.b_mn, d.ldb = B.data_ptr(), b_mn, (N if b_mn else K)
    d.M, d.N, d.K = M, N, K
    d.c, d.ldc, d.c_type, d.alpha = Cc.data_ptr(), N, 1, 1.0
    d.splits, d.bn, d.cta2 = splits, bn, cta2
    keep = (A, B, Cc)
    def f():
        rc = lib.hp_kernel_gemm(C.byref(d), None)
        assert rc == 0, last_error()
    return f, keep

def conv_fn(B, Cin, H, F, R, pad):
    x = torch.randn(B, H, H, Cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(F, R, R, Cin, device="cuda") * 0.1).to(torch.bfloat16)
    OH = H + 2 * pad - R + 1
    y = torch.empty(B * OH * OH, F, device="cuda")
    keep = (x, w, y)
    def f():
        assert lib.hp_kernel_conv_fprop(0, x.data_ptr(), B, H, H, Cin, w.data_ptr(), F, R, R, 1, pad, y.data_ptr(), None) == 0, last_error()
    return f, keep, 2.0 * B * OH * OH * F * R * R * Cin

print("shape                          variant          ms     TF/s")
for (M, N, K) in [(8192, 8192, 8192), (16384, 256, 4096), (93312, 192, 1600), (21632, 384, 3456)]:
    flops = 2.0 * M * N * K
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16); b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    t = timeit(lambda: a @ b)
    print(f"{str((M,N,K)):30s} cublas        {t:7.3f}  {flops/t/1e9:7.0f}")
    for cta2 in (0, 1):
        for bn in ((192, 256) if cta2 else (192, 256)):
            if N % bn and N < bn: continue
            f, keep = gemm_fn(M, N, K, bn=bn, cta2=cta2)
            t = timeit(f)
            print(f"{str((M,N,K)):30s} cta2={cta2} bn={bn:3d}  {t:7.3f}  {flops/t/1e9:7.0f}", flush=True)
for args in [(128, 64, 27, 192, 5, 2), (128, 192, 13, 384, 3, 1), (128, 384, 13, 384, 3, 1), (128, 384, 13, 256, 3, 1)]:
    for cta2, bn in ((-1, 0), (0, 192), (0, 256), (1, 192), (1, 256)):
        lib.hp_debug_gemm_force(cta2, bn)
        f, keep, flops = conv_fn(*args)
        t = timeit(f)
        print(f"conv {str(args):25s} cta2={cta2:2d} bn={bn:3d} {t:7.3f}  {flops/t/1e9:7.0f}", flush=True)
    lib.hp_debug_gemm_force(-1, 0)
