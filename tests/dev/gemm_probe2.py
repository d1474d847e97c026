"""Dev: mainloop-only vs full GEMM timing (dbg flag 1 skips epilogue stores)."""
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

def gemm_fn(M, N, K, bn=0, cta2=-1):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Cc = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    d = HpGemmDesc(); d.math = 0
    d.a, d.a_mn, d.lda = A.data_ptr(), 0, K
    d.b, d.b_mn, d.ldb = B.data_ptr(), 0, K
    d.M, d.N, d.K = M, N, K
    d.c, d.ldc, d.c_type, d.alpha = Cc.data_ptr(), N, 1, 1.0
    d.splits, d.bn, d.cta2 = 1, bn, cta2
    keep = (A, B, Cc)
    def f():
        rc = lib.hp_kernel_gemm(C.byref(d), None)
        assert rc == 0, last_error()
    return f, keep

def conv_shift(B, Cin, H, F, R):
    p = (R - 1) // 2
    rows = B * (H + p) * (H + p)
    x = torch.randn(rows, Cin, device="cuda").to(torch.bfloat16)
    w = (torch.randn(F, R * R * Cin, device="cuda") * 0.1).to(torch.bfloat16)
    y = torch.empty(rows, F, device="cuda")
    def f():
        assert lib.hp_kernel_conv_shift(x.data_ptr(), rows, Cin, R, R, H + p, w.data_ptr(), F, y.data_ptr(), 0, None) == 0, last_error()
    return f, (x, w, y), 2.0 * rows * F * R * R * Cin

if __name__ == "__main__":
  for flags in (0, 1):
      lib.hp_debug_gemm_flags(flags)
      for (M, N, K) in [(8192, 8192, 8192), (93312, 192, 1600), (21632, 384, 3456)]:
          for cta2, bn in ((1, 256), (1, 192), (0, 256)):
              f, keep = gemm_fn(M, N, K, bn, cta2)
              t = timeit(f)
              print(f"flags={flags} gemm {str((M,N,K)):22s} cta2={cta2} bn={bn}: {t:.4f} ms {2*M*N*K/t/1e9:7.0f} TF/s", flush=True)
      for args in [(128, 384, 13, 384, 3), (128, 192, 13, 384, 3), (128, 64, 27, 192, 5)]:
          f, keep, fl = conv_shift(*args)
          t = timeit(f)
          print(f"flags={flags} shift {str(args):22s}: {t:.4f} ms {fl/t/1e9:7.0f} TF/s", flush=True)
  lib.hp_debug_gemm_flags(0)
