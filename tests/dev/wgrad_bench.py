"""Dev microbenchmark: the conv-wgrad GEMM shapes (huge K, small M x N) on the plain
GEMM path, across operand major-ness, tile kernels and split-K, vs cuBLAS."""
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


WS = torch.empty(64 * 1024 * 1024, device="cuda")


def gemm_fn(M, N, K, a_mn, b_mn, bn, cta2, splits):
    A = torch.randn(K, M, device="cuda").to(torch.bfloat16) if a_mn else torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(K, N, device="cuda").to(torch.bfloat16) if b_mn else torch.randn(N, K, device="cuda").to(torch.bfloat16)
    Cc = torch.empty(M, N, device="cuda", dtype=torch.float32)
    d = HpGemmDesc(); d.math = 0
    d.a, d.a_mn, d.lda = A.data_ptr(), a_mn, (M if a_mn else K)
    d.b, d.b_mn, d.ldb = B.data_ptr(), b_mn, (N if b_mn else K)
    d.M, d.N, d.K = M, N, K
    d.c, d.ldc, d.c_type, d.alpha = Cc.data_ptr(), N, 0, 1.0
    d.splits, d.bn, d.cta2, d.ws = splits, bn, cta2, WS.data_ptr()
    s = lib.hp_kernel_gemm_splits(C.byref(d))
    keep = (A, B, Cc, d)
    def f():
        rc = lib.hp_kernel_gemm(C.byref(d), None)
        assert rc == 0, last_error()
    return f, keep, s


VARIANTS = ((-1, 0), (0, 128), (0, 192), (0, 256), (1, 128), (1, 256))
if os.environ.get("WGRAD_AUTO_ONLY"):
    VARIANTS = ((-1, 0),)
if os.environ.get("WGRAD_VARIANTS"):  # "cta2:bn,..."
    VARIANTS = tuple(tuple(int(v) for v in x.split(":")) for x in os.environ["WGRAD_VARIANTS"].split(","))
SPLITS = tuple(int(v) for v in os.environ.get("WGRAD_SPLITS", "0").split(","))
MAJORS = tuple(tuple(int(c) for c in m) for m in os.environ.get("WGRAD_MAJORS", "11,00").split(","))
shapes = [(384, 3456, 25088), (384, 1728, 25088), (256, 3456, 25088), (1600, 192, 107648), (64, 576, 387200)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1:]]
print("shape                     major  cta2  bn  splits    ms    TF/s")
for (M, N, K) in shapes:
    flops = 2.0 * M * N * K
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16); b = torch.randn(K, N, device="cuda", dtype=torch.bfloat16)
    t = timeit(lambda: a @ b)
    print(f"{str((M, N, K)):25s} cublas                 {t:7.3f} {flops / t / 1e9:7.0f}", flush=True)
    del a, b
    for (a_mn, b_mn) in MAJORS:
        for cta2, bn in VARIANTS:
            for splits in SPLITS:
                try:
                    f, keep, s = gemm_fn(M, N, K, a_mn, b_mn, bn, cta2, splits)
                    t = timeit(f)
                except AssertionError as e:
                    print(f"{str((M, N, K)):25s} {a_mn}{b_mn}    {cta2:3d} {bn:4d}  failed {e}")
                    continue
                print(f"{str((M, N, K)):25s} {a_mn}{b_mn}    {cta2:3d} {bn:4d} {s:5d} {t:7.3f} {flops / t / 1e9:7.0f}",
                      flush=True)
