"""GPU probe: tcgen05 GEMM vs torch fp64 on rounded inputs, all layouts/modes."""
import sys, os, ctypes as C, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from paper_1404_5997_b200._lib import lib, HpGemmDesc, last_error

def tf32_trunc(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)

def run(math, M, N, K, a_mn, b_mn, epi=None, splits=1, bn=0, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    dt = torch.bfloat16 if math == 0 else torch.float32
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    pad = 64
    def store(X, mn):  # X is [rows][K] logical
        rows, k = X.shape
        if mn:
            ld = ((rows + pad - 1) // pad) * pad
            buf = torch.zeros(k, ld, device="cuda", dtype=torch.float32)
            buf[:, :rows] = X.t()
        else:
            ld = ((k + pad - 1) // pad) * pad
            buf = torch.zeros(rows, ld, device="cuda", dtype=torch.float32)
            buf[:, :k] = X
        return buf.to(dt).contiguous(), ld
    Ab, lda = store(A, a_mn)
    Bb, ldb = store(B, b_mn)
    alo = blo = None
    if math == 2:
        alo = (Ab - tf32_trunc(Ab)).contiguous(); blo = (Bb - tf32_trunc(Bb)).contiguous()
    if math == 0:
        Ar, Br = A.to(torch.bfloat16).double(), B.to(torch.bfloat16).double()
    elif math == 1:
        Ar, Br = tf32_trunc(A).double(), tf32_trunc(B).double()
    else:
        Ar, Br = A.double(), B.double()
    ref = Ar @ Br.t()
    ldc = ((N + 63) // 64) * 64
    Cb = torch.full((M, ldc), float("nan"), device="cuda", dtype=torch.float32)
    d = HpGemmDesc()
    d.math = math
    d.a = Ab.data_ptr(); d.a_mn = a_mn; d.lda = lda
    d.b = Bb.data_ptr(); d.b_mn = b_mn; d.ldb = ldb
    d.M, d.N, d.K = M, N, K
    d.c = Cb.data_ptr(); d.ldc = ldc; d.c_type = 0; d.c_trans = 0; d.alpha = 1.0
    d.splits = splits; d.bn = bn
    ws = None
    s = lib.hp_kernel_gemm_splits(C.byref(d)) if splits <= 0 else splits
    if s > 1:
        ws = torch.empty(s * M * N + 1024, device="cuda", dtype=torch.float32)
        d.ws = ws.data_ptr()
    rc = lib.hp_kernel_gemm(C.byref(d), None)
    if rc != 0:
        return f"rc={rc} {last_error()}"
    torch.cuda.synchronize()
    out = Cb[:, :N].double()
    err = (out - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
    return err

torch.cuda.init()
print("device", torch.cuda.get_device_name())
fails = 0
for math in [int(x) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["0","1","2"])]:
    for a_mn, b_mn in itertools.product((0, 1), (0, 1)):
        for (M, N, K, bn, sp) in [(128, 64, 64, 64, 1), (256, 128, 512, 128, 1), (300, 200, 333, 0, 1),
                                  (128, 256, 1024, 256, 1), (384, 192, 640, 192, 1), (128, 512, 4096, 128, 0),
                                  (1000, 130, 70, 0, 1)]:
            try:
                e = run(math, M, N, K, a_mn, b_mn, splits=sp, bn=bn)
            except Exception as ex:
                e = f"EXC {ex}"
            tol = {0: 1e-5, 1: 1e-5, 2: 1e-5}[math]
            ok = isinstance(e, float) and e < tol
            fails += 0 if ok else 1
            print(f"math={math} a_mn={a_mn} b_mn={b_mn} M={M} N={N} K={K} bn={bn} splits={sp}: err={e} {'OK' if ok else 'FAIL'}", flush=True)
print("FAILS", fails)
