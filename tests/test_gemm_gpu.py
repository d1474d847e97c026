"""tcgen05 GEMM kernel (hp_kernel_gemm) against a float64 torch reference of
the same op on identically rounded inputs: every operand major-ness, bf16 /
tf32 / 3xTF32, tails, split-K and the fused epilogue. These GEMMs replace
matmul / matmul_tn / matmul_nt (tensor.cpp:254-305) and the conv loops."""
import ctypes as C
import itertools

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1404_5997_b200._lib import HpGemmDesc, last_error, lib  # noqa: E402

TOL = {0: 2e-5, 1: 2e-5, 2: 5e-5}  # vs fp64 on the operands the tensor core sees


def tf32_trunc(x):
    return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)


def store(X, mn, dt):
    rows, k = X.shape
    if mn:
        ld = (rows + 63) // 64 * 64
        buf = torch.zeros(k, ld, device="cuda")
        buf[:, :rows] = X.t()
    else:
        ld = (k + 63) // 64 * 64
        buf = torch.zeros(rows, ld, device="cuda")
        buf[:, :k] = X
    return buf.to(dt).contiguous(), ld


def gemm(math, A, B, a_mn, b_mn, M, N, K, splits=1, bn=0, cta2=-1, **epi):
    dt = torch.bfloat16 if math == 0 else torch.float32
    Ab, lda = store(A, a_mn, dt)
    Bb, ldb = store(B, b_mn, dt)
    ldc = (M if epi.get("c_trans") else N + 63) // 64 * 64 if not epi.get("c_trans") else (M + 63) // 64 * 64
    rows = N if epi.get("c_trans") else M
    Cb = epi.pop("C_init", None)
    c_type = int(epi.get("c_type", 0))
    if Cb is None:
        Cb = torch.full((rows, ldc), float("nan"), device="cuda",
                        dtype=torch.bfloat16 if c_type else torch.float32)
    d = HpGemmDesc()
    d.math = math
    d.a, d.a_mn, d.lda = Ab.data_ptr(), a_mn, lda
    d.b, d.b_mn, d.ldb = Bb.data_ptr(), b_mn, ldb
    d.M, d.N, d.K = M, N, K
    d.c, d.ldc, d.c_type, d.c_trans = Cb.data_ptr(), ldc, c_type, int(epi.get("c_trans", 0))
    mask = epi.get("mask")
    if mask is not None:
        d.mask, d.ldmask = mask.data_ptr(), mask.shape[1]
        d.mask_type = 1 if mask.dtype == torch.bfloat16 else 0
    d.alpha = epi.get("alpha", 1.0)
    d.beta = int(epi.get("beta", 0))
    bias = epi.get("bias")
    d.bias = bias.data_ptr() if bias is not None else None
    d.bias_mode = epi.get("bias_mode", 0)
    d.relu = int(epi.get("relu", 0))
    d.splits, d.bn, d.cta2 = splits, bn, cta2
    s = lib.hp_kernel_gemm_splits(C.byref(d))
    ws = None
    if s > 1:
        ws = torch.empty(s * M * N, device="cuda")
        d.ws = ws.data_ptr()
    assert lib.hp_kernel_gemm(C.byref(d), None) == 0, last_error()
    torch.cuda.synchronize()
    return Cb, (Ab, Bb)


def ref_inputs(math, A, B):
    if math == 0:
        return A.to(torch.bfloat16).double(), B.to(torch.bfloat16).double()
    if math == 1:
        return tf32_trunc(A).double(), tf32_trunc(B).double()
    return A.double(), B.double()


SHAPES = [(128, 64, 64, 64, 1), (300, 200, 333, 0, 1), (384, 192, 640, 192, 1), (128, 256, 1024, 256, 1),
          (128, 512, 4096, 128, 0), (1000, 130, 70, 0, 1), (64, 363, 4000, 128, 0)]


@pytest.mark.parametrize("math", [0, 1, 2])
@pytest.mark.parametrize("a_mn,b_mn", list(itertools.product((0, 1), (0, 1))))
@pytest.mark.parametrize("cta2", [0, 1])
def test_gemm_layouts(math, a_mn, b_mn, cta2):
    """cta2=1: CTA-pair kernel (tcgen05.mma.cta_group::2, 256-row tiles)."""
    if cta2 and math == 2:
        pytest.skip("3xTF32 runs on the single-CTA kernel")
    g = torch.Generator(device="cuda").manual_seed(1)
    for M, N, K, bn, sp in SHAPES:
        if cta2:
            bn = 128 if bn in (64, 128, 192) else bn
            if b_mn and bn not in (0, 128, 256):
                bn = 128
        A = torch.randn(M, K, device="cuda", generator=g)
        B = torch.randn(N, K, device="cuda", generator=g)
        out, _ = gemm(math, A, B, a_mn, b_mn, M, N, K, splits=sp, bn=bn, cta2=cta2)
        Ar, Br = ref_inputs(math, A, B)
        ref = Ar @ Br.t()
        err = (out[:, :N].double() - ref).abs().max().item() / ref.abs().max().item()
        assert err < TOL[math], (M, N, K, err)


def test_gemm_f32x3_is_near_fp32():
    """3xTF32 (in-kernel hi/lo split) reaches fp32-class accuracy on raw fp32 inputs."""
    g = torch.Generator(device="cuda").manual_seed(2)
    A = torch.randn(256, 2048, device="cuda", generator=g)
    B = torch.randn(192, 2048, device="cuda", generator=g)
    out, _ = gemm(2, A, B, 0, 1, 256, 192, 2048, splits=0)
    ref = A.double() @ B.double().t()
    err = (out[:, :192].double() - ref).abs().max().item() / ref.abs().max().item()
    assert err < 5e-6  # chains bounded to 128 products (split-K, fp32 RN reduce)
    out1, _ = gemm(1, A, B, 0, 1, 256, 192, 2048)
    err1 = (out1[:, :192].double() - ref).abs().max().item() / ref.abs().max().item()
    assert err1 > 4 * err  # plain tf32 is measurably coarser


@pytest.mark.parametrize("math", [0, 2])
def test_gemm_epilogue(math):
    """bias (per row / per column), ReLU, alpha, beta accumulation, transposed store."""
    g = torch.Generator(device="cuda").manual_seed(3)
    M, N, K = 200, 96, 160
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    Ar, Br = ref_inputs(math, A, B)
    ref = Ar @ Br.t()
    tol = 3e-5 if math == 0 else 2e-5
    bc = torch.randn(N, device="cuda", generator=g)
    out, _ = gemm(math, A, B, 0, 0, M, N, K, bias=bc, bias_mode=2, relu=1, alpha=0.5)
    r = torch.relu(0.5 * ref + bc.double())
    assert (out[:, :N].double() - r).abs().max().item() / r.abs().max().item() < tol
    br = torch.randn(M, device="cuda", generator=g)
    out, _ = gemm(math, A, B, 1, 1, M, N, K, bias=br, bias_mode=1)
    r = ref + br.double()[:, None]
    assert (out[:, :N].double() - r).abs().max().item() / r.abs().max().item() < tol
    init = torch.randn(M, (N + 63) // 64 * 64, device="cuda", generator=g)
    out, _ = gemm(math, A, B, 0, 1, M, N, K, beta=1, C_init=init.clone())
    r = ref + init[:, :N].double()
    assert (out[:, :N].double() - r).abs().max().item() / r.abs().max().item() < tol
    out, _ = gemm(math, A, B, 0, 0, M, N, K, c_trans=1)
    assert (out[:N, :M].double() - ref.t()).abs().max().item() / ref.abs().max().item() < tol


@pytest.mark.parametrize("cta2", [0, 1])
def test_gemm_epilogue_mask_bf16_ragged(cta2):
    """ReLU-backward mask (bf16 and fp32) and bf16 output through the staged,
    coalesced epilogue, with ragged M and N edges (rows past M, columns past N)."""
    g = torch.Generator(device="cuda").manual_seed(4)
    M, N, K = 300, 200, 192
    A = torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g)
    Ar, Br = ref_inputs(0, A, B)
    ref = Ar @ Br.t()
    for mdt in (torch.bfloat16, torch.float32):
        mask = torch.randn(M, 256, device="cuda", generator=g).to(mdt)
        out, _ = gemm(0, A, B, 0, 0, M, N, K, mask=mask, cta2=cta2)
        r = torch.where(mask[:, :N].double() > 0, ref, torch.zeros_like(ref))
        assert (out[:, :N].double() - r).abs().max().item() / ref.abs().max().item() < 3e-5
    out, _ = gemm(0, A, B, 1, 0, M, N, K, c_type=1, relu=1, cta2=cta2)
    r = torch.relu(ref)
    assert (out[:, :N].double() - r).abs().max().item() / r.abs().max().item() < 8e-3  # bf16 store
    for n in (193, 197, 199):  # column counts that end inside a 4-wide group
        out, _ = gemm(0, A[:, :K], B[:n], 0, 0, M, n, K, cta2=cta2)
        r = ref[:, :n]
        assert (out[:, :n].double() - r).abs().max().item() / r.abs().max().item() < 3e-5
        assert torch.isnan(out[:, n:].float()).all()  # nothing written past N
