"""Kernel parity: the step's fused LRN + max-pool kernels (forward and backward)
and its momentum-SGD kernel, called through the C ABI on identical inputs,
against the oracle's restatement (oracle/hpsim_oracle.c or_lrn_* /
or_maxpool_* / or_momentum_update_f32; the pool/LRN restatement is
torch-checked in tests/test_oracle_extensions.py, the SGD one pinned to the
compiled reference).

Integer work is bit-exact:
* pool argmax -- the GPU's 1-byte window offset r*pk+q, mapped to the oracle's
  in-plane index -- must equal the oracle's index in EVERY window when both
  pool the same values (LRN with alpha = 0, k = 1 is the identity on fp32:
  pow(1, -beta) == 1 exactly in the kernel's lg2/ex2 form), ties, zeros and
  NaN included;
* with a real LRN the GPU's fp32 LRN differs from the double one by rounding,
  so the argmax must match wherever the oracle's winner leads the runner-up by
  more than that rounding (1e-5 relative), and otherwise point at a value
  within it.
Floating point: pooled values within 2e-6 (fp32) / bf16 rounding (4e-3) of
max |ref|; the backward is fed the GPU's own argmax so both route the same
windows, dz within 1e-5 (fp32) / 1e-2 (bf16: dz is stored as bf16) of max |ref|.
Pool-only backward: routed to exactly the oracle's pixels, sums within 1e-6 /
4e-3. SGD: bit-identical to the reference's four rounded float passes.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import oracle as O  # noqa: E402
import paper_1404_5997_b200 as hp  # noqa: E402
from paper_1404_5997_b200._lib import last_error, lib  # noqa: E402

torch = pytest.importorskip("torch")

BF16, F32 = int(hp.MathMode.BF16), int(hp.MathMode.TF32)  # TF32 mode keeps fp32 activations


def _dev(a, math):
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    return t.to(torch.bfloat16) if math == BF16 else t


def _host(t):
    return t.float().cpu().numpy()


def _oracle_fwd(a_nchw, n, alpha, beta, k, pk, ps):
    B, Cc, H, W = a_nchw.shape
    if n > 0:
        b = np.empty_like(a_nchw)
        d = np.empty_like(a_nchw)
        O.oracle_lib().or_lrn_forward(O._dp(a_nchw), B, Cc, H * W, n, alpha, beta, k, O._dp(b), O._dp(d))
    else:
        b, d = a_nchw, None
    PH, PW = (H - pk) // ps + 1, (W - pk) // ps + 1
    y = np.empty((B, Cc, PH, PW))
    idx = np.empty((B, Cc, PH, PW), dtype=np.int32)
    O.oracle_lib().or_maxpool_forward(O._dp(np.ascontiguousarray(b)), B, Cc, H, W, pk, ps, O._dp(y),
                                      idx.ctypes.data_as(C.POINTER(C.c_int32)))
    return b, d, y, idx


def _gpu_idx_to_plane(widx_nhwc, H, W, pk, ps):
    """[B][PH][PW][C] window offsets -> [B][C][PH][PW] in-plane indices h*W+w."""
    B, PH, PW, Cc = widx_nhwc.shape
    r, q = widx_nhwc // pk, widx_nhwc % pk
    oh = np.arange(PH)[None, :, None, None]
    ow = np.arange(PW)[None, None, :, None]
    plane = (oh * ps + r) * W + (ow * ps + q)
    return plane.transpose(0, 3, 1, 2).astype(np.int32)


def _runner_up_gap(b_nchw, idx, pk, ps):
    """Per window: (max - second max) / max|b| over the window's other entries."""
    B, Cc, H, W = b_nchw.shape
    PH, PW = idx.shape[2:]
    wins = np.stack([b_nchw[:, :, r:r + ps * (PH - 1) + 1:ps, q:q + ps * (PW - 1) + 1:ps]
                     for r in range(pk) for q in range(pk)], axis=-1)
    s = np.sort(wins, axis=-1)
    return (s[..., -1] - s[..., -2]) / max(np.abs(b_nchw).max(), 1e-30), wins


def _run(math, B, H, W, Cc, n, alpha, beta, k, pk, ps, relu=True, seed=0, ties=False, scale=1.0):
    rng = np.random.default_rng(seed)
    a = scale * (np.maximum(rng.normal(size=(B, H, W, Cc)), 0.0) if relu else rng.normal(size=(B, H, W, Cc)))
    if ties:  # exact ties inside windows, plus a NaN
        a[:, 1, 1, :] = a[:, 1, 2, :]
        a[:, 3, 3, :] = a[:, 2, 3, :]
        a[0, 4, 4, 0] = np.nan
    ad = _dev(a, math)
    a_used = _host(ad).astype(np.float64)  # the values the GPU sees (bf16-rounded in bf16 mode)
    PH, PW = (H - pk) // ps + 1, (W - pk) // ps + 1
    y = torch.empty((B, PH, PW, Cc), device="cuda", dtype=ad.dtype)
    widx = torch.empty((B, PH, PW, Cc), device="cuda", dtype=torch.uint8)
    rc = lib.hp_kernel_lrn_pool_fwd(math, ad.data_ptr(), B, H, W, Cc, n, alpha, beta, k, pk, ps, y.data_ptr(),
                                    widx.data_ptr(), None)
    assert rc == 0, last_error()
    torch.cuda.synchronize()
    a_nchw = np.ascontiguousarray(a_used.transpose(0, 3, 1, 2))
    b, d, yo, io = _oracle_fwd(a_nchw, n, alpha, beta, k, pk, ps)
    gi = _gpu_idx_to_plane(widx.cpu().numpy().astype(np.int32), H, W, pk, ps)
    yg = _host(y).transpose(0, 3, 1, 2)
    return a_used, a_nchw, ad, b, d, yo, io, gi, yg, y, widx


@pytest.mark.parametrize("math", [F32, BF16])
@pytest.mark.parametrize("shape", [(4, 55, 55, 64), (4, 27, 27, 192), (2, 13, 13, 256), (2, 9, 11, 32)])
def test_pool_argmax_bit_exact(math, shape):
    """Identity LRN (alpha=0, k=1) and pool-only: the GPU pools exactly the
    oracle's values, so every window's argmax must be identical -- ties
    (first maximum, strict >), ReLU zeros and NaN (first NaN wins) included.
    Shapes: AlexNet conv1 / conv2 (row-streaming kernels), conv5 (pool-only kernel), and
    an odd one (smem-band kernel)."""
    B, H, W, Cc = shape
    for n in (5, 0):
        _, _, _, _, _, yo, io, gi, yg, _, _ = _run(math, B, H, W, Cc, n, 0.0, 0.75, 1.0, 3, 2, ties=True)
        assert np.array_equal(gi, io), (n, int((gi != io).sum()))
        fin = ~np.isnan(yo)
        assert np.array_equal(np.isnan(yg), ~fin)
        assert np.array_equal(yg[fin], yo[fin])  # y is the (rounded) input value itself


@pytest.mark.parametrize("math", [F32, BF16])
@pytest.mark.parametrize("shape", [(4, 55, 55, 64), (4, 27, 27, 192), (2, 9, 11, 32)])
def test_lrn_pool_forward_backward(math, shape):
    """LRN (n=5, beta=0.75, k=2) + pool 3/2 vs the double oracle; alpha and the
    input scale chosen so the normaliser is far from constant (alpha*sum a^2 ~ 0.2;
    AlexNet's own alpha=1e-4 runs in the step parity tests)."""
    B, H, W, Cc = shape
    n, alpha, beta, k, pk, ps = 5, 1e-2, 0.75, 2.0, 3, 2
    a_used, a_nchw, ad, b, d, yo, io, gi, yg, y, widx = _run(math, B, H, W, Cc, n, alpha, beta, k, pk, ps, seed=1,
                                                             scale=3.0)
    ytol = 2e-6 if math == F32 else 4e-3
    assert np.abs(yg - yo).max() / np.abs(yo).max() <= ytol
    gap, wins = _runner_up_gap(b, io, pk, ps)
    # a clear winner, or an all-zero (ReLU) window where both take the first zero
    clear = (gap > 1e-5) | (yo == 0.0)
    assert clear.mean() > 0.99
    assert np.array_equal(gi[clear], io[clear]), int((gi[clear] != io[clear]).sum())
    # near-ties: the GPU's pick is within rounding of the window maximum
    Bq, Cq, PH, PW = io.shape
    picked = np.take_along_axis(b.reshape(Bq, Cq, -1), gi.reshape(Bq, Cq, -1).astype(np.int64), axis=2)
    assert np.abs(picked.reshape(io.shape) - yo).max() <= 1e-5 * np.abs(b).max()
    # backward with the GPU's routing
    rng = np.random.default_rng(2)
    gy = rng.normal(size=(B, PH, PW, Cc))
    gyd = torch.from_numpy(gy.astype(np.float32)).cuda()
    dz = torch.empty_like(ad)
    bias = torch.full((Cc,), float("nan"), device="cuda")
    rc = lib.hp_kernel_lrn_pool_bwd(math, gyd.data_ptr(), widx.data_ptr(), ad.data_ptr(), B, H, W, Cc, n, alpha,
                                    beta, k, pk, ps, 1, dz.data_ptr(), bias.data_ptr(), None)
    assert rc == 0
    torch.cuda.synchronize()
    # fused bias gradient = channel sums of the STORED dz (fp32 sums vs double)
    dsum = _host(dz).astype(np.float64).sum(axis=(0, 1, 2))
    assert np.abs(bias.cpu().numpy() - dsum).max() <= 1e-5 * np.abs(_host(dz)).sum(axis=(0, 1, 2)).max()
    gb = np.zeros_like(a_nchw)
    gyo = np.ascontiguousarray(gy.astype(np.float32).astype(np.float64).transpose(0, 3, 1, 2))
    O.oracle_lib().or_maxpool_backward(O._dp(gyo), np.ascontiguousarray(gi).ctypes.data_as(C.POINTER(C.c_int32)),
                                       B, Cc, H, W, pk, ps, O._dp(gb))
    ga = np.empty_like(a_nchw)
    O.oracle_lib().or_lrn_backward(O._dp(a_nchw), O._dp(d), O._dp(gb), B, Cc, H * W, n, alpha, beta, O._dp(ga))
    ga *= a_nchw > 0  # the fused ReLU mask
    dg = _host(dz).transpose(0, 3, 1, 2)
    tol = 1e-5 if math == F32 else 1e-2
    assert np.abs(dg - ga).max() / np.abs(ga).max() <= tol


@pytest.mark.parametrize("math", [F32, BF16])
def test_maxpool_backward_routes_exactly(math):
    """Pool-only backward (conv5): the gradient lands on the argmax (sum over
    overlapping windows), exactly as or_maxpool_backward with the same indices;
    fp32 sums of at most 4 terms in the same order -> bit-identical in fp32."""
    B, H, W, Cc = 2, 13, 13, 256
    a_used, a_nchw, ad, b, d, yo, io, gi, yg, y, widx = _run(math, B, H, W, Cc, 0, 0.0, 0.75, 1.0, 3, 2, seed=3)
    rng = np.random.default_rng(4)
    gy = rng.normal(size=(B, 6, 6, Cc)).astype(np.float32)
    gyd = torch.from_numpy(gy).cuda()
    dz = torch.empty_like(ad)
    assert lib.hp_kernel_lrn_pool_bwd(math, gyd.data_ptr(), widx.data_ptr(), ad.data_ptr(), B, H, W, Cc, 0, 0.0,
                                      0.75, 1.0, 3, 2, 1, dz.data_ptr(), None, None) == 0
    torch.cuda.synchronize()
    gx = np.zeros_like(a_nchw)
    O.oracle_lib().or_maxpool_backward(O._dp(np.ascontiguousarray(gy.astype(np.float64).transpose(0, 3, 1, 2))),
                                       io.ctypes.data_as(C.POINTER(C.c_int32)), B, Cc, H, W, 3, 2, O._dp(gx))
    gx *= a_nchw > 0
    dg = _host(dz).transpose(0, 3, 1, 2)
    assert np.array_equal(dg != 0, gx != 0)  # routed to exactly the same pixels
    tol = 1e-6 if math == F32 else 4e-3  # up to 4 overlapping windows summed in fp32 vs double
    assert np.abs(dg - gx).max() <= tol * np.abs(gx).max()


@pytest.mark.parametrize("has_gscale", [0, 1])
@pytest.mark.parametrize("n", [1, 1000, 3207104])
def test_sgd_kernel_bit_exact(n, has_gscale):
    """momentum_update (optimizer.cpp:19-31) in float: the GPU kernel must give
    the reference's bits (four rounded passes, no FMA, scalars rounded once)."""
    rng = np.random.default_rng(n)
    w = (0.01 * rng.normal(size=n)).astype(np.float32)
    m = (1e-3 * rng.normal(size=n)).astype(np.float32)
    g = rng.normal(size=n).astype(np.float32)
    lr, mu, wd, gs = 0.01, 0.9, 5e-4, np.float32(0.25 if has_gscale else 1.0)
    wd_, md_, gd_ = (torch.from_numpy(v.copy()).cuda() for v in (w, m, g))
    cp = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    assert lib.hp_kernel_sgd(wd_.data_ptr(), md_.data_ptr(), gd_.data_ptr(), n, lr, mu, wd, float(gs), has_gscale,
                             cp.data_ptr(), None) == 0
    torch.cuda.synchronize()
    wo, mo = w.copy(), m.copy()
    go = (g * gs).astype(np.float32) if has_gscale else g
    F = C.POINTER(C.c_float)
    O.oracle_lib().or_momentum_update_f32(wo.ctypes.data_as(F), mo.ctypes.data_as(F), go.ctypes.data_as(F), n, lr,
                                          mu, wd)
    assert np.array_equal(wd_.cpu().numpy(), wo)
    assert np.array_equal(md_.cpu().numpy(), mo)
    assert torch.equal(cp, torch.from_numpy(wo).cuda().to(torch.bfloat16))


@pytest.mark.parametrize("math", [hp.MathMode.F32X3, hp.MathMode.BF16])
@pytest.mark.parametrize("K,scheme,var", [(1, "B", False), (2, "C", True), (3, "B", False)])
def test_fused_fc_sgd_epilogue_bit_identical(math, K, scheme, var):
    """The FC weight update fused into the wgrad GEMM epilogue gives the same
    bits as storing the gradient and running the SGD kernel (itself bit-exact
    to the reference's float update above), split-K plans included."""
    spec = hp.tiny_cnn()
    res = []
    for fuse in (True, False):
        g = hp.Cluster(spec, hp.ClusterConfig(workers=K, per_worker_batch=12 if K == 3 else 16,
                                              scheme=hp.Scheme.from_string(scheme), variable_batch=var, seed=4,
                                              math_mode=math))
        g.set_fuse_fc_sgd(fuse)
        b = g.config.per_worker_batch
        for s in range(2):
            xs, ts = zip(*[hp.synthetic_batch(spec, b, step=s, worker=w) for w in range(K)])
            g.run_step(list(xs), list(ts), hp.HyperParams(momentum=0.9, lr=0.05, weight_decay=5e-4))
        res.append([g.param(w, which, l) for w in range(K) for which in (2, 3, 6, 7) for l in range(2)])
    for a, b in zip(*res):
        assert np.array_equal(a, b)
