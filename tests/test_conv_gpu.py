"""Implicit-GEMM convolutions (tcgen05 + TMA im2col) against torch float64
convolutions on the same rounded inputs: fprop, wgrad, and the stride-1
dgrad-as-rotated-conv. These replace conv2d_forward / conv2d_backward
(tensor.cpp:419-516) on the AlexNet conv2-5 shapes."""
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.nn.functional as F  # noqa: E402

from paper_1404_5997_b200._lib import last_error, lib  # noqa: E402

SHAPES = [  # B, C, H, F, R, stride, pad
    (2, 64, 27, 192, 5, 1, 2),     # AlexNet conv2
    (2, 192, 13, 384, 3, 1, 1),    # conv3
    (3, 384, 13, 256, 3, 1, 1),    # conv5
    (2, 64, 14, 96, 3, 2, 1),      # strided fprop/wgrad
    (1, 128, 9, 64, 1, 1, 0),      # 1x1
]


def ops(math, x, w):
    dt = torch.bfloat16 if math == 0 else torch.float32
    return x.to(dt), w.to(dt), (x.to(dt).double() if math == 0 else x.double()), \
        (w.to(dt).double() if math == 0 else w.double())


@pytest.mark.parametrize("math", [0, 2])
@pytest.mark.parametrize("shape", SHAPES)
def test_fprop_wgrad_dgrad(math, shape):
    B, Cc, H, Fo, R, st, pad = shape
    g = torch.Generator(device="cuda").manual_seed(sum(shape))
    x = torch.randn(B, H, H, Cc, device="cuda", generator=g)          # NHWC
    w = torch.randn(Fo, R, R, Cc, device="cuda", generator=g) * 0.1    # FRSC
    xd, wd, xr, wr = ops(math, x, w)
    OH = (H + 2 * pad - R) // st + 1
    # bf16: vs fp64 on bf16-rounded operands; 3xTF32: the tensor core accumulates
    # tf32 products with round-toward-zero, bounding it near 1e-5 (stated 5e-5)
    tol = 2e-5 if math == 0 else 5e-5
    # fprop
    y = torch.empty(B * OH * OH, Fo, device="cuda")
    assert lib.hp_kernel_conv_fprop(math, xd.data_ptr(), B, H, H, Cc, wd.data_ptr(), Fo, R, R, st, pad,
                                    y.data_ptr(), None) == 0, last_error()
    torch.cuda.synchronize()
    ref = F.conv2d(xr.permute(0, 3, 1, 2), wr.permute(0, 3, 1, 2), stride=st, padding=pad)
    ref = ref.permute(0, 2, 3, 1).reshape(B * OH * OH, Fo)
    assert (y.double() - ref).abs().max().item() / ref.abs().max().item() < tol
    # wgrad
    dy = torch.randn(B * OH * OH, Fo, device="cuda", generator=g)
    dyd = dy.to(xd.dtype)
    dyr = dyd.double()
    dw = torch.full((Fo, R * R * Cc), float("nan"), device="cuda")
    ws = torch.empty(64 * Fo * R * R * Cc, device="cuda")
    assert lib.hp_kernel_conv_wgrad(math, xd.data_ptr(), B, H, H, Cc, dyd.data_ptr(), Fo, R, R, st, pad,
                                    dw.data_ptr(), ws.data_ptr(), ws.numel(), None) == 0, last_error()
    torch.cuda.synchronize()
    xt = xr.permute(0, 3, 1, 2).requires_grad_()
    wt = wr.permute(0, 3, 1, 2).clone().requires_grad_()
    out = F.conv2d(xt, wt, stride=st, padding=pad)
    out.backward(dyr.reshape(B, OH, OH, Fo).permute(0, 3, 1, 2))
    rdw = wt.grad.permute(0, 2, 3, 1).reshape(Fo, -1)
    assert (dw.double() - rdw).abs().max().item() / rdw.abs().max().item() < tol
    # dgrad (stride 1 only: rotated-weight conv)
    if st == 1:
        wrot = w.reshape(Fo, R, R, Cc).flip(1).flip(2).permute(3, 1, 2, 0).contiguous()  # [C][R][S][F]
        wrotd = wrot.to(xd.dtype)
        dx = torch.full((B * H * H, Cc), float("nan"), device="cuda")
        assert lib.hp_kernel_conv_dgrad(math, dyd.data_ptr(), B, OH, OH, Fo, wrotd.data_ptr(), Cc, R, R, pad,
                                        dx.data_ptr(), None) == 0, last_error()
        torch.cuda.synchronize()
        rdx = xt.grad.permute(0, 2, 3, 1).reshape(B * H * H, Cc)
        assert (dx.double() - rdx).abs().max().item() / rdx.abs().max().item() < tol


def to_q(x, p):
    """NHWC [B][H][W][C] -> q-layout rows [(B*(H+p)*(W+p))][C]: pixel (h, w) at
    slot (h+p, w+p) of its image's (H+p) x (W+p) block, zeros elsewhere."""
    B, H, W, C = x.shape
    q = torch.zeros(B, H + p, W + p, C, dtype=x.dtype, device=x.device)
    q[:, p:, p:, :] = x
    return q.reshape(-1, C).contiguous()


SHIFT_SHAPES = [  # B, C, H, F, R (stride 1, same padding)
    (2, 64, 27, 192, 5),    # AlexNet conv2 fprop
    (2, 192, 13, 384, 3),   # conv3
    (3, 384, 13, 256, 3),   # conv5
    (2, 192, 27, 64, 5),    # conv2 dgrad shape (N = 64)
    (1, 128, 9, 128, 1),    # 1x1
]


@pytest.mark.parametrize("shape", SHIFT_SHAPES)
def test_conv_shift_q_layout(shape):
    """Flat-shift implicit GEMM (one smem halo per channel block, row-shifted
    UMMA descriptors per tap) on a q-layout input == torch conv2d (fp64 on the
    bf16-rounded operands) at every valid output position."""
    B, C, H, Fo, R = shape
    p = (R - 1) // 2
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(B, H, H, C, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(Fo, R, R, C, device="cuda", generator=g) * 0.1).to(torch.bfloat16)
    xq = to_q(x, p)
    rows = xq.shape[0]
    y = torch.full((rows, Fo), float("nan"), device="cuda")
    rc = lib.hp_kernel_conv_shift(xq.data_ptr(), rows, C, R, R, H + p, w.data_ptr(), Fo, y.data_ptr(), 0, None)
    assert rc == 0, last_error()
    torch.cuda.synchronize()
    ref = F.conv2d(x.double().permute(0, 3, 1, 2), w.double().permute(0, 3, 1, 2), padding=p)
    ref = ref.permute(0, 2, 3, 1)  # B, H, W, F
    got = y.reshape(B, H + p, H + p, Fo)[:, :H, :H, :].double()
    err = (got - ref).abs().max().item() / ref.abs().max().item()
    assert err < 2e-5, err
