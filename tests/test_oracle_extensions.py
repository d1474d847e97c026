"""The AlexNet superset the reference cannot express (floor-mode geometry,
cross-channel LRN, overlapping max-pool): parity UNPINNED by the reference,
so the oracle's restatement is cross-checked against torch.nn.functional on
CPU (float64), forward and autograd backward. Integer pool indices must match
torch's exactly (first maximum in row-major window order)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle as O


def _pool(x, k, s):
    B, C, H, W = x.shape
    OH, OW = (H - k) // s + 1, (W - k) // s + 1
    y = np.empty((B, C, OH, OW)); idx = np.empty((B, C, OH, OW), dtype=np.int32)
    O.oracle_lib().or_maxpool_forward(O._dp(x), B, C, H, W, k, s, O._dp(y), idx.ctypes.data_as(O.C.POINTER(O.C.c_int32)))
    return y, idx


@pytest.mark.parametrize("shape", [(2, 3, 13, 13), (1, 4, 27, 27), (2, 2, 6, 6)])
def test_maxpool_matches_torch(shape):
    rng = np.random.default_rng(0)
    x = rng.normal(size=shape)
    x[0, 0, 1, 1] = x[0, 0, 1, 2]  # an exact tie inside a window
    y, idx = _pool(x, 3, 2)
    ty, tidx = F.max_pool2d(torch.from_numpy(x), 3, 2, return_indices=True)
    assert np.array_equal(y, ty.numpy())
    assert np.array_equal(idx, tidx.numpy().astype(np.int32))
    gy = rng.normal(size=y.shape)
    gx = np.empty_like(x)
    O.oracle_lib().or_maxpool_backward(O._dp(gy), idx.ctypes.data_as(O.C.POINTER(O.C.c_int32)), *shape, 3, 2, O._dp(gx))
    t = torch.from_numpy(x).requires_grad_()
    F.max_pool2d(t, 3, 2).backward(torch.from_numpy(gy))
    assert np.allclose(gx, t.grad.numpy(), rtol=0, atol=1e-14)


@pytest.mark.parametrize("C,n", [(8, 5), (64, 5), (5, 3), (6, 4)])
def test_lrn_matches_torch(C, n):
    """Krizhevsky LRN with alpha NOT divided by n == torch LRN(size=n, alpha=alpha*n)."""
    rng = np.random.default_rng(C)
    B, H, W = 2, 5, 4
    a = np.abs(rng.normal(size=(B, C, H, W)))
    alpha, beta, k = 1e-2, 0.75, 2.0
    b = np.empty_like(a); d = np.empty_like(a)
    O.oracle_lib().or_lrn_forward(O._dp(a), B, C, H * W, n, alpha, beta, k, O._dp(b), O._dp(d))
    t = torch.from_numpy(a).requires_grad_()
    tb = F.local_response_norm(t, n, alpha=alpha * n, beta=beta, k=k)
    assert np.allclose(b, tb.detach().numpy(), rtol=1e-12, atol=0)
    gb = rng.normal(size=a.shape)
    tb.backward(torch.from_numpy(gb))
    ga = np.empty_like(a)
    O.oracle_lib().or_lrn_backward(O._dp(a), O._dp(d), O._dp(gb), B, C, H * W, n, alpha, beta, O._dp(ga))
    assert np.allclose(ga, t.grad.numpy(), rtol=1e-10, atol=1e-13)


def test_alexnet_geometry():
    """floor-mode conv1 224 -> 55, pools 55->27->13->6, flat 9216; the
    reference's exact-division rule rejects it."""
    import paper_1404_5997_b200 as hp
    from oracle import make_spec_c
    spec = hp.alexnet_1col()
    sc = make_spec_c(spec)
    hw = (O.C.c_int64 * 10)()
    assert O.oracle_lib().or_conv_output_sizes(O.C.byref(sc), hw) == 0
    assert list(hw) == [27, 27, 13, 13, 13, 13, 13, 13, 6, 6]
    assert O.oracle_lib().or_flattened_conv_size(O.C.byref(sc)) == 9216
    spec.conv_layers[0].floor_mode = False
    assert O.oracle_lib().or_validate(O.C.byref(make_spec_c(spec))) == 1
    assert "not a positive integer" in O.oracle_lib().or_last_error().decode()


def test_alexnet_conv_stack_vs_torch():
    """Oracle AlexNet conv forward+backward at tiny batch vs torch autograd (double)."""
    import paper_1404_5997_b200 as hp
    spec = hp.alexnet_1col(num_classes=16)
    spec.fc_layers[0].out_dim = 32; spec.fc_layers[1].in_dim = 32; spec.fc_layers[1].out_dim = 32
    spec.fc_layers[2].in_dim = 32
    c = O.OracleCluster(spec, workers=1, per_worker_batch=1, scheme="B", precision="double", seed=4)
    rng = np.random.default_rng(1)
    for which in (0, 2):
        for l in range(len(spec.conv_layers) if which == 0 else 3):
            c.write_param(0, which, l, c.param(0, which, l) * 20.0)
    params = {(w, l): c.param(0, w, l) for w in range(4) for l in range(5 if w < 2 else 3)}
    x = rng.normal(size=(1, 3, 224, 224)); t = np.zeros((1, 16)); t[0, 3] = 1.0
    m = c.run_step([x], [t], O.make_hyper_c(0.0, 1.0, 0.0))  # w' = w - g
    # torch double reference of the same network
    X = torch.from_numpy(x)
    ws = []
    h = X
    for l, L in enumerate(spec.conv_layers):
        k = torch.from_numpy(params[(0, l)].reshape(L.out_channels, L.in_channels, L.kernel, L.kernel)).requires_grad_()
        bb = torch.from_numpy(params[(1, l)]).requires_grad_()
        ws.append(k)
        h = torch.relu(F.conv2d(h, k, bb, stride=L.stride, padding=L.pad))
        if L.lrn_size:
            h = F.local_response_norm(h, L.lrn_size, alpha=L.lrn_alpha * L.lrn_size, beta=L.lrn_beta, k=L.lrn_k)
        if L.pool_kernel:
            h = F.max_pool2d(h, L.pool_kernel, L.pool_stride)
    h = h.reshape(1, -1)
    for l, L in enumerate(spec.fc_layers):
        W = torch.from_numpy(params[(2, l)].reshape(L.in_dim, L.out_dim))
        h = h @ W + torch.from_numpy(params[(3, l)])
        if L.relu:
            h = torch.relu(h)
    T = torch.from_numpy(t)
    loss = (F.softplus(-h) + (1 - T) * h).sum()
    loss.backward()
    assert abs(loss.item() - m.loss) < 1e-9 * abs(loss.item())
    for l in range(5):
        g_oracle = params[(0, l)] - c.param(0, 0, l)
        g_torch = ws[l].grad.numpy().ravel()
        assert np.abs(g_oracle - g_torch).max() <= 1e-9 * np.abs(g_torch).max()
