"""Shared helpers for the parity tests (test infrastructure)."""
import types

import numpy as np


def conv(i, o, k, s=1, p=0, relu=True, **kw):
    return types.SimpleNamespace(in_channels=i, out_channels=o, kernel=k, stride=s, pad=p, relu=relu, **kw)


def fc(i, o, relu=False):
    return types.SimpleNamespace(in_dim=i, out_dim=o, relu=relu)


def toy_spec():
    """SPEC.md toy spec."""
    return types.SimpleNamespace(conv_layers=[conv(2, 3, 3, 1, 1), conv(3, 4, 2, 2, 0)],
                                 fc_layers=[fc(36, 8, True), fc(8, 4)], input_shape=[2, 6, 6], num_classes=4)


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def one_hot(labels, L):
    t = np.zeros((len(labels), L))
    t[np.arange(len(labels)), labels] = 1.0
    return t
