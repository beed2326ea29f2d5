"""ctypes binding of oracle/gacer_oracle.c (fp64, NCHW).  TEST INFRASTRUCTURE.

Each wrapper allocates the fp64 output and calls the plain C loop.  Shapes
follow PyTorch: floor((H + 2p - k) / s) + 1.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gacer_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "gacer_oracle_train.c")]   # forward ops, training backward ops
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc -O2 -fopenmp (no fast-math: IEEE fp64)."""
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(f) for f in _SRCS):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared",
                               "-fno-fast-math", "-ffp-contract=off",
                               "-o", _LIB, *_SRCS, "-lm"])
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
        D = ctypes.POINTER(ctypes.c_double)
        i, d, sz = ctypes.c_int, ctypes.c_double, ctypes.c_size_t
        _lib.oracle_conv2d.argtypes = [D, D, D] + [i] * 13 + [D]
        _lib.oracle_batchnorm.argtypes = [D, i, i, i, D, D, D, D, d, D]
        _lib.oracle_relu.argtypes = [D, sz, i, D]
        _lib.oracle_maxpool.argtypes = [D] + [i] * 11 + [D]
        _lib.oracle_avgpool.argtypes = [D] + [i] * 12 + [D]
        _lib.oracle_gap.argtypes = [D, i, i, i, D]
        _lib.oracle_linear.argtypes = [D, D, D, i, i, i, D]
        _lib.oracle_add.argtypes = [D, D, sz, D]
        _lib.oracle_hardswish.argtypes = [D, sz, D]
        _lib.oracle_hardsigmoid.argtypes = [D, sz, D]
        _lib.oracle_scale_channels.argtypes = [D, D, i, i, i, D]
        _lib.oracle_num_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def out_size(n, k, s, p):
    return (n + 2 * p - k) // s + 1


def conv2d(x, w, b=None, stride=1, pad=(0, 0), groups=1):
    x, w = _f64(x), _f64(w)
    b = None if b is None else _f64(b)
    N, Cin, H, W = x.shape
    Cout, _, KH, KW = w.shape
    ph, pw = pad if isinstance(pad, (tuple, list)) else (pad, pad)
    Ho, Wo = out_size(H, KH, stride, ph), out_size(W, KW, stride, pw)
    y = np.empty((N, Cout, Ho, Wo), dtype=np.float64)
    lib().oracle_conv2d(_p(x), _p(w), _p(b), N, Cin, H, W, Cout, KH, KW,
                        stride, ph, pw, groups, Ho, Wo, _p(y))
    return y


def batchnorm(x, gamma, beta, mean, var, eps):
    x = _f64(x)
    N, C = x.shape[:2]
    HW = int(np.prod(x.shape[2:])) if x.ndim > 2 else 1
    y = np.empty_like(x)
    g, b, m, v = (_f64(a) for a in (gamma, beta, mean, var))
    lib().oracle_batchnorm(_p(x), N, C, HW, _p(g), _p(b), _p(m), _p(v), float(eps), _p(y))
    return y


def relu(x, six=False):
    x = _f64(x)
    y = np.empty_like(x)
    lib().oracle_relu(_p(x), x.size, int(six), _p(y))
    return y


def maxpool(x, k, stride, pad=(0, 0)):
    x = _f64(x)
    N, C, H, W = x.shape
    KH, KW = (k, k) if isinstance(k, int) else k
    ph, pw = pad if isinstance(pad, (tuple, list)) else (pad, pad)
    Ho, Wo = out_size(H, KH, stride, ph), out_size(W, KW, stride, pw)
    y = np.empty((N, C, Ho, Wo), dtype=np.float64)
    lib().oracle_maxpool(_p(x), N, C, H, W, KH, KW, stride, ph, pw, Ho, Wo, _p(y))
    return y


def avgpool(x, k, stride, pad=(0, 0), count_include_pad=True):
    x = _f64(x)
    N, C, H, W = x.shape
    KH, KW = (k, k) if isinstance(k, int) else k
    ph, pw = pad if isinstance(pad, (tuple, list)) else (pad, pad)
    Ho, Wo = out_size(H, KH, stride, ph), out_size(W, KW, stride, pw)
    y = np.empty((N, C, Ho, Wo), dtype=np.float64)
    lib().oracle_avgpool(_p(x), N, C, H, W, KH, KW, stride, ph, pw,
                         int(count_include_pad), Ho, Wo, _p(y))
    return y


def gap(x):
    x = _f64(x)
    N, C, H, W = x.shape
    y = np.empty((N, C, 1, 1), dtype=np.float64)
    lib().oracle_gap(_p(x), N, C, H * W, _p(y))
    return y


def linear(x, w, b=None):
    x, w = _f64(x), _f64(w)
    b = None if b is None else _f64(b)
    N, K = x.shape
    O = w.shape[0]
    y = np.empty((N, O), dtype=np.float64)
    lib().oracle_linear(_p(x), _p(w), _p(b), N, K, O, _p(y))
    return y


def add(a, b):
    a, b = _f64(a), _f64(b)
    assert a.shape == b.shape
    y = np.empty_like(a)
    lib().oracle_add(_p(a), _p(b), a.size, _p(y))
    return y


def hardswish(x):
    x = _f64(x)
    y = np.empty_like(x)
    lib().oracle_hardswish(_p(x), x.size, _p(y))
    return y


def hardsigmoid(x):
    x = _f64(x)
    y = np.empty_like(x)
    lib().oracle_hardsigmoid(_p(x), x.size, _p(y))
    return y


def scale_channels(x, s):
    """y[n, c, ...] = x[n, c, ...] * s[n, c] (s: [N, C] or [N, C, 1, 1])."""
    x = _f64(x)
    N, C = x.shape[:2]
    s = _f64(s).reshape(N, C)
    HW = int(np.prod(x.shape[2:])) if x.ndim > 2 else 1
    y = np.empty_like(x)
    lib().oracle_scale_channels(_p(x), _p(s), N, C, HW, _p(y))
    return y


def num_threads() -> int:
    return lib().oracle_num_threads()
