"""ctypes binding of the product's C-ABI (include/tie_cuda.h) -- exactly what a reference
maintainer's ctypes/cffi stub would bind.  The GPU parity tests call the
CUDA path through this, not through the pybind layer."""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2604_00499_b200", "_lib", "libtie_b200.so")
HEADER = os.path.join(ROOT, "include", "tie_cuda.h")

_d, _u64, _i, _p, _u = ctypes.c_double, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p, ctypes.c_uint
TIE_SCORE_MOMENT, TIE_SCORE_EXACT, TIE_SCORE_RAW = 0, 1, 2


class TieError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(tie_[a-z0-9_]+)\s*\(", txt)))


def _ptr(a):
    return None if a is None else a.ctypes.data


class CAbi:
    def __init__(self, path=LIB):
        self.lib = L = ctypes.CDLL(path)
        L.tie_last_error.restype = ctypes.c_char_p
        L.tie_ctx_create.argtypes = [_i, _p, _i, _d, _d, ctypes.POINTER(_p)]
        L.tie_ctx_create_mc.argtypes = [_i, _d, _i, _u64, ctypes.POINTER(_p)]
        L.tie_ctx_destroy.argtypes = [_p]
        L.tie_ctx_destroy.restype = None
        L.tie_sync.argtypes = [_p, _p]
        L.tie_score_host.argtypes = [_p, _p, _p, _p, _u64, _d, _d, _p, _p, _p, _u]
        L.tie_score_rank_host.argtypes = [_p, _p, _p, _p, _u64, _d, _d, _p, _p, _u]
        L.tie_rank_host.argtypes = [_p, _p, _p, _u64, _p]
        L.tie_fit_host.argtypes = [_p, _p, _u64, _u64, _d, _p, _p, _p, _p, _p, _p]
        L.tie_fit_report_host.argtypes = [_p, _p, _u64, _u64, _d, _u, _p, _p]
        L.tie_fit_report_ragged_host.argtypes = [_p, _p, _p, _u64, _d, _u, _p, _p]
        L.tie_t_quantile.argtypes = [_d, _d]
        L.tie_t_quantile.restype = _d
        L.tie_compute_beta.argtypes = [_i, _d, _d, _d, _u64, ctypes.POINTER(_d)]
        L.tie_launch_count.argtypes = [_i]
        L.tie_launch_count.restype = _u64

    def check(self, rc):
        if rc:
            raise TieError(rc, self.lib.tie_last_error().decode())

    def ctx(self, samples=None, nu=3.5, sigma_table_max=0.0, device=0):
        h = _p()
        if samples is None:
            self.check(self.lib.tie_ctx_create_mc(device, nu, 10000, 12, ctypes.byref(h)))
        else:
            s = np.ascontiguousarray(samples, np.float64)
            self.check(self.lib.tie_ctx_create(device, _ptr(s), len(s), nu, sigma_table_max,
                                               ctypes.byref(h)))
        return h

    def destroy(self, h):
        self.lib.tie_ctx_destroy(h)

    def score(self, h, mu, sigma, x_max, alpha=0.9, beta=0.5, flags=TIE_SCORE_MOMENT):
        mu = np.ascontiguousarray(mu, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        x_max = np.ascontiguousarray(x_max, np.float64)
        n = len(mu)
        E, C, S = np.empty(n), np.empty(n), np.empty(n)
        self.check(self.lib.tie_score_host(h, _ptr(mu), _ptr(sigma), _ptr(x_max), n, alpha, beta,
                                           _ptr(E), _ptr(C), _ptr(S), flags))
        return E, C, S

    def score_rank(self, h, mu, sigma, max_tokens, alpha=0.9, beta=0.5, flags=TIE_SCORE_MOMENT):
        mu = np.ascontiguousarray(mu, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        mt = np.ascontiguousarray(max_tokens, np.uint32)
        n = len(mu)
        S = np.empty(n)
        order = np.empty(n, np.uint64)
        self.check(self.lib.tie_score_rank_host(h, _ptr(mu), _ptr(sigma), _ptr(mt), n, alpha,
                                                beta, _ptr(S), _ptr(order), flags))
        return S, order

    def rank(self, h, key, ids=None):
        key = np.ascontiguousarray(key, np.float64)
        ids = None if ids is None else np.ascontiguousarray(ids, np.uint64)
        order = np.empty(len(key), np.uint64)
        self.check(self.lib.tie_rank_host(h, _ptr(key), _ptr(ids), len(key), _ptr(order)))
        return order

    def fit(self, h, x, nu=3.5):
        x = np.ascontiguousarray(x, np.float64)
        P, K = x.shape
        mu, sg, ll = np.empty(P), np.empty(P), np.empty(P)
        it = np.empty(P, np.int32)
        cv = np.empty(P, np.uint8)
        dg = np.empty(P, np.uint8)
        self.check(self.lib.tie_fit_host(h, _ptr(x), P, K, nu, _ptr(mu), _ptr(sg), _ptr(ll),
                                         _ptr(it), _ptr(cv), _ptr(dg)))
        return dict(mu=mu, sigma=sg, log_likelihood=ll, iterations=it,
                    converged=cv.astype(bool), degenerate=dg.astype(bool))

    def fit_report_raw(self, h, x, nu=3.5, families=15):
        x = np.ascontiguousarray(x, np.float64)
        P, K = x.shape
        fits = np.full((4, 10, P), np.nan)
        tail = np.full((5, P), np.nan)
        self.check(self.lib.tie_fit_report_host(h, _ptr(x), P, K, nu, families, _ptr(fits),
                                                _ptr(tail)))
        return fits, tail

    def fit_report_ragged_raw(self, h, lengths, offsets, nu=3.5, families=15):
        lengths = np.ascontiguousarray(lengths, np.float64)
        offsets = np.ascontiguousarray(offsets, np.uint64)
        P = len(offsets) - 1
        fits = np.full((4, 10, P), np.nan)
        tail = np.full((5, P), np.nan)
        self.check(self.lib.tie_fit_report_ragged_host(h, _ptr(lengths), _ptr(offsets), P, nu,
                                                       families, _ptr(fits), _ptr(tail)))
        return fits, tail

    def launches(self, reset=False):
        return int(self.lib.tie_launch_count(1 if reset else 0))


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.maximum(np.abs(b), np.finfo(np.float64).tiny)
    return np.abs(a - b) / den


def order_check(order, key_ref, ids=None, tol=1e-12):
    """Is `order` a permutation sorted by (reference key, id) except among adjacent pairs whose
    reference keys differ by <= tol relative?  Returns (ok, n_violations, n_exempt)."""
    order = np.asarray(order, np.int64)
    n = len(key_ref)
    if len(order) != n or not np.array_equal(np.sort(order), np.arange(n)):
        return False, -1, 0
    k = np.asarray(key_ref)[order]
    idv = order if ids is None else np.asarray(ids)[order]
    ka, kb = k[:-1], k[1:]
    ok_pair = (ka < kb) | ((ka == kb) & (idv[:-1] < idv[1:]))
    close = np.abs(kb - ka) <= tol * np.maximum(np.abs(ka), np.abs(kb))
    bad = ~ok_pair & ~close
    exempt = ~ok_pair & close
    return not bad.any(), int(bad.sum()), int(exempt.sum())
