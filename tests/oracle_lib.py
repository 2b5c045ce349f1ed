"""ctypes wrappers over the CHECKERS (test infrastructure only).

* ``Oracle``  -- oracle/_build/libtie_oracle.so, the plain-C restatement (oracle/tie_oracle.c).
* ``RefLib``  -- oracle/_ref/libtie_ref.so, the untouched reference sources compiled by
  ``make -C oracle ref`` (only present where /root/reference was available at build time).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "_build", "libtie_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libtie_ref.so")

_d = ctypes.c_double
_u64 = ctypes.c_uint64
_i32 = ctypes.c_int
_p = ctypes.c_void_p


def _ptr(a):
    return None if a is None else a.ctypes.data


def _threads(threads):
    return int(threads) if threads else (os.cpu_count() or 1)


class _Base:
    prefix = ""

    def _fn(self, name, argtypes, restype=ctypes.c_int):
        f = getattr(self.lib, self.prefix + name)
        f.argtypes = argtypes
        f.restype = restype
        return f

    def _check(self, rc, what):
        if rc:
            msg = self._err().decode()
            if rc == 1:
                raise ValueError(f"{what}: domain_error: {msg}")
            if rc == 2:
                raise ValueError(f"{what}: invalid_argument: {msg}")
            raise RuntimeError(f"{what}: rc={rc}: {msg}")

    # -- common API ------------------------------------------------------------------
    def mc_samples(self, nu=3.5, n=10000, seed=12):
        out = np.empty(n, np.float64)
        self._check(self._mc(nu, n, seed, _ptr(out)), "mc_samples")
        return out

    def gen_workload(self, n, seed=1, mu_range=(3.0, 5.0), sigma_range=(0.5, 1.2), nu=3.5,
                     max_tokens=2048, rps=100.0, extras=False):
        mu = np.empty(n, np.float64)
        sg = np.empty(n, np.float64)
        mt = np.empty(n, np.uint32)
        arr = np.empty(n, np.float64) if extras else None
        pt = np.empty(n, np.uint32) if extras else None
        tl = np.empty(n, np.uint32) if extras else None
        rc = self._gw(n, seed, mu_range[0], mu_range[1], sigma_range[0], sigma_range[1], nu,
                      max_tokens, rps, _ptr(mu), _ptr(sg), _ptr(mt), _ptr(arr), _ptr(pt),
                      _ptr(tl))
        self._check(rc, "gen_workload")
        if extras:
            return mu, sg, mt, arr, pt, tl
        return mu, sg, mt

    def rank(self, key, ids=None):
        key = np.ascontiguousarray(key, np.float64)
        ids = None if ids is None else np.ascontiguousarray(ids, np.uint64)
        out = np.empty(len(key), np.uint64)
        self._check(self._rank(_ptr(key), _ptr(ids), len(key), _ptr(out)), "rank")
        return out

    def fit(self, x, nu=3.5, threads=None):
        x = np.ascontiguousarray(x, np.float64)
        P, K = x.shape
        mu = np.empty(P)
        sg = np.empty(P)
        ll = np.empty(P)
        it = np.empty(P, np.int32)
        cv = np.empty(P, np.uint8)
        dg = np.empty(P, np.uint8)
        rc = self._fit(_ptr(x), P, K, nu, _ptr(mu), _ptr(sg), _ptr(ll), _ptr(it), _ptr(cv),
                       _ptr(dg), _threads(threads))
        self._check(rc, "fit")
        return dict(mu=mu, sigma=sg, log_likelihood=ll, iterations=it,
                    converged=cv.astype(bool), degenerate=dg.astype(bool))


    FIT_FAMILIES = ("logt", "logt_free_nu", "lognormal", "exponential")
    FIT_FIELDS = ("mu", "sigma", "nu", "rate", "log_likelihood", "iterations", "converged",
                  "degenerate", "ks_statistic", "ks_p_value")
    TAIL_FIELDS = ("skewness", "cv", "p90_over_p50", "p99_over_p50", "top10_share")

    def fit_report_raw(self, x, nu=3.5, families=15, threads=None):
        """cmd_fit's per-prompt analysis -> (fits[4][10][P], tail[5][P]) arrays."""
        x = np.ascontiguousarray(x, np.float64)
        P, K = x.shape
        fits = np.full((4, 10, P), np.nan)
        tail = np.full((5, P), np.nan)
        self._check(self._report(_ptr(x), P, K, nu, families, _ptr(fits), _ptr(tail),
                                 _threads(threads)), "fit_report")
        return fits, tail

    def fit_report(self, x, nu=3.5, families=15, threads=None):
        """-> ({family: {field: array[P]}}, {field: array[P]})."""
        return unpack_report(*self.fit_report_raw(x, nu, families, threads), families)


def unpack_report(fits, tail, families):
    out = {}
    for f, name in enumerate(_Base.FIT_FAMILIES):
        if families >> f & 1:
            out[name] = {k: fits[f, j] for j, k in enumerate(_Base.FIT_FIELDS)}
    return out, {k: tail[j] for j, k in enumerate(_Base.TAIL_FIELDS)}


class Oracle(_Base):
    """The C restatement (the parity checker)."""

    prefix = "tor_"

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)
        self.lib = ctypes.CDLL(path)
        self._err = self._fn("last_error", [], ctypes.c_char_p)
        self._mc = self._fn("mc_samples", [_d, _i32, _u64, _p])
        self.t_cdf = self._fn("t_cdf", [_d, _d], _d)
        self.t_pdf = self._fn("t_pdf", [_d, _d], _d)
        self.t_quantile = self._fn("t_quantile", [_d, _d], _d)
        self.mix64 = self._fn("mix64", [_u64, _u64], _u64)
        self.regularized_incomplete_beta = self._fn("regularized_incomplete_beta",
                                                    [_d, _d, _d], _d)
        self._score = self._fn("score", [_p, _i32, _d, _p, _p, _p, _u64, _d, _d, _p, _p, _p,
                                         ctypes.POINTER(_u64), _i32])
        self._beta = self._fn("compute_beta", [_i32, _d, _d, _d, _u64, ctypes.POINTER(_d)])
        self._rank = self._fn("rank", [_p, _p, _u64, _p])
        self._fit = self._fn("fit", [_p, _u64, _u64, _d, _p, _p, _p, _p, _p, _p, _i32])
        self._report = self._fn("fit_report", [_p, _u64, _u64, _d, ctypes.c_uint, _p, _p,
                                               _i32])
        self.logt_loglik_raw = self._fn("logt_loglik", [_p, _u64, _d, _d, _d], _d)
        self._gw = self._fn("gen_workload", [_u64, _u64, _d, _d, _d, _d, _d, ctypes.c_uint32,
                                             _d, _p, _p, _p, _p, _p, _p])
        self._gf = self._fn("gen_fit_data", [_u64, _u64, _u64, _d, _d, _d, _d, _d, _i32, _p,
                                             _p, _p, _i32])
        self._sl = self._fn("sample_logt", [_d, _d, _d, _u64, _u64, _p])
        self._sched = self._fn("scheduler_script", [_i32, _i32, _d, _d, _d, _d, _u64, _p, _p,
                                                    _p, _p, _p, ctypes.POINTER(_u64)])

    def sim_scores(self, mu, sigma, ids, max_tokens, predictor=0, mu_sd=0.0, ls_sd=0.0,
                   seed=0, family=0, alpha=0.9, samples=None):
        f = self._fn("sim_scores", [_p, _i32, _d, _p, _p, _p, _p, _u64, _i32, _d, _d, _u64,
                                    _i32, _d, _p, _p])
        Y = self.mc_samples() if samples is None else np.ascontiguousarray(samples, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        ids = np.ascontiguousarray(ids, np.uint64)
        xm = np.ascontiguousarray(max_tokens, np.float64)
        E, C = np.empty(len(mu)), np.empty(len(mu))
        self._check(f(_ptr(Y), len(Y), 3.5, _ptr(mu), _ptr(sigma), _ptr(ids), _ptr(xm),
                      len(mu), predictor, mu_sd, ls_sd, seed, family, alpha, _ptr(E),
                      _ptr(C)), "sim_scores")
        return E, C

    def scheduler_script(self, policy, ops, ids, a, b, adaptive=True, beta_fixed=0.1,
                         beta_max=0.5, q_sat=128.0, rebuild_threshold=0.1):
        ops = np.ascontiguousarray(ops, np.int32)
        ids = np.ascontiguousarray(ids, np.uint64)
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty(max(len(ops), 1), np.uint64)
        n_out = _u64(0)
        rc = self._sched(policy, int(adaptive), beta_fixed, beta_max, q_sat, rebuild_threshold,
                         len(ops), _ptr(ops), _ptr(ids), _ptr(a), _ptr(b), _ptr(out),
                         ctypes.byref(n_out))
        self._check(rc, "scheduler_script")
        return out[: n_out.value]

    def score(self, samples, mu, sigma, x_max, alpha=0.9, beta=0.5, nu=3.5, threads=None):
        samples = np.ascontiguousarray(samples, np.float64)
        mu = np.ascontiguousarray(mu, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        x_max = np.ascontiguousarray(x_max, np.float64)
        n = len(mu)
        E = np.empty(n)
        C = np.empty(n)
        S = np.empty(n)
        bad = _u64(0)
        rc = self._score(_ptr(samples), len(samples), nu, _ptr(mu), _ptr(sigma), _ptr(x_max),
                         n, alpha, beta, _ptr(E), _ptr(C), _ptr(S), ctypes.byref(bad),
                         _threads(threads))
        self._check(rc, f"score (request {bad.value})")
        return E, C, S

    def compute_beta(self, adaptive, beta_fixed, beta_max, q_sat, queue_len):
        out = _d(0)
        self._check(self._beta(int(adaptive), beta_fixed, beta_max, q_sat, queue_len,
                               ctypes.byref(out)), "compute_beta")
        return out.value

    def gen_fit_data(self, P, K=16, seed=1, mu_range=(3.0, 5.0), sigma_range=(0.5, 1.2),
                     nu=3.5, integerise=True, threads=None):
        x = np.empty((P, K), np.float64)
        tm = np.empty(P)
        ts = np.empty(P)
        rc = self._gf(P, K, seed, mu_range[0], mu_range[1], sigma_range[0], sigma_range[1], nu,
                      int(integerise), _ptr(x), _ptr(tm), _ptr(ts), _threads(threads))
        self._check(rc, "gen_fit_data")
        return x, tm, ts

    def sample_logt(self, mu, sigma, nu, n, seed):
        out = np.empty(n)
        self._sl(mu, sigma, nu, n, seed, _ptr(out))
        return out

    def logt_loglik(self, x, mu, sigma, nu):
        x = np.ascontiguousarray(x, np.float64)
        return self.logt_loglik_raw(_ptr(x), len(x), mu, sigma, nu)

    def logt_loglik_grad(self, x, mu, sigma, nu):
        f = self._fn("logt_loglik_grad", [_p, _u64, _d, _d, _d, _p], None)
        x = np.ascontiguousarray(x, np.float64)
        g = np.empty(2)
        f(_ptr(x), len(x), mu, sigma, nu, _ptr(g))
        return g


def ref_available():
    return os.path.exists(REF_SO)


class RefLib(_Base):
    """The untouched reference library behind oracle/ref_harness.cpp."""

    prefix = "ref_"

    def __init__(self, path=REF_SO):
        self.lib = ctypes.CDLL(path)
        self._err = self._fn("last_error", [], ctypes.c_char_p)
        self._mc = self._fn("mc_samples", [_d, _i32, _u64, _p])
        self.t_cdf = self._fn("t_cdf", [_d, _d], _d)
        self.t_pdf = self._fn("t_pdf", [_d, _d], _d)
        self.t_quantile = self._fn("t_quantile", [_d, _d], _d)
        self.mix64 = self._fn("mix64", [_u64, _u64], _u64)
        self.hw_threads = self._fn("hw_threads", [], _i32)
        self._score = self._fn("score", [_p, _p, _p, _u64, _d, _i32, _u64, _d, _d, _p, _p, _p,
                                         _i32])
        self.compute_beta_raw = self._fn("compute_beta", [_i32, _d, _d, _d, _u64], _d)
        self._rank = self._fn("rank", [_p, _p, _u64, _p])
        self._fit = self._fn("fit", [_p, _u64, _u64, _d, _p, _p, _p, _p, _p, _p, _i32])
        self._report = self._fn("fit_report", [_p, _u64, _u64, _d, ctypes.c_uint, _p, _p,
                                               _i32])
        self.logt_loglik_raw = self._fn("logt_loglik", [_p, _u64, _d, _d, _d], _d)
        self._gw = self._fn("gen_workload", [_u64, _u64, _d, _d, _d, _d, _d, ctypes.c_uint32,
                                             _d, _p, _p, _p, _p, _p, _p])
        self._gf = self._fn("gen_fit_data", [_u64, _u64, _u64, _d, _d, _d, _d, _d, _i32, _p,
                                             _p, _p])
        self._sched = self._fn("scheduler_script", [_i32, _i32, _d, _d, _d, _d, _u64, _p, _p,
                                                    _p, _p, _p, ctypes.POINTER(_u64)])

    def score(self, mu, sigma, x_max, alpha=0.9, beta=0.5, nu=3.5, mc_n=10000, mc_seed=12,
              threads=None):
        mu = np.ascontiguousarray(mu, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        x_max = np.ascontiguousarray(x_max, np.float64)
        n = len(mu)
        E = np.empty(n)
        C = np.empty(n)
        S = np.empty(n)
        rc = self._score(_ptr(mu), _ptr(sigma), _ptr(x_max), n, nu, mc_n, mc_seed, alpha, beta,
                         _ptr(E), _ptr(C), _ptr(S), _threads(threads))
        self._check(rc, "score")
        return E, C, S

    def gen_fit_data(self, P, K=16, seed=1, mu_range=(3.0, 5.0), sigma_range=(0.5, 1.2),
                     nu=3.5, integerise=True):
        x = np.empty((P, K), np.float64)
        tm = np.empty(P)
        ts = np.empty(P)
        rc = self._gf(P, K, seed, mu_range[0], mu_range[1], sigma_range[0], sigma_range[1], nu,
                      int(integerise), _ptr(x), _ptr(tm), _ptr(ts))
        self._check(rc, "gen_fit_data")
        return x, tm, ts

    def logt_loglik(self, x, mu, sigma, nu):
        x = np.ascontiguousarray(x, np.float64)
        return self.logt_loglik_raw(_ptr(x), len(x), mu, sigma, nu)

    def logt_loglik_grad(self, x, mu, sigma, nu):
        f = self._fn("logt_loglik_grad", [_p, _u64, _d, _d, _d, _p], None)
        x = np.ascontiguousarray(x, np.float64)
        g = np.empty(2)
        f(_ptr(x), len(x), mu, sigma, nu, _ptr(g))
        return g

    def sim_scores(self, mu, sigma, ids, max_tokens, predictor=0, mu_sd=0.0, ls_sd=0.0,
                   seed=0, family=0, alpha=0.9, threads=None):
        f = self._fn("sim_scores", [_p, _p, _p, _p, _u64, _i32, _d, _d, _u64, _i32, _d, _p, _p,
                                    _i32])
        mu = np.ascontiguousarray(mu, np.float64)
        sigma = np.ascontiguousarray(sigma, np.float64)
        ids = np.ascontiguousarray(ids, np.uint64)
        mt = np.ascontiguousarray(max_tokens, np.uint32)
        E, C = np.empty(len(mu)), np.empty(len(mu))
        self._check(f(_ptr(mu), _ptr(sigma), _ptr(ids), _ptr(mt), len(mu), predictor, mu_sd,
                      ls_sd, seed, family, alpha, _ptr(E), _ptr(C), _threads(threads)),
                    "sim_scores")
        return E, C

    def scheduler_script(self, policy, ops, ids, a, b, adaptive=True, beta_fixed=0.1,
                         beta_max=0.5, q_sat=128.0, rebuild_threshold=0.1):
        ops = np.ascontiguousarray(ops, np.int32)
        ids = np.ascontiguousarray(ids, np.uint64)
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        out = np.empty(len(ops), np.uint64)
        n_out = _u64(0)
        rc = self._sched(policy, int(adaptive), beta_fixed, beta_max, q_sat, rebuild_threshold,
                         len(ops), _ptr(ops), _ptr(ids), _ptr(a), _ptr(b), _ptr(out),
                         ctypes.byref(n_out))
        self._check(rc, "scheduler_script")
        return out[: n_out.value]


def fnv1a64(buf: bytes) -> str:
    h = 0xCBF29CE484222325
    for byte in buf:
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def fnv1a64_np(arr) -> str:
    """FNV-1a-64 over the raw little-endian bytes of an array (vectorised over 8-byte words
    would change the definition, so this hashes bytes; fine for <= a few MB)."""
    a = np.ascontiguousarray(arr)
    b = a.view(np.uint8)
    h = np.uint64(0xCBF29CE484222325)
    prime = np.uint64(0x100000001B3)
    with np.errstate(over="ignore"):
        for byte in b:
            h = (h ^ np.uint64(byte)) * prime
    return f"{int(h):016x}"


# ---- the reference's per-item API, run_sim and ks_test_fit (oracle/ref_harness.cpp)
EVAL_OPS = {"psi": 1, "regularized_incomplete_beta": 2, "t_pdf": 3, "t_cdf": 4, "logt_pdf": 5,
            "logt_cdf": 6, "normal_cdf": 7, "normal_quantile": 8,
            "lognormal_censored_expectation": 9, "lognormal_censored_cvar": 10}


def ref_eval(R, fn, a, b=None, c=None, param=0.0):
    f = R._fn("eval", [_i32, _p, _p, _p, _u64, _d, _p])
    a = np.ascontiguousarray(a, np.float64)
    b = np.zeros_like(a) if b is None else np.ascontiguousarray(b, np.float64)
    c = np.zeros_like(a) if c is None else np.ascontiguousarray(c, np.float64)
    out = np.empty_like(a)
    R._check(f(EVAL_OPS[fn], _ptr(a), _ptr(b), _ptr(c), len(a), param, _ptr(out)), "eval")
    return out


def ref_ks_test_fit(R, x, family, mu=0.0, sigma=0.0, nu=0.0, rate=0.0):
    f = R._fn("ks_test_fit", [_p, _u64, _i32, _d, _d, _d, _d, _p, _p])
    x = np.ascontiguousarray(x, np.float64)
    st, p = ctypes.c_double(), ctypes.c_double()
    R._check(f(_ptr(x), len(x), family, mu, sigma, nu, rate, ctypes.byref(st), ctypes.byref(p)),
             "ks_test_fit")
    return st.value, p.value


# canonical.json (proj/configs/canonical.json:1-29) as run_sim arguments
CANONICAL = dict(n=8000, rps=100.0, mu_range=(0.1, 2.7), sigma_range=(0.4, 1.2),
                 prompt_range=(16, 128), max_tokens=512, alpha=0.9, adaptive=True,
                 beta_fixed=0.1, beta_max=0.5, q_sat=128.0, threshold=0.1, slots=8, c0=0.02,
                 c1=0.002, c2=1e-4, kind=1, family=0, mu_sd=0.0, ls_sd=0.0, batched=True)


def ref_run_sim(R, wseed, policy, seed, **kw):
    """run_sim of the reference on gen_logt_workload(spec, wseed): per-event arrays (id order),
    metrics (ttft_avg, ttft_p90, ptla_avg, ptla_p90) and run_sim's own wall seconds."""
    a = dict(CANONICAL)
    a.update(kw)
    f = R._fn("run_sim", [_u64, _d, _d, _d, _d, _d, ctypes.c_uint32, ctypes.c_uint32,
                          ctypes.c_uint32, _u64, _i32, _d, _i32, _d, _d, _d, _d, _i32, _d, _d,
                          _d, _i32, _i32, _d, _d, _i32, _u64] + [_p] * 8)
    n = a["n"]
    ev = {k: np.empty(n) for k in ("arrival_s", "predict_ready_s", "admit_s", "first_token_s",
                                   "completion_s")}
    emitted = np.empty(n, np.uint32)
    metrics = np.empty(4)
    secs = ctypes.c_double()
    rc = f(n, a["rps"], a["mu_range"][0], a["mu_range"][1], a["sigma_range"][0],
           a["sigma_range"][1], a["prompt_range"][0], a["prompt_range"][1], a["max_tokens"],
           wseed, policy, a["alpha"], int(a["adaptive"]), a["beta_fixed"], a["beta_max"],
           a["q_sat"], a["threshold"], a["slots"], a["c0"], a["c1"], a["c2"], a["kind"],
           a["family"], a["mu_sd"], a["ls_sd"], int(a["batched"]), seed,
           _ptr(ev["arrival_s"]), _ptr(ev["predict_ready_s"]), _ptr(ev["admit_s"]),
           _ptr(ev["first_token_s"]), _ptr(ev["completion_s"]), _ptr(emitted), _ptr(metrics),
           ctypes.byref(secs))
    R._check(rc, "run_sim")
    ev["emitted_tokens"] = emitted
    return ev, metrics, secs.value
