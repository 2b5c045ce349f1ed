"""CPU: the drop-in boundary itself -- libtie_b200.so loads, exports every entry point that
include/tie_cuda.h declares, the host-side helpers match the reference, and the device path
fails loudly (never silently on the CPU) when no GPU is present."""
import ctypes
import math

import numpy as np
import pytest
import torch

from cabi import LIB, CAbi, TieError, header_symbols


def test_header_symbols_exported():
    lib = ctypes.CDLL(LIB)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_host_helpers_match_reference(oracle):
    abi = CAbi()
    L = abi.lib
    assert L.tie_t_quantile(0.9, 3.5) == oracle.t_quantile(0.9, 3.5)
    b = ctypes.c_double()
    for adaptive, q in [(1, 0), (1, 64), (1, 128), (1, 10**6), (0, 5)]:
        assert L.tie_compute_beta(adaptive, 0.1, 0.5, 128.0, q, ctypes.byref(b)) == 0
        assert b.value == oracle.compute_beta(adaptive, 0.1, 0.5, 128.0, q)
    assert L.tie_compute_beta(0, -0.1, 0.5, 128.0, 1, ctypes.byref(b)) == 1  # domain_error
    assert L.tie_compute_beta(1, 0.1, 0.5, 0.0, 1, ctypes.byref(b)) == 1


def test_pybind_surface_mirrors_reference(tie):
    # the names the reference's tiesched module exposes on this path (module.cpp:22-83,171-172)
    for name in ["LogTParams", "CensoredLogT", "McContext", "t_pdf", "t_cdf", "t_quantile",
                 "sample_logt", "censored_expectation", "censored_cvar", "FitFamily",
                 "FitResult", "logt_loglik", "logt_loglik_grad", "fit_logt_fixed_nu", "Policy",
                 "BetaMode", "ScoreConfig", "compute_beta", "compute_score"]:
        assert hasattr(tie, name), name
    p = tie.LogTParams(1.0, 1e-12, 3.5)
    assert p.sigma == 1e-9 and p.sigma_clamped
    with pytest.raises(ValueError):
        tie.LogTParams(0.0, -1.0, 3.5)
    with pytest.raises(ValueError):
        tie.CensoredLogT(tie.LogTParams(4.0, 0.8, 3.5), 0.0)
    assert tie.compute_score(100.0, 400.0, 0.3) == pytest.approx(220.0, rel=1e-15)
    with pytest.raises(ValueError):
        tie.compute_score(200.0, 100.0, 0.3)
    cfg = tie.ScoreConfig()
    assert cfg.alpha == 0.9 and cfg.beta_max == 0.5 and cfg.q_sat == 128.0
    assert tie.compute_beta(cfg, 64) == pytest.approx(0.25, rel=1e-15)
    assert math.isclose(tie.t_cdf(tie.t_quantile(0.9, 3.5), 3.5), 0.9, abs_tol=1e-10)


def test_workload_generator_matches_reference(tie, oracle):
    w = tie.gen_logt_workload_soa(5000, 1)
    mu, sg, mt, arr, pt, tl = oracle.gen_workload(5000, seed=1, extras=True)
    for a, b in [(w["mu"], mu), (w["sigma"], sg), (w["max_tokens"], mt), (w["arrival_s"], arr),
                 (w["prompt_tokens"], pt), (w["true_output_tokens"], tl)]:
        assert np.array_equal(a, b)
    x, tm, ts = tie.gen_fit_data(500, 16, 3)
    xo, tmo, tso = oracle.gen_fit_data(500, 16, seed=3)
    assert np.array_equal(x, xo) and np.array_equal(tm, tmo)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_gpu_fails_loudly(tie):
    abi = CAbi()
    with pytest.raises(TieError) as ei:
        abi.ctx()
    assert ei.value.code == 3 and "no CUDA device" in str(ei.value)
    with pytest.raises(RuntimeError):
        tie.McContext(3.5)
