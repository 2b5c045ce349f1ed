"""GPU parity: K1 score (moment-table and exact paths) against the oracle and the reference's
golden fixtures, through the C-ABI.

Tolerances: the north star's bar is 1e-6 relative for E / CVaR / score.  Both device paths
are held to 1e-12 here (they agree with the reference to ~1e-15), and
case-1 CVaR cells must equal x_max bit-for-bit."""
import numpy as np
import pytest

from cabi import TIE_SCORE_EXACT, TIE_SCORE_MOMENT, TIE_SCORE_RAW, CAbi, TieError, rel_err
from conftest import golden

pytestmark = pytest.mark.gpu

TOL = 1e-12     # held by both paths on well-conditioned cells
TOL_ILL = 1e-10 # CVaR at alpha=0.99 / tiny sigma: psi(y_max) - psi(y_alpha) cancels ~100x
BAR = 1e-6      # the north star's stated tolerance
MODES = [TIE_SCORE_MOMENT, TIE_SCORE_EXACT]


@pytest.fixture(scope="module")
def abi():
    return CAbi()


@pytest.fixture(scope="module")
def h(abi):
    ctx = abi.ctx()
    yield ctx
    abi.destroy(ctx)


@pytest.mark.parametrize("flags", MODES)
def test_grid27(abi, h, flags):
    g = golden("grid27.npz")
    E, C, S = abi.score(h, g["mu"], g["sigma"], g["x_max"], 0.9, 0.5, flags)
    for got, ref in ((E, g["E"]), (C, g["C"]), (S, g["S"])):
        assert rel_err(got, ref).max() <= TOL
    sat = g["C"] == g["x_max"]
    assert sat.any() and np.array_equal(C[sat], g["x_max"][sat])  # case 1: bit-exact x_max
    E0, C0, _ = abi.score(h, g["mu"], g["sigma"], g["x_max"], 0.0, 0.3, flags)
    assert np.array_equal(E0, C0)  # cvar(0) == E
    assert rel_err(E0, g["E_a0"]).max() <= TOL


@pytest.mark.parametrize("flags", MODES)
def test_edge_cells(abi, h, flags):
    g = golden("edges.npz")
    E, C, S = abi.score(h, g["mu"], g["sigma"], g["x_max"], 0.9, 0.5, flags)
    for got, ref in ((E, g["E"]), (C, g["C"]), (S, g["S"])):
        assert rel_err(got, ref).max() <= TOL, rel_err(got, ref)
    sat = g["C"] == g["x_max"]
    assert np.array_equal(C[sat], g["x_max"][sat])


@pytest.mark.parametrize("flags", MODES)
def test_config1_scores_and_order(abi, h, flags):
    g = golden("config1.npz")
    S, order = abi.score_rank(h, g["mu"], g["sigma"], g["max_tokens"], 0.9, 0.5, flags)
    assert rel_err(S, g["S"]).max() <= TOL
    assert np.array_equal(order, g["order"])  # bit-exact dispatch order
    assert order[:8].tolist() == [25, 142, 172, 568, 266, 840, 699, 270]


@pytest.mark.parametrize("flags", MODES)
def test_config2_full_order_bit_exact(abi, h, oracle, flags):
    """Config 2: the 1M-request queue's complete dispatch order equals the reference's
    (WaitingQueue pop order, sha256 of the u64 id sequence in tests/golden/golden.json)."""
    import hashlib

    g = golden("golden.json")["config2"]
    mu, sg, mt = oracle.gen_workload(1_000_000, seed=1)
    S, order = abi.score_rank(h, mu, sg, mt, 0.9, 0.5, flags)
    assert hashlib.sha256(order.tobytes()).hexdigest() == g["sha256_order"]
    smp = golden("config2_sample.npz")
    assert rel_err(S[smp["idx"]], smp["S"]).max() <= TOL
    assert np.array_equal(order[:4096], smp["order_head"])


def test_canonical_config_queue(abi, h):
    g = golden("canonical20k.npz")
    from oracle_lib import Oracle

    mu, sg, mt = Oracle().gen_workload(20000, seed=1, mu_range=(0.1, 2.7),
                                       sigma_range=(0.4, 1.2), max_tokens=512)
    E, C, S = abi.score(h, mu, sg, mt.astype(float), 0.9, 0.5)
    assert rel_err(E, g["E"]).max() <= TOL and rel_err(C, g["C"]).max() <= TOL
    _, order = abi.score_rank(h, mu, sg, mt, 0.9, 0.5)
    assert np.array_equal(order, g["order"])


@pytest.mark.parametrize("flags", MODES)
def test_random_wide_ranges_vs_oracle(abi, h, oracle, samples, flags):
    rng = np.random.default_rng(2026 + flags)
    n = 40000 if flags == TIE_SCORE_EXACT else 200000
    mu = rng.uniform(-2.0, 9.0, n)
    sg = np.exp(rng.uniform(np.log(1e-3), np.log(6.0), n))  # spans the table edge (4.0)
    xm = np.floor(np.exp(rng.uniform(0.0, 12.0, n))) + 1.0
    for alpha, beta in [(0.9, 0.5), (0.5, 0.1), (0.0, 0.7), (0.99, 2.0)]:
        Eo, Co, So = oracle.score(samples, mu, sg, xm, alpha=alpha, beta=beta)
        E, C, S = abi.score(h, mu, sg, xm, alpha, beta, flags)
        tol = TOL_ILL if alpha >= 0.99 else TOL
        for got, ref in ((E, Eo), (C, Co), (S, So)):
            err = rel_err(got, ref)
            assert err.max() <= tol, (alpha, beta, err.max(), int(err.argmax()))
        sat = Co == xm
        assert np.array_equal(C[sat], xm[sat])


def test_per_item_raw_semantics(abi, h, oracle, samples):
    """censored_expectation / censored_cvar per item (no max, no compute_score checks)."""
    mu = np.array([4.0, 4.0, 2.0])
    sg = np.array([0.8, 0.8, 1e-12])
    xm = np.array([512.0, np.exp(4.0), 64.0])
    E, C, _ = abi.score(h, mu, sg, xm, 0.9, 0.0, TIE_SCORE_RAW)
    Eo, Co, _ = oracle.score(samples, mu, sg, xm, alpha=0.9, beta=0.0)
    assert rel_err(E, Eo).max() <= TOL
    assert C[1] == np.exp(4.0)  # case 1 exactly (test_dist.cpp:218-219)
    assert abs(C[0] - 353.8733877) / 353.8733877 < 0.02  # frozen brute force (test_dist.cpp:228)


def test_validation_errors(abi, h):
    good = np.array([4.0, 4.0]), np.array([0.8, 0.8]), np.array([512.0, 512.0])
    for which, bad, msg in [(0, np.nan, "mu must be finite"), (1, -1.0, "sigma"),
                            (1, 0.0, "sigma"), (2, 0.0, "x_max"), (2, np.inf, "x_max")]:
        args = [a.copy() for a in good]
        args[which][1] = bad
        with pytest.raises(TieError) as ei:
            abi.score(h, *args)
        assert ei.value.code == 1 and msg in str(ei.value) and "item 1" in str(ei.value)
    with pytest.raises(TieError) as ei:
        abi.score(h, *good, alpha=1.0)
    assert "alpha" in str(ei.value)
    E, C, S = abi.score(h, *good)  # the context recovers after an error
    assert np.all(np.isfinite(S))


def test_expectation_nonpositive_is_domain_error(abi, h):
    # every included term underflows and the censor mass is 0 -> E == 0 -> compute_score throws
    with pytest.raises(TieError) as ei:
        abi.score(h, np.array([3.0, -800.0]), np.array([0.5, 0.01]), np.array([64.0, 1.0]))
    assert ei.value.code == 1 and "expectation must be > 0" in str(ei.value)
    assert "item 1" in str(ei.value)


def test_other_sample_sets(abi, oracle):
    """A context built from a caller-provided McContext (different nu / N / seed)."""
    for nu, n, seed in [(1.5, 3000, 5), (8.0, 20000, 9), (3.5, 1, 1)]:
        Y = oracle.mc_samples(nu, n, seed)
        h2 = abi.ctx(Y, nu=nu)
        try:
            rng = np.random.default_rng(seed)
            mu = rng.uniform(1, 6, 5000)
            sg = rng.uniform(0.1, 2.0, 5000)
            xm = np.full(5000, 1024.0)
            Eo, Co, So = oracle.score(Y, mu, sg, xm, alpha=0.9, beta=0.5, nu=nu)
            for flags in MODES:
                E, C, S = abi.score(h2, mu, sg, xm, 0.9, 0.5, flags)
                assert rel_err(S, So).max() <= TOL, (nu, n, flags)
        finally:
            abi.destroy(h2)


def test_sigma_table_boundary(abi, oracle, samples):
    """sigma just inside / outside the moment table (default 4.0) and a tiny table."""
    h2 = abi.ctx(samples, sigma_table_max=0.5)
    try:
        sg = np.array([0.49, 0.5, 0.5156, 0.52, 3.99, 4.0, 4.01, 1e-9, 1e-5])
        mu = np.full(len(sg), 3.0)
        xm = np.full(len(sg), 2048.0)
        Eo, Co, So = oracle.score(samples, mu, sg, xm, alpha=0.9, beta=0.5)
        E, C, S = abi.score(h2, mu, sg, xm, 0.9, 0.5)
        assert rel_err(S, So).max() <= TOL
    finally:
        abi.destroy(h2)


@pytest.mark.parametrize("n", [1000, 300_001, 1_000_000, 2_500_003])
def test_host_call_pinned_zero_copy_equals_pageable(tie, mc, n):
    """tie_score_rank_host on pinned buffers (the score kernel reads the inputs and the sort
    writes the order through UVA-mapped host memory) == the same call on pageable NumPy
    buffers (staged copies), scores and order bitwise; plus the error path (a bad request is
    reported with its index from the zero-copy kernel)"""
    import torch

    w = tie.gen_logt_workload_soa(n, 5)
    mu, sg, mt = w["mu"].copy(), w["sigma"].copy(), w["max_tokens"].copy()
    pin = lambda a: torch.from_numpy(a).pin_memory()
    mu_p, sg_p, mt_p = pin(mu), pin(sg), pin(mt.view(np.int32))
    s_p = torch.empty(n, dtype=torch.float64).pin_memory()
    o_p = torch.empty(n, dtype=torch.int64).pin_memory()
    tie.score_rank_host_ptr(mc.handle, mu_p.data_ptr(), sg_p.data_ptr(), mt_p.data_ptr(), n,
                            0.9, 0.5, s_p.data_ptr(), o_p.data_ptr(), 0)
    s_h = np.empty(n)
    o_h = np.empty(n, np.uint64)
    tie.score_rank_host_ptr(mc.handle, mu.ctypes.data, sg.ctypes.data, mt.ctypes.data, n, 0.9,
                            0.5, s_h.ctypes.data, o_h.ctypes.data, 0)
    assert np.array_equal(s_p.numpy().view(np.uint64), s_h.view(np.uint64))
    assert np.array_equal(o_p.numpy().view(np.uint64), o_h)
    # pinned inputs with a pageable order (staged output only), and the reverse
    o_h2 = np.empty(n, np.uint64)
    tie.score_rank_host_ptr(mc.handle, mu_p.data_ptr(), sg_p.data_ptr(), mt_p.data_ptr(), n,
                            0.9, 0.5, 0, o_h2.ctypes.data, 0)
    assert np.array_equal(o_h2, o_h)
    o_p2 = torch.zeros(n, dtype=torch.int64).pin_memory()
    tie.score_rank_host_ptr(mc.handle, mu.ctypes.data, sg.ctypes.data, mt.ctypes.data, n, 0.9,
                            0.5, 0, o_p2.data_ptr(), 0)
    assert np.array_equal(o_p2.numpy().view(np.uint64), o_h)
    bad = sg.copy()
    bad[n // 3] = -1.0  # the staged (pageable) inputs report the same item index
    with pytest.raises(ValueError, match=f"item {n // 3}"):
        tie.score_rank_host_ptr(mc.handle, mu.ctypes.data, bad.ctypes.data, mt.ctypes.data, n,
                                0.9, 0.5, 0, o_h2.ctypes.data, 0)
    with pytest.raises(ValueError, match="null pointer"):  # not a crash in the staging copies
        tie.score_rank_host_ptr(mc.handle, mu.ctypes.data, 0, mt.ctypes.data, n, 0.9, 0.5, 0,
                                o_h2.ctypes.data, 0)
    sg_p[n // 2] = -1.0  # LogTParams: sigma must be finite and > 0
    with pytest.raises(ValueError, match=f"item {n // 2}"):
        tie.score_rank_host_ptr(mc.handle, mu_p.data_ptr(), sg_p.data_ptr(), mt_p.data_ptr(),
                                n, 0.9, 0.5, s_p.data_ptr(), o_p.data_ptr(), 0)
