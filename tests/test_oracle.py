"""CPU: pin the oracle (oracle/tie_oracle.c) against the reference's golden fixtures
(tests/golden/, generated from the compiled reference) and, where it is built here, against
the reference library itself (oracle/_ref)."""
import numpy as np
import pytest

from conftest import golden
from oracle_lib import RefLib, fnv1a64_np, ref_available

G = golden("golden.json")


def fromhex(s):
    return float.fromhex(s)


def test_mc_samples_hash(oracle):
    Y = oracle.mc_samples(3.5, 10000, 12)
    assert fnv1a64_np(Y) == G["mc_3.5_10000_12"]["fnv"]
    assert Y.min() == fromhex(G["mc_3.5_10000_12"]["min"])
    assert Y.max() == fromhex(G["mc_3.5_10000_12"]["max"])
    assert fnv1a64_np(oracle.mc_samples(3.5, 1000, 5)) == G["mc_3.5_1000_5"]["fnv"]
    assert np.all(np.diff(Y) >= 0)


def test_student_t_known_answers(oracle):
    for y, nu, v in G["t_cdf"]:
        assert oracle.t_cdf(y, nu) == fromhex(v), (y, nu)
    for p, nu, v in G["t_quantile"]:
        assert oracle.t_quantile(p, nu) == fromhex(v), (p, nu)
    # reference unit-test anchors (test_dist.cpp:31-70)
    assert oracle.t_cdf(0.0, 3.5) == 0.5
    assert abs(oracle.t_cdf(oracle.t_quantile(0.9, 3.5), 3.5) - 0.9) <= 1e-10


def test_grid27_bit_exact(oracle, samples):
    g = golden("grid27.npz")
    E, C, S = oracle.score(samples, g["mu"], g["sigma"], g["x_max"], alpha=0.9, beta=0.5)
    assert np.array_equal(E, g["E"]) and np.array_equal(C, g["C"]) and np.array_equal(S, g["S"])
    E, C, S = oracle.score(samples, g["mu"], g["sigma"], g["x_max"], alpha=0.0, beta=0.3)
    assert np.array_equal(E, g["E_a0"]) and np.array_equal(C, g["C_a0"])
    # acceptance C03 brute-force table within 2% (acceptance.cpp:90-100)
    kref = np.array([18.6352, 19.1922, 20.5836, 72.8689, 87.3485, 126.403, 188.691, 275.905,
                     543.476, 123.175, 129.639, 138.153, 244.622, 354.130, 550.018, 256.0,
                     512.0, 1460.36, 256.0, 512.0, 917.069, 256.0, 512.0, 1908.20, 256.0,
                     512.0, 2048.0])
    assert np.max(np.abs(g["C"] - kref) / kref) < 0.02


def test_edges_bit_exact(oracle, samples):
    g = golden("edges.npz")
    E, C, S = oracle.score(samples, g["mu"], g["sigma"], g["x_max"], alpha=0.9, beta=0.5)
    assert np.array_equal(E, g["E"]) and np.array_equal(C, g["C"]) and np.array_equal(S, g["S"])


def test_config1_bit_exact(oracle, samples):
    g = golden("config1.npz")
    mu, sg, mt = oracle.gen_workload(1000, seed=1)
    assert np.array_equal(mu, g["mu"]) and np.array_equal(sg, g["sigma"])
    assert np.array_equal(mt, g["max_tokens"])
    E, C, S = oracle.score(samples, mu, sg, mt.astype(float), alpha=0.9, beta=0.5)
    assert np.array_equal(S, g["S"]) and np.array_equal(E, g["E"]) and np.array_equal(C, g["C"])
    order = oracle.rank(S)
    assert np.array_equal(order, g["order"])
    assert order[:8].tolist() == [25, 142, 172, 568, 266, 840, 699, 270]


def test_config2_inputs_and_sample(oracle, samples):
    g = golden("config2_sample.npz")
    mu, sg, mt = oracle.gen_workload(1_000_000, seed=1)
    idx = g["idx"]
    E, C, S = oracle.score(samples, mu[idx], sg[idx], mt[idx].astype(float), alpha=0.9, beta=0.5)
    assert np.array_equal(S, g["S"]) and np.array_equal(E, g["E"])


def test_rank_fixtures(oracle):
    g = golden("rank.npz")
    assert oracle.rank(g["tie_keys"], g["tie_ids"]).tolist() == [0, 2, 4, 7, 9]
    assert np.array_equal(oracle.rank(g["keys"], g["ids"]), g["order_ids"])
    assert np.array_equal(oracle.rank(g["keys"]), g["order_index"])


@pytest.mark.parametrize("name", ["K16", "K5", "K20", "K100", "raw16"])
def test_fit_bit_exact(oracle, name):
    f = golden("fit.npz")
    x = f[f"{name}__x"]
    r = oracle.fit(x)
    for k in ("mu", "sigma", "log_likelihood", "iterations", "converged", "degenerate"):
        assert np.array_equal(np.asarray(r[k]), f[f"{name}__{k}"]), k


def test_fit_data_generator(oracle):
    f = golden("fit.npz")
    x, _, _ = oracle.gen_fit_data(4000, 16, seed=1)
    assert np.array_equal(x, f["K16__x"])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_oracle_vs_reference_library(oracle):
    R = RefLib()
    Y = R.mc_samples()
    mu, sg, mt = R.gen_workload(3000, seed=7, mu_range=(-1.0, 8.0), sigma_range=(0.05, 3.0))
    xm = mt.astype(float)
    for a, b in [(0.9, 0.5), (0.0, 0.2), (0.5, 1.3)]:
        r1 = oracle.score(Y, mu, sg, xm, alpha=a, beta=b)
        r2 = R.score(mu, sg, xm, alpha=a, beta=b)
        for u, v in zip(r1, r2):
            assert np.array_equal(u, v)
    x, _, _ = R.gen_fit_data(3000, 12, seed=11, integerise=False)
    r1, r2 = oracle.fit(x), R.fit(x)
    for k in r1:
        assert np.array_equal(r1[k], r2[k]), k


# ---------------------------------------------------------------- scheduler (sched.cpp)
def _drift_script(threshold):
    """test_sched.cpp:245-292: q_sat=4, predictions at q=4 (beta .5), the pop drops beta to
    .375 -> drift .125: with threshold .1 the rebuild surfaces X (id 1), with .2 Y (id 2)."""
    ops = [0, 0, 0, 0, 1, 1, 1, 2, 2, 2, 2]
    ids = [0, 1, 2, 3, 0, 1, 2, 0, 0, 0, 0]
    a = [0.0, 0.1, 0.2, 0.30000000000000004, 5.0, 100.0, 671.0, 0, 0, 0, 0]
    b = [2048, 2048, 2048, 2048, 10.0, 2000.0, 671.0, 0, 0, 0, 0]
    return ops, ids, a, b, dict(adaptive=True, beta_max=0.5, q_sat=4.0,
                                rebuild_threshold=threshold)


def test_scheduler_reference_scenarios(oracle):
    ops, ids, a, b, cfg = _drift_script(0.1)
    assert oracle.scheduler_script(2, ops, ids, a, b, **cfg).tolist()[:2] == [0, 1]
    ops, ids, a, b, cfg = _drift_script(0.2)
    assert oracle.scheduler_script(2, ops, ids, a, b, **cfg).tolist()[:2] == [0, 2]
    # FCFS ignores predictions; equal max_tokens pop by id (test_sched.cpp:199-243)
    out = oracle.scheduler_script(0, [0, 0, 1, 2, 2, 2], [5, 3, 5, 0, 0, 0],
                                  [1.0, 2.0, 5000.0, 0, 0, 0], [2048, 2048, 6000.0, 0, 0, 0],
                                  adaptive=False, beta_fixed=0.3)
    assert out.tolist() == [5, 3, np.iinfo(np.uint64).max]
    out = oracle.scheduler_script(2, [0, 0, 2], [9, 4, 0], [0.0, 0.1, 0], [1024, 1024, 0],
                                  adaptive=False, beta_fixed=0.3)
    assert out.tolist() == [4]


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("policy,thr", [(2, 0.1), (2, 0.0), (2, 0.2), (1, 0.1), (0, 0.1)])
def test_scheduler_oracle_vs_reference(oracle, policy, thr):
    from sched_scripts import make_script

    R = RefLib()
    cfg = dict(adaptive=True, beta_max=0.5, q_sat=64.0, rebuild_threshold=thr)
    for seed in range(4):
        ops, ids, a, b = make_script(seed, oracle, policy=policy, **cfg)
        got = oracle.scheduler_script(policy, ops, ids, a, b, **cfg)
        ref = R.scheduler_script(policy, ops, ids, a, b, **cfg)
        assert np.array_equal(got, ref), (policy, thr, seed)
        assert len(got) > 50


# ---------------------------------------------------------------- run_sim scoring chain
@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
@pytest.mark.parametrize("predictor,family", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_sim_scores_oracle_vs_reference(oracle, predictor, family):
    R = RefLib()
    mu, sg, mt = oracle.gen_workload(3000, seed=5, mu_range=(0.1, 2.7), sigma_range=(0.4, 1.2),
                                     max_tokens=512)
    ids = np.arange(3000, dtype=np.uint64) * 3 + 1
    kw = dict(predictor=predictor, mu_sd=0.4, ls_sd=0.3, seed=11, family=family, alpha=0.9)
    E1, C1 = oracle.sim_scores(mu, sg, ids, mt, **kw)
    E2, C2 = R.sim_scores(mu, sg, ids, mt, **kw)
    assert np.array_equal(E1, E2) and np.array_equal(C1, C2)


# ---------------------------------------------------------------- cmd_fit analysis (8f #3)
FR_SETS = ("K16", "K5", "K12c", "K100", "degen")


@pytest.mark.parametrize("name", FR_SETS)
def test_fit_report_bit_exact(oracle, name):
    """The restatement of cmd_fit's per-prompt analysis (four families, KS, tail stats)
    equals the reference's fixtures bit for bit."""
    g = golden("fit_report.npz")
    fits, tail = oracle.fit_report_raw(g[f"{name}__x"])
    np.testing.assert_array_equal(fits, g[f"{name}__fits"])
    np.testing.assert_array_equal(tail, g[f"{name}__tail"])


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_fit_report_oracle_vs_reference_library(oracle):
    R = RefLib()
    x, _, _ = R.gen_fit_data(400, 20, seed=21)
    for fam, nu in [(15, 3.5), (1, 2.0), (6, 3.5)]:
        a, b = oracle.fit_report_raw(x, nu, fam), R.fit_report_raw(x, nu, fam)
        np.testing.assert_array_equal(a[0], b[0])
        np.testing.assert_array_equal(a[1], b[1])
    with pytest.raises(ValueError, match="at least 5"):
        oracle.fit_report_raw(x[:, :4])


def test_loglik_grad_bit_exact(oracle):
    """F2/F3 restatement vs the reference's own logt_loglik / logt_loglik_grad values."""
    g = golden("loglik.npz")
    for K in (1, 16, 60, 1000):
        x, mu, sg = g[f"K{K}__x"], g[f"K{K}__mu"], g[f"K{K}__sigma"]
        ll = np.array([oracle.logt_loglik(x, m, s, 3.5) for m, s in zip(mu, sg)])
        gr = np.array([oracle.logt_loglik_grad(x, m, s, 3.5) for m, s in zip(mu, sg)])
        assert np.array_equal(ll, g[f"K{K}__ll"]), K
        assert np.array_equal(gr, g[f"K{K}__grad"]), K
