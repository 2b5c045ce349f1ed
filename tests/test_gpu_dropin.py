"""GPU parity of the drop-in API surface beyond score/rank/fit (VERDICT r1 "What's missing" #1,
#2, #5, #6):

* the per-item distribution functions (psi, regularized_incomplete_beta, logt_pdf / logt_cdf,
  normal_cdf / normal_quantile, lognormal_censored_*; dist.hpp:47-88, module.cpp:48-60) on the
  GPU against the reference's own functions (oracle/_ref) on grids, plus their errors;
* ks_test_fit (module.cpp:117-123) against the reference;
* the Python WaitingQueue / Scheduler classes (sched.hpp:43-90);
* the reference's own Python smoke tests (proj/tests/python/test_smoke.py:8-62) restated
  against paper_2604_00499_b200 -- tests 1, 2, 3, 5 and 6 (test 4, the tail-law estimator,
  is SURVEY.md sec. 2 row 5, out of scope);
* run_sim (sim.cpp:39-185, module.cpp:269-271) event-for-event against the reference's
  run_sim: BASELINE config 5 (canonical.json, seeds 1..10, rebuild_threshold 0) and the
  policy / predictor / family / batching variants.
"""
import math

import zlib

import numpy as np
import pytest

from conftest import golden
from oracle_lib import RefLib, ref_available, ref_eval, ref_ks_test_fit, ref_run_sim, CANONICAL

pytestmark = pytest.mark.gpu
needs_ref = pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def R():
    return RefLib()


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return np.abs(a - b) / np.maximum(np.abs(b), 1e-300)


# ---------------------------------------------------------------- per-item functions
@needs_ref
def test_psi_matches_reference(tie, mc, R):
    rng = np.random.default_rng(3)
    n = 400
    y = np.concatenate([rng.uniform(-16, 19, n - 4), [-20.0, 20.0, -np.inf, np.inf]])
    mu = rng.uniform(-1, 7, n)
    sg = np.concatenate([rng.uniform(0.05, 2.5, n - 2), [1e-12, 3.0]])
    got = tie.dist_eval("psi", y, mu, sg, 3.5, mc)
    ref = ref_eval(R, "psi", y, mu, sg, 3.5)
    assert rel(got, ref).max() <= 1e-13
    # per-item form and the censored-moment identity E = Psi(y_max) + x_max (1 - T(y_max))
    p = tie.LogTParams(4.0, 0.8, 3.5)
    ym = (math.log(512.0) - 4.0) / 0.8
    e = tie.censored_expectation(tie.CensoredLogT(p, 512.0), mc)
    assert abs(tie.psi(ym, p, mc) + 512.0 * (1 - tie.t_cdf(ym, 3.5)) - e) <= 1e-12 * e


def _dist_inputs(fn, rng, n=2000):
    """the inputs of one dist-function parity case (the reference's valid domains)"""
    if fn == "regularized_incomplete_beta":
        a, b, c = rng.uniform(0.05, 30, n), rng.uniform(0.05, 30, n), rng.uniform(0, 1, n)
        c[:3] = [0.0, 1.0, 0.5]
    elif fn in ("t_pdf", "t_cdf"):
        a, b, c = rng.uniform(-40, 40, n), None, None
    elif fn.startswith("logt"):
        a, b, c = np.exp(rng.uniform(-3, 12, n)), rng.uniform(-1, 8, n), rng.uniform(1e-3, 3, n)
    elif fn == "normal_cdf":
        a, b, c = rng.uniform(-12, 12, n), None, None
    elif fn == "normal_quantile":
        a, b, c = np.concatenate([rng.uniform(0, 1, n - 4), [1e-300, 0.01, 0.99, 1 - 1e-16]]), None, None
    else:
        a, b, c = rng.uniform(-1, 8, n), rng.uniform(0.05, 3, n), rng.uniform(1, 4096, n)
    return a, b, c


def _dist_err(fn, got, ref):
    """relative error; absolute where the reference underflows.  normal_quantile is measured
    against max(|x|, 1): near p = 1/2 the quantile is ~0 and its last-ulp difference (device
    vs glibc erfc in the Newton step, dist.cpp:193-225) is an absolute ~1e-16"""
    scale = np.maximum(np.abs(ref), 1.0) if fn == "normal_quantile" else np.abs(ref)
    return np.where(np.abs(ref) < 1e-280, np.abs(got - ref),
                    np.abs(got - ref) / np.maximum(scale, 1e-300))


@needs_ref
@pytest.mark.parametrize("fn,nargs,param", [
    ("regularized_incomplete_beta", 3, 0.0), ("t_pdf", 1, 3.5), ("t_cdf", 1, 2.5),
    ("logt_pdf", 3, 3.5), ("logt_cdf", 3, 1.5), ("normal_cdf", 1, 0.0),
    ("normal_quantile", 1, 0.0), ("lognormal_censored_expectation", 3, 0.0),
    ("lognormal_censored_cvar", 3, 0.9), ("lognormal_censored_cvar", 3, 0.0)])
def test_dist_functions_match_reference(tie, R, fn, nargs, param):
    # a fixed seed per function (hash(str) is salted per process: inputs must not vary run
    # to run)
    a, b, c = _dist_inputs(fn, np.random.default_rng(zlib.crc32(fn.encode()) % 1000))
    got = tie.dist_eval(fn, a, b, c, param)
    ref = ref_eval(R, fn, a, b, c, param)
    # device vs glibc libm (lgamma / exp / log / erfc): a few ulp, amplified by cancellation in
    # 1 - F near F -> 1; the north star's bar is 1e-6 (worst over 100 input seeds:
    # tools/dist_eval_probe.py)
    tol = 1e-9 if fn in ("regularized_incomplete_beta", "t_cdf", "logt_cdf", "normal_cdf") else 1e-12
    err = _dist_err(fn, got, ref)
    assert err.max() <= tol, (fn, float(err.max()), int(err.argmax()))


def test_dist_function_errors(tie, mc):
    with pytest.raises(ValueError, match="x must lie in"):
        tie.regularized_incomplete_beta(1.0, 1.0, 1.5)
    with pytest.raises(ValueError, match="a and b must be finite"):
        tie.regularized_incomplete_beta(0.0, 1.0, 0.5)
    with pytest.raises(ValueError, match="logt_cdf: x must be finite and > 0"):
        tie.logt_cdf(0.0, tie.LogTParams(1.0, 1.0, 3.5))
    with pytest.raises(ValueError, match="normal_quantile: p must lie in"):
        tie.normal_quantile(1.0)
    with pytest.raises(ValueError, match="psi: McContext nu does not match"):
        tie.psi(1.0, tie.LogTParams(1.0, 1.0, 2.5), mc)
    with pytest.raises(ValueError, match="lognormal_censored_cvar: alpha"):
        tie.lognormal_censored_cvar(1.0, 1.0, 100.0, 1.0)
    with pytest.raises(ValueError, match="x_max must be finite"):
        tie.lognormal_censored_expectation(1.0, 1.0, -1.0)


# ---------------------------------------------------------------- ks_test_fit
@needs_ref
def test_ks_test_fit_matches_reference(tie, R):
    rng = np.random.default_rng(9)
    for trial in range(20):
        K = int(rng.integers(5, 80))
        x = np.exp(rng.normal(3.0, 1.0, K))
        fam = trial % 4
        f = [tie.fit_logt_fixed_nu(list(x), 3.5)]
        mu, sg = float(f[0].mu), float(f[0].sigma)
        nu = 3.5 if fam == 0 else 2.0 + 0.5 * (trial % 5)
        rate = 1.0 / float(np.mean(x))
        st, p = ref_ks_test_fit(R, x, fam, mu, sg, nu, rate)
        got = tie.ks_test_fit_raw(x, fam, mu, sg, nu, rate)
        assert abs(got[0] - st) <= 1e-12 and abs(got[1] - p) <= 1e-9, (trial, got, (st, p))
    with pytest.raises(ValueError, match="need at least 5 samples"):
        tie.ks_test_fit([1.0, 2.0], tie.fit_logt_fixed_nu([1.0, 2.0, 3.0], 3.5))


# ---------------------------------------------------------------- WaitingQueue / Scheduler
def test_waiting_queue_python(tie):
    q = tie.WaitingQueue()
    assert q.pop_min() is None and q.empty()
    for i in (7, 2, 9, 4, 0):
        q.push(tie.QueueEntry(i, 2048.0))
    assert [q.pop_min().req_id for _ in range(5)] == [0, 2, 4, 7, 9]
    rng = np.random.default_rng(1)
    ids = np.arange(20000, dtype=np.uint64)
    keys = rng.integers(0, 300, 20000).astype(float)
    q.push_batch(ids, keys)
    q.update_batch(ids[:5000], keys[:5000] + 0.5)
    keys[:5000] += 0.5
    assert q.validate()
    got, gk = q.pop_batch(20000)
    order = np.lexsort((ids, keys))
    np.testing.assert_array_equal(got, ids[order])
    np.testing.assert_array_equal(gk, keys[order])
    with pytest.raises(ValueError, match="already queued"):
        q.push_batch(np.array([1, 1], np.uint64), np.array([1.0, 2.0]))
    with pytest.raises(ValueError, match="not queued"):
        q.update(123456, 1.0)


def test_waiting_queue_growth_and_compaction(tie):
    """slots are append-only; pushes beyond the capacity grow the queue or compact the popped
    slots, with the pop order unchanged"""
    q = tie.WaitingQueue(None, 64)
    rng = np.random.default_rng(2)
    live = {}
    nid = 0
    for rnd in range(40):
        m = int(rng.integers(1, 200))
        ids = np.arange(nid, nid + m, dtype=np.uint64)
        nid += m
        keys = rng.uniform(0, 50, m)
        q.push_batch(ids, keys)
        live.update(zip(ids.tolist(), keys.tolist()))
        k = int(rng.integers(0, len(live) + 1))
        got, gk = q.pop_batch(k)
        want = sorted(live.items(), key=lambda t: (t[1], t[0]))[:k]
        assert got.tolist() == [w[0] for w in want]
        for i in got.tolist():
            del live[i]
        assert len(q) == len(live) and q.validate()


def test_scheduler_python_drift(tie):
    """test_sched.cpp:246-292 through the Python Scheduler class"""
    cfg = tie.ScoreConfig()
    cfg.beta_max, cfg.q_sat, cfg.rebuild_threshold = 0.5, 4.0, 0.1

    def build():
        s = tie.Scheduler(tie.Policy.TIE, cfg)
        for i in range(4):
            r = tie.Request()
            r.id, r.arrival_s, r.max_tokens = i, 0.1 * i, 2048
            s.on_arrival(r)
        s.on_prediction(0, 5.0, 10.0)
        s.on_prediction(1, 100.0, 2000.0)
        s.on_prediction(2, 671.0, 671.0)
        return s

    s = build()
    assert s.next_request() == 0
    assert s.queue().at(1).key == pytest.approx(1100.0, rel=1e-15)
    assert s.rebuild_if_drifted()
    assert s.queue().at(2).key == pytest.approx(922.625, rel=1e-15)
    assert s.queue().at(3).key == 2048.0 and s.queue().validate()
    assert s.next_request() == 1
    a = build()
    assert [a.next_request(), a.next_request()] == [0, 1]


# ---------------------------------------------------------------- reference smoke tests
# proj/tests/python/test_smoke.py restated against the drop-in package
def test_smoke_censored_moment_invariants(tie):  # test_smoke.py:8-17
    mc = tie.McContext(3.5)
    cl = tie.CensoredLogT(tie.LogTParams(4.0, 0.8, 3.5), 512.0)
    e = tie.censored_expectation(cl, mc)
    assert 0.0 < e <= 512.0
    assert tie.censored_cvar(cl, mc, 0.0) == e
    c = tie.censored_cvar(cl, mc, 0.9)
    assert e <= c <= 512.0
    assert tie.censored_cvar(cl, mc, 0.999) == 512.0


def test_smoke_student_t_roundtrip(tie):  # test_smoke.py:20-22
    for p in (0.05, 0.5, 0.9, 0.975):
        assert math.isclose(tie.t_cdf(tie.t_quantile(p, 3.5), 3.5), p, abs_tol=1e-9)


def test_smoke_fit_recovers_truth(tie):  # test_smoke.py:25-31
    x = tie.sample_logt(tie.LogTParams(5.0, 0.7, 3.5), 400, 7)
    f = tie.fit_logt_fixed_nu(x, 3.5)
    assert f.converged
    assert abs(f.mu - 5.0) < 0.15
    assert abs(f.sigma - 0.7) < 0.15
    assert tie.ks_test_fit(x, f).p_value > 0.05


def test_smoke_score_monotone_in_beta(tie):  # test_smoke.py:40-44
    assert tie.compute_score(10.0, 40.0, 0.0) == 10.0
    assert tie.compute_score(10.0, 40.0, 0.3) == pytest.approx(22.0)
    with pytest.raises(Exception):
        tie.compute_score(10.0, 5.0, 0.1)


def test_smoke_sim_policies_and_determinism(tie):  # test_smoke.py:47-62
    ws = tie.WorkloadSpec()
    ws.n_requests = 400
    ws.rps = 80.0
    ws.mu_range = (0.5, 2.5)
    ws.sigma_range = (0.4, 1.2)
    ws.prompt_range = (16, 128)
    ws.max_tokens = 512
    w = tie.gen_logt_workload(ws, 11)
    sc, eng, pc = tie.ScoreConfig(), tie.EngineConfig(), tie.PredictorConfig()
    tie_r = tie.run_sim(w, tie.Policy.TIE, sc, eng, pc, 11)
    fcfs_r = tie.run_sim(w, tie.Policy.FCFS, sc, eng, pc, 11)
    assert len(tie_r.events) == 400
    assert tie_r.metrics.ptla_avg < fcfs_r.metrics.ptla_avg
    again = tie.run_sim(w, tie.Policy.TIE, sc, eng, pc, 11)
    assert [e.completion_s for e in again.events] == [e.completion_s for e in tie_r.events]


# ---------------------------------------------------------------- run_sim parity
def _ours(tie, wseed, policy, seed, **kw):
    a = dict(CANONICAL)
    a.update(kw)
    ws = tie.WorkloadSpec()
    ws.n_requests, ws.rps = a["n"], a["rps"]
    ws.mu_range, ws.sigma_range = a["mu_range"], a["sigma_range"]
    ws.prompt_range, ws.max_tokens = a["prompt_range"], a["max_tokens"]
    w = tie.gen_logt_workload(ws, wseed)
    sc = tie.ScoreConfig()
    sc.alpha = a["alpha"]
    sc.beta_mode = tie.BetaMode.AdaptiveLinear if a["adaptive"] else tie.BetaMode.Fixed
    sc.beta_fixed, sc.beta_max, sc.q_sat = a["beta_fixed"], a["beta_max"], a["q_sat"]
    sc.rebuild_threshold = a["threshold"]
    ec = tie.EngineConfig()
    ec.batch_slots, ec.c0, ec.c1, ec.c2 = a["slots"], a["c0"], a["c1"], a["c2"]
    pc = tie.PredictorConfig()
    pc.kind = [tie.PredictorKind.NoPredictor, tie.PredictorKind.Oracle,
               tie.PredictorKind.Noisy][a["kind"]]
    pc.family = [tie.ScoreFamily.LogT, tie.ScoreFamily.LogNormal][a["family"]]
    ns = tie.NoiseSpec()
    ns.mu_sd, ns.log_sigma_sd = a["mu_sd"], a["ls_sd"]
    pc.noise = ns
    pc.batched = a["batched"]
    pol = [tie.Policy.FCFS, tie.Policy.SEPT, tie.Policy.TIE][policy]
    r = tie.run_sim(w, pol, sc, ec, pc, seed)
    ev = {k: np.array([getattr(e, k) if getattr(e, k) is not None else np.nan
                       for e in r.events])
          for k in ("arrival_s", "predict_ready_s", "admit_s", "first_token_s", "completion_s",
                    "emitted_tokens")}
    m = np.array([r.metrics.ttft_avg, r.metrics.ttft_p90, r.metrics.ptla_avg,
                  r.metrics.ptla_p90])
    return ev, m


def _same(ev, ref):
    for k in ("arrival_s", "predict_ready_s", "admit_s", "first_token_s", "completion_s",
              "emitted_tokens"):
        a, b = np.asarray(ev[k], float), np.asarray(ref[k], float)
        assert np.array_equal(a, b, equal_nan=True), (k, int(np.flatnonzero(a != b)[0]))


@needs_ref
@pytest.mark.parametrize("seed", range(1, 11))
def test_config5_canonical_threshold0_matches_reference(tie, R, seed):
    """BASELINE config 5: canonical.json, re-scoring every step (rebuild_threshold 0)"""
    ev, m = _ours(tie, seed, 2, seed, threshold=0.0)
    ref, rm, _ = ref_run_sim(R, seed, 2, seed, threshold=0.0)
    _same(ev, ref)
    np.testing.assert_array_equal(m, rm)
    g = golden("config5.json")["seeds"][str(seed)]
    assert m.tolist() == g["metrics"]


@needs_ref
@pytest.mark.parametrize("policy,kw", [
    (2, {}), (0, {}), (1, {}), (2, dict(kind=2, mu_sd=0.4, ls_sd=0.3)),
    (2, dict(family=1)), (2, dict(batched=False)), (2, dict(kind=0)),
    (2, dict(adaptive=False, beta_fixed=0.3)), (1, dict(kind=2, mu_sd=0.2, ls_sd=0.2))])
def test_run_sim_variants_match_reference(tie, R, policy, kw):
    kw = dict(kw, n=3000)
    ev, m = _ours(tie, 5, policy, 7, **kw)
    ref, rm, _ = ref_run_sim(R, 5, policy, 7, **kw)
    _same(ev, ref)
    np.testing.assert_array_equal(m, rm)


def test_run_sim_errors(tie):
    w = tie.gen_logt_workload(tie.WorkloadSpec(), 1)[:10]
    ec = tie.EngineConfig()
    ec.batch_slots = 0
    with pytest.raises(ValueError, match="batch_slots must be >= 1"):
        tie.run_sim(w, tie.Policy.TIE, tie.ScoreConfig(), ec, tie.PredictorConfig(), 1)
    w[3].id = w[1].id
    with pytest.raises(ValueError, match="duplicate request id"):
        tie.run_sim(w, tie.Policy.TIE, tie.ScoreConfig(), tie.EngineConfig(),
                    tie.PredictorConfig(), 1)
    r = tie.Request()
    r.id, r.arrival_s, r.prompt_tokens, r.true_output_tokens, r.max_tokens = 0, 0.0, 8, 4, 64
    with pytest.raises(ValueError, match="carries no ground-truth parameters"):
        tie.run_sim([r], tie.Policy.TIE, tie.ScoreConfig(), tie.EngineConfig(),
                    tie.PredictorConfig(), 1)
