"""GPU parity: the GPU-resident Scheduler (tie_queue_*) pops exactly the
reference Scheduler's sequence (oracle restatement, pinned to the reference in
test_oracle.py) across FCFS / SEPT / TIE, drift rebuilds, key ties and id tie-breaks."""
import numpy as np
import pytest

from sched_scripts import make_script, runs_of

pytestmark = pytest.mark.gpu
U64MAX = np.iinfo(np.uint64).max


def run_gpu(tie, mc, policy, ops, ids, a, b, cfg):
    sc = tie.ScoreConfig()
    sc.beta_mode = tie.BetaMode.AdaptiveLinear if cfg["adaptive"] else tie.BetaMode.Fixed
    sc.beta_max = cfg.get("beta_max", 0.5)
    sc.beta_fixed = cfg.get("beta_fixed", 0.1)
    sc.q_sat = cfg.get("q_sat", 128.0)
    sc.rebuild_threshold = cfg.get("rebuild_threshold", 0.1)
    pol = [tie.Policy.FCFS, tie.Policy.SEPT, tie.Policy.TIE][policy]
    q = tie.GpuScheduler(mc, pol, sc, max(len(ops), 1))
    out = []
    for kind, s, e in runs_of(ops):
        if kind == 0:
            q.on_arrival_batch(ids[s:e], a[s:e], b[s:e].astype(np.uint32))
        elif kind == 1:
            q.on_prediction_batch(ids[s:e], a[s:e], b[s:e])
        else:
            got = q.next_requests(e - s).tolist()
            out += got + [U64MAX] * ((e - s) - len(got))
    return np.array(out, np.uint64)


@pytest.mark.parametrize("policy,thr,q_sat", [(2, 0.1, 64.0), (2, 0.0, 64.0), (2, 0.2, 16.0),
                                              (2, 0.1, 1e9), (1, 0.1, 64.0), (0, 0.1, 64.0)])
def test_pop_sequence_matches_reference(tie, mc, oracle, policy, thr, q_sat):
    cfg = dict(adaptive=True, beta_max=0.5, q_sat=q_sat, rebuild_threshold=thr)
    for seed in range(3):
        ops, ids, a, b = make_script(100 + seed, oracle, policy=policy, **cfg)
        ref = oracle.scheduler_script(policy, ops, ids, a, b, **cfg)
        got = run_gpu(tie, mc, policy, ops, ids, a, b, cfg)
        assert np.array_equal(got, ref), (policy, thr, q_sat, seed)


def test_drift_rebuild_scenario(tie, mc):
    """test_sched.cpp:245-292 on the GPU queue."""
    for thr, second in [(0.1, 1), (0.2, 2)]:
        sc = tie.ScoreConfig()
        sc.q_sat = 4.0
        sc.rebuild_threshold = thr
        q = tie.GpuScheduler(mc, tie.Policy.TIE, sc, 16)
        q.on_arrival_batch(np.arange(4, dtype=np.uint64), np.arange(4) * 0.1,
                           np.full(4, 2048, np.uint32))
        q.on_prediction_batch(np.array([0, 1, 2], np.uint64), np.array([5.0, 100.0, 671.0]),
                              np.array([10.0, 2000.0, 671.0]))
        assert q.next_request() == 0
        assert q.next_request() == second
        assert q.waiting() == 2


def test_logt_predictions_and_errors(tie, mc, oracle, samples):
    sc = tie.ScoreConfig()
    q = tie.GpuScheduler(mc, tie.Policy.TIE, sc, 1000)
    mu, sg, mt = oracle.gen_workload(300, seed=3)
    ids = np.arange(300, dtype=np.uint64) * 7 + 11
    q.on_arrival_batch(ids, np.zeros(300), mt)
    q.on_prediction_logt(ids, mu, sg, mt)
    E, C, _ = oracle.score(samples, mu, sg, mt.astype(float), alpha=0.9, beta=0.0)
    C = np.maximum(C, E)
    # the reference Scheduler fed the same events (drift rebuilds fire as the queue drains
    # below q_sat = 128)
    ops = np.r_[np.zeros(300), np.ones(300), np.full(300, 2)].astype(np.int32)
    sids = np.r_[ids, ids, np.zeros(300, np.uint64)]
    ref = oracle.scheduler_script(2, ops, sids, np.r_[np.zeros(300), E, np.zeros(300)],
                                  np.r_[mt.astype(float), C, np.zeros(300)])
    assert np.array_equal(q.next_requests(300), ref)
    with pytest.raises(ValueError, match="not waiting"):
        q.on_prediction_batch(np.array([5], np.uint64), np.array([1.0]), np.array([2.0]))
    q.on_arrival_batch(np.array([1], np.uint64), np.zeros(1), np.array([64], np.uint32))
    with pytest.raises(ValueError, match="already queued"):
        q.on_arrival_batch(np.array([1], np.uint64), np.zeros(1), np.array([64], np.uint32))
    with pytest.raises(ValueError, match="cvar below expectation"):
        q.on_prediction_batch(np.array([1], np.uint64), np.array([10.0]), np.array([5.0]))
    assert q.next_requests(5).tolist() == [1]
    assert q.next_request() is None


# ---- fused scheduler iteration (tie_queue_step): one device round trip per step
def _cfg(tie, q_sat=128.0, thr=0.1):
    sc = tie.ScoreConfig()
    sc.q_sat = q_sat
    sc.rebuild_threshold = thr
    return sc


@pytest.mark.parametrize("policy,q_sat,thr", [(2, 128.0, 0.1), (2, 1e9, 0.0), (2, 64.0, 0.05),
                                              (1, 128.0, 0.1), (0, 128.0, 0.1)])
def test_step_equals_separate_calls(tie, mc, oracle, policy, q_sat, thr):
    pol = [tie.Policy.FCFS, tie.Policy.SEPT, tie.Policy.TIE][policy]
    n0, steps, per, pops = 3000, 40, 32, 8
    tot = n0 + steps * per
    mu, sg, mt = oracle.gen_workload(tot, seed=11)
    ids = np.random.default_rng(5).permutation(tot * 3)[:tot].astype(np.uint64)
    arr = np.arange(tot, dtype=np.float64) * 0.01
    qa = tie.GpuScheduler(mc, pol, _cfg(tie, q_sat, thr), tot)
    qb = tie.GpuScheduler(mc, pol, _cfg(tie, q_sat, thr), tot)
    for q in (qa, qb):
        q.on_arrival_batch(ids[:n0], arr[:n0], mt[:n0])
        q.on_prediction_logt(ids[:n0 // 2], mu[:n0 // 2], sg[:n0 // 2], mt[:n0 // 2])
    pending = list(range(n0 // 2, n0))  # predicted one step after they arrive
    for s in range(steps):
        lo, hi = n0 + s * per, n0 + (s + 1) * per
        pa = np.array(pending[:per], np.int64)
        got_a = qa.step(ids[lo:hi], arr[lo:hi], mt[lo:hi], ids[pa], mu[pa], sg[pa], mt[pa], pops)
        qb.on_arrival_batch(ids[lo:hi], arr[lo:hi], mt[lo:hi])
        qb.on_prediction_logt(ids[pa], mu[pa], sg[pa], mt[pa])
        got_b = qb.next_requests(pops)
        assert np.array_equal(got_a, got_b), (s, got_a, got_b)
        popped = set(got_a.tolist())
        pending = [p for p in pending[per:] if ids[p] not in popped] + \
                  [p for p in range(lo, hi) if ids[p] not in popped]
    assert qa.waiting() == qb.waiting()
    assert np.array_equal(qa.next_requests(500), qb.next_requests(500))


def test_step_errors_leave_reference_state(tie, mc):
    q = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), 100)
    q.step(np.array([1, 2, 3], np.uint64), np.zeros(3), np.full(3, 512, np.uint32),
           np.array([], np.uint64), np.array([]), np.array([]), np.array([], np.uint32), 0)
    with pytest.raises(ValueError, match="sigma"):  # LogTParams check of prediction 1
        q.step(np.array([4], np.uint64), np.zeros(1), np.array([64], np.uint32),
               np.array([1, 2], np.uint64), np.array([3.0, 3.0]), np.array([0.5, -1.0]),
               np.array([512, 512], np.uint32), 4)
    assert q.waiting() == 4  # the arrival applied, no prediction, no pop
    with pytest.raises(ValueError, match="not waiting"):
        q.step(np.array([], np.uint64), np.array([]), np.array([], np.uint32),
               np.array([9], np.uint64), np.array([3.0]), np.array([0.5]),
               np.array([512], np.uint32), 1)
    with pytest.raises(ValueError, match="already queued"):
        q.step(np.array([4], np.uint64), np.zeros(1), np.array([64], np.uint32),
               np.array([], np.uint64), np.array([]), np.array([]), np.array([], np.uint32), 1)
    # unpredicted keys are max_tokens: 4 (64) first, then 1, 2, 3 (512) by id
    assert q.step(np.array([], np.uint64), np.array([]), np.array([], np.uint32),
                  np.array([], np.uint64), np.array([]), np.array([]),
                  np.array([], np.uint32), 10).tolist() == [4, 1, 2, 3]


def test_topb_pop_candidate_overflow_path(tie, mc):
    """Equal keys, ids ascending with the slot: every chosen block is full of candidates, so
    the top-B pop takes its per-pop fallback; the order is still by id."""
    n = 20_000
    q = tie.GpuScheduler(mc, tie.Policy.SEPT, _cfg(tie), n)
    q.on_arrival_batch(np.arange(n, dtype=np.uint64), np.zeros(n), np.full(n, 100, np.uint32))
    assert q.next_requests(32).tolist() == list(range(32))
    assert q.next_requests(40).tolist() == list(range(32, 72))
