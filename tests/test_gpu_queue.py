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
