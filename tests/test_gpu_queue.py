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


def _empty_step_args():
    return (np.array([], np.uint64), np.array([]), np.array([], np.uint32))


def test_step_prediction_error_keeps_arrivals_poppable(tie, mc):
    """a prediction-validation error in a fused step leaves the step's
    arrivals applied ON THE DEVICE too (reference: on_arrival calls stay applied when a later
    on_prediction throws), so they pop with their ids and a later prediction re-keys them."""
    for bad in ("not waiting", "already predicted"):
        q = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), 100)
        q.on_arrival_batch(np.array([1], np.uint64), np.zeros(1), np.array([512], np.uint32))
        q.on_prediction_batch(np.array([1], np.uint64), np.array([50.0]), np.array([80.0]))
        pid = np.array([99], np.uint64) if bad == "not waiting" else np.array([1], np.uint64)
        with pytest.raises(ValueError, match=bad):
            q.step(np.array([5, 6], np.uint64), np.zeros(2), np.array([300, 200], np.uint32),
                   pid, np.array([3.0]), np.array([0.5]), np.array([512], np.uint32), 3)
        assert q.waiting() == 3
        # the arrival 6 (key 200) gets a prediction now: key 10 + beta * 20 < 50 + beta * 80
        q.on_prediction_batch(np.array([6], np.uint64), np.array([10.0]), np.array([20.0]))
        assert q.next_requests(3).tolist() == [6, 1, 5]


def test_step_prediction_of_same_step_arrival(tie, mc):
    """A prediction may name an arrival of the same step (it is waiting by then)."""
    q = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), 100)
    got = q.step(np.array([7, 8], np.uint64), np.zeros(2), np.array([512, 512], np.uint32),
                 np.array([8], np.uint64), np.array([3.0]), np.array([0.5]),
                 np.array([512], np.uint32), 1)
    assert got.tolist() == [8]


def test_arrive_rejected_batch_leaves_queue_usable(tie, mc):
    """a batch rejected part-way (non-finite key / duplicate) changes nothing, so
    later arrivals are accepted and every id pops exactly once."""
    q = tie.GpuScheduler(mc, tie.Policy.FCFS, _cfg(tie), 100)
    with pytest.raises(ValueError, match="finite"):
        q.on_arrival_batch(np.array([1, 2, 3], np.uint64), np.array([0.1, 0.2, np.inf]),
                           np.full(3, 512, np.uint32))
    with pytest.raises(ValueError, match="id 2 already queued"):
        q.on_arrival_batch(np.array([1, 2, 2], np.uint64), np.array([0.1, 0.2, 0.3]),
                           np.full(3, 512, np.uint32))
    assert q.waiting() == 0
    q.on_arrival_batch(np.array([1, 2, 3], np.uint64), np.array([0.3, 0.2, 0.1]),
                       np.full(3, 512, np.uint32))
    assert q.next_requests(5).tolist() == [3, 2, 1]


def test_predict_duplicate_far_apart_rejected(tie, mc):
    """an id repeated anywhere in one prediction batch is 'already predicted'
    (the reference's second on_prediction throws), and the queue is unchanged."""
    n = 200
    q = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), n)
    q.on_arrival_batch(np.arange(n, dtype=np.uint64), np.zeros(n), np.full(n, 512, np.uint32))
    ids = np.arange(100, dtype=np.uint64)
    ids[99] = 3  # 96 positions after the first 3
    with pytest.raises(ValueError, match="id 3 already predicted"):
        q.on_prediction_batch(ids, np.full(100, 10.0), np.full(100, 20.0))
    assert q.beta_range()[2] == 0  # betas_in_use_ untouched
    q.on_prediction_batch(np.array([150], np.uint64), np.array([10.0]), np.array([20.0]))
    assert q.next_requests(2).tolist() == [150, 0]


def test_invalid_beta_config_raises_domain_error(tie, mc):
    """compute_beta's std::domain_error on an invalid ScoreConfig surfaces at
    on_prediction (sched.cpp:10-15, 139) instead of running with beta = 0."""
    for field, val in [("q_sat", 0.0), ("beta_max", -1.0)]:
        sc = _cfg(tie)
        setattr(sc, field, val)
        q = tie.GpuScheduler(mc, tie.Policy.TIE, sc, 10)
        q.on_arrival_batch(np.array([1], np.uint64), np.zeros(1), np.array([512], np.uint32))
        with pytest.raises(ValueError, match="compute_beta"):
            q.on_prediction_batch(np.array([1], np.uint64), np.array([10.0]), np.array([20.0]))
        with pytest.raises(ValueError, match="compute_beta"):
            q.step(*_empty_step_args(), np.array([1], np.uint64), np.array([3.0]),
                   np.array([0.5]), np.array([512], np.uint32), 0)
        assert q.next_requests(1).tolist() == [1]
    sc = _cfg(tie)
    sc.beta_mode = tie.BetaMode.Fixed
    sc.beta_fixed = -0.5
    q = tie.GpuScheduler(mc, tie.Policy.TIE, sc, 10)
    q.on_arrival_batch(np.array([1], np.uint64), np.zeros(1), np.array([512], np.uint32))
    with pytest.raises(ValueError, match="beta_fixed"):
        q.on_prediction_batch(np.array([1], np.uint64), np.array([10.0]), np.array([20.0]))


def test_batch_length_mismatch_is_value_error(tie, mc):
    q = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), 10)
    with pytest.raises(ValueError, match="lengths"):
        q.on_arrival_batch(np.array([1, 2], np.uint64), np.zeros(1), np.full(2, 5, np.uint32))
    q.on_arrival_batch(np.array([1, 2], np.uint64), np.zeros(2), np.full(2, 5, np.uint32))
    with pytest.raises(ValueError, match="lengths"):
        q.on_prediction_batch(np.array([1, 2], np.uint64), np.array([1.0, 2.0]), np.ones(1))
    with pytest.raises(ValueError, match="lengths"):
        q.on_prediction_logt(np.array([1, 2], np.uint64), np.ones(2), np.ones(1),
                             np.full(2, 5, np.uint32))


def _many_block_keys(n, seed):
    """keys for n slots (1024-slot blocks, 4+ blocks per thread of the 1024-thread pop CTA):
    uniform background, the smallest keys packed into the blocks of ONE pop thread (blocks
    5, 1029, 2053, ...: it wins many rounds and must rescan its share), a few more in other
    blocks, and tied keys across blocks (id tie-break)"""
    rng = np.random.default_rng(seed)
    keys = rng.uniform(100.0, 200.0, n)
    nb = n // 1024
    own = [b for b in range(5, nb, 1024)]
    small = np.arange(1.0, 1.0 + 3 * len(own))
    for j, k in enumerate(small):  # three tiny keys per block of thread 5
        b = own[j % len(own)]
        keys[b * 1024 + 17 * (j // len(own)) + 3] = k
    keys[7 * 1024 + 9] = 2.5
    keys[(nb - 1) * 1024 + 1000] = 1.5
    tied = rng.choice(n, 64, replace=False)
    keys[tied] = 50.0
    return keys


def test_pop_many_blocks_per_thread_waiting_queue(tie):
    """4M slots = 4 blocks per thread of the top-B scan (the two-best-per-thread registers and
    the rescan after a third win; config 4's 64M queue has 64 per thread): pop order equals
    the (key, id) sort"""
    n = 4 * 2 ** 20
    keys = _many_block_keys(n, 3)
    ids = np.arange(n, dtype=np.uint64)
    q = tie.WaitingQueue(None, n)
    q.push_batch(ids, keys)
    want = np.lexsort((ids, keys))
    got = []
    for m in (8, 32, 1, 3, 32, 100, 8, 500, 1000):
        g, _ = q.pop_batch(m)
        got += g.tolist()
    np.testing.assert_array_equal(np.array(got, np.uint64), ids[want[:len(got)]])
    assert q.validate()


def test_pop_many_blocks_per_thread_scheduler(tie, mc):
    """the Scheduler's pop path (the fused apply kernel) on the same layout: SEPT keys = E"""
    n = 4 * 2 ** 20
    E = _many_block_keys(n, 4)
    ids = np.arange(n, dtype=np.uint64)
    q = tie.GpuScheduler(mc, tie.Policy.SEPT, _cfg(tie), n)
    q.on_arrival_batch(ids, np.zeros(n), np.full(n, 512, np.uint32))
    q.on_prediction_batch(ids, E, E)
    want = ids[np.lexsort((ids, E))]
    got = []
    for m in (8, 8, 32, 1, 8, 64, 8):
        got += q.next_requests(m).tolist()
    np.testing.assert_array_equal(np.array(got, np.uint64), want[:len(got)])


def _rekey_expected(tie, sc, pred, E, C, mkey, ids, pops):
    """the reference's pop sequence at rebuild_threshold 0 with beta moving at every pop
    (sched.cpp:152-175): before pop j every predicted key is re-made at beta(Q_j) =
    compute_beta(Q_j) (E + beta * C, the same IEEE operations), then the (key, id) minimum"""
    alive = np.ones(len(ids), bool)
    out = []
    q = len(ids)
    for _ in range(pops):
        b = tie.compute_beta(sc, q)
        keys = np.where(pred, E + b * C, mkey)
        keys = np.where(alive, keys, np.inf)
        j = np.lexsort((ids, keys))[0]
        out.append(int(ids[j]))
        alive[j] = False
        q -= 1
    return out


@pytest.mark.parametrize("ties,q_sat_gap", [(False, None), (True, None), (False, 40)])
def test_rekey_every_pop_one_pass_matches_reference(tie, mc, ties, q_sat_gap):
    """the one-pass re-key + pop kernel (>= 512 blocks; a run of (rebuild, pop) segments): pops
    at rebuild_threshold 0 with beta moving every pop equal the reference's re-key-then-pop
    sequence; mixed unpredicted entries (constant keys) pop among the predicted ones; with
    `ties`, 3,000 identical (E, C) pairs at the front make the candidate list overflow (the
    in-launch per-segment fallback) and pop in id order"""
    n = 600_000
    rng = np.random.default_rng(11 + ties)
    ids = rng.permutation(np.arange(10, 10 + n, dtype=np.uint64))
    E = rng.uniform(50.0, 500.0, n)
    C = E * rng.uniform(1.0, 3.0, n)
    pred = rng.random(n) > 0.05
    mt = rng.integers(60, 4000, n).astype(np.uint32)
    if ties:
        E[:3000], C[:3000] = 20.0, 30.0
        pred[:3000] = True
    # q_sat_gap: beta saturated (constant, no rebuilds) for the first pops, then moving with
    # every pop -- the plan switches from fixed-key pops to (rebuild, pop) runs
    sc = _cfg(tie, q_sat=1e9 if q_sat_gap is None else float(n - q_sat_gap), thr=0.0)
    q = tie.GpuScheduler(mc, tie.Policy.TIE, sc, n)
    q.on_arrival_batch(ids, np.zeros(n), mt)
    q.on_prediction_batch(ids[pred], E[pred], C[pred])
    mkey = mt.astype(np.float64)  # unpredicted TIE entries are keyed at max_tokens
    got = []
    for m in (8, 8, 32, 5, 32, 32, 3):
        got += q.next_requests(m).tolist()
    want = _rekey_expected(tie, sc, pred, E, C, mkey, ids, len(got))
    assert got == want


@pytest.mark.parametrize("policy,q_sat,thr", [(2, 128.0, 0.1), (2, 1e9, 0.0), (1, 128.0, 0.1),
                                              (0, 128.0, 0.1)])
def test_step_ec_equals_separate_calls(tie, mc, oracle, policy, q_sat, thr):
    """tie_queue_step_ec (Scheduler::step: on_prediction's (E, C) pairs) == on_arrival_batch +
    on_prediction_batch + next_requests; a C < E prediction raises the reference's error
    (compute_score, sched.cpp:19-26) with the step's arrivals applied"""
    pol = [tie.Policy.FCFS, tie.Policy.SEPT, tie.Policy.TIE][policy]
    n0, steps, per, pops = 3000, 30, 32, 8
    tot = n0 + steps * per
    rng = np.random.default_rng(9)
    ids = rng.permutation(tot * 3)[:tot].astype(np.uint64)
    arr = np.arange(tot, dtype=np.float64) * 0.01
    mt = rng.integers(64, 4096, tot).astype(np.uint32)
    E = rng.uniform(10.0, 800.0, tot)
    C = E * rng.uniform(1.0, 2.5, tot)
    qa = tie.GpuScheduler(mc, pol, _cfg(tie, q_sat, thr), tot)
    qb = tie.GpuScheduler(mc, pol, _cfg(tie, q_sat, thr), tot)
    for q in (qa, qb):
        q.on_arrival_batch(ids[:n0], arr[:n0], mt[:n0])
        q.on_prediction_batch(ids[:n0 // 2], E[:n0 // 2], C[:n0 // 2])
    pending = list(range(n0 // 2, n0))
    for s in range(steps):
        lo, hi = n0 + s * per, n0 + (s + 1) * per
        pa = np.array(pending[:per] + list(range(lo, lo + 4)), np.int64)  # + same-step arrivals
        got_a = qa.step_ec(ids[lo:hi], arr[lo:hi], mt[lo:hi], ids[pa], E[pa], C[pa], pops)
        qb.on_arrival_batch(ids[lo:hi], arr[lo:hi], mt[lo:hi])
        qb.on_prediction_batch(ids[pa], E[pa], C[pa])
        got_b = qb.next_requests(pops)
        assert np.array_equal(got_a, got_b), (s, got_a, got_b)
        popped = set(got_a.tolist())
        pending = [p for p in pending[per:] if ids[p] not in popped] + \
                  [p for p in range(lo + 4, hi) if ids[p] not in popped]
    assert np.array_equal(qa.next_requests(500), qb.next_requests(500))
    if policy != 0:  # FCFS validates too, but a bad prediction never reaches a key there
        nid = np.array([10 ** 9], np.uint64)
        with pytest.raises(ValueError):
            qa.step_ec(nid, np.zeros(1), np.array([64], np.uint32), nid, np.array([5.0]),
                       np.array([4.0]), 1)
        assert nid[0] in qa.next_requests(qa.waiting()).tolist()  # the arrival stayed


@pytest.mark.parametrize("policy,thr,q_sat", [(2, 0.0, 1e9), (2, 0.05, 4096.0), (1, 0.1, 64.0)])
def test_pop_sequence_matches_reference_multi_block(tie, mc, oracle, policy, thr, q_sat):
    """random event scripts whose queue grows to ~10 blocks (arrival runs of up to 400): the
    multi-CTA re-key + pop runs, multi-block top-B pops and drift rebuilds against the
    reference Scheduler (oracle restatement)"""
    cfg = dict(adaptive=True, beta_max=0.5, q_sat=q_sat, rebuild_threshold=thr)
    ops, ids, a, b = make_script(7, oracle, policy=policy, n_req=12_000, runs=160,
                                 arr_max=400, **cfg)
    ref = oracle.scheduler_script(policy, ops, ids, a, b, **cfg)
    got = run_gpu(tie, mc, policy, ops, ids, a, b, cfg)
    assert np.array_equal(got, ref), (policy, thr, q_sat)


@pytest.mark.parametrize("q_sat,thr", [(1e9, 0.0), (128.0, 0.1)])
def test_large_step_equals_separate_calls(tie, mc, oracle, q_sat, thr):
    """a step above the small-step limits (> 16,384 arrivals / predictions: one packed H2D and
    the multi-kernel apply path) == on_arrival_batch + on_prediction_logt + next_requests"""
    n0, big, pops = 5000, 20_000, 24
    tot = n0 + 2 * big
    mu, sg, mt = oracle.gen_workload(tot, seed=12)
    ids = np.random.default_rng(8).permutation(tot * 2)[:tot].astype(np.uint64)
    arr = np.arange(tot, dtype=np.float64) * 0.001
    cfg = _cfg(tie, q_sat=q_sat, thr=thr)  # q_sat 1e9: beta moves, the pops are rebuild segments
    qa = tie.GpuScheduler(mc, tie.Policy.TIE, cfg, tot)
    qb = tie.GpuScheduler(mc, tie.Policy.TIE, cfg, tot)
    for q in (qa, qb):
        q.on_arrival_batch(ids[:n0], arr[:n0], mt[:n0])
    popped, done = set(), 0
    for s in range(2):
        lo, hi = n0 + s * big, n0 + (s + 1) * big
        pr = np.array([p for p in range(done, hi - 1000) if int(ids[p]) not in popped], np.int64)
        done = hi - 1000  # old ids + ids arriving in this same step
        got_a = qa.step(ids[lo:hi], arr[lo:hi], mt[lo:hi], ids[pr], mu[pr], sg[pr], mt[pr],
                        pops)
        qb.on_arrival_batch(ids[lo:hi], arr[lo:hi], mt[lo:hi])
        qb.on_prediction_logt(ids[pr], mu[pr], sg[pr], mt[pr])
        got_b = qb.next_requests(pops)
        assert len(pr) > 16_384 and np.array_equal(got_a, got_b), s
        popped |= set(got_a.tolist())
    assert qa.waiting() == qb.waiting()
    assert np.array_equal(qa.next_requests(300), qb.next_requests(300))


# ---- tie_queue_step_ec_runs: a run of interleaved (arrivals, predictions) then pops ----------
def _ec(rng, m):
    e = rng.uniform(10.0, 500.0, m)
    return e, e * rng.uniform(1.0, 3.0, m)


def _seq_runs(q, ids, arr, mt, ae, pids, E, C, pe, k):
    """the definition: consecutive step_ec calls, the last one popping"""
    got, a0, p0 = np.zeros(0, np.uint64), 0, 0
    for r in range(len(ae)):
        got = q.step_ec(ids[a0:ae[r]], arr[a0:ae[r]], mt[a0:ae[r]], pids[p0:pe[r]], E[p0:pe[r]],
                        C[p0:pe[r]], k if r + 1 == len(ae) else 0)
        a0, p0 = ae[r], pe[r]
    return got


@pytest.mark.parametrize("policy,q_sat,thr", [(2, 128.0, 0.1), (2, 1e9, 0.0), (2, 40.0, 0.05),
                                              (1, 128.0, 0.1), (0, 128.0, 0.1)])
def test_step_ec_runs_equals_step_sequence(tie, mc, policy, q_sat, thr):
    pol = [tie.Policy.FCFS, tie.Policy.SEPT, tie.Policy.TIE][policy]
    rng = np.random.default_rng(31 + policy)
    tot = 6000
    ids = rng.permutation(tot * 4)[:tot].astype(np.uint64)
    arr = np.arange(tot, dtype=np.float64) * 0.01
    mt = rng.integers(16, 4096, tot).astype(np.uint32)
    Eall, Call = _ec(rng, tot)
    qa = tie.GpuScheduler(mc, pol, _cfg(tie, q_sat, thr), tot)
    qb = tie.GpuScheduler(mc, pol, _cfg(tie, q_sat, thr), tot)
    nxt, unpred, popped = 0, [], set()
    for f in range(80):
        a_ids, p_idx, ae, pe = [], [], [], []
        for _ in range(int(rng.integers(1, 7))):
            na = int(rng.integers(0, 9)) if nxt < tot - 10 else 0
            a_ids += range(nxt, nxt + na)
            unpred += range(nxt, nxt + na)
            nxt += na
            ae.append(len(a_ids))
            npd = min(len(unpred), int(rng.integers(0, 9)))
            pick = sorted(rng.choice(len(unpred), npd, replace=False).tolist(), reverse=True)
            p_idx += [unpred.pop(j) for j in pick]
            pe.append(len(p_idx))
        a = np.array(a_ids, np.int64)
        p = np.array(p_idx, np.int64)
        k = int(rng.integers(0, 9))
        args = (ids[a], arr[a], mt[a], np.array(ae, np.uint64), ids[p], Eall[p], Call[p],
                np.array(pe, np.uint64), k)
        got_a = qa.step_ec_runs(*args)
        got_b = _seq_runs(qb, ids[a], arr[a], mt[a], ae, ids[p], Eall[p], Call[p], pe, k)
        assert np.array_equal(got_a, got_b), (f, got_a, got_b)
        popped |= set(got_a.tolist())
        unpred = [u for u in unpred if int(ids[u]) not in popped]
    assert qa.waiting() == qb.waiting()
    assert np.array_equal(qa.next_requests(tot), qb.next_requests(tot))


@pytest.mark.parametrize("case", ["pred_before_arrival", "pred_twice", "arrival_twice",
                                  "bad_cvar"])
def test_step_ec_runs_errors_match_step_sequence(tie, mc, case):
    """an invalid sequence raises the error of the first failing call, with the calls before it
    applied -- exactly as consecutive step_ec calls"""
    rng = np.random.default_rng(5)
    ids = np.arange(100, 160, dtype=np.uint64)
    arr = np.arange(60, dtype=np.float64)
    mt = np.full(60, 512, np.uint32)
    E, C = _ec(rng, 60)
    a = np.arange(10, 30)  # arrivals of the step, 4 runs of 5
    ae = [5, 10, 15, 20]
    p = {"pred_before_arrival": [0, 1, 5, 12, 16],   # 16 arrives in run 3, predicted in run 2
         "pred_twice": [0, 1, 5, 1, 14],
         "arrival_twice": [0, 1, 5, 12, 14],           # arrival 17 repeats 3: run 3 fails
         "bad_cvar": [0, 1, 5, 12, 14]}[case]
    pe = [2, 3, 5, 5]
    aid = ids[a].copy()
    if case == "arrival_twice":
        aid[17] = aid[3]
    pid = aid[p]
    Ec, Cc = E[:5].copy(), C[:5].copy()
    if case == "bad_cvar":
        Cc[3] = Ec[3] * 0.5
    qa = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), 64)
    qb = tie.GpuScheduler(mc, tie.Policy.TIE, _cfg(tie), 64)
    for q in (qa, qb):
        q.on_arrival_batch(ids[:10], arr[:10], mt[:10])
    with pytest.raises(Exception) as ea:
        qa.step_ec_runs(aid, arr[a], mt[a], np.array(ae, np.uint64), pid, Ec, Cc,
                        np.array(pe, np.uint64), 4)
    with pytest.raises(Exception) as eb:
        _seq_runs(qb, aid, arr[a], mt[a], ae, pid, Ec, Cc, pe, 4)
    assert type(ea.value) is type(eb.value) and str(ea.value) == str(eb.value), (ea, eb)
    assert qa.waiting() == qb.waiting()
    assert np.array_equal(qa.next_requests(64), qb.next_requests(64))
