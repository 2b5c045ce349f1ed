import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_2604_00499_b200 as tie
mc = tie.McContext(3.5, 10000, 12, 0)
sc = tie.ScoreConfig(); sc.q_sat = 1e9; sc.rebuild_threshold = 0.0
q = tie.GpuScheduler(mc, tie.Policy.TIE, sc, 200000)
rng = np.random.default_rng(1)
nid = 0
def arrive(m):
    global nid
    ids = np.arange(nid, nid + m, dtype=np.uint64); nid += m
    return ids
q.on_arrival_batch(arrive(300), np.zeros(300), np.full(300, 512, np.uint32))
E0 = np.array([]); U = np.array([], np.uint64)
for label, na, npd, k in (("arr1_k0", 1, 0, 0), ("arr1_k1", 1, 0, 1), ("arr1_pred1_k0", 1, 1, 0),
                          ("arr1_pred1_k1", 1, 1, 1), ("empty_k1", 0, 0, 1), ("empty_k0", 0, 0, 0)):
    ts = []
    for it in range(400):
        ids = arrive(na)
        pid = ids[:npd]
        e = rng.uniform(10, 500, npd); c = e * 1.5
        t0 = time.perf_counter()
        q.step_ec(ids, np.zeros(na), np.full(na, 512, np.uint32), pid, e, c, k)
        ts.append(time.perf_counter() - t0)
    print(label, round(1e6 * float(np.median(ts[50:])), 1), "us")
