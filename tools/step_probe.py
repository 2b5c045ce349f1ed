"""schedule-step latency breakdown (development tool): p50 of tie_queue_step variants."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie

n, steps, per = (int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000), 200, 32
mc = tie.McContext(3.5)
w = tie.gen_logt_workload_soa(n + steps * per * 4, 7)
mu, sg, mt = w["mu"], w["sigma"], w["max_tokens"]
ids = np.arange(len(mu), dtype=np.uint64)
cfg = tie.ScoreConfig()
E, C, _ = tie.score_batch(mu[:n], sg[:n], mt[:n].astype(np.float64), mc, cfg)
q = tie.GpuScheduler(mc, tie.Policy.TIE, cfg, len(mu))
q.on_arrival_batch(ids[:n], np.zeros(n), mt[:n])
q.on_prediction_batch(ids[:n], E, C)
e64, e32 = np.empty(0, np.uint64), np.empty(0, np.uint32)
z = np.zeros(per)
cur = n
res = {}
for name, (na, npred, pops) in {"empty": (0, 0, 0), "arrive": (per, 0, 0), "arrive+pred": (per, per, 0),
                                "pops_only": (0, 0, 8), "full": (per, per, 8)}.items():
    lat = []
    for s in range(steps):
        a = slice(cur, cur + na)
        t0 = time.perf_counter()
        q.step(ids[a], z[:na], mt[a], ids[a][:npred], mu[a][:npred], sg[a][:npred], mt[a][:npred], pops)
        lat.append(time.perf_counter() - t0)
        cur += na
    res[name] = round(1e6 * float(np.median(lat)), 1)
print(res)
