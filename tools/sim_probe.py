"""config-5 run_sim timing probe (development tool): per-sim wall time of tie.run_sim on the
canonical trace, median of 5, with the flush statistics when TIE_SIM_STATS is set."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
if os.environ.get("WITH_TORCH"):
    import torch  # noqa: F401
    torch.zeros(1).cuda()
import paper_2604_00499_b200 as tie  # noqa: E402
from oracle_lib import CANONICAL as c  # noqa: E402

ws = tie.WorkloadSpec()
ws.n_requests, ws.rps = c["n"], c["rps"]
ws.mu_range, ws.sigma_range = c["mu_range"], c["sigma_range"]
ws.prompt_range, ws.max_tokens = c["prompt_range"], c["max_tokens"]
sc = tie.ScoreConfig()
sc.rebuild_threshold = float(os.environ.get("THR", "0"))
ec, pc = tie.EngineConfig(), tie.PredictorConfig()
seed = int(os.environ.get("SEED", "1"))
w = tie.gen_logt_workload(ws, seed)
tie.run_sim(w, tie.Policy.TIE, sc, ec, pc, seed)
if os.environ.get("WITH_REF"):
    from oracle_lib import RefLib, ref_run_sim
    ref_run_sim(RefLib(), 1, 2, 1, threshold=0.0)
tie.launch_count(True)
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    r = tie.run_sim(w, tie.Policy.TIE, sc, ec, pc, seed)
    ts.append(time.perf_counter() - t0)
print(json.dumps({"tag": os.environ.get("TAG", ""), "seed": seed,
                  "launches_per_sim": tie.launch_count(False) / 5,
                  "ms_per_sim": round(1e3 * float(np.median(ts)), 1),
                  "all_ms": [round(1e3 * t, 1) for t in ts],
                  "admit_sum": float(sum(e.admit_s for e in r.events))}))
