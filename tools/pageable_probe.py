"""Pageable-buffer e2e of tie_score_rank_host (development tool): NumPy inputs / order, 1M
requests, median of 15 wall-clocked calls, checked against the pinned call."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00499_b200 as tie  # noqa: E402

n = 1_000_000
mc = tie.McContext(3.5, 10000, 12, 0)
w = tie.gen_logt_workload_soa(n, 1)
mu, sg, mt = w["mu"].copy(), w["sigma"].copy(), w["max_tokens"].copy()
o = np.empty(n, np.uint64)
ts = []
for i in range(18):
    t0 = time.perf_counter()
    tie.score_rank_host_ptr(mc.handle, mu.ctypes.data, sg.ctypes.data, mt.ctypes.data, n, 0.9,
                            0.5, 0, o.ctypes.data, 0)
    if i >= 3:
        ts.append(time.perf_counter() - t0)
print(json.dumps({"tag": os.environ.get("TAG", ""), "pageable_us": round(1e6 * float(np.median(ts)), 1),
                  "min_us": round(1e6 * min(ts), 1)}))
