"""Pageable-buffer e2e of tie_fit_host (development tool): config 3 (1M x 16) samples and
results in NumPy arrays, median of 7 wall-clocked calls."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00499_b200 as tie  # noqa: E402

P, K = 1_000_000, 16
mc = tie.McContext(3.5, 10000, 12, 0)
x, _, _ = tie.gen_fit_data(P, K, 1)
x = np.ascontiguousarray(x)
outs = [np.zeros(P), np.zeros(P), np.zeros(P), np.zeros(P, np.int32), np.zeros(P, np.uint8),
        np.zeros(P, np.uint8)]
ts = []
for i in range(9):
    t0 = time.perf_counter()
    tie.fit_host_ptr(mc.handle, x.ctypes.data, P, K, 3.5, *[o.ctypes.data for o in outs])
    if i >= 2:
        ts.append(time.perf_counter() - t0)
print(json.dumps({"tag": os.environ.get("TAG", ""), "fit_pageable_ms": round(1e3 * float(np.median(ts)), 2)}))
