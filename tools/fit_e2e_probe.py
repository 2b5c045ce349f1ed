"""config-3 fits through the C-ABI host call on pinned buffers (e2e), median of 10 calls, next
to the device-only fit (development tool; env vars select host-path A/B switches)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie  # noqa: E402

P, K = 1_000_000, 16
mc = tie.McContext(3.5)
x, _, _ = tie.gen_fit_data(P, K, 1)
xp = torch.from_numpy(x).pin_memory()
outs = [torch.empty(P, dtype=t).pin_memory() for t in
        (torch.float64, torch.float64, torch.float64, torch.int32, torch.uint8, torch.uint8)]
f = lambda: tie.fit_host_ptr(mc.handle, xp.data_ptr(), P, K, 3.5, *[o.data_ptr() for o in outs])
f()
ts = []
for _ in range(10):
    t0 = time.perf_counter()
    f()
    ts.append(time.perf_counter() - t0)
print({"e2e_ms": round(1e3 * float(np.median(ts)), 3), "mu0": float(outs[0][0]),
       "env": {k: v for k, v in os.environ.items() if k.startswith("TIE_")}})
