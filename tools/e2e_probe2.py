"""e2e interaction probe: the host-API score+rank call measured alone, then after the
device-pointer path has run on torch's stream, then after tie.sync (development tool)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00499_b200 as tie  # noqa: E402

n = 1_000_000
mc = tie.McContext(3.5, 10000, 12, 0)
ctx = mc.handle
w = tie.gen_logt_workload_soa(n, 1)
pin = lambda a: torch.from_numpy(a).pin_memory()
mu_p, sg_p, mt_p = pin(w["mu"]), pin(w["sigma"]), pin(w["max_tokens"].view(np.int32))
ord_p = torch.empty(n, dtype=torch.int64).pin_memory()
dev = torch.device("cuda", 0)
mu, sg, mt = mu_p.to(dev), sg_p.to(dev), mt_p.to(dev)
S = torch.empty(n, dtype=torch.float64, device=dev)
order = torch.empty(n, dtype=torch.int64, device=dev)
sh = torch.cuda.current_stream().cuda_stream


def e2e(reps=30):
    ts = []
    for i in range(reps + 5):
        t0 = time.perf_counter()
        tie.score_rank_host_ptr(ctx, mu_p.data_ptr(), sg_p.data_ptr(), mt_p.data_ptr(), n, 0.9,
                                0.5, 0, ord_p.data_ptr(), 0)
        if i >= 5:
            ts.append(time.perf_counter() - t0)
    return round(float(np.median(ts)) * 1e3, 3), round(float(np.max(ts)) * 1e3, 3)


out = {"alone": e2e()}
for _ in range(50):
    tie.score_rank_device(ctx, mu.data_ptr(), sg.data_ptr(), mt.data_ptr(), n, 0.9, 0.5, 0, 0,
                          S.data_ptr(), order.data_ptr(), 0, sh)
torch.cuda.synchronize()
out["after_device_path"] = e2e()
tie.sync(ctx, sh)
out["after_sync"] = e2e()
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
flush.zero_()
torch.cuda.synchronize()
out["after_flush_alloc"] = e2e()
print(json.dumps(out))
