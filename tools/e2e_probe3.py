"""e2e breakdown (development tool): the fused score+rank device call with its inputs and/or
its order in pinned host memory (UVA zero-copy) vs in HBM, CUDA-event timed, next to the
host-API call (tie_score_rank_host) -- what of the e2e time is PCIe, kernels and host work."""
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
h = {"mu": pin(w["mu"]), "sg": pin(w["sigma"]), "mt": pin(w["max_tokens"].view(np.int32))}
d = {k: v.cuda() for k, v in h.items()}
o_h = torch.empty(n, dtype=torch.int64).pin_memory()
o_d = torch.empty(n, dtype=torch.int64, device="cuda")
S = torch.empty(n, dtype=torch.float64, device="cuda")
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
sh = st.cuda_stream


def dev_call(src, out):
    tie.score_rank_device(ctx, src["mu"].data_ptr(), src["sg"].data_ptr(), src["mt"].data_ptr(),
                          n, 0.9, 0.5, 0, 0, S.data_ptr(), out.data_ptr(), 0, sh)


res = {}
for name, src, out in (("hbm_in_hbm_out", d, o_d), ("pinned_in_hbm_out", h, o_d),
                       ("hbm_in_pinned_out", d, o_h), ("pinned_in_pinned_out", h, o_h)):
    for _ in range(3):
        dev_call(src, out)
    ts = []
    for _ in range(20):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        dev_call(src, out)
        b.record(st)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    res[name + "_us"] = round(float(np.median(ts)), 1)
tie.sync(ctx, sh)
ts = []
for i in range(40):
    t0 = time.perf_counter()
    tie.score_rank_host_ptr(ctx, h["mu"].data_ptr(), h["sg"].data_ptr(), h["mt"].data_ptr(), n,
                            0.9, 0.5, 0, o_h.data_ptr(), 0)
    if i >= 5:
        ts.append(time.perf_counter() - t0)
res["host_api_us"] = round(1e6 * float(np.median(ts)), 1)
print(json.dumps(res))
