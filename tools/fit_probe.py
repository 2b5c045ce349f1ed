"""Probe (not a test): time the fit kernel on config-3 prompts at several sizes / K.
    python tools/fit_probe.py [P]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2604_00499_b200 as tie  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
ctx = tie.default_context()
for K in (16,):
    x, _, _ = tie.gen_fit_data(P, K, 1)
    xd = torch.from_numpy(x).cuda()
    outs = [torch.empty(P, dtype=t, device="cuda") for t in
            (torch.float64, torch.float64, torch.float64, torch.int32, torch.uint8, torch.uint8)]
    s = torch.cuda.current_stream().cuda_stream
    args = (ctx, xd.data_ptr(), P, K, 3.5, *[o.data_ptr() for o in outs], s)
    tie.fit_device(*args)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    tie.fit_device(*args)
    b.record()
    torch.cuda.synchronize()
    it = outs[3].cpu().numpy()
    print(f"K={K} P={P}: {a.elapsed_time(b):.2f} ms; iterations mean {it.mean():.2f} "
          f"max {it.max()} (>=100: {(it >= 100).sum()}, 500: {(it >= 500).sum()})")
