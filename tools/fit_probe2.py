"""config-3 fit run for profiling (development tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie

P, K = 1_000_000, 16
mc = tie.McContext(3.5)
x, _, _ = tie.gen_fit_data(P, K, 1)
xd = torch.from_numpy(x).cuda()
outs = [torch.empty(P, dtype=t, device="cuda") for t in (torch.float64, torch.float64, torch.float64, torch.int32, torch.uint8, torch.uint8)]
sh = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    tie.fit_device(mc.handle, xd.data_ptr(), P, K, 3.5, *[o.data_ptr() for o in outs], sh)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    tie.fit_device(mc.handle, xd.data_ptr(), P, K, 3.5, *[o.data_ptr() for o in outs], sh)
b.record()
torch.cuda.synchronize()
tie.sync(mc.handle, sh)
print("fit ms", a.elapsed_time(b) / 3, "mu[:3]", outs[0][:3].tolist())
