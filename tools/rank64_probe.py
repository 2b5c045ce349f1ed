"""Config-4 size (64M) score+rank on one GPU: per-kernel device time (ProfScope events) and the
step time (development tool)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64 * 2 ** 20
mc = tie.McContext(3.5)
ctx = mc.handle
w = tie.gen_logt_workload_soa(n, 1)
mu = torch.from_numpy(w["mu"]).cuda()
sg = torch.from_numpy(w["sigma"]).cuda()
mt = torch.from_numpy(w["max_tokens"].view(np.int32)).cuda()
S = torch.empty(n, dtype=torch.float64, device="cuda")
order = torch.empty(n, dtype=torch.int64, device="cuda")
sh = torch.cuda.current_stream().cuda_stream
step = lambda: tie.score_rank_device(ctx, mu.data_ptr(), sg.data_ptr(), mt.data_ptr(), n, 0.9,
                                     0.5, 0, 0, S.data_ptr(), order.data_ptr(), 0, sh)
for _ in range(2):
    step()
torch.cuda.synchronize()
tie.profile(ctx, True)
step()
torch.cuda.synchronize()
print({k: round(v[1], 3) for k, v in tie.profile_report(ctx).items()})
tie.profile(ctx, False)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    step()
b.record()
torch.cuda.synchronize()
print("n", n, "step ms", a.elapsed_time(b) / 5)
