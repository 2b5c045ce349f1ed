"""k-way merge probe: 8 sorted 1M runs merged by tie_merge_runs (development tool)."""
import sys, os
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie
from paper_2604_00499_b200.dist import DeviceOps

G, L = 8, 1_000_000
rng = np.random.default_rng(1)
k = np.sort(rng.lognormal(5, 0.5, (G, L)), axis=1)
i = np.arange(G * L, dtype=np.int64).reshape(G, L)
ops = DeviceOps(tie.McContext(3.5), 0.9)
kd, idd = torch.from_numpy(k).cuda(), torch.from_numpy(i).cuda()
for _ in range(3):
    ops.merge_runs(kd, idd, [L] * G)
torch.cuda.synchronize()
ops.sync()
print("ok")
