"""Partition-size statistics of the rank path's bucket mappings on the config-2 (1M) and
config-4 (64M) queues (development tool): the power-of-two shift mapping vs an exact-span
(multiply-high) mapping, at the level-1 / level-2 partition granularities."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie  # noqa: E402


def stats(name, counts, cap=1408):
    c = counts[counts > 0]
    print(f"  {name}: P={len(counts)} used={len(c)} mean={c.mean():.0f} p50={np.median(c):.0f} "
          f"p99={np.percentile(c, 99):.0f} max={c.max()} frac>{cap}={np.mean(c > cap):.3f} "
          f"keys_in>{cap}={c[c > cap].sum() / c.sum():.3f}")


mc = tie.McContext(3.5)
for n, B in ((1_000_000, 10), (64 * 2 ** 20, 16)):
    w = tie.gen_logt_workload_soa(n, 1)
    mu = torch.from_numpy(w["mu"]).cuda()
    sg = torch.from_numpy(w["sigma"]).cuda()
    mt = torch.from_numpy(w["max_tokens"].view(np.int32)).cuda()
    S = torch.empty(n, dtype=torch.float64, device="cuda")
    sh = torch.cuda.current_stream().cuda_stream
    tie.score_device(mc.handle, mu.data_ptr(), sg.data_ptr(), mt.data_ptr(), True, n, 0.9, 0.5,
                     0, 0, S.data_ptr(), 0, sh)
    torch.cuda.synchronize()
    k = (S.cpu().numpy().view(np.uint64) | np.uint64(1 << 63))
    kmin, kmax = int(k.min()), int(k.max())
    span = kmax - kmin
    bits = span.bit_length()
    print(f"n={n} span bits={bits} used fraction of 2^bits: {span / 2 ** bits:.3f}")
    d = (k - np.uint64(kmin)).astype(np.uint64)
    pw = (d >> np.uint64(bits - B)).astype(np.int64)
    stats(f"shift  B={B}", np.bincount(pw, minlength=1 << B))
    ex = np.floor(d.astype(np.float64) / (span + 1.0) * (1 << B)).astype(np.int64)
    stats(f"exact  B={B}", np.bincount(ex, minlength=1 << B))
    del mu, sg, mt, S
