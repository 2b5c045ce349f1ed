"""e2e probe: PCIe copy rates next to the score+rank host-API call (tie_score_rank_host) on the
config-2 queue, median over many calls.  Development tool (env vars select internal A/B
switches of the host path)."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00499_b200 as tie  # noqa: E402


def med(f, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3


def main():
    n = 1_000_000
    mc = tie.McContext(3.5, 10000, 12, 0)
    w = tie.gen_logt_workload_soa(n, 1)
    pin = lambda a: torch.from_numpy(a).pin_memory()
    mu, sg, mt = pin(w["mu"]), pin(w["sigma"]), pin(w["max_tokens"].view(np.int32))
    order = torch.empty(n, dtype=torch.int64).pin_memory()
    big_h = torch.empty(20_000_000 // 4, dtype=torch.float32).pin_memory()
    big_d = torch.empty_like(big_h, device="cuda")
    o_h = torch.empty(8_000_000 // 4, dtype=torch.float32).pin_memory()
    o_d = torch.empty_like(o_h, device="cuda")

    def h2d():
        big_d.copy_(big_h, non_blocking=True)
        torch.cuda.synchronize()

    def d2h():
        o_h.copy_(o_d, non_blocking=True)
        torch.cuda.synchronize()

    def e2e():
        tie.score_rank_host_ptr(mc.handle, mu.data_ptr(), sg.data_ptr(), mt.data_ptr(), n, 0.9,
                                0.5, 0, order.data_ptr(), 0)

    for f in (h2d, d2h, e2e):
        med(f, 5)
    res = {}
    for rnd in range(3):
        res[f"h2d_20MB_ms_{rnd}"] = med(h2d, 30)
        res[f"d2h_8MB_ms_{rnd}"] = med(d2h, 30)
        res[f"e2e_ms_{rnd}"] = med(e2e, 50)
    res["env"] = {k: v for k, v in os.environ.items() if k.startswith("TIE_")}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
