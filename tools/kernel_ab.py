"""A/B timing of the score kernel variants (flags) and the fused score+rank step on the
config-2 queue (1M requests, seed 1), CUDA events on the launching stream, L2 flushed before
every timed launch.  Development tool: `python tools/kernel_ab.py [flags ...]`."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00499_b200 as tie  # noqa: E402


def main():
    flags_list = [int(a, 0) for a in sys.argv[1:]] or [0]
    n = 1_000_000
    dev = torch.device("cuda", 0)
    mc = tie.McContext(3.5, 10000, 12, 0)
    w = tie.gen_logt_workload_soa(n, 1)
    mu = torch.from_numpy(w["mu"]).to(dev)
    sg = torch.from_numpy(w["sigma"]).to(dev)
    mt = torch.from_numpy(w["max_tokens"].view(np.int32)).to(dev)
    S = torch.empty(n, dtype=torch.float64, device=dev)
    ref = torch.empty_like(S)
    order = torch.empty(n, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = torch.cuda.current_stream()
    sh = st.cuda_stream
    out = {}
    for fl in flags_list:
        def score():
            tie.score_device(mc.handle, mu.data_ptr(), sg.data_ptr(), mt.data_ptr(), True, n,
                             0.9, 0.5, 0, 0, S.data_ptr(), fl, sh)

        def step():
            tie.score_rank_device(mc.handle, mu.data_ptr(), sg.data_ptr(), mt.data_ptr(), n,
                                  0.9, 0.5, 0, 0, S.data_ptr(), order.data_ptr(), fl, sh)

        res = {}
        for name, fn in (("score", score), ("score_rank", step)):
            for _ in range(3):
                fn()
            ts = []
            for _ in range(20):
                if not os.environ.get("AB_NO_FLUSH"):
                    flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(st)
                fn()
                b.record(st)
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3)
            res[name + "_us_median"] = float(np.median(ts))
            res[name + "_us_min"] = float(np.min(ts))
        tie.sync(mc.handle, sh)
        if fl == flags_list[0]:
            ref.copy_(S)
        res["max_abs_diff_vs_first"] = float((S - ref).abs().max().item())
        out[hex(fl)] = res
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
