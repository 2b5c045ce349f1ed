"""Schedule-step p50 of the package next to this script's parent (development tool: same-box
A/B of two builds -- python tools/sched_ab.py [root]): bench_sched.run steady + rekey, no CPU
side, sizes 1k / 1M / 10M."""
import json
import os
import sys

root = os.path.abspath(sys.argv[1]) if len(sys.argv) > 1 else \
    os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import bench_sched  # noqa: E402
import paper_2604_00499_b200 as tie  # noqa: E402

assert os.path.dirname(tie.__file__).startswith(root), tie.__file__
mc = tie.McContext(3.5)
r = bench_sched.run(tie, mc, sizes=(1000, 1_000_000, 10_000_000), cpu=False)
print(json.dumps({"root": os.path.basename(root) or root,
                  **{v: {n: round(x["gpu_p50_us"], 1) for n, x in rr.items()}
                     for v, rr in r.items()}}))
