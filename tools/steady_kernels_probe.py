"""Kernels of the steady scheduler step (development tool, run under ncu): bench_sched's steady
variant at a 1k queue, 60 steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench_sched  # noqa: E402
import paper_2604_00499_b200 as tie  # noqa: E402

mc = tie.McContext(3.5)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
bench_sched.run(tie, mc, sizes=(n,), steps=60, variants=("steady",), cpu=False)
