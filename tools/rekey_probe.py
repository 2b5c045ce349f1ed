"""Schedule-step p50 in the re-key-every-pop regime (rebuild_threshold 0) at given queue
sizes (development tool): python tools/rekey_probe.py 1000000,10000000 <cpu_max_n>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench_sched  # noqa: E402
import paper_2604_00499_b200 as tie  # noqa: E402

sizes = tuple(int(x) for x in sys.argv[1].split(","))
r = bench_sched.run(tie, tie.McContext(3.5), sizes=sizes, variants=("rekey",),
                    cpu_max_n=int(sys.argv[2]) if len(sys.argv) > 2 else 0)
print(json.dumps({k: (round(v["gpu_p50_us"], 1), v.get("pops_identical"))
                  for k, v in r["rekey"].items()}))
