"""profiles/ncu_*_summary.json (tools/ncu_summary.py) -> the per-kernel traffic / limiter file
bench.py reads (profiles/ncu_traffic_*.json).  Usage:
    python tools/make_traffic.py profiles/ncu_traffic_r02x.json summary.json:N [summary.json:N ...]
(N = the requests / prompts per launch of that capture; the first summary naming a kernel wins)
"""
import json
import sys

NAMES = {"score_coop": "score.moment", "part_fused": "rank.fused", "part_count": "rank.count",
         "part_scatter": "rank.scatter", "part_sort": "rank.local", "part_l2": "rank.local",
         "onesweep": "rank.onesweep", "fit_lanes": "fit.lanes", "step_apply": "queue.step_apply"}


def main(dst, *srcs):
    out = {"note": "dram__bytes_read.sum + dram__bytes_write.sum per launch and the limiter "
                   "metrics from `ncu --set full --clock-control none` (" +
                   ", ".join(s.rsplit(":", 1)[0] for s in srcs) + "); ncu flushes caches "
                   "before each replayed kernel, so reads come from DRAM."}
    for spec in srcs:
        src, n = spec.rsplit(":", 1)
        d = json.load(open(src))
        for k in d["kernels"]:
            for frag, nm in NAMES.items():
                if frag not in k["kernel"] or nm in out:
                    continue
                out[nm] = {"n": int(n),
                           "dram_read_bytes": k.get("dram_read_bytes"),
                           "dram_write_bytes": k.get("dram_write_bytes"),
                           "duration_us": round(k["duration_us"], 2),
                           "l1_throughput_pct": round(k.get("l1_throughput_pct", 0), 1),
                           "issue_active_pct": round(k.get("issue_active_pct", 0), 1),
                           "fp64_pipe_pct": round(k.get("fp64_pipe_pct", 0), 1),
                           "inst_executed": k.get("inst_executed"),
                           "registers": k.get("registers"),
                           "achieved_occupancy_pct": round(k.get("achieved_occupancy_pct", 0), 1),
                           "top_stalls": k.get("top_stalls_cycles_per_issue"),
                           "capture": f"{src} id {k['id']} ({d.get('report', '?')})"}
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
