"""profiles/ncu_*_summary.json (tools/ncu_summary.py) -> the per-kernel traffic / limiter file
bench.py reads (profiles/ncu_traffic_*.json).  Usage:
    python tools/make_traffic.py profiles/ncu_r01h_summary.json profiles/ncu_traffic_r01h.json N
"""
import json
import sys

NAMES = {"score_coop": "score.moment", "part_fused": "rank.fused", "part_count": "rank.count",
         "part_scatter": "rank.scatter", "part_sort": "rank.local", "onesweep": "rank.onesweep"}


def main(src, dst, n):
    d = json.load(open(src))
    out = {"note": "dram__bytes_read.sum + dram__bytes_write.sum per launch and the limiter "
                   "metrics from `ncu --set full --clock-control none` (" + src + "); ncu "
                   "flushes caches before each replayed kernel, so reads come from DRAM.",
           "n": int(n)}
    for k in d["kernels"]:
        for frag, nm in NAMES.items():
            if frag in k["kernel"] and nm not in out:
                out[nm] = {"dram_read_bytes": k.get("dram_read_bytes"),
                           "dram_write_bytes": k.get("dram_write_bytes"),
                           "duration_us": round(k["duration_us"], 2),
                           "l1_throughput_pct": round(k.get("l1_throughput_pct", 0), 1),
                           "issue_active_pct": round(k.get("issue_active_pct", 0), 1),
                           "fp64_pipe_pct": round(k.get("fp64_pipe_pct", 0), 1),
                           "top_stalls": k.get("top_stalls_cycles_per_issue"),
                           "capture": f"{src} id {k['id']}" + (f" ({k['report']})" if "report" in k else "")}
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:4])
