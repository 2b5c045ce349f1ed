"""Summarise an ncu --set full report (.ncu-rep) into per-kernel JSON: duration, DRAM bytes,
throughput fractions, issue / occupancy, FP64 pipe, top stall reasons.  Development tool:
`python tools/ncu_summary.py gpurun_out/prof.ncu-rep > profiles/ncu_X.json`."""
import csv
import io
import json
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,  # -> us
        "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6,
        "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}                 # -> bytes
METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l2_throughput_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l1_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "inst_executed": ("smsp__inst_executed.sum", 1),
}


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, body = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    out = []
    for r in body:
        d = {"kernel": r[col["Kernel Name"]][:120], "id": r[col["ID"]]}
        for k, (m, scale) in METRICS.items():
            if m in col and r[col[m]] not in ("", "n/a"):
                try:
                    d[k] = float(r[col[m]].replace(",", "")) * scale * UNIT.get(
                        units[col[m]], 1.0)
                except ValueError:
                    pass
        stalls = []
        for h, i in col.items():
            if h.startswith("smsp__average_warps_issue_stalled_") and \
                    h.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h[len("smsp__average_warps_issue_stalled_"):
                                                  -len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        d["top_stalls_cycles_per_issue"] = {n: round(v, 2) for v, n in sorted(stalls)[::-1][:4]}
        out.append(d)
    print(json.dumps({"report": path, "kernels": out}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
