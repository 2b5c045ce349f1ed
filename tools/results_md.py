"""Render profiles/RESULTS.md from a bench.py JSON line and the reference arm's line
(development tool): python tools/results_md.py profiles/bench_rXX.json profiles/bench_ref_rXX.json
profiles/gpu_tests_rXX.txt > profiles/RESULTS.md"""
import json
import sys


def fmt(x):
    return f"{x:.3e}"


def main(bench, ref, tests):
    d = json.load(open(bench))
    r = json.load(open(ref)) if ref else None
    c = d["clocks"]
    L = [f"# Results (round 2)", "",
         f"1x B200 via gpurun, `python bench.py` ({bench}); reference arm `python bench.py "
         f"--impl reference` ({ref}).",
         "Config 2 = 1M-request queue (gen_logt_workload seed 1), McContext(3.5, 10000, 12), "
         "alpha 0.9, beta 0.5; L2 flushed between timed steps.",
         f"Clocks during the timed region: {c['sm_mhz']} MHz median (max {c['sm_max_mhz']}), "
         f"throttle reasons: {', '.join(c['reasons']) or 'none'}.", "",
         "| metric | value |", "|---|---|",
         f"| score+rank, inputs in HBM (`value`) | {fmt(d['value'])} req/s "
         f"({1e3 * d['ms_per_step']:.1f} us/step) |",
         f"| score+rank end to end, C-ABI host call, pinned (`e2e`) | {fmt(d['e2e']['value'])} "
         f"req/s ({1e3 * d['e2e']['ms_per_step']:.0f} us, {d['e2e']['statistic']}; 20 MB H2D + "
         f"8 MB D2H per call) |"]
    pg = d["e2e"].get("pageable")
    if pg:
        L.append(f"| e2e on pageable NumPy buffers | {fmt(pg['value'])} req/s "
                 f"({1e3 * pg['ms_per_step']:.0f} us) |")
    if d.get("context"):
        L.append(f"| McContext creation (once per process, excluded from steps) | "
                 f"{d['context']['create_ms']:.0f} ms, {d['context']['device_bytes'] / 1e6:.0f} MB |")
    if r and "value" in r:
        L += [f"| reference arm (`--impl reference`: oracle/_ref, {r['cpu_baseline']['cores']} "
              f"cores, the full 1M queue per step) | {fmt(r['value'])} req/s |",
              f"| e2e / reference arm | {d['e2e']['value'] / r['value']:.0f}x |"]
    cb = d["cpu_baseline"]
    L += [f"| `cpu_baseline` in the bench line ({cb['kind']}, {cb['cores']} cores) | "
          f"{fmt(cb['value'])} req/s |",
          f"| exact per-term score path + rank | {fmt(d['exact_path']['value'])} req/s |",
          f"| config 3 fits (1M x 16), device | {fmt(d['fit']['value'])} fits/s "
          f"({d['fit']['ms']:.1f} ms) |",
          f"| config 3 fits, e2e (host buffers) | {fmt(d['fit']['e2e']['value'])} fits/s |",
          *([f"| config 3 fits, e2e on pageable NumPy buffers | "
             f"{fmt(d['fit']['e2e']['pageable']['value'])} fits/s "
             f"({d['fit']['e2e']['pageable']['ms']:.1f} ms) |"]
            if 'pageable' in d['fit']['e2e'] else []),
          f"| north-star fits, 10M x 16, one GPU | {fmt(d['fit_10M']['value'])} fits/s "
          f"({d['fit_10M']['ms']:.0f} ms) |",
          f"| config 5 trace simulation (run_sim, canonical.json, rebuild_threshold 0) | "
          f"{d['config5_sim']['ms_per_sim']:.0f} ms/sim vs reference "
          f"{d['config5_sim']['reference']['ms_per_sim']:.0f} ms "
          f"({d['config5_sim']['speedup_vs_reference']:.1f}x), events identical: "
          f"{d['config5_sim']['events_identical_to_reference']} |",
          f"| `tie fit` analysis (4 families + KS + tail), 1M x 16 | "
          f"{fmt(d['fit_report']['value'])} prompts/s ({d['fit_report']['ms']:.0f} ms) |",
          f"| config 4 size (64M requests) on one GPU | "
          f"{fmt(d['config4_single_gpu']['value'])} req/s "
          f"({d['config4_single_gpu']['ms_per_step']:.1f} ms) |"]
    rm = d["rank0_merge"]
    L.append("| rank-0 final step, G x 1M runs: k-way merge / re-sort (ms) | " + ", ".join(
        f"{g} {rm[g]['kmerge_ms']:.3f} / {rm[g]['stable_resort_ms']:.3f}"
        for g in ("G2", "G4", "G8")) + " |")
    ss = d["schedule_step"]["results"]
    L += ["", "Schedule step p50 (32 arrivals + 32 scored predictions + 8 pops per step through "
          "`tie_queue_step`, wall clock incl. host I/O) vs resident queue size; steady = beta "
          "saturated (q_sat 128), rekey = rebuild_threshold 0 with beta moving every pop (the "
          "survey's \"re-scoring every step\"); CPU = the reference Scheduler, 1 thread (sizes "
          "above 1M: GPU only):", "",
          "| variant | n | GPU p50 us | CPU p50 us | speed-up | pops identical |",
          "|---|---|---|---|---|---|"]
    for v in ("steady", "rekey"):
        for n, x in ss[v].items():
            cpu, gpu = x.get("cpu_p50_us"), x["gpu_p50_us"]
            cpu_s = f"{cpu:.0f}" if cpu else "-"
            sp = f"{cpu / gpu:.0f}x" if cpu else "-"
            L.append(f"| {v} | {int(n):,} | {gpu:.1f} | {cpu_s} | {sp} | "
                     f"{x.get('pops_identical', '-')} |")
    k = d["kernels_ms_per_step"]
    L += ["", "Per-kernel device time per step (event-bracketed): " + ", ".join(
        f"{n} {1e3 * v:.1f} us" for n, v in k.items()), ""]
    for ro in [d["roofline"]] + list(d.get("roofline_other_kernels", {}).values()):
        lim = ro.get("limiter", {})
        L.append(f"Roofline {ro['kernel']}: {ro['algorithmic_bytes_per_unit']:.0f} B/request "
                 f"algorithmic -> {ro['achieved']:.0f} {ro['unit']} = {100 * ro['frac']:.1f}% of "
                 f"the measured {ro['peak']} {ro['unit']}; DRAM traffic "
                 f"{(ro['traffic'] or 0) / 1e6:.1f} MB/launch (ncu); limiter: L1 "
                 f"{lim.get('l1_throughput_pct')}%, issue {lim.get('issue_active_pct')}%, FP64 "
                 f"pipe {lim.get('fp64_pipe_pct')}%, top stalls {lim.get('top_stalls')}.")
        if "fp64_pipe" in ro:
            fp = ro["fp64_pipe"]
            L.append(f"  FP64-pipe roofline (SURVEY 8d K1, ncu-executed): {100 * fp['frac']:.1f}% "
                     f"of the FP64 pipe, issue {100 * fp['issue_frac']:.1f}%, "
                     f"{fp['inst_executed_per_request']:.1f} warp-instructions per request.")
        L.append("")
    fe = d.get("score_effective")
    if fe:
        L += [f"Effective rate vs the reference arithmetic: {fe['sample_terms_per_launch']:.3e} "
              f"sample-terms x {fe['flops_per_term']} flops per launch = "
              f"{fe['effective_tflops']:.0f} TFLOP/s equivalent -- the moment tables replace "
              f"~9,900 exp per request with two table rows (not executed flops).", ""]
    fr = d.get("fit", {}).get("roofline")
    if fr:
        L += [f"Roofline fit.lanes (SURVEY 8d K3, FP64 pipe, ncu): {100 * fr['frac']:.1f}% of the "
              f"FP64 pipe, issue {100 * fr['issue_frac']:.1f}%, top stalls {fr['top_stalls']}.", ""]
    if tests:
        last = open(tests).read().strip().splitlines()[-1]
        L.append(f"Parity on the same box: {tests} (`pytest tests -m gpu`: {last.strip()}).")
    print("\n".join(L))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None,
         sys.argv[3] if len(sys.argv) > 3 else None)
