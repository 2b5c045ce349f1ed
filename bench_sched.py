"""Schedule-step latency vs queue size (the second half of BASELINE.json's metric; SURVEY.md
8d "Schedule-step latency", config 5's "re-scoring every step").

A step is one scheduler iteration of the reference's run_sim loop at a resident queue of n
predicted requests: 32 arrivals (Scheduler::on_arrival), their predictions scored and
applied (run_sim's chain sim.cpp:85-94 + Scheduler::on_prediction), then up to B = 8
next_request() pops (the engine's batch slots, sim.hpp:15-20).  Variants:

  steady : ScoreConfig{} (q_sat = 128): beta is saturated at 0.5, no drift rebuilds.
  rekey  : q_sat = 1e9, rebuild_threshold = 0: beta moves with every queue-length change, so
           the reference re-keys and re-heapifies the whole queue before EVERY pop.

GPU side: tie_queue (paper_2604_00499_b200.GpuScheduler.step -> tie_queue_step: the whole
iteration in one packed H2D, the kernels, one packed D2H and one sync), wall-clocked per step
including H2D/D2H.  CPU side: the untouched reference Scheduler (oracle/_ref, one thread -- the
reference scheduler is single-threaded) through oracle/ref_harness.cpp:ref_sched_bench,
timed per step with steady_clock.  Both see identical inputs; the popped id sequences are
compared (parity).
"""
from __future__ import annotations

import ctypes
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import REF_SO, ref_available

    if not ref_available():
        return None
    L = ctypes.CDLL(REF_SO)
    d, u64, p, i32, u32 = ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32
    L.ref_sched_bench.argtypes = [i32, i32, d, d, d, d, u64, p, p, p, p, u64, u64, p, p, p, p,
                                  u32, p, p, ctypes.POINTER(u64)]
    L.ref_last_error.restype = ctypes.c_char_p
    return L


def run(tie, mc, sizes=(1000, 10_000, 100_000, 1_000_000, 10_000_000, 64 * 2 ** 20), steps=120,
        per_step=32, pops=8,
        variants=("steady", "rekey"), cpu=True, cpu_max_n=1_000_000):
    ptr = lambda a: a.ctypes.data
    L = _ref() if cpu else None
    out = {v: {} for v in variants}
    for n in sizes:  # one workload per queue size, shared by the variants
        tot = n + steps * per_step
        w = tie.gen_logt_workload_soa(tot, 7)
        mu, sg, mt = w["mu"], w["sigma"], w["max_tokens"]
        ids = np.arange(tot, dtype=np.uint64)
        for variant in variants:
            q_sat = 128.0 if variant == "steady" else 1e9
            thr = 0.1 if variant == "steady" else 0.0
            res = out[variant]
            cfg = tie.ScoreConfig()
            cfg.q_sat = q_sat
            cfg.rebuild_threshold = thr
            # preload n resident predicted requests (untimed); E/CVaR from the GPU score path
            E, C, _ = tie.score_batch(mu[:n], sg[:n], mt[:n].astype(np.float64), mc, cfg)
            q = tie.GpuScheduler(mc, tie.Policy.TIE, cfg, tot)
            q.on_arrival_batch(ids[:n], np.zeros(n), mt[:n])
            q.on_prediction_batch(ids[:n], E, C)
            lat, popped = [], []
            zeros = np.zeros(per_step)
            for s in range(steps):
                lo, hi = n + s * per_step, n + (s + 1) * per_step
                t0 = time.perf_counter()
                # one fused device round trip (tie_queue_step) == on_arrival_batch +
                # on_prediction_logt + next_requests (tests/test_gpu_queue.py)
                got = q.step(ids[lo:hi], zeros, mt[lo:hi], ids[lo:hi], mu[lo:hi], sg[lo:hi],
                             mt[lo:hi], pops)
                lat.append(time.perf_counter() - t0)
                popped.append(got)
            gpu_pop = np.concatenate(popped)
            r = {"gpu_p50_us": 1e6 * float(np.median(lat)),
                 "gpu_p90_us": 1e6 * float(np.percentile(lat, 90)), "steps": steps}
            if L is not None and n <= cpu_max_n:
                cpu_steps = (steps if (variant == "steady" or n <= 100_000)
                             else max(20, steps // 6))
                secs = np.empty(cpu_steps)
                pop_ref = np.empty(cpu_steps * pops, np.uint64)
                npop = ctypes.c_uint64(0)
                rc = L.ref_sched_bench(2, 1, 0.5, q_sat, thr, 0.9, n, ptr(ids), ptr(mt),
                                       ptr(E), ptr(C), cpu_steps, per_step, ptr(ids[n:]),
                                       ptr(mu[n:]), ptr(sg[n:]), ptr(mt[n:]), pops, ptr(secs),
                                       ptr(pop_ref), ctypes.byref(npop))
                if rc:
                    r["cpu_error"] = L.ref_last_error().decode()
                else:
                    ref_pop = pop_ref[: npop.value]
                    ref_pop = ref_pop[ref_pop != np.iinfo(np.uint64).max]
                    m = min(len(ref_pop), len(gpu_pop))
                    r.update({"cpu_p50_us": 1e6 * float(np.median(secs)),
                              "cpu_p90_us": 1e6 * float(np.percentile(secs, 90)),
                              "cpu_steps": cpu_steps,
                              "pops_identical": bool(np.array_equal(ref_pop[:m], gpu_pop[:m])),
                              "pops_compared": int(m)})
            res[str(n)] = r
    return out


if __name__ == "__main__":
    import json

    import paper_2604_00499_b200 as tie

    mc = tie.McContext(3.5)
    sizes = tuple(int(x) for x in sys.argv[1].split(",")) if len(sys.argv) > 1 else (1000, 10000)
    print(json.dumps(run(tie, mc, sizes=sizes), indent=1))
