"""Generate the committed golden fixtures from the REAL reference (oracle/_ref/libtie_ref.so,
the untouched /root/reference/proj sources compiled by `make -C oracle ref`).

    python tests/golden/make_golden.py          # writes tests/golden/*.npz + golden.json

Every array here is produced by the reference's own functions through oracle/ref_harness.cpp;
nothing is computed by the restatement or by the CUDA path.  Hashes are FNV-1a-64 over the
raw little-endian bytes.
"""
from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib, fnv1a64_np  # noqa: E402

GRID_MU = [2.0, 4.0, 6.0]
GRID_SIGMA = [0.3, 0.8, 1.5]
GRID_XMAX = [256.0, 512.0, 2048.0]


def fnv_fast(arr) -> str:
    """FNV-1a-64 over bytes, chunked through numpy for MB-sized arrays."""
    b = np.ascontiguousarray(arr).view(np.uint8)
    h = 0xCBF29CE484222325
    prime = 0x100000001B3
    mask = 0xFFFFFFFFFFFFFFFF
    for byte in b.tobytes():
        h = ((h ^ byte) * prime) & mask
    return f"{h:016x}"


def edge_cases():
    """(mu, sigma, x_max) cells exercising the reference's branches."""
    rows = []
    # zero-uncertainty requests (acceptance.cpp:360-376): mu = ln(len), sigma = 1e-9
    for L in [3, 7, 34, 55, 120, 260, 511, 512, 513, 2048]:
        rows.append((math.log(L), 1e-9, 512.0))
    # sigma below the clamp, tiny and huge x_max, case-1 (x_max at the median)
    rows += [(4.0, 1e-12, 512.0), (4.0, 0.8, math.exp(4.0)), (4.0, 0.8, 1.0),
             (4.0, 0.8, 1e6), (0.0, 2.5, 2048.0), (-3.0, 0.5, 16.0), (9.0, 0.05, 4096.0),
             (2.0, 3.9, 2048.0), (2.0, 4.2, 2048.0), (3.0, 7.5, 1e5), (650.0, 1.0, 1e300),
             (-20.0, 3.0, 1.0), (5.0, 1.2, 4294967295.0), (1.0, 0.0312499, 64.0),
             (1.0, 0.03125, 64.0), (1.0, 0.0156250001, 64.0)]
    return np.array(rows, dtype=np.float64)


def main():
    R = RefLib()
    out = {"generator": "tests/golden/make_golden.py", "reference": "/root/reference/proj",
           "hash": "fnv1a64 over raw little-endian bytes"}
    t0 = time.time()

    # ---- McContext(3.5, 10000, 12) and a second set
    Y = R.mc_samples(3.5, 10000, 12)
    out["mc_3.5_10000_12"] = {"fnv": fnv_fast(Y), "min": Y.min().hex(), "max": Y.max().hex(),
                              "first": Y[:4].tolist(), "last": Y[-4:].tolist()}
    Y5 = R.mc_samples(3.5, 1000, 5)
    out["mc_3.5_1000_5"] = {"fnv": fnv_fast(Y5)}

    # ---- Student-t values
    pts = [(2.0, 3.5), (-1.3, 2.5), (7.0, 5.0), (0.0, 3.5), (1e-5, 3.5), (30.0, 3.5),
           (0.9, 3.5), (-0.8, 3.5), (0.76, 0.5), (2.2, 100.0)]
    out["t_cdf"] = [[y, nu, R.t_cdf(y, nu).hex()] for y, nu in pts]
    out["t_quantile"] = [[p, nu, R.t_quantile(p, nu).hex()]
                         for p, nu in [(0.9, 3.5), (0.5, 3.5), (0.05, 3.5), (0.999999, 10.0)]]

    # ---- acceptance 3x3x3 grid (acceptance.cpp:79-100) at alpha 0.9, beta 0.5
    g = np.array([(m, s, x) for m in GRID_MU for s in GRID_SIGMA for x in GRID_XMAX])
    E, C, S = R.score(g[:, 0], g[:, 1], g[:, 2], alpha=0.9, beta=0.5)
    E0, C0, S0 = R.score(g[:, 0], g[:, 1], g[:, 2], alpha=0.0, beta=0.3)
    np.savez(os.path.join(HERE, "grid27.npz"), mu=g[:, 0], sigma=g[:, 1], x_max=g[:, 2], E=E,
             C=C, S=S, E_a0=E0, C_a0=C0, S_a0=S0)

    # ---- edge cells
    ec = edge_cases()
    E, C, S = R.score(ec[:, 0], ec[:, 1], ec[:, 2], alpha=0.9, beta=0.5)
    np.savez(os.path.join(HERE, "edges.npz"), mu=ec[:, 0], sigma=ec[:, 1], x_max=ec[:, 2], E=E,
             C=C, S=S)

    # ---- config 1: 1k queue, seed 1, full arrays
    mu, sg, mt = R.gen_workload(1000, seed=1)
    E, C, S = R.score(mu, sg, mt.astype(np.float64), alpha=0.9,
                      beta=R.compute_beta_raw(1, 0.1, 0.5, 128.0, 1000))
    order = R.rank(S)
    np.savez(os.path.join(HERE, "config1.npz"), mu=mu, sigma=sg, max_tokens=mt, E=E, C=C, S=S,
             order=order)
    out["config1"] = {"order_prefix": order[:8].tolist(), "fnv_order": fnv_fast(order),
                      "fnv_mu": fnv_fast(mu), "fnv_sigma": fnv_fast(sg)}

    # ---- canonical-config queue (configs/canonical.json: mu U[0.1,2.7], sigma U[0.4,1.2],
    #      x_max 512), 20k requests
    mu, sg, mt = R.gen_workload(20000, seed=1, mu_range=(0.1, 2.7), sigma_range=(0.4, 1.2),
                                max_tokens=512)
    E, C, S = R.score(mu, sg, mt.astype(np.float64), alpha=0.9, beta=0.5)
    np.savez(os.path.join(HERE, "canonical20k.npz"), E=E, C=C, S=S, order=R.rank(S))

    # ---- config 2: 1M queue, seed 1 -- hashes + a strided sample (the arrays are 8 MB each)
    n2 = 1_000_000
    mu, sg, mt = R.gen_workload(n2, seed=1)
    t1 = time.time()
    E, C, S = R.score(mu, sg, mt.astype(np.float64), alpha=0.9, beta=0.5)
    t_score = time.time() - t1
    t1 = time.time()
    order = R.rank(S)
    t_rank = time.time() - t1
    idx = np.arange(0, n2, 997, dtype=np.int64)
    srt = np.sort(S)
    rel_gap = np.diff(srt) / srt[1:]
    np.savez(os.path.join(HERE, "config2_sample.npz"), idx=idx, E=E[idx], C=C[idx], S=S[idx],
             order_head=order[:4096], order_tail=order[-4096:])
    out["config2"] = {"n": n2, "fnv_order": fnv_fast(order), "fnv_S": fnv_fast(S),
                      "sha256_order": hashlib.sha256(order.tobytes()).hexdigest(),
                      "sha256_E": hashlib.sha256(E.tobytes()).hexdigest(),
                      "fnv_mu": fnv_fast(mu), "fnv_sigma": fnv_fast(sg),
                      "sum_S": float(S.sum()), "pairs_rel_gap_lt_1e-12": int((rel_gap < 1e-12).sum()),
                      "pairs_rel_gap_lt_1e-9": int((rel_gap < 1e-9).sum()),
                      "pairs_rel_gap_lt_1e-6": int((rel_gap < 1e-6).sum()),
                      "ref_seconds_score": t_score, "ref_seconds_rank": t_rank,
                      "ref_threads": int(R.hw_threads())}

    # ---- rank fixtures: heap tie-break (test_sched.cpp:124-135), arbitrary ids, neg/zero keys
    keys = np.array([2048.0] * 5)
    ids = np.array([7, 2, 9, 4, 0], dtype=np.uint64)
    rng = np.random.default_rng(404)
    rk = np.round(rng.uniform(-50, 50, 5000), 1)  # many exact ties
    rk[::97] = 0.0
    rk[1::97] = -0.0
    rids = rng.permutation(np.arange(10_000, 20_000, dtype=np.uint64))[:5000]
    np.savez(os.path.join(HERE, "rank.npz"), tie_keys=keys, tie_ids=ids,
             tie_order=R.rank(keys, ids), keys=rk, ids=rids, order_ids=R.rank(rk, rids),
             order_index=R.rank(rk))

    # ---- fit: config-3 style prompts, P=4000 x K=16 (+ K=5, K=20, K=100 subsets)
    fits = {}
    for P, K, seed in [(4000, 16, 1), (2000, 5, 2), (2000, 20, 3), (300, 100, 4)]:
        x, tm, ts = R.gen_fit_data(P, K, seed=seed)
        r = R.fit(x)
        fits[f"K{K}"] = dict(x=x, **{k: np.asarray(v) for k, v in r.items()})
    # non-integer draws + degenerate prompts + scaled copies (fit invariances)
    x, _, _ = R.gen_fit_data(1000, 16, seed=9, integerise=False)
    x[:7] = 100.0
    x[7, :] = np.exp(3.0)
    r = R.fit(x)
    fits["raw16"] = dict(x=x, **{k: np.asarray(v) for k, v in r.items()})
    flat = {}
    for name, d in fits.items():
        for k, v in d.items():
            flat[f"{name}__{k}"] = v
    np.savez_compressed(os.path.join(HERE, "fit.npz"), **flat)
    out["fit_summary"] = {name: {"iters_max": int(d["iterations"].max()),
                                 "nonconverged": int((~d["converged"]).sum()),
                                 "degenerate": int(d["degenerate"].sum())}
                          for name, d in fits.items()}

    out["seconds"] = time.time() - t0
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("config1", "config2", "fit_summary", "seconds")},
                     indent=1))


if __name__ == "__main__":
    main()
