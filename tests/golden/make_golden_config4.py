"""Pin BASELINE config 4 (64M-request queue, gen_logt_workload seed 1, beta 0.5) to the REAL
reference: oracle/_ref/libtie_ref.so (the untouched /root/reference/proj sources built by
`make -C oracle ref`).

    python tests/golden/make_golden_config4.py      # ~40 min on 8 cores; writes config4.json

The reference scores every request with its own censored_expectation / censored_cvar /
compute_score chain (threaded over host cores, pure functions) and orders the queue with its
own WaitingQueue (push x n, pop_min until empty).  The 512 MB score vector and order are
cached under _cache/config4/ (git- and gpurun-ignored); only digests are committed:

* sha256 of the complete reference dispatch order (u64 ids);
* the tie runs of the reference order at the survey's tolerance (and the reference's ids
  inside each run, to count the runs another implementation orders differently) (SURVEY.md 8d "parity
  checks": adjacent reference scores within 1e-12 relative) as (start, length) -- a GPU order
  that differs from the reference only by permutations inside these runs is within the bar,
  and its run-canonicalised sha256 (ids sorted inside each run) must equal the reference's;
* per-2^20-chunk order sha256s (to localise a mismatch) and per-chunk math.fsum of the
  reference scores in id order (a checksum of checksums for the score vector);
* near-tie counts at 1e-12 / 1e-9 / 1e-6 relative.
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
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib  # noqa: E402

N4 = 64 * 2 ** 20
CHUNK = 2 ** 20
TOL = 1e-12
CACHE = os.path.join(ROOT, "_cache", "config4")


def tie_runs(S_sorted, tol=TOL):
    """Maximal runs of consecutive positions whose adjacent scores are within tol relative."""
    a, b = S_sorted[:-1], S_sorted[1:]
    near = np.abs(b - a) <= tol * np.maximum(np.abs(a), np.abs(b))
    # run boundaries: positions i where near[i] starts/ends a True stretch
    idx = np.flatnonzero(near)
    if idx.size == 0:
        return np.zeros((0, 2), np.int64)
    brk = np.flatnonzero(np.diff(idx) != 1)
    starts = np.concatenate([[idx[0]], idx[brk + 1]])
    ends = np.concatenate([idx[brk], [idx[-1]]])  # last "near" pair index in the run
    return np.stack([starts, ends - starts + 2], axis=1).astype(np.int64)


def canonicalise(order, runs):
    out = np.array(order, copy=True)
    for s, n in runs:
        out[s:s + n] = np.sort(out[s:s + n])
    return out


def main():
    os.makedirs(CACHE, exist_ok=True)
    R = RefLib()
    t0 = time.time()
    mu, sg, mt = R.gen_workload(N4, seed=1)
    t_gen = time.time() - t0
    beta = R.compute_beta_raw(1, 0.1, 0.5, 128.0, N4)
    sp = os.path.join(CACHE, "S.npy")
    if os.path.exists(sp):
        S = np.load(sp)
        t_score = None
    else:
        t1 = time.time()
        _, _, S = R.score(mu, sg, mt.astype(np.float64), alpha=0.9, beta=beta)
        t_score = time.time() - t1
        np.save(sp, S)
    op = os.path.join(CACHE, "order.npy")
    if os.path.exists(op):
        order = np.load(op)
        t_rank = None
    else:
        t1 = time.time()
        order = R.rank(S)
        t_rank = time.time() - t1
        np.save(op, order)
    Ss = S[order.astype(np.int64)]
    runs = tie_runs(Ss)
    rel_gap = np.diff(Ss) / np.maximum(Ss[1:], Ss[:-1])
    canon = canonicalise(order, runs)
    out = {
        "generator": "tests/golden/make_golden_config4.py",
        "reference": "/root/reference/proj via oracle/_ref/libtie_ref.so",
        "n": N4, "seed": 1, "alpha": 0.9, "beta": beta, "tol": TOL,
        "sha256_order": hashlib.sha256(order.tobytes()).hexdigest(),
        "sha256_order_canonical": hashlib.sha256(canon.tobytes()).hexdigest(),
        "tie_runs": runs.tolist(),
        "tie_run_ids_ref": [order[s:s + n].astype(np.int64).tolist() for s, n in runs],
        "chunk": CHUNK,
        "chunk_sha256_order": [hashlib.sha256(order[i:i + CHUNK].tobytes()).hexdigest()[:16]
                               for i in range(0, N4, CHUNK)],
        "chunk_fsum_S": [math.fsum(S[i:i + CHUNK].tolist()) for i in range(0, N4, CHUNK)],
        "S_min": float(S.min()), "S_max": float(S.max()),
        "pairs_rel_gap_lt_1e-12": int((rel_gap < 1e-12).sum()),
        "pairs_rel_gap_lt_1e-9": int((rel_gap < 1e-9).sum()),
        "pairs_rel_gap_lt_1e-6": int((rel_gap < 1e-6).sum()),
        "pairs_exact_ties": int((rel_gap == 0).sum()),
        "ref_seconds_gen": t_gen, "ref_seconds_score": t_score, "ref_seconds_rank": t_rank,
        "ref_threads": int(R.hw_threads()),
    }
    with open(os.path.join(HERE, "config4.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k not in
                      ("tie_runs", "tie_run_ids_ref", "chunk_sha256_order", "chunk_fsum_S")},
                     indent=1))


if __name__ == "__main__":
    main()
