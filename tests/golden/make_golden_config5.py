"""Pin BASELINE config 5 to the REAL reference: run_sim of oracle/_ref/libtie_ref.so (the
untouched /root/reference/proj sources, `make -C oracle ref`) on configs/canonical.json
(proj/configs/canonical.json:1-29: 8000 requests, Poisson 100 RPS, mu~U[0.1,2.7],
sigma~U[0.4,1.2], x_max 512, prompts U{16..128}, EngineConfig 8 / 0.02 / 0.002 / 1e-4, batched
oracle predictor, TIE policy) with rebuild_threshold = 0 ("re-scoring every step"), workload
and simulation seeds 1..10.

    python tests/golden/make_golden_config5.py     # ~25 s; writes config5.json

Committed: per seed the four metrics and the sha256 of each per-event array (id order).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib, ref_run_sim  # noqa: E402


def digest(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def main():
    R = RefLib()
    out = {"generator": "tests/golden/make_golden_config5.py", "policy": "TIE",
           "rebuild_threshold": 0.0, "seeds": {}}
    for seed in range(1, 11):
        ev, m, secs = ref_run_sim(R, seed, 2, seed, threshold=0.0)
        out["seeds"][str(seed)] = {
            "metrics": m.tolist(), "ref_seconds": secs,
            "sha256": {k: digest(v) for k, v in ev.items()}}
        print(seed, m.tolist(), round(secs, 3))
    with open(os.path.join(HERE, "config5.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
