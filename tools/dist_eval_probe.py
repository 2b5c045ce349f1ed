"""Worst-case error of the per-item dist functions vs the reference over many input seeds
(development tool for tests/test_gpu_dropin.py's tolerances)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_00499_b200 as tie  # noqa: E402
from oracle_lib import RefLib, ref_eval  # noqa: E402
from test_gpu_dropin import _dist_inputs, _dist_err  # noqa: E402

R = RefLib()
for fn, nargs, param in [("regularized_incomplete_beta", 3, 0.0), ("t_pdf", 1, 3.5),
                         ("t_cdf", 1, 2.5), ("logt_pdf", 3, 3.5), ("logt_cdf", 3, 1.5),
                         ("normal_cdf", 1, 0.0), ("normal_quantile", 1, 0.0),
                         ("lognormal_censored_expectation", 3, 0.0),
                         ("lognormal_censored_cvar", 3, 0.9), ("lognormal_censored_cvar", 3, 0.0)]:
    worst = 0.0
    for seed in range(100):
        a, b, c = _dist_inputs(fn, np.random.default_rng(seed))
        got = tie.dist_eval(fn, a, b, c, param)
        ref = ref_eval(R, fn, a, b, c, param)
        worst = max(worst, float(_dist_err(fn, got, ref).max()))
    print(f"{fn:34s} {param:4.1f} worst {worst:.3e}")
