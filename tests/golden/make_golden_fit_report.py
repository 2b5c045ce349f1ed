"""Golden fixtures for cmd_fit's per-prompt analysis from the REAL
reference (oracle/_ref/libtie_ref.so: fit_logt_fixed_nu, fit_logt_free_nu, fit_lognormal,
fit_exponential, ks_test(fit_cdf), tail_stats -- tools/main.cpp:527-562 per prompt).

    python tests/golden/make_golden_fit_report.py     # writes tests/golden/fit_report.npz
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib  # noqa: E402


def input_sets(R):
    sets = {}
    sets["K16"], _, _ = R.gen_fit_data(1000, 16, seed=3)                 # config-3 style
    sets["K5"], _, _ = R.gen_fit_data(300, 5, seed=4)                    # KS minimum, no tail
    sets["K12c"], _, _ = R.gen_fit_data(300, 12, seed=5, integerise=False)
    sets["K100"], _, _ = R.gen_fit_data(60, 100, seed=6)                 # > 64: scratch rows
    rng = np.random.default_rng(7)
    degen = np.repeat(rng.integers(1, 500, (20, 1)).astype(float), 10, axis=1)
    degen[10:, :3] += 1.0                                                # two distinct values
    sets["degen"] = degen
    return sets


def main():
    R = RefLib()
    out = {}
    for name, x in input_sets(R).items():
        fits, tail = R.fit_report_raw(x)
        out[f"{name}__x"] = x
        out[f"{name}__fits"] = fits
        out[f"{name}__tail"] = tail
    np.savez_compressed(os.path.join(HERE, "fit_report.npz"), **out)
    print("wrote", os.path.join(HERE, "fit_report.npz"))


if __name__ == "__main__":
    main()
