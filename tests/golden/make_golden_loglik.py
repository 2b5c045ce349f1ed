"""Golden log-likelihood / gradient values (fit.cpp:44-71) from the REAL reference
(oracle/_ref/libtie_ref.so):  python tests/golden/make_golden_loglik.py -> loglik.npz"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import RefLib  # noqa: E402


def main():
    R = RefLib()
    rng = np.random.default_rng(2024)
    out = {}
    for K, seed in [(1, 3), (16, 5), (60, 123), (1000, 9)]:
        x, _, _ = R.gen_fit_data(1, K, seed=seed, integerise=False)
        x = x[0]
        mu = rng.uniform(1.0, 7.0, 64)
        sg = np.exp(rng.uniform(np.log(0.05), np.log(5.0), 64))
        out[f"K{K}__x"] = x
        out[f"K{K}__mu"] = mu
        out[f"K{K}__sigma"] = sg
        out[f"K{K}__ll"] = np.array([R.logt_loglik(x, m, s, 3.5) for m, s in zip(mu, sg)])
        out[f"K{K}__grad"] = np.array([R.logt_loglik_grad(x, m, s, 3.5) for m, s in zip(mu, sg)])
    np.savez(os.path.join(HERE, "loglik.npz"), **out)


if __name__ == "__main__":
    main()
