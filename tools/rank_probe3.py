"""rank a continuous 3M-key queue through the C-ABI (two-level partition path; debugging)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from cabi import CAbi
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3_000_000
abi = CAbi()
h = abi.ctx()
sd = float(sys.argv[2]) if len(sys.argv) > 2 else 0.6
key = np.random.default_rng(3).lognormal(5.0, sd, n) + (50.0 if sd == 0.6 else 0.0)
if len(sys.argv) > 3:
    key = np.round(np.random.default_rng(77).lognormal(5.0, 0.7, n), 1)
o = abi.rank(h, key)
print("sorted", bool(np.all(np.diff(key[o.astype(np.int64)]) >= 0)))
