"""Diagnostic (not a test): where do GPU fits differ from the reference's golden fits?
Writes gpurun_out/diag_fit.json."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from cabi import CAbi, rel_err  # noqa: E402
from conftest import golden  # noqa: E402
from oracle_lib import Oracle  # noqa: E402

abi = CAbi()
h = abi.ctx()
f = golden("fit.npz")
O = Oracle()
out = {}
sets = {n: f[f"{n}__x"] for n in ["K16", "K5", "K20", "K100", "raw16"]}
for K in (33, 64):
    sets[f"gen{K}"] = O.gen_fit_data(3000, K, seed=K)[0]
for name, x in sets.items():
    ref = O.fit(x)
    got = abi.fit(h, x)
    conv = ref["converged"]
    e_mu = rel_err(got["mu"], ref["mu"])
    e_sg = rel_err(got["sigma"], ref["sigma"])
    d = {
        "P": int(len(conv)),
        "max_rel_mu_conv": float(e_mu[conv].max(initial=0)),
        "max_rel_sigma_conv": float(e_sg[conv].max(initial=0)),
        "max_rel_mu_all": float(e_mu.max()),
        "bitwise_mu": int((got["mu"] == ref["mu"]).sum()),
        "iter_mismatch": int((got["iterations"] != ref["iterations"]).sum()),
        "conv_mismatch": int((got["converged"] != conv).sum()),
        "degen_mismatch": int((got["degenerate"] != ref["degenerate"]).sum()),
        "ref_nonconv": int((~conv).sum()),
        "gpu_nonconv": int((~got["converged"]).sum()),
    }
    bad = np.where((got["converged"] != conv) | (e_mu > 1e-6) | (e_sg > 1e-6))[0][:10]
    d["examples"] = [{"p": int(p), "ref": [float(ref["mu"][p]), float(ref["sigma"][p]),
                                         int(ref["iterations"][p]), bool(conv[p])],
                      "gpu": [float(got["mu"][p]), float(got["sigma"][p]),
                              int(got["iterations"][p]), bool(got["converged"][p])]}
                     for p in bad]
    out[name] = d
    print(name, json.dumps({k: v for k, v in d.items() if k != "examples"}))
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/diag_fit.json", "w") as fp:
    json.dump(out, fp, indent=1)
