"""GPU parity: K3 batched fit_logt_fixed_nu against the reference's golden fits and the
oracle, through the C-ABI.  Bar: fitted (mu, sigma) within 1e-6 relative; converged /
degenerate flags equal; iteration-count mismatches are counted and reported."""
import numpy as np
import pytest

from cabi import CAbi, TieError, rel_err
from conftest import golden

pytestmark = pytest.mark.gpu

BAR = 1e-6


@pytest.fixture(scope="module")
def abi():
    return CAbi()


@pytest.fixture(scope="module")
def h(abi):
    ctx = abi.ctx()
    yield ctx
    abi.destroy(ctx)


def _compare(got, ref, name):
    conv = ref["converged"]
    e_mu = rel_err(got["mu"], ref["mu"])
    e_sg = rel_err(got["sigma"], ref["sigma"])
    # converged fits: the 1e-6 bar (typically ~1e-13); non-converged ones stopped at 500
    # iterations on flat likelihoods and are reported, not gated, beyond the flag check
    assert e_mu[conv].max(initial=0) <= BAR, (name, e_mu.max())
    assert e_sg[conv].max(initial=0) <= BAR, (name, e_sg.max())
    # flags must agree wherever the reference stopped before the 500-iteration cap; at the
    # cap the reference itself is still hovering at |g| ~ gtol (flat likelihood), so the flag
    # can legitimately flip on a 1-ulp difference -- those are counted, values still gated
    capped = (ref["iterations"] >= 500) | (got["iterations"] >= 500)
    assert np.array_equal(got["converged"][~capped], conv[~capped]), name
    assert np.array_equal(got["degenerate"], ref["degenerate"]), name
    assert np.max(e_mu, initial=0) <= 1e-6 and np.max(e_sg, initial=0) <= 1e-6, name
    ll_err = np.abs(got["log_likelihood"] - ref["log_likelihood"]) / np.maximum(
        1.0, np.abs(ref["log_likelihood"]))
    assert ll_err[conv].max(initial=0) <= BAR
    mism = int((got["iterations"] != ref["iterations"]).sum())
    print(f"{name}: max rel mu {e_mu.max():.2e} sigma {e_sg.max():.2e}; "
          f"iteration mismatches {mism}/{len(conv)}; bitwise-equal mu "
          f"{int((got['mu'] == ref['mu']).sum())}/{len(conv)}")
    return mism


@pytest.mark.parametrize("name", ["K16", "K5", "K20", "K100", "raw16"])
def test_golden_fits(abi, h, name):
    f = golden("fit.npz")
    ref = {k: f[f"{name}__{k}"] for k in ("mu", "sigma", "log_likelihood", "iterations",
                                          "converged", "degenerate")}
    got = abi.fit(h, f[f"{name}__x"])
    mism = _compare(got, ref, name)
    # libdevice vs glibc log1p/exp differ by <= 1 ulp; near the gtol = 1e-8 exit that can move
    # the stop by one BFGS iteration (reported, bounded, not a value mismatch)
    assert mism <= max(2, len(ref["mu"]) // 10)


def test_config3_100k_vs_oracle(abi, h, oracle):
    x, _, _ = oracle.gen_fit_data(100_000, 16, seed=1)
    ref = oracle.fit(x)
    got = abi.fit(h, x)
    _compare(got, ref, "config3-100k")


def test_fit_invariances(abi, h, oracle):
    """test_fit.cpp:85-115: order invariance, duplication, scaling, degenerate point mass."""
    y = oracle.sample_logt(5.0, 0.7, 3.5, 100, 9001)
    rng = np.random.default_rng(5)
    batch = np.stack([y, rng.permutation(y)])
    r = abi.fit(h, batch)
    assert abs(r["mu"][1] - r["mu"][0]) <= 1e-8 * abs(r["mu"][0])
    assert abs(r["sigma"][1] - r["sigma"][0]) <= 1e-8 * r["sigma"][0]
    d = abi.fit(h, np.concatenate([y, y])[None, :])
    assert abs(d["mu"][0] - r["mu"][0]) <= 1e-6 * abs(r["mu"][0])
    s = abi.fit(h, (y * 10.0)[None, :])
    assert abs(s["mu"][0] - (r["mu"][0] + np.log(10.0))) <= 1e-6 * abs(s["mu"][0])
    deg = abi.fit(h, np.array([[100.0, 100.0, 100.0]]))
    assert deg["degenerate"][0] and deg["converged"][0]
    assert abs(deg["mu"][0] - np.log(100.0)) <= 1e-12 * np.log(100.0)
    assert deg["sigma"][0] == 1e-6


def test_generic_k_path(abi, h, oracle):
    for K in (3, 7, 33, 64):
        x, _, _ = oracle.gen_fit_data(3000, K, seed=K)
        _compare(abi.fit(h, x), oracle.fit(x), f"K{K}")


def test_errors(abi, h):
    with pytest.raises(TieError) as ei:
        abi.fit(h, np.ones((4, 2)))
    assert ei.value.code == 2
    x = np.full((3, 5), 10.0)
    x[2, 3] = -1.0
    with pytest.raises(TieError) as ei:
        abi.fit(h, x)
    assert ei.value.code == 1 and "item 2" in str(ei.value)
    with pytest.raises(TieError) as ei:
        abi.fit(h, np.full((2, 5), 3.0), nu=-1.0)
    assert ei.value.code == 1


def test_chunked_host_pipeline(abi, h, oracle):
    """tie_fit_host pipelines >= 2^18 prompts in 4 chunks (H2D / fit / D2H overlapped):
    results equal the one-shot device fits and errors name the global prompt index."""
    x, _, _ = oracle.gen_fit_data(300_001, 16, seed=4)
    got = abi.fit(h, x)
    _compare(got, oracle.fit(x), "chunked-300k")
    x[290_000, 7] = 0.0
    with pytest.raises(TieError) as ei:
        abi.fit(h, x)
    assert ei.value.code == 1 and "item 290000" in str(ei.value)


def test_device_fit_ops_for_sharded_fit(tie, mc, oracle):
    """dist.DeviceFitOps (the per-rank op of dist.ShardedFit) on the GPU vs the reference"""
    import torch

    from paper_2604_00499_b200.dist import FIT_FIELDS, DeviceFitOps, ShardedFit

    x, _, _ = oracle.gen_fit_data(5000, 16, seed=8)
    local, glob = ShardedFit(DeviceFitOps(mc), gather="all")(torch.from_numpy(x).cuda(), 5000)
    got = {f: local[f].cpu().numpy() for f in FIT_FIELDS}
    got["converged"] = got["converged"].astype(bool)
    got["degenerate"] = got["degenerate"].astype(bool)
    _compare(got, oracle.fit(x), "device-fit-ops")
    assert glob is local  # one rank: the gathered result is the local one
