"""GPU parity: cmd_fit's per-prompt analysis (tools/main.cpp:527-562) --
fixed-nu and free-nu log-t BFGS fits, log-normal and exponential fits, the KS test of every
fit and the tail statistics -- through the C-ABI (tie_fit_report_host) against the oracle
(pinned to the reference's fixtures in test_oracle.py).

Tolerances: fitted (mu, sigma) 1e-6 relative (the north star's; observed ~1e-8, the BFGS
paths' libdevice-vs-glibc rounding), the selected free-nu grid point exact, closed-form
families and tail statistics 1e-12, KS statistic / p-value 1e-6 absolute (they inherit the
fitted parameters' differences through the CDF)."""
import numpy as np
import pytest

from cabi import CAbi, TieError, rel_err
from conftest import golden

pytestmark = pytest.mark.gpu
F_MU, F_SIGMA, F_NU, F_RATE, F_LL, F_IT, F_CONV, F_DEG, F_KSD, F_KSP = range(10)


@pytest.fixture(scope="module")
def abi():
    return CAbi()


@pytest.fixture(scope="module")
def h(abi):
    ctx = abi.ctx()
    yield ctx
    abi.destroy(ctx)


def check(got, ref, tail_got, tail_ref, families=15):
    for f in range(4):
        if not families >> f & 1:
            continue
        g, r = got[f], ref[f]
        assert rel_err(g[F_MU], r[F_MU]).max() <= 1e-6, f
        assert rel_err(g[F_SIGMA], r[F_SIGMA]).max() <= 1e-6, f
        assert np.array_equal(g[F_NU], r[F_NU]), f           # incl. the free-nu grid point
        assert rel_err(g[F_RATE], r[F_RATE]).max() <= 1e-12, f
        assert rel_err(g[F_LL], r[F_LL]).max() <= 1e-9, f
        assert np.array_equal(g[F_DEG], r[F_DEG]), f
        if f >= 2:  # closed forms: exact up to libm rounding
            for k in (F_MU, F_SIGMA, F_LL, F_RATE):
                assert rel_err(g[k], r[k]).max() <= 1e-12, (f, k)
        assert np.abs(g[F_KSD] - r[F_KSD]).max() <= 1e-6, f
        assert np.abs(g[F_KSP] - r[F_KSP]).max() <= 1e-6, f
    both = ~np.isnan(tail_ref)
    assert np.array_equal(both, ~np.isnan(tail_got))
    if both.any():
        assert rel_err(tail_got[both], tail_ref[both]).max() <= 1e-12


@pytest.mark.parametrize("name", ["K16", "K5", "K12c", "K100", "degen"])
def test_fit_report_golden_sets(abi, h, name):
    g = golden("fit_report.npz")
    fits, tail = abi.fit_report_raw(h, g[f"{name}__x"])
    check(fits, g[f"{name}__fits"], tail, g[f"{name}__tail"])


def test_fit_report_family_subsets_and_nu(abi, h, oracle):
    x, _, _ = oracle.gen_fit_data(3000, 20, seed=9)
    for fam, nu in [(1, 2.5), (2, 3.5), (12, 3.5), (5, 6.0)]:
        fits, tail = abi.fit_report_raw(h, x, nu, fam)
        rf, rt = oracle.fit_report_raw(x, nu, fam)
        check(fits, rf, tail, rt, fam)
        for f in range(4):  # families not requested are left as passed in (NaN)
            if not fam >> f & 1:
                assert np.isnan(fits[f]).all()


def test_fit_report_errors(abi, h):
    x = np.full((3, 4), 10.0)
    with pytest.raises(TieError, match="at least 5"):
        abi.fit_report_raw(h, x)
    x = np.full((3, 6), 10.0)
    x[1, 2] = -1.0
    with pytest.raises(TieError, match="finite and > 0"):
        abi.fit_report_raw(h, x)


def test_fit_report_ragged_prompts(abi, h, oracle):
    """`tie fit` inputs are ragged: prompts with 5..40 samples, grouped by count on the host,
    one GPU batch per group; each prompt equals the oracle's report of its own row."""
    rng = np.random.default_rng(12)
    Ks = rng.integers(5, 41, 700)
    rows = [oracle.gen_fit_data(1, int(k), seed=100 + i)[0][0] for i, k in enumerate(Ks)]
    offsets = np.r_[0, np.cumsum(Ks)].astype(np.uint64)
    fits, tail = abi.fit_report_ragged_raw(h, np.concatenate(rows), offsets)
    for k in np.unique(Ks):
        sel = np.flatnonzero(Ks == k)
        rf, rt = oracle.fit_report_raw(np.stack([rows[i] for i in sel]))
        check(fits[:, :, sel], rf, tail[:, sel], rt)
