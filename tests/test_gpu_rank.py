"""GPU parity: K2 dispatch order (stable LSD radix sort by (key, id)) against the reference's
WaitingQueue pop order (golden fixtures) and the oracle, through the C-ABI.  Integer/index
work: bit-exact."""
import numpy as np
import pytest

from cabi import CAbi, TieError, order_check
from conftest import golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def abi():
    return CAbi()


@pytest.fixture(scope="module")
def h(abi):
    ctx = abi.ctx()
    yield ctx
    abi.destroy(ctx)


def test_heap_tie_break_by_id(abi, h):
    g = golden("rank.npz")  # test_sched.cpp:124-135
    assert abi.rank(h, g["tie_keys"], g["tie_ids"]).tolist() == [0, 2, 4, 7, 9]


def test_golden_orders(abi, h):
    g = golden("rank.npz")  # ties, -0.0 == +0.0, negative keys, unsorted ids
    assert np.array_equal(abi.rank(h, g["keys"], g["ids"]), g["order_ids"])
    assert np.array_equal(abi.rank(h, g["keys"]), g["order_index"])


@pytest.mark.parametrize("n", [0, 1, 2, 4095, 4096, 4097, 65537, 1_000_003])
def test_sizes_vs_oracle(abi, h, oracle, n):
    rng = np.random.default_rng(n)
    key = rng.lognormal(4.0, 1.0, n) + 80.0
    key[rng.integers(0, max(n, 1), n // 7)] = 123.5  # exact ties
    got = abi.rank(h, key)
    assert np.array_equal(got, oracle.rank(key))


def test_explicit_ids_sorted_and_unsorted(abi, h, oracle):
    rng = np.random.default_rng(7)
    n = 300_000
    key = np.round(rng.normal(0, 100, n), 2)
    ids_sorted = np.cumsum(rng.integers(1, 5, n)).astype(np.uint64)
    assert np.array_equal(abi.rank(h, key, ids_sorted), oracle.rank(key, ids_sorted))
    ids_perm = rng.permutation(ids_sorted)
    assert np.array_equal(abi.rank(h, key, ids_perm), oracle.rank(key, ids_perm))


def test_constant_and_degenerate_keys(abi, h, oracle):
    for key in [np.full(10000, 7.0), np.zeros(5000), np.array([1e-300, -1e-300, 0.0, -0.0]),
                np.array([np.finfo(float).max, -np.finfo(float).max, 1.0])]:
        ids = np.random.default_rng(1).permutation(len(key)).astype(np.uint64)
        assert np.array_equal(abi.rank(h, key), oracle.rank(key))
        assert np.array_equal(abi.rank(h, key, ids), oracle.rank(key, ids))


def test_errors(abi, h):
    with pytest.raises(TieError) as ei:
        abi.rank(h, np.array([1.0, np.nan, 3.0]))
    assert ei.value.code == 1 and "item 1" in str(ei.value)
    with pytest.raises(TieError) as ei:
        abi.rank(h, np.array([1.0, 2.0, 3.0, 4.0]), np.array([5, 9, 5, 1], np.uint64))
    assert ei.value.code == 2 and "already queued" in str(ei.value)
    assert "item 2" in str(ei.value)  # the second push of id 5 is the one that throws


def test_order_check_helper_exempts_near_ties():
    key = np.array([1.0, 1.0 + 1e-15, 2.0])
    ok, bad, exempt = order_check(np.array([1, 0, 2]), key, tol=1e-12)
    assert ok and bad == 0 and exempt == 1


# ---- bucket path (default): range bucketing + per-bucket shared-memory ranking, with the
# device-side LSD fallback when one bucket exceeds a local-sort CTA's capacity
@pytest.mark.parametrize("n", [4096 * 3 + 5, 262_144, 2_000_000, 3_000_000])  # partition | bucket path
def test_bucket_path_continuous_keys(abi, h, oracle, n):
    rng = np.random.default_rng(n + 11)
    key = rng.lognormal(5.0, 0.6, n) + 50.0  # score-like: no bucket overflows
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))


def test_bucket_path_moderate_ties_and_signs(abi, h, oracle):
    rng = np.random.default_rng(3)
    n = 600_000
    key = np.round(rng.normal(0.0, 300.0, n), 0)  # ~600 distinct values: ties inside buckets
    key[::97] = -0.0
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))
    ids = np.arange(n, dtype=np.uint64) * 3 + 1  # ascending explicit ids: bucket path too
    assert np.array_equal(abi.rank(h, key, ids), oracle.rank(key, ids))


@pytest.mark.parametrize("distinct", [1, 2, 5])
def test_bucket_overflow_falls_back_exactly(abi, h, oracle, distinct):
    rng = np.random.default_rng(distinct)
    n = 300_000
    key = rng.integers(0, distinct, n).astype(np.float64) * 17.25 + 100.0
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))
    ids = np.arange(n, dtype=np.uint64) + 1000
    assert np.array_equal(abi.rank(h, key, ids), oracle.rank(key, ids))


def test_bucket_extreme_range(abi, h, oracle):
    rng = np.random.default_rng(5)
    n = 100_000
    key = rng.standard_normal(n) * np.exp(rng.uniform(-600, 600, n))  # span of all exponents
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))


@pytest.mark.parametrize("n", [2_500_000, 6_600_000])  # bucket path | two-level path
@pytest.mark.parametrize("distinct", [1, 3])
def test_large_n_overflow_falls_back_exactly(abi, h, oracle, distinct, n):
    """2^21 < n < 6M takes the bucket path, n >= 6M the two-level partition path (tiled
    level-1 scatter); massive ties overflow a bucket / sub-partition and the device-side LSD
    fallback must still give the heap's order."""
    rng = np.random.default_rng(distinct + 50)
    key = rng.integers(0, distinct, n).astype(np.float64) * 3.5 + 10.0
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))


@pytest.mark.parametrize("n", [4_200_000, 6_600_000, 9_000_001])
def test_large_n_moderate_ties(abi, h, oracle, n):
    rng = np.random.default_rng(77)
    key = np.round(rng.lognormal(5.0, 0.7, n), 1)  # many small tie groups, no overflow
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))


def test_two_level_path_continuous_keys(abi, h, oracle):
    """two-level path with score-like keys: skewed partition sizes, tiles ending mid-chunk"""
    rng = np.random.default_rng(123)
    n = 7_000_003
    key = rng.lognormal(5.0, 0.6, n) + 50.0
    assert np.array_equal(abi.rank(h, key), oracle.rank(key))
