"""GPU parity: the k-way merge of sorted (score, id) runs (tie_merge_runs) --
the sharded score+rank's final step -- against NumPy's lexsort, incl. cross-run ties (broken
by id, as the reference heap does, sched.cpp:28-31), empty and uneven runs, -0.0 / +0.0."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def make_runs(rng, G, lens, tie_frac=0.3):
    stride = max(max(lens), 1)
    ids = rng.permutation(sum(lens) * 2)[: sum(lens)].astype(np.int64)
    keys = np.full((G, stride), np.finfo(np.float64).max)
    idm = np.full((G, stride), -1, np.int64)
    o = 0
    for g, L in enumerate(lens):
        k = np.round(rng.lognormal(5.0, 0.5, L), 0 if rng.random() < tie_frac else 6)
        k[rng.random(L) < 0.01] = -0.0
        i = ids[o:o + L]
        srt = np.lexsort((i, np.where(k == 0.0, 0.0, k)))
        keys[g, :L], idm[g, :L] = k[srt], i[srt]
        o += L
    return keys, idm


@pytest.mark.parametrize("G,lens", [(1, [1000]), (2, [5000, 4999]), (3, [0, 7000, 123]),
                                    (5, [2048, 2049, 1, 0, 30000]),
                                    (8, [125_000] * 8), (7, [100_003] * 7)])
def test_merge_runs_vs_lexsort(tie, mc, G, lens):
    import torch

    from paper_2604_00499_b200.dist import DeviceOps

    rng = np.random.default_rng(G * 1000 + sum(lens) % 997)
    keys, ids = make_runs(rng, G, lens)
    ops = DeviceOps(mc, 0.9)
    out = ops.merge_runs(torch.from_numpy(keys).cuda(), torch.from_numpy(ids).cuda(), lens)
    ops.sync()
    k = np.concatenate([keys[g, :L] for g, L in enumerate(lens)])
    i = np.concatenate([ids[g, :L] for g, L in enumerate(lens)])
    k = np.where(k == 0.0, 0.0, k)  # the heap compares with ==: -0.0 ties +0.0
    ref = i[np.lexsort((i, k))]
    assert np.array_equal(out.cpu().numpy(), ref)
