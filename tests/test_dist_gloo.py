"""CPU, world_size 2 (gloo): the sharded score+rank host logic of paper_2604_00499_b200.dist --
shard bounds, global-queue beta, run padding, all-gather and the stable merge -- must yield
exactly the reference's single-queue dispatch order.  Device kernels are replaced by
reference-semantics NumPy ops (the oracle) so the collective plumbing is what is tested."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_00499_b200.dist import SENTINEL, ShardedScoreRank, shard_bounds


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleOps:
    """score_sort / stable_sort with the reference's semantics, on CPU tensors."""

    def __init__(self, alpha=0.9):
        from oracle_lib import Oracle

        self.o = Oracle()
        self.Y = self.o.mc_samples()
        self.alpha = alpha

    def score_sort(self, mu, sigma, mt, beta):
        _, _, S = self.o.score(self.Y, mu.numpy(), sigma.numpy(), mt.numpy().astype(float),
                               alpha=self.alpha, beta=beta, threads=2)
        order = self.o.rank(S).astype(np.int64)
        return torch.from_numpy(S), torch.from_numpy(order)

    def merge_runs(self, keys, ids, lens):
        """reference semantics of the k-way merge: (key, id) order of the valid prefixes"""
        import torch

        k = np.concatenate([keys[g, :L].numpy() for g, L in enumerate(lens)])
        i = np.concatenate([ids[g, :L].numpy() for g, L in enumerate(lens)])
        return torch.from_numpy(i[np.lexsort((i, k))])

    def stable_sort(self, keys):
        return torch.from_numpy(np.argsort(keys.numpy(), kind="stable").astype(np.int64))


def _worker(rank, world, port, n_global, case, out_q):
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle_lib import Oracle

        o = Oracle()
        if case == "workload":
            mu, sg, mt = o.gen_workload(n_global, seed=1)
        else:  # every request identical: all cross-shard ties must break by id
            mu = np.full(n_global, 4.0)
            sg = np.full(n_global, 0.8)
            mt = np.full(n_global, 2048, np.uint32)
        lo, hi = shard_bounds(n_global, world, rank)
        beta = o.compute_beta(True, 0.1, 0.5, 128.0, n_global)  # GLOBAL queue length
        ops = OracleOps()
        for bad in ({"transport": "p2p"}, {"transport": "p2p", "merge_on": "range"},
                    {"transport": "nvlink"}):  # p2p needs device ops and the range exchange
            try:
                ShardedScoreRank(ops, beta, **bad)
                out_q.put((rank, "bad-config-accepted", bad))
            except ValueError:
                pass
        for merge_on, kway in (("root", "auto"), ("all", "auto"), ("root", "always"),
                               ("range", "auto"), ("range", "always")):
            res = ShardedScoreRank(ops, beta, merge_on=merge_on, kway=kway)(
                torch.from_numpy(mu[lo:hi].copy()), torch.from_numpy(sg[lo:hi].copy()),
                torch.from_numpy(mt[lo:hi].copy()), n_global)
            if merge_on == "range":  # this rank's slice of the global order
                out_q.put((rank, merge_on + "/" + kway,
                           (res.offset, res.global_order.numpy().tolist())))
            elif res.global_order is not None:
                out_q.put((rank, merge_on + "/" + kway, res.global_order.numpy().tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n_global,case", [(2001, "workload"), (64, "ties"), (3, "workload")])
def test_two_rank_order_matches_single_queue(n_global, case, oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_global, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
        assert p.exitcode == 0
    # k-way root merge and re-sort root merge on rank 0, all-merge on both ranks, and the
    # splitter exchange's two slices per variant
    got = [q.get(timeout=5) for _ in range(8)]
    # the reference: one queue, one heap
    if case == "workload":
        mu, sg, mt = oracle.gen_workload(n_global, seed=1)
    else:
        mu, sg, mt = np.full(n_global, 4.0), np.full(n_global, 0.8), np.full(n_global, 2048)
    beta = oracle.compute_beta(True, 0.1, 0.5, 128.0, n_global)
    _, _, S = oracle.score(oracle.mc_samples(), mu, sg, np.asarray(mt, float), alpha=0.9,
                           beta=beta)
    ref = oracle.rank(S).tolist()
    slices = {}
    for rank, merge_on, order in got:
        if merge_on.startswith("range"):
            slices.setdefault(merge_on, []).append(order)
            continue
        assert order == ref, (rank, merge_on)
    assert len(slices) == 2
    for variant, parts in slices.items():
        parts.sort()
        assert parts[0][0] == 0 and parts[1][0] == len(parts[0][1]), variant
        assert parts[0][1] + parts[1][1] == ref, variant
        if n_global > 100:  # the regular sample balances the ranges
            assert min(len(p[1]) for p in parts) > n_global // 4, variant
    if case == "ties":
        assert ref == list(range(n_global))


def test_shard_bounds_cover_queue():
    for n in (0, 1, 7, 1000, 1001):
        for w in (1, 2, 3, 8):
            spans = [shard_bounds(n, w, r) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(ValueError):
        shard_bounds(10, 2, 2)
    assert SENTINEL > 1e300
