"""Request-sharded score + rank over G GPUs: one process per GPU, NCCL.

The reference is single-process (a binary heap in one thread, proj/src/sched.cpp:28-94); the
order it defines -- (score asc, request id asc) over the whole queue -- is reproduced here
exactly across shards:

1. shard the queue into contiguous id ranges [lo_g, hi_g)  (``shard_bounds``);
2. beta = compute_beta(cfg, GLOBAL queue length)  (sched.cpp:9-17 -- NOT the shard length);
3. each rank scores its shard and sorts it locally (fused K1+K2 on its GPU);
4. the sorted (score, id) runs are all-gathered over NCCL (NVLink / NVSwitch), padded to
   the longest shard with DBL_MAX sentinels (scores are finite, so sentinels sort last);
5. rank 0 k-way merges the G runs (tie_merge_runs: a tree of merge-path rounds comparing
   (score, id), so cross-shard ties break by id exactly as the reference heap does,
   sched.cpp:28-31).  Ops without ``merge_runs`` fall back to a stable sort of the
   concatenation: runs are concatenated in rank order over contiguous ascending id ranges,
   so among equal scores the concatenation order IS ascending id order.

``merge_on="range"`` replaces steps 4-5 by a splitter exchange (the preferred
alternative for scaling): every rank contributes a regular sample of its sorted run, all ranks
pick the same G-1 (score, id) splitters from the gathered sample, cut their run at the
splitters (lexicographic binary search), and one variable-size all-to-all sends cut j to rank
j.  Rank j then orders the G pieces it received and owns global positions
[offset_j, offset_j + len_j): the global order is the concatenation over ranks, and no rank
receives more than its range (no redundant all-gather, no single-rank merge).

Device work is behind ``DeviceOps`` (the C-ABI through ``_core``); tests substitute
reference-semantics NumPy ops to exercise the sharding / padding / gather / merge logic on
CPU with the gloo backend.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SENTINEL = np.finfo(np.float64).max


def shard_bounds(n_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous id range of ``rank``; sizes differ by at most one (the first n % world
    ranks take one extra request)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("shard_bounds: bad world/rank")
    base, extra = divmod(int(n_global), world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_beta(cfg, n_global: int) -> float:
    """beta from the GLOBAL queue length (sched.cpp:9-17)."""
    from . import _core

    return _core.compute_beta(cfg, int(n_global))


class Comm:
    """The collectives the sharded paths use, on ``group``.  Under NCCL (one process per GPU,
    NVLink / NVSwitch) device tensors go straight to the collective; under gloo (the CPU test
    transport, and the one-GPU multi-process tests) CUDA tensors are staged through host
    memory, since gloo's all-gather / all-to-all take CPU tensors only."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.stage = dist.get_backend(group) == "gloo"

    def _h(self, t):
        return t.cpu() if self.stage and t.is_cuda else t

    def all_gather(self, outs, t):
        if not (self.stage and t.is_cuda):
            self.dist.all_gather(outs, t, group=self.group)
            return
        hs = [torch_empty_like_cpu(o) for o in outs]
        self.dist.all_gather(hs, t.cpu(), group=self.group)
        for o, h in zip(outs, hs):
            o.copy_(h)

    def all_to_all_single(self, out, inp, out_splits=None, in_splits=None):
        if not (self.stage and inp.is_cuda):
            self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
            return
        ho = torch_empty_like_cpu(out)
        self.dist.all_to_all_single(ho, inp.cpu(), out_splits, in_splits, group=self.group)
        out.copy_(ho)

    def all_reduce(self, t):
        if not (self.stage and t.is_cuda):
            self.dist.all_reduce(t, group=self.group)
            return
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h)


def torch_empty_like_cpu(t):
    import torch

    return torch.empty(t.shape, dtype=t.dtype)


class DeviceOps:
    """K1+K2 on this rank's GPU through the C-ABI (torch CUDA tensors in and out)."""

    def __init__(self, mc, alpha: float, exact: bool = False):
        import torch

        from . import _core

        self.torch = torch
        self.core = _core
        self.mc = mc  # keeps the context (and its device tables) alive with the ops
        self.ctx = mc.handle
        self.alpha = alpha
        self.flags = 1 if exact else 0

    def _stream(self, t):
        return self.torch.cuda.current_stream(t.device).cuda_stream

    def score_sort(self, mu, sigma, max_tokens, beta):
        """-> (scores in queue order, local order (int64 indices sorted by (score, index)))."""
        torch = self.torch
        n = mu.numel()
        S = torch.empty(n, dtype=torch.float64, device=mu.device)
        order = torch.empty(n, dtype=torch.int64, device=mu.device)
        self.core.score_rank_device(self.ctx, mu.data_ptr(), sigma.data_ptr(),
                                    max_tokens.data_ptr(), n, self.alpha, beta, 0, 0,
                                    S.data_ptr(), order.data_ptr(), self.flags,
                                    self._stream(mu))
        return S, order

    def sorted_run(self, mu, sigma, max_tokens, beta, run_keys, run_ids):
        """score + rank the shard, writing its sorted run straight from the device path
        (tie_score_rank_run): run_keys (f64) / run_ids (int32 shard-local index) views of the
        caller's exchange buffer -> (scores, local order)."""
        torch = self.torch
        n = mu.numel()
        S = torch.empty(n, dtype=torch.float64, device=mu.device)
        order = torch.empty(n, dtype=torch.int64, device=mu.device)
        self.core.score_rank_run_device(self.ctx, mu.data_ptr(), sigma.data_ptr(),
                                        max_tokens.data_ptr(), n, self.alpha, beta,
                                        S.data_ptr(), order.data_ptr(), run_keys.data_ptr(),
                                        run_ids.data_ptr(), self.flags, self._stream(mu))
        return S, order

    def shard_cuts(self, run_keys, run_ids, id_base, sample_keys, sample_ids, G, s):
        """-> int64 send counts [G] (device) of the splitter exchange (tie_shard_cuts)."""
        torch = self.torch
        out = torch.empty(G, dtype=torch.int64, device=run_keys.device)
        self.core.shard_cuts_device(self.ctx, run_keys.data_ptr(), run_ids.data_ptr(),
                                    int(id_base), run_keys.numel(), sample_keys.data_ptr(),
                                    sample_ids.data_ptr(), G, s, out.data_ptr(), 0, 0,
                                    self._stream(run_keys))
        return out

    def stable_sort(self, keys):
        """-> int64 permutation sorting ``keys`` by (key, position)."""
        torch = self.torch
        n = keys.numel()
        order = torch.empty(n, dtype=torch.int64, device=keys.device)
        self.core.rank_device(self.ctx, keys.data_ptr(), 0, n, order.data_ptr(),
                              self._stream(keys))
        return order

    def merge_runs(self, keys, ids, lens):
        """k-way merge (tie_merge_runs) of G padded runs keys/ids [G, stride], run g valid for
        lens[g], each sorted by (key, id) -> the merged ids (int64, sum(lens))."""
        torch = self.torch
        G, stride = keys.shape
        out = torch.empty(int(sum(lens)), dtype=torch.int64, device=keys.device)
        self.core.merge_runs_device(self.ctx, keys.data_ptr(), ids.data_ptr(), stride,
                                    [int(x) for x in lens], out.data_ptr(), self._stream(keys))
        return out

    def sync(self):
        stream = self.torch.cuda.current_stream().cuda_stream
        self.core.sync(self.ctx, stream)


def _host_shard_cuts(run_keys, run_ids, id_base, sample_keys, sample_ids, G, s):
    """tie_shard_cuts' semantics in NumPy (ops without a device implementation)."""
    import torch

    sk = sample_keys.cpu().numpy()
    si = sample_ids.cpu().numpy()
    valid = si >= 0
    k, i = sk[valid], si[valid]
    o = np.lexsort((i, k))
    k, i = k[o], i[o]
    t = len(k)
    rk = run_keys.cpu().numpy()
    ri = run_ids.cpu().numpy().astype(np.int64) + int(id_base)
    n = len(rk)
    cuts = [0]
    for j in range(1, G):
        c = (j * t) // G
        if c >= t:
            cuts.append(n)
            continue
        lo = int(np.searchsorted(rk, k[c], side="left"))
        hi = int(np.searchsorted(rk, k[c], side="right"))
        cuts.append(lo + int(np.searchsorted(ri[lo:hi], i[c], side="left")))
    cuts.append(n)
    return torch.tensor(np.diff(cuts), dtype=torch.int64, device=run_keys.device)


class _DevArray:
    """a raw device allocation as a torch tensor (__cuda_array_interface__, no copy)"""

    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2,
                                         "strides": None}


class PeerExchange:
    """The range exchange's records over peer memory (NVLink / NVSwitch between
    the GPUs of a node): every rank owns one receive buffer [cap x f64 keys | cap x u32 ids]
    allocated by ``tie_ipc_alloc`` and mapped into every other rank with ``tie_ipc_open``
    (CUDA IPC handles exchanged once with ``all_gather_object``), and ONE launch of
    ``tie_peer_put_runs`` writes this rank's sorted run pieces straight into the destinations
    at their final offsets -- no staging buffer, no NCCL all-to-all of keys and ids.  Completion
    is ordered by a stream synchronisation and a barrier before any rank reads its buffer.
    Capacity grows collectively (every rank re-allocates and re-exchanges handles together)."""

    def __init__(self, ops, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.ops = ops
        self.core = ops.core
        self.ctx = ops.ctx
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cap = 0
        self.mine = 0          # this rank's buffer (device pointer)
        self.peers = []        # every rank's buffer base in THIS address space
        self.opened = []

    def _release(self):
        for ptr in self.opened:
            self.core.ipc_close(self.ctx, ptr)
        if self.mine:
            self.core.ipc_free(self.ctx, self.mine)
        self.opened, self.peers, self.mine, self.cap = [], [], 0, 0

    def _agree(self, ok: bool, what: str):
        """collective: every rank learns whether ALL ranks succeeded (a failure on one rank
        must not leave the others waiting in the next collective); raises on every rank"""
        import torch

        t = torch.tensor([1 if ok else 0], dtype=torch.int64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(t.item()) == 0:
            raise RuntimeError(f"PeerExchange: {what} failed on some rank")

    def ensure(self, need: int):
        """collective: every rank's buffer holds >= max over ranks of ``need`` records"""
        import torch

        t = torch.tensor([int(need)], dtype=torch.int64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        want = int(t.item())
        if want <= self.cap:
            return
        self.ops.torch.cuda.synchronize()
        self.dist.barrier(group=self.group)  # nobody still writes into the old buffers
        self._release()
        cap = max(want + want // 8, 1 << 16)
        ptr, handle, ok = 0, b"", True
        try:
            ptr, handle = self.core.ipc_alloc(self.ctx, 12 * cap)
        except Exception:  # noqa: BLE001 -- reported collectively below
            ok = False
        handles = [None] * self.world
        self.dist.all_gather_object(handles, handle if ok else None, group=self.group)
        peers = []
        ok = ok and all(h is not None for h in handles)
        if ok:
            try:
                for g, h in enumerate(handles):
                    if g == self.rank:
                        peers.append(ptr)
                    else:
                        q = self.core.ipc_open(self.ctx, h)
                        self.opened.append(q)
                        peers.append(q)
            except Exception:  # noqa: BLE001
                ok = False
        self.mine, self.peers, self.cap = ptr, peers, cap
        try:
            self._agree(ok, "CUDA IPC buffer mapping")
        except RuntimeError:
            self._release()
            raise

    def views(self, total: int):
        """this rank's received (keys f64, ids int32) records as torch tensors"""
        torch = self.ops.torch
        k = torch.as_tensor(_DevArray(self.mine, total, "<f8"), device="cuda")
        i = torch.as_tensor(_DevArray(self.mine + 8 * self.cap, total, "<i4"), device="cuda")
        return k, i

    def put(self, rk, ri, send_l, dst_l):
        """write the sorted run's pieces (send_l records each) into the peers at dst_l"""
        ok = True
        try:
            stream = self.ops.torch.cuda.current_stream(rk.device).cuda_stream
            self.core.peer_put_runs_device(
                self.ctx, rk.data_ptr(), ri.data_ptr(), rk.numel(), [int(x) for x in send_l],
                [int(x) for x in dst_l], [int(p) for p in self.peers],
                [int(p) + 8 * self.cap for p in self.peers], stream)
            self.ops.torch.cuda.current_stream(rk.device).synchronize()
        except Exception:  # noqa: BLE001 -- reported collectively
            ok = False
        # the all-reduce is also the barrier: every piece has landed in every buffer
        self._agree(ok, "peer put")

    def close(self):
        self._release()


@dataclass
class ShardResult:
    scores: object            # this rank's scores, queue order (device tensor)
    local_order: object       # this rank's sorted local indices
    global_order: object      # rank 0 (or every rank with merge_on="all"): global ids; else None
                              # merge_on="range": this rank's slice of the global order
    offset: int = 0           # merge_on="range": global position of global_order[0]


class ShardedScoreRank:
    """score + rank a globally-indexed queue sharded over the ranks of ``group``.

    The exchange moves 12-byte records (f64 score + u32 shard-local index; the sender's id
    base is implied by its rank): the root / all variants all-gather one packed
    [keys | ids] byte buffer per rank; the range variant all-to-alls keys and ids.  Device
    ops emit the sorted run directly (tie_score_rank_run) and compute the splitter cuts on the
    device (tie_shard_cuts), so a root / all step has no host synchronisation and a range step
    has exactly one (the send / receive counts the all-to-all's host split sizes need)."""

    def __init__(self, ops, cfg_beta: float, group=None, merge_on: str = "root",
                 kway: str = "auto", transport: str = "collective"):
        import torch.distributed as dist

        self.dist = dist
        self.ops = ops
        self.beta = cfg_beta
        self.group = group
        if transport not in ("collective", "p2p"):
            raise ValueError("transport must be 'collective' or 'p2p'")
        # "p2p": the range exchange writes the records into the destinations' buffers over
        # peer memory (PeerExchange); needs device ops and merge_on="range"
        if transport == "p2p" and merge_on != "range":
            raise ValueError("transport='p2p' moves the range exchange (merge_on='range')")
        if transport == "p2p" and not hasattr(ops, "core"):
            raise ValueError("transport='p2p' needs device ops (DeviceOps): the records move "
                             "between GPU buffers")
        self.peer = PeerExchange(ops, group) if transport == "p2p" else None
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.comm = Comm(group) if dist.is_initialized() else None
        if merge_on not in ("root", "all", "range"):
            raise ValueError("merge_on must be 'root', 'all' or 'range'")
        self.merge_on = merge_on
        if kway not in ("auto", "always", "never"):
            raise ValueError("kway must be 'auto', 'always' or 'never'")
        self.kway = kway
        self.host_syncs = 0  # host round trips of the last call (diagnostics)
        self.last_counts = None  # (send, receive) record counts of the last range exchange

    oversample = 32  # regular-sample points per rank and destination range

    def _run(self, mu, sigma, max_tokens, keys_view, ids_view):
        """the sorted run into keys_view (f64) / ids_view (int32): fused on device ops"""
        if hasattr(self.ops, "sorted_run"):
            return self.ops.sorted_run(mu, sigma, max_tokens, self.beta, keys_view, ids_view)
        S, order = self.ops.score_sort(mu, sigma, max_tokens, self.beta)
        keys_view.copy_(S[order])
        ids_view.copy_(order.to(ids_view.dtype))
        return S, order

    def __call__(self, mu, sigma, max_tokens, n_global: int) -> ShardResult:
        import torch

        self.host_syncs = 0
        lo, hi = shard_bounds(n_global, self.world, self.rank)
        m = hi - lo
        if mu.numel() != m:
            raise ValueError(f"rank {self.rank}: shard holds {mu.numel()} requests, expected "
                             f"{m} (ids [{lo}, {hi}))")
        if self.world == 1:
            S, order = self.ops.score_sort(mu, sigma, max_tokens, self.beta)
            return ShardResult(S, order, order)
        dev = mu.device
        if self.merge_on == "range":
            rk = torch.empty(m, dtype=torch.float64, device=dev)
            ri = torch.empty(m, dtype=torch.int32, device=dev)
            S, order = self._run(mu, sigma, max_tokens, rk, ri)
            return self._range_exchange(S, order, rk, ri, lo, n_global)
        # root / all: one packed record buffer per rank, [width x f64 keys | width x i32 ids],
        # padded to the longest shard with (+max, -1) sentinels
        G = self.world
        width = shard_bounds(n_global, G, 0)[1]
        rec = torch.empty(12 * width, dtype=torch.uint8, device=dev)
        rkeys = rec[:8 * width].view(torch.float64)
        rids = rec[8 * width:].view(torch.int32)
        if m < width:
            rkeys[m:].fill_(SENTINEL)
            rids[m:].fill_(-1)
        S, order = self._run(mu, sigma, max_tokens, rkeys[:m], rids[:m])
        recs = [torch.empty_like(rec) for _ in range(G)]
        self.comm.all_gather(recs, rec)
        merged = None
        if self.merge_on == "all" or self.rank == 0:
            bounds = [shard_bounds(n_global, G, g) for g in range(G)]
            lens = [b - a for a, b in bounds]
            gk = torch.stack([r[:8 * width].view(torch.float64) for r in recs])
            base = torch.tensor([a for a, _ in bounds], dtype=torch.int64, device=dev)
            gi = torch.stack([r[8 * width:].view(torch.int32) for r in recs]).to(torch.int64)
            gi += base[:, None]  # shard-local -> global ids (sentinels: base - 1, never read)
            # k-way merge of the sorted runs, or a re-sort of the concatenation: both give the
            # identical order; measured on one B200 for G x 1M runs (bench.py "rank0_merge"):
            # G=2 73 vs 71 us re-sort, G=4 213 vs 179, G=8 490 vs 322 -- the range-partition
            # sort is at least as fast, so "auto" re-sorts and the merge tree is opt-in
            if hasattr(self.ops, "merge_runs") and self.kway == "always":
                merged = self.ops.merge_runs(gk, gi, lens)
            else:  # stable re-sort of the concatenation (sentinels sort last)
                perm = self.ops.stable_sort(gk.reshape(-1))
                merged = gi.reshape(-1)[perm][:n_global]
        return ShardResult(S, order, merged)

    def _range_exchange(self, S, order, rk, ri, lo, n_global):
        import torch

        G, dev, m = self.world, rk.device, rk.numel()
        s = self.oversample * G
        take = min(m, s)
        # regular sample of the sorted run (device), sentinel-padded to s entries
        pos = ((torch.arange(take, device=dev, dtype=torch.float64) + 0.5) * (m / max(take, 1)))
        pos = pos.to(torch.int64).clamp_(max=max(m - 1, 0))
        sk = torch.full((s,), SENTINEL, dtype=torch.float64, device=dev)
        si = torch.full((s,), -1, dtype=torch.int64, device=dev)
        sk[:take] = rk[pos]
        si[:take] = ri[pos].to(torch.int64) + lo
        gk = torch.empty(G * s, dtype=torch.float64, device=dev)
        gi = torch.empty(G * s, dtype=torch.int64, device=dev)
        self.comm.all_gather(list(gk.view(G, s).unbind(0)), sk)
        self.comm.all_gather(list(gi.view(G, s).unbind(0)), si)
        cuts = getattr(self.ops, "shard_cuts", None) or \
            (lambda *a: _host_shard_cuts(*a))
        send = cuts(rk, ri, lo, gk, gi, G, s)
        if self.peer is not None:
            # the G x G send matrix (one all-gather, ONE host read): the receive counts are
            # its column, a piece's landing offset in its destination the column sum above
            # this rank, the destinations' global offsets its prefix sums; then one launch of
            # peer stores moves every piece (PeerExchange)
            mat = torch.empty((G, G), dtype=torch.int64, device=dev)
            self.comm.all_gather(list(mat.unbind(0)), send)
            M = mat.cpu().numpy()
            self.host_syncs += 1
            send_l = [int(x) for x in M[self.rank]]
            recv_l = [int(x) for x in M[:, self.rank]]
            below_l = [int(M[:, :g].sum()) for g in range(G)]
            dst_l = [int(M[:self.rank, g].sum()) for g in range(G)]
            self.last_counts = (send_l, recv_l)
            total = int(sum(recv_l))
            self.peer.ensure(total)
            self.peer.put(rk, ri, send_l, dst_l)
            keys, ids = self.peer.views(total)
        else:
            # receive counts, and every destination's global offset (the records all ranks
            # send to destinations below it): one all-to-all + one all-reduce, ONE host read
            recv = torch.empty(G, dtype=torch.int64, device=dev)
            self.comm.all_to_all_single(recv, send)
            below = torch.zeros(G, dtype=torch.int64, device=dev)
            below[1:] = torch.cumsum(send, 0)[:-1]
            self.comm.all_reduce(below)
            counts = torch.cat([send, recv, below]).cpu().tolist()  # the one host sync
            self.host_syncs += 1
            send_l, recv_l, below_l = counts[:G], counts[G:2 * G], counts[2 * G:]
            self.last_counts = (send_l, recv_l)
            total = int(sum(recv_l))
            keys = torch.empty(total, dtype=torch.float64, device=dev)
            ids = torch.empty(total, dtype=torch.int32, device=dev)
            self.comm.all_to_all_single(keys, rk, recv_l, send_l)
            self.comm.all_to_all_single(ids, ri, recv_l, send_l)
        # shard-local -> global ids: piece g came from rank g (its id base)
        bases = torch.tensor([shard_bounds(n_global, G, g)[0] for g in range(G)],
                             dtype=torch.int64, device=dev)
        gids = ids.to(torch.int64) + torch.repeat_interleave(
            bases, torch.tensor(recv_l, device=dev), output_size=total)
        # pieces arrive in source-rank order = ascending id ranges, each sorted by (k, i): a
        # stable sort by k alone (or the k-way merge) yields the (k, i) order
        if hasattr(self.ops, "merge_runs") and self.kway == "always" and total:
            width = max(recv_l)
            pk = torch.full((G, width), SENTINEL, dtype=torch.float64, device=dev)
            pi = torch.full((G, width), -1, dtype=torch.int64, device=dev)
            o = 0
            for g in range(G):
                pk[g, :recv_l[g]] = keys[o:o + recv_l[g]]
                pi[g, :recv_l[g]] = gids[o:o + recv_l[g]]
                o += recv_l[g]
            mine = self.ops.merge_runs(pk, pi, recv_l)
        elif total:
            mine = gids[self.ops.stable_sort(keys)]
        else:
            mine = gids
        return ShardResult(S, order, mine, int(below_l[self.rank]))


U64_MAX = np.iinfo(np.uint64).max


class ShardedScheduler:
    """ONE reference Scheduler (sched.cpp:125-175) over requests sharded across ranks
    ("queue-resident scheduler"): each rank's ``local`` queue (a
    ``GpuScheduler``) holds the (E, CVaR, key) of the requests it owns, and every method is a
    collective that all ranks call with their own slice of the events.  The shards together
    pop exactly the reference's sequence:

    * beta at a prediction or pop is compute_beta of the GLOBAL waiting count (sched.cpp:136,
      154): each rank tells its queue how many requests the others hold
      (``set_peer_waiting``) after one all-gather of the shard sizes;
    * rebuild_if_drifted (sched.cpp:152-167) is a global decision: drift is taken over the
      union of the shards' betas_in_use_, whose extremes are the extremes of the per-shard
      extremes (``beta_range``), and a rebuild re-keys every shard at the same beta
      (``rebuild_at``);
    * pops: the multiset only loses entries as pops proceed, so its range only shrinks; the
      pops for which no rebuild is possible under the current range are selected in ONE
      exchange -- every rank peeks its next L (key, id) entries, one all-gather of G x L
      candidates, the L smallest in (key, id) order are the next L global pops, and shard g
      pops its share with ``next_requests`` (its own top entries, in order).  A rebuild that
      must fire is applied on every shard and the exchange repeats.

    Every rank returns the same global pop sequence.  ``beta_fn(queue_len)`` is compute_beta
    for the queue's ScoreConfig; ``policy`` 0 FCFS / 1 SEPT / 2 TIE."""

    def __init__(self, local, policy: int, beta_fn, rebuild_threshold: float, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.local = local
        self.policy = int(policy)
        self.beta_fn = beta_fn
        self.threshold = float(rebuild_threshold)
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.exchanges = 0  # all-gathers issued (diagnostics)

    # ---- collectives over small host arrays (device tensors under NCCL)
    def _gather(self, arr):
        import torch

        a = np.ascontiguousarray(arr)
        wire = a.view(np.int64) if a.dtype == np.uint64 else a
        dev = "cpu"
        if self.dist.get_backend(self.group) == "nccl":
            dev = torch.device("cuda", torch.cuda.current_device())
        t = torch.from_numpy(wire.copy()).to(dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        self.exchanges += 1
        res = np.stack([o.cpu().numpy() for o in out])
        return res.view(np.uint64) if a.dtype == np.uint64 else res

    def _collective(self, fn):
        """run the local part, then agree on success: a failure on any rank raises on all"""
        err = None
        try:
            out = fn()
        except Exception as e:  # noqa: BLE001 -- re-raised below
            err, out = e, None
        flags = self._gather(np.array([0 if err is None else 1], np.int64))
        if err is not None:
            raise err
        if flags.any():
            bad = [int(r) for r in np.nonzero(flags[:, 0])[0]]
            raise RuntimeError(f"ShardedScheduler: the event batch failed on rank(s) {bad}")
        return out

    def _sync_sizes(self, extra: int = 0) -> int:
        """global waiting count (after this rank adds ``extra``); sets the peer count"""
        mine = self.local.waiting() + int(extra)
        sizes = self._gather(np.array([mine], np.int64))[:, 0]
        total = int(sizes.sum())
        self.local.set_peer_waiting(total - mine)
        return total

    # ---- Scheduler entry points (each a collective)
    def waiting(self) -> int:
        return int(self._gather(np.array([self.local.waiting()], np.int64)).sum())

    def on_arrival_batch(self, ids, arrival_s, max_tokens):
        self._collective(lambda: self.local.on_arrival_batch(ids, arrival_s, max_tokens))

    def on_prediction_batch(self, ids, expectation, cvar):
        self._sync_sizes()
        self._collective(lambda: self.local.on_prediction_batch(ids, expectation, cvar))

    def on_prediction_logt(self, ids, mu, sigma, max_tokens):
        self._sync_sizes()
        self._collective(lambda: self.local.on_prediction_logt(ids, mu, sigma, max_tokens))

    def step(self, arr_ids, arrival_s, arr_max_tokens, pred_ids, mu, sigma, pred_max_tokens,
             k: int):
        """one iteration: every rank's arrivals, then every rank's predictions (beta of the
        global queue after all arrivals), then k global pops"""
        self._sync_sizes(extra=len(arr_ids))
        self._collective(lambda: self.local.step(arr_ids, arrival_s, arr_max_tokens, pred_ids,
                                                 mu, sigma, pred_max_tokens, 0))
        return self.next_requests(k)

    def next_requests(self, k: int):
        """next_request() x k over the union of the shards -> global pop ids (uint64)"""
        out = []
        while len(out) < k:
            mine = self.local.waiting()
            lo, hi, n_in_use = self.local.beta_range()
            st = self._gather(np.array([mine, lo, hi, n_in_use], np.float64))
            sizes = st[:, 0].astype(np.int64)
            Q = int(sizes.sum())
            if Q == 0:
                break
            left = min(k - len(out), Q)
            used = st[:, 3] > 0
            pred = self.policy == 2 and bool(used.any())
            if pred:
                glo, ghi = float(st[used, 1].min()), float(st[used, 2].max())
            # pops with no possible rebuild before them: the range only shrinks as pops go
            L = 0
            while L < left:
                if pred:
                    now = self.beta_fn(Q - L)
                    if max(abs(now - glo), abs(now - ghi)) > self.threshold:
                        break
                L += 1
            if L == 0:  # the range is exact now: this rebuild fires (sched.cpp:156-166)
                now = self.beta_fn(Q)
                self.local.set_peer_waiting(Q - mine)
                self._collective(lambda: self.local.rebuild_at(now))
                continue
            keys, ids = self.local.peek(L)
            ck = np.full(L, U64_MAX, np.uint64)
            ci = np.full(L, U64_MAX, np.uint64)
            ck[:len(keys)] = keys
            ci[:len(ids)] = ids
            g = self._gather(np.stack([ck, ci]))  # [G, 2, L]: one exchange
            owner = np.repeat(np.arange(self.world), L)
            fk, fi = g[:, 0].reshape(-1), g[:, 1].reshape(-1)
            o = np.lexsort((fi, fk))[:L]
            win_ids, win_owner = fi[o], owner[o]
            take = int((win_owner == self.rank).sum())
            self.local.set_peer_waiting(Q - mine)
            got = np.asarray(self.local.next_requests(take), np.uint64) if take else \
                np.empty(0, np.uint64)
            if not np.array_equal(got, win_ids[win_owner == self.rank]):
                raise RuntimeError(f"ShardedScheduler: rank {self.rank} popped {got.tolist()}, "
                                   f"expected {win_ids[win_owner == self.rank].tolist()}")
            out.extend(int(x) for x in win_ids)
            # peers after this batch: (Q - L) global, (mine - take) here
            self.local.set_peer_waiting((Q - L) - (mine - take))
        return np.array(out, np.uint64)


FIT_FIELDS = ("mu", "sigma", "log_likelihood", "iterations", "converged", "degenerate")


class DeviceFitOps:
    """K3 (fit_logt_fixed_nu per prompt) on this rank's GPU through the C-ABI."""

    def __init__(self, mc, nu: float = 3.5):
        import torch

        from . import _core

        self.torch, self.core, self.mc, self.nu = torch, _core, mc, nu

    def fit(self, x):
        """x: [P, K] float64 device tensor -> dict of device tensors (FIT_FIELDS)"""
        torch = self.torch
        P, K = x.shape
        dev = x.device
        out = {"mu": torch.empty(P, dtype=torch.float64, device=dev),
               "sigma": torch.empty(P, dtype=torch.float64, device=dev),
               "log_likelihood": torch.empty(P, dtype=torch.float64, device=dev),
               "iterations": torch.empty(P, dtype=torch.int32, device=dev),
               "converged": torch.empty(P, dtype=torch.uint8, device=dev),
               "degenerate": torch.empty(P, dtype=torch.uint8, device=dev)}
        stream = torch.cuda.current_stream(dev).cuda_stream
        self.core.fit_device(self.mc.handle, x.contiguous().data_ptr(), P, K, self.nu,
                             *[out[f].data_ptr() for f in FIT_FIELDS], stream)
        self.core.sync(self.mc.handle, stream)
        return out


class ShardedFit:
    """Config 3 over the ranks of ``group`` ("Fit K3: embarrassingly parallel
    by prompt"): prompts are sharded contiguously (``shard_bounds``), every rank fits its own
    shard, and the only collective is the optional result gather -- ``gather="root"`` (rank
    0) or ``"all"`` returns the fits of every prompt in global order, ``"none"`` only the
    local ones."""

    def __init__(self, ops, group=None, gather: str = "none"):
        import torch.distributed as dist

        if gather not in ("none", "root", "all"):
            raise ValueError("gather must be 'none', 'root' or 'all'")
        self.dist, self.ops, self.group, self.gather = dist, ops, group, gather
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0

    def __call__(self, x_local, P_global: int):
        import torch

        lo, hi = shard_bounds(P_global, self.world, self.rank)
        if x_local.shape[0] != hi - lo:
            raise ValueError(f"rank {self.rank}: shard holds {x_local.shape[0]} prompts, "
                             f"expected {hi - lo} (prompts [{lo}, {hi}))")
        local = self.ops.fit(x_local)
        if self.gather == "none" or self.world == 1:
            return local, (local if self.gather != "none" else None)
        lens = [b - a for a, b in (shard_bounds(P_global, self.world, g)
                                   for g in range(self.world))]
        width = lens[0]
        glob = {}
        for f in FIT_FIELDS:
            t = local[f]
            wire = t.to(torch.int32) if t.dtype == torch.uint8 else t  # gloo / NCCL friendly
            pad = torch.zeros(width, dtype=wire.dtype, device=wire.device)
            pad[:wire.numel()] = wire
            parts = [torch.empty_like(pad) for _ in range(self.world)]
            self.dist.all_gather(parts, pad, group=self.group)
            if self.gather == "all" or self.rank == 0:
                cat = torch.cat([p[:L] for p, L in zip(parts, lens)])
                glob[f] = cat.to(t.dtype)
        return local, (glob if glob else None)
