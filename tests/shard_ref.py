"""Reference-semantics shard of a Scheduler (test infrastructure for the sharded scheduler's
host protocol on CPU): the per-shard state of sched.cpp:28-175 -- entries keyed as
on_arrival / on_prediction key them, betas_in_use_ -- plus the shard primitives the
GpuScheduler exports (set_peer_waiting, beta_range, rebuild_at, peek).  Plain Python over a
few hundred entries; the pop order is the WaitingQueue's (key, id) order (sched.cpp:28-31)."""
import struct
from collections import Counter

import numpy as np


def order_bits(x: float) -> int:
    """order-preserving u64 image of a double (what the device keys hold)"""
    b = struct.unpack("<Q", struct.pack("<d", float(x)))[0]
    return (~b) & 0xFFFFFFFFFFFFFFFF if b >> 63 else b | (1 << 63)


class RefShard:
    def __init__(self, policy, beta_fn, threshold):
        self.policy = policy
        self.beta_fn = beta_fn
        self.thr = threshold
        self.e = {}          # id -> [key, predicted, E, C, beta]
        self.betas = Counter()
        self.peers = 0

    def waiting(self):
        return len(self.e)

    def set_peer_waiting(self, peers):
        self.peers = int(peers)

    def beta_range(self):
        if not self.betas:
            return 0.0, 0.0, 0
        return min(self.betas), max(self.betas), sum(self.betas.values())

    def on_arrival_batch(self, ids, arrival_s, max_tokens):
        for i, t, m in zip(ids, arrival_s, max_tokens):
            if int(i) in self.e:
                raise ValueError("WaitingQueue::push: id already queued")
            key = float(t) if self.policy == 0 else float(np.uint32(m))
            self.e[int(i)] = [key, False, 0.0, 0.0, 0.0]

    def on_prediction_batch(self, ids, E, C):
        for i, a, b in zip(ids, E, C):
            ent = self.e.get(int(i))
            if ent is None:
                raise ValueError("Scheduler::on_prediction: id not waiting")
            if self.policy == 0:
                continue
            if ent[1]:
                raise ValueError("Scheduler::on_prediction: id already predicted")
            beta = self.beta_fn(len(self.e) + self.peers) if self.policy == 2 else 0.0
            ent[:] = [float(a) + beta * float(b) if self.policy == 2 else float(a), True,
                      float(a), float(b), beta]
            if self.policy == 2:
                self.betas[beta] += 1

    def rebuild_at(self, beta):
        if self.policy != 2 or not self.betas:
            return
        self.betas = Counter()
        for ent in self.e.values():
            if ent[1]:
                ent[0] = ent[2] + beta * ent[3]
                ent[4] = beta
                self.betas[beta] += 1

    def _order(self):
        return sorted(self.e, key=lambda i: (self.e[i][0], i))

    def peek(self, k):
        top = self._order()[:k]
        return (np.array([order_bits(self.e[i][0]) for i in top], np.uint64),
                np.array(top, np.uint64))

    def next_requests(self, k):
        """next_request() x k with this shard's own drift check (sched.cpp:152-175)"""
        out = []
        for _ in range(k):
            if not self.e:
                break
            if self.policy == 2 and self.betas:
                now = self.beta_fn(len(self.e) + self.peers)
                if max(abs(now - min(self.betas)), abs(now - max(self.betas))) > self.thr:
                    self.rebuild_at(now)
            i = self._order()[0]
            ent = self.e.pop(i)
            if ent[1] and self.policy == 2:
                self.betas[ent[4]] -= 1
                if not self.betas[ent[4]]:
                    del self.betas[ent[4]]
            out.append(i)
        return np.array(out, np.uint64)
