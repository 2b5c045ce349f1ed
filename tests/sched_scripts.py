"""Random Scheduler event scripts (test infrastructure): arrivals, predictions and pops in
runs, shaped so that drift rebuilds, ties and the FCFS / SEPT / TIE policies all occur."""
import numpy as np

ARRIVE, PREDICT, POP = 0, 1, 2


def make_script(seed, oracle, policy=2, n_req=600, max_tokens_choices=(256, 512, 2048),
                runs=80, arr_max=24, **cfg):
    """`oracle` replays the prefix after every pop run so predictions only name requests
    that are still waiting (the simulator drops stale predictions the same way)."""
    rng = np.random.default_rng(seed)
    ids = rng.permutation(np.arange(10_000, 10_000 + n_req, dtype=np.uint64))
    ops, oid, a, b = [], [], [], []
    waiting, unpredicted = [], []
    nxt, t = 0, 0.0
    for _ in range(runs):
        kind = rng.choice(3, p=[0.4, 0.35, 0.25])
        if kind == 0 and nxt < n_req:
            for _ in range(int(rng.integers(1, arr_max))):
                if nxt >= n_req:
                    break
                t += float(rng.exponential(0.01))
                ops.append(ARRIVE)
                oid.append(ids[nxt])
                a.append(round(t, 3))  # coarse arrivals: FCFS ties
                b.append(float(rng.choice(max_tokens_choices)))  # size ties
                waiting.append(ids[nxt])
                unpredicted.append(ids[nxt])
                nxt += 1
        elif kind == 1 and unpredicted:
            k = int(rng.integers(1, min(16, len(unpredicted)) + 1))
            pick = rng.choice(len(unpredicted), size=k, replace=False)
            for j in sorted(pick, reverse=True):
                rid = unpredicted.pop(j)
                E = float(np.round(rng.lognormal(4.0, 0.8), 1)) + 1.0
                C = E * float(rng.choice([1.0, 1.5, 3.0, 10.0]))
                ops.append(PREDICT)
                oid.append(rid)
                a.append(E)
                b.append(C)
        else:
            for _ in range(int(rng.integers(1, 9))):
                ops.append(POP)
                oid.append(0)
                a.append(0.0)
                b.append(0.0)
            popped = set(int(x) for x in oracle.scheduler_script(
                policy, ops, oid, a, b, **cfg) if x != np.iinfo(np.uint64).max)
            unpredicted = [r for r in unpredicted if int(r) not in popped]
    return np.array(ops, np.int32), np.array(oid, np.uint64), np.array(a), np.array(b)


def runs_of(ops):
    """Consecutive same-kind op groups: [(kind, start, stop), ...]."""
    out, start = [], 0
    for i in range(1, len(ops) + 1):
        if i == len(ops) or ops[i] != ops[start]:
            out.append((int(ops[start]), start, i))
            start = i
    return out
