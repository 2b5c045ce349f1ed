"""CPU: the input formats either side of the path, through the product's
C-ABI host calls (no GPU needed: these are host-only):
  * request traces (JSONL) -- tie_trace_load / tie_trace_save against the reference's own
    load_trace / save_trace (proj/src/workload.cpp:82-161, compiled into oracle/_ref);
  * `tie fit` inputs (CSV prompt_id,length / JSONL {"prompt_id","lengths"}) -- against a
    restatement of load_fit_input (proj/tools/main.cpp:432-495; the CLI itself cannot be
    built here: CLI11 is not vendored), below as `ref_load_fit_input`."""
import ctypes
import json
import os

import numpy as np
import pytest

from cabi import LIB
from oracle_lib import REF_SO, ref_available

_p, _u64, _d, _u32p = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_double, ctypes.c_void_p


@pytest.fixture(scope="module")
def lib():
    L = ctypes.CDLL(LIB)
    L.tie_last_error.restype = ctypes.c_char_p
    L.tie_trace_load.argtypes = [ctypes.c_char_p, _d, _u64, ctypes.POINTER(_p)]
    L.tie_trace_size.argtypes = [_p]
    L.tie_trace_size.restype = _u64
    for nm, ct in [("ids", ctypes.c_uint64), ("arrival", ctypes.c_double),
                   ("prompt_tokens", ctypes.c_uint32), ("output_tokens", ctypes.c_uint32),
                   ("max_tokens", ctypes.c_uint32), ("mu", ctypes.c_double),
                   ("sigma", ctypes.c_double)]:
        f = getattr(L, "tie_trace_" + nm)
        f.argtypes = [_p]
        f.restype = ctypes.POINTER(ct)
    L.tie_trace_free.argtypes = [_p]
    L.tie_trace_free.restype = None
    L.tie_trace_save.argtypes = [ctypes.c_char_p, _u64, _p, _p, _p, _p, _p, _p, _p]
    L.tie_fit_input_load.argtypes = [ctypes.c_char_p, ctypes.POINTER(_p)]
    L.tie_fit_input_count.argtypes = [_p]
    L.tie_fit_input_count.restype = _u64
    L.tie_fit_input_prompt_id.argtypes = [_p, _u64]
    L.tie_fit_input_prompt_id.restype = ctypes.c_char_p
    L.tie_fit_input_offsets.argtypes = [_p]
    L.tie_fit_input_offsets.restype = ctypes.POINTER(ctypes.c_uint64)
    L.tie_fit_input_lengths.argtypes = [_p]
    L.tie_fit_input_lengths.restype = ctypes.POINTER(ctypes.c_double)
    L.tie_fit_input_free.argtypes = [_p]
    L.tie_fit_input_free.restype = None
    return L


FIELDS = ("ids", "arrival", "prompt_tokens", "output_tokens", "max_tokens", "mu", "sigma")
DT = (np.uint64, np.float64, np.uint32, np.uint32, np.uint32, np.float64, np.float64)


def load_trace(L, path, fill_rps=0.0, seed=0):
    h = _p()
    rc = L.tie_trace_load(str(path).encode(), fill_rps, seed, ctypes.byref(h))
    if rc:
        raise ValueError(L.tie_last_error().decode())
    n = L.tie_trace_size(h)
    out = {f: np.ctypeslib.as_array(getattr(L, "tie_trace_" + f)(h), (n,)).astype(dt).copy()
           if n else np.empty(0, dt) for f, dt in zip(FIELDS, DT)}
    L.tie_trace_free(h)
    return out


def save_trace(L, path, t):
    a = [np.ascontiguousarray(t[f], dt) for f, dt in zip(FIELDS, DT)]
    rc = L.tie_trace_save(str(path).encode(), len(a[0]), *[x.ctypes.data for x in a])
    assert rc == 0, L.tie_last_error().decode()


def ref_lib():
    R = ctypes.CDLL(REF_SO)
    R.ref_last_error.restype = ctypes.c_char_p
    R.ref_save_trace.argtypes = [ctypes.c_char_p, _u64] + [_p] * 7
    R.ref_load_trace.argtypes = [ctypes.c_char_p, _d, _u64, _u64] + [_p] * 7 + [
        ctypes.POINTER(_u64)]
    return R


def ref_save(R, path, t):
    a = [np.ascontiguousarray(t[f], dt) for f, dt in zip(FIELDS, DT)]
    assert R.ref_save_trace(str(path).encode(), len(a[0]), *[x.ctypes.data for x in a]) == 0


def ref_load(R, path, fill_rps=0.0, seed=0, cap=100000):
    out = [np.empty(cap, dt) for dt in DT]
    n = _u64(0)
    rc = R.ref_load_trace(str(path).encode(), fill_rps, seed, cap,
                          *[x.ctypes.data for x in out], ctypes.byref(n))
    if rc:
        raise ValueError(R.ref_last_error().decode())
    return {f: x[: n.value] for f, x in zip(FIELDS, out)}


def same(a, b):
    for f in FIELDS:
        np.testing.assert_array_equal(a[f], b[f], err_msg=f)


def synth_trace(n, seed):
    rng = np.random.default_rng(seed)
    t = {"ids": rng.permutation(n * 3)[:n].astype(np.uint64),
         "arrival": np.round(rng.exponential(0.01, n).cumsum(), 6) * rng.choice([1, 1.0000001], n),
         "prompt_tokens": rng.integers(16, 512, n).astype(np.uint32),
         "output_tokens": rng.integers(1, 2048, n).astype(np.uint32),
         "max_tokens": np.full(n, 2048, np.uint32),
         "mu": rng.uniform(0.1, 5.0, n), "sigma": rng.uniform(0.3, 1.2, n)}
    t["mu"][::7] = np.nan  # records without the log-t truth
    t["sigma"][::7] = np.nan
    t["arrival"][5] = t["arrival"][4]  # arrival ties: the stable sort keeps file order
    rng.shuffle(t["arrival"][:50])     # out-of-order arrivals: load sorts them
    return t


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_trace_roundtrips_match_reference(lib, tmp_path):
    R = ref_lib()
    t = synth_trace(3000, 1)
    p1, p2 = tmp_path / "ref.jsonl", tmp_path / "ours.jsonl"
    ref_save(R, p1, t)                       # written by the reference
    same(load_trace(lib, p1), ref_load(R, p1))
    save_trace(lib, p2, t)                   # written by us, read by the reference
    same(ref_load(R, p2), ref_load(R, p1))
    same(load_trace(lib, p2), ref_load(R, p1))


@pytest.mark.skipif(not ref_available(), reason="oracle/_ref not built (no /root/reference)")
def test_trace_missing_arrivals_fill_and_errors(lib, tmp_path):
    R = ref_lib()
    recs = [{"id": i, "prompt_tokens": 10 + i, "output_tokens": 5 * i + 1, "max_tokens": 512}
            for i in range(40)]
    for i in range(0, 40, 3):
        recs[i]["arrival_s"] = 0.05 * i
    p = tmp_path / "fill.jsonl"
    p.write_text("\n".join(json.dumps(r) for r in recs) + "\n\n")
    same(load_trace(lib, p, 50.0, 9), ref_load(R, p, 50.0, 9))
    with pytest.raises(ValueError, match="no fill rate"):
        load_trace(lib, p)
    with pytest.raises(ValueError, match="no fill rate"):
        ref_load(R, p)
    cases = {"dup": (recs[:3] + [recs[1]], "duplicate id 1"),
             "missing": ([{"id": 1, "prompt_tokens": 2, "output_tokens": 3}], "max_tokens")}
    for name, (rs, msg) in cases.items():
        q = tmp_path / f"{name}.jsonl"
        q.write_text("\n".join(json.dumps(r) for r in rs) + "\n")
        for loader in (lambda: load_trace(lib, q, 10.0), lambda: ref_load(R, q, 10.0)):
            with pytest.raises(ValueError, match=msg):
                loader()
    q = tmp_path / "bad.jsonl"
    q.write_text('{"id": 1, "prompt_tokens": 2,\n')
    with pytest.raises(ValueError, match="bad JSON"):
        load_trace(lib, q, 10.0)


# ---- `tie fit` inputs (main.cpp:432-495)
def ref_load_fit_input(path):
    """Restatement of load_fit_input (tools/main.cpp:432-495) -- test infrastructure."""
    prompts, index = [], {}
    with open(path, newline="") as f:
        lines = f.read().split("\n")
    if path.endswith(".csv"):
        if not lines or lines == [""]:
            raise ValueError(f"{path}: empty file")
        if lines[0].rstrip("\r") != "prompt_id,length":
            raise ValueError(f"{path}:1: expected header prompt_id,length")
        for no, line in enumerate(lines[1:], start=2):
            line = line.rstrip("\r")
            if not line:
                continue
            if "," not in line:
                raise ValueError(f"{path}:{no}: expected prompt_id,length")
            pid, num = line.split(",", 1)
            s = num.lstrip(" \t\n\v\f\r")
            body = s[1:] if s[:1] in "+-" else s
            if not body or not body.isdigit():
                raise ValueError(f"{path}:{no}: length must be an integer")
            val = int(s)
            if val < 1:
                raise ValueError(f"{path}:{no}: length must be >= 1")
            if pid not in index:
                index[pid] = len(prompts)
                prompts.append((pid, []))
            prompts[index[pid]][1].append(float(val))
    else:
        for no, line in enumerate(lines, start=1):
            line = line.rstrip("\r")
            if not line:
                continue
            rec = json.loads(line)
            pid, lens = rec["prompt_id"], rec["lengths"]
            if pid in index:
                raise ValueError(f"{path}:{no}: duplicate prompt_id {pid}")
            index[pid] = len(prompts)
            if any((not isinstance(v, int)) or isinstance(v, bool) or v < 1 for v in lens):
                raise ValueError(f"{path}:{no}: lengths must be integers >= 1")
            prompts.append((pid, [float(v) for v in lens]))
    if not prompts:
        raise ValueError(f"{path}: no prompts found")
    return prompts


def load_fit_input(L, path):
    h = _p()
    if L.tie_fit_input_load(str(path).encode(), ctypes.byref(h)):
        raise ValueError(L.tie_last_error().decode())
    n = L.tie_fit_input_count(h)
    off = np.ctypeslib.as_array(L.tie_fit_input_offsets(h), (n + 1,)).copy()
    lens = np.ctypeslib.as_array(L.tie_fit_input_lengths(h), (int(off[-1]),)).copy()
    out = [(L.tie_fit_input_prompt_id(h, i).decode(), lens[off[i]:off[i + 1]].tolist())
           for i in range(n)]
    L.tie_fit_input_free(h)
    return out


def test_fit_input_csv_and_jsonl(lib, tmp_path):
    rng = np.random.default_rng(3)
    rows = [(f"p{rng.integers(0, 40)}", int(rng.integers(1, 5000))) for _ in range(900)]
    c = tmp_path / "in.csv"
    c.write_text("prompt_id,length\r\n" + "".join(f"{a},{b}\r\n" for a, b in rows) + "\n")
    assert load_fit_input(lib, c) == ref_load_fit_input(str(c))
    j = tmp_path / "in.jsonl"
    recs = [{"prompt_id": f"q{i}", "lengths": [int(v) for v in rng.integers(1, 900, 5 + i % 7)]}
            for i in range(60)]
    j.write_text("\n".join(json.dumps(r) for r in recs) + "\n")
    assert load_fit_input(lib, j) == ref_load_fit_input(str(j))


@pytest.mark.parametrize("name,text,msg", [
    ("a.csv", "prompt,length\nx,1\n", "expected header"),
    ("b.csv", "prompt_id,length\nx,1.5\n", "length must be an integer"),
    ("c.csv", "prompt_id,length\nx,0\n", "length must be >= 1"),
    ("d.csv", "prompt_id,length\nnocomma\n", "expected prompt_id,length"),
    ("e.jsonl", '{"prompt_id": "a", "lengths": [1, 2.0]}\n', "integers >= 1"),
    ("f.jsonl", '{"prompt_id": "a", "lengths": [1]}\n{"prompt_id": "a", "lengths": [2]}\n',
     "duplicate prompt_id a"),
    ("g.jsonl", "\n\n", "no prompts found"),
])
def test_fit_input_errors(lib, tmp_path, name, text, msg):
    p = tmp_path / name
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        load_fit_input(lib, p)
    with pytest.raises(ValueError, match=msg):
        ref_load_fit_input(str(p))


def test_python_api_trace_and_fit_input(tie, tmp_path):
    t = synth_trace(500, 2)
    p = tmp_path / "t.jsonl"
    tie.save_trace_soa(str(p), t["ids"], t["arrival"], t["prompt_tokens"], t["output_tokens"],
                       t["max_tokens"], t["mu"], t["sigma"])
    d = tie.load_trace_soa(str(p))
    order = np.argsort(t["arrival"], kind="stable")
    np.testing.assert_array_equal(d["id"], t["ids"][order])
    np.testing.assert_array_equal(d["mu"], t["mu"][order])
    # the reference's list-of-Request form (module.cpp:154-156): round trip through both
    reqs = tie.load_trace(str(p))
    assert [r.id for r in reqs] == d["id"].tolist()
    assert [r.true_mu for r in reqs] == [None if np.isnan(v) else v for v in d["mu"]]
    p2 = tmp_path / "t2.jsonl"
    tie.save_trace(reqs, str(p2))
    d2 = tie.load_trace_soa(str(p2))
    for k in ("id", "arrival_s", "prompt_tokens", "output_tokens", "max_tokens"):
        np.testing.assert_array_equal(d2[k], d[k])
    c = tmp_path / "f.csv"
    c.write_text("prompt_id,length\na,3\nb,4\na,5\n")
    ids, off, lens = tie.load_fit_input(str(c))
    assert ids == ["a", "b"] and off.tolist() == [0, 2, 3] and lens.tolist() == [3, 5, 4]
