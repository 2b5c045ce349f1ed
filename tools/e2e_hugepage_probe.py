"""e2e score+rank (1M) with the host buffers from torch pin_memory (cudaHostAlloc) vs 2 MB
aligned anonymous memory advised for transparent huge pages and registered with
cudaHostRegister (development tool: per-process DMA throughput variance)."""
import ctypes
import json
import mmap
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_00499_b200 as tie  # noqa: E402

libc = ctypes.CDLL("libc.so.6", use_errno=True)
MADV_HUGEPAGE = 14


def thp_array(nbytes):
    size = (nbytes + (2 << 20) - 1) & ~((2 << 20) - 1)
    m = mmap.mmap(-1, size + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(m))
    al = (base + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(al), ctypes.c_size_t(size), MADV_HUGEPAGE)
    arr = np.frombuffer(m, dtype=np.uint8, count=size, offset=al - base)
    arr[:] = 0  # fault in (huge pages when THP allows)
    rc = torch.cuda.cudart().cudaHostRegister(al, size, 0)
    assert int(rc) == 0, rc
    return m, arr


def main(mode):
    n = 1_000_000
    mc = tie.McContext(3.5, 10000, 12, 0)
    w = tie.gen_logt_workload_soa(n, 1)
    keep = []
    if mode == "torch":
        pin = lambda a: torch.from_numpy(a).pin_memory()
        mu, sg, mt = pin(w["mu"]), pin(w["sigma"]), pin(w["max_tokens"].view(np.int32))
        order = torch.empty(n, dtype=torch.int64).pin_memory()
        ptrs = [t.data_ptr() for t in (mu, sg, mt, order)]
    else:
        ptrs = []
        for a in (w["mu"], w["sigma"], w["max_tokens"], np.empty(n, np.int64)):
            m, buf = thp_array(a.nbytes)
            buf[:a.nbytes] = a.view(np.uint8)
            keep.append(m)
            ptrs.append(buf.ctypes.data)
    f = lambda: tie.score_rank_host_ptr(mc.handle, ptrs[0], ptrs[1], ptrs[2], n, 0.9, 0.5, 0,
                                        ptrs[3], 0)
    for _ in range(5):
        f()
    if os.environ.get("WITH_SAMPLER"):  # bench.py's nvidia-smi clock sampler around a soak
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench

        cs = bench.ClockSampler(0)
        cs.start()
        x = torch.empty(64 << 20, device="cuda")
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 1.5:
            x.mul_(1.0001)
        torch.cuda.synchronize()
        cs.stop()
    ts = []
    for _ in range(40):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    thp = open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip()
    print(json.dumps({"mode": mode, "sampler": bool(os.environ.get("WITH_SAMPLER")),
                      "e2e_ms_median": 1e3 * float(np.median(ts)), "thp": thp}))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "torch")
