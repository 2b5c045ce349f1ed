"""Patch a COPY of queue.cu with %globaltimer phase stamps of the scheduler step's apply
kernel (development tool; used on _ab/<variant>/ sources, built with -DTIE_APPLY_TIMING):
    python tools/apply_timing_patch.py _ab/timing/paper_2604_00499_b200/csrc/queue.cu
Thread 0 prints "APPLY_TS ... idx:ns" for every 16th step; stamps 2 arrivals, 4 predictions,
6 key writes + refresh, 10 pop start, 14 block rounds done, 11 register-path loads + sort done,
12 its rounds done, 13 after its barrier, 8 pops done, 9 completion record written."""
import sys

p = sys.argv[1]
s = open(p).read()


def rep(a, b):
    global s
    assert s.count(a) == 1, a[:70]
    s = s.replace(a, b)


macro = r'''#ifdef TIE_APPLY_TIMING
__shared__ unsigned long long tie_ts[16];
#define TIE_TS(n)                                                        \
  do {                                                                   \
    if (threadIdx.x == 0) {                                              \
      unsigned long long t_;                                             \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));             \
      tie_ts[n] = t_;                                                    \
    }                                                                    \
  } while (0)
#else
#define TIE_TS(n) \
  do {            \
  } while (0)
#endif

'''
anchor = "// Up to `pops` pop_min()s with fixed keys in ONE pass"
rep(anchor, macro + anchor)
rep("  scan_top2(0, 0xffffffffu);" if "scan_top2(0, 0xffffffffu);" in s else "  scan_top2(0);",
    "  TIE_TS(10);\n" + ("  scan_top2(0, 0xffffffffu);" if "scan_top2(0, 0xffffffffu);" in s
                         else "  scan_top2(0);"))
rep("  if (kSmallPath && nchosen < pops && nchosen <= 8 && blockDim.x == 1024) {",
    "  TIE_TS(14);\n  if (kSmallPath && nchosen < pops && nchosen <= 8 && blockDim.x == 1024) {")
i = s.index("__device__ __forceinline__ void pop_from_blocks_regs(")
j = s.index("  uint32_t done = 0;\n  for (; done < pops; ++done) {", i)
s = s[:j] + "  TIE_TS(11);\n" + s[j:]
rep("  if (threadIdx.x == 0) *out_n = done;\n  __syncthreads();\n  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n  for (uint32_t e = warp; e < nchosen; e += blockDim.x >> 5) {",
    "  TIE_TS(12);\n  if (threadIdx.x == 0) *out_n = done;\n  __syncthreads();\n  TIE_TS(13);\n  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n  for (uint32_t e = warp; e < nchosen; e += blockDim.x >> 5) {")
rep("  cudaGridDependencySynchronize();\n  for (uint64_t t = threadIdx.x; t < np; t += blockDim.x) {",
    "  TIE_TS(2);\n  cudaGridDependencySynchronize();\n  for (uint64_t t = threadIdx.x; t < np; t += blockDim.x) {")
rep("  const bool skip = bad ||", "  TIE_TS(4);\n  const bool skip = bad ||")
rep("  if (skip || pops == 0) {\n    if (threadIdx.x == 0) *out_n = 0;",
    "  TIE_TS(6);\n  if (skip || pops == 0) {\n    if (threadIdx.x == 0) *out_n = 0;")
rep("  if (status_seq) {  // the step's last kernel",
    "  TIE_TS(8);\n  if (status_seq) {  // the step's last kernel")
i = s.index("__global__ void __launch_bounds__(1024) step_apply_kernel(")
j = s.index("  __shared__ int bad;\n  if (threadIdx.x == 0) bad = 0;\n", i)
k = j + len("  __shared__ int bad;\n  if (threadIdx.x == 0) bad = 0;\n")
s = s[:k] + "#ifdef TIE_APPLY_TIMING\n  if (threadIdx.x == 0)\n    for (int x = 0; x < 16; ++x) tie_ts[x] = 0;\n#endif\n  TIE_TS(0);\n" + s[k:]
e = s.index("      *status_seq = seq | (failed ? kStatusErrBit : 0u);\n    }\n  }\n}", i)
e2 = e + len("      *status_seq = seq | (failed ? kStatusErrBit : 0u);\n    }\n  }\n")
s = s[:e2] + r'''#ifdef TIE_APPLY_TIMING
  __syncthreads();
  TIE_TS(9);
  if (threadIdx.x == 0 && seq % 16 == 0) {
    printf("APPLY_TS n_arr=%llu np=%llu nblk=%u nblocks=%u pops=%u", (unsigned long long)n_arr,
           (unsigned long long)np, nblk, nblocks, pops);
    for (int x = 1; x < 16; ++x)
      printf(" %d:%lld", x, tie_ts[x] ? (long long)(tie_ts[x] - tie_ts[0]) : -1ll);
    printf("\n");
  }
#endif
''' + s[e2:]
open(p, "w").write(s)
print("patched", p)
