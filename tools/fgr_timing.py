"""Phase timeline of the c4 fgr kernel (debug build with -DKLE_FGR_TIMING; SM clock cycles).
usage: KLE_B200_LIB=.../libkle_ftim.so python tools/fgr_timing.py [M]"""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "131072"]
import runpy
g = runpy.run_path("tools/tune_c4.py", run_name="prof")
import torch
from paper_2510_26180_b200 import _lib
lib = _lib.load()
buf = (ctypes.c_longlong * (4096 * 16))()
g["fgr"](); torch.cuda.synchronize()
assert lib.kle_debug_fgr_timing(buf) == 0
t = np.frombuffer(buf, dtype=np.int64).reshape(4096, 16).astype(np.float64)
t = t[t[:, 0] > 0]
names = ["issue loads+blob+chunk products", "wait start rows", "smem -> registers", "J steps", "epilogue math + stage",
         "stores"]
d = np.diff(t[:, :7], axis=1)
print("CTAs", len(t), "mean CTA life cycles", np.mean(t[:, 6] - t[:, 0]))
for i, n in enumerate(names):
    print(f"{n:34s} median {np.median(d[:, i]):9.0f} cyc  p10 {np.percentile(d[:, i], 10):9.0f}  p90 {np.percentile(d[:, i], 90):9.0f}")
# per-SM slot turnaround: gap between one CTA's end and the start of the next CTA launched on that SM
sm = t[:, 7].astype(int)
gaps = []
for q in np.unique(sm):
    a = t[sm == q]
    starts = np.sort(a[:, 0]); ends = np.sort(a[:, 6])
    # with 8 slots per SM the k-th start follows the k-th end (FIFO refill); ends before the first start are other CTAs
    for st_ in starts:
        prev = ends[ends <= st_]
        if len(prev):
            gaps.append(st_ - prev[-1])
gaps = np.array(gaps)
if len(gaps):
    print(f"start - latest earlier end on the same SM: median {np.median(gaps):.0f} cyc  p90 {np.percentile(gaps, 90):.0f}")

if t[:, 8].max() > 0:  # in-step stamps of step 1 (eager be_steps_cs builds)
    names2 = ["fwd local", "fwd scan", "fwd stitch", "bwd local", "bwd scan", "bwd stitch"]
    d2 = np.diff(t[:, 8:15], axis=1)
    for i, n in enumerate(names2):
        print(f"  step 1: {n:12s} median {np.median(d2[:, i]):7.0f} cyc  p10 {np.percentile(d2[:, i], 10):7.0f}  p90 {np.percentile(d2[:, i], 90):7.0f}")
    print(f"  step 1 total median {np.median(t[:, 14] - t[:, 8]):.0f}")

# warp slots: which SM sub-partition (warpid % 4) the concurrently resident one-warp CTAs sit on
wid = t[:, 15].astype(int)
import collections
print("warpid histogram:", sorted(collections.Counter(wid.tolist()).items()))
occ = []
for q in np.unique(sm)[:40]:
    a = t[sm == q]
    # at the start time of each CTA, which other CTAs of this SM are alive?
    for row in a[:8]:
        alive = a[(a[:, 0] <= row[0]) & (a[:, 6] > row[0])]
        c = collections.Counter((alive[:, 15].astype(int) % 4).tolist())
        occ.append(tuple(c.get(i, 0) for i in range(4)))
print("resident CTAs per sub-partition (samples):", collections.Counter(occ).most_common(8))
