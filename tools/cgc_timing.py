"""Phase timeline of the cluster CGC kernel (debug build with -DKLE_CGC_TIMING).
usage: KLE_B200_LIB=.../libkle_tim.so python tools/cgc_timing.py [M]"""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "4096", "cgc"]
import runpy
g = runpy.run_path("tools/prof_kernels.py", run_name="prof")
import torch
from paper_2510_26180_b200 import _lib
lib = _lib.load()
buf = (ctypes.c_ulonglong * (4096 * 10))()
g["cgc"](g["sfac"]); torch.cuda.synchronize()
assert lib.kle_debug_cgc_timing(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 10).astype(np.float64)
t = t[t[:, 0] > 0]
t0 = t[:, 0].min()
names = ["prefetch", "fft_fwd", "solve_fwd", "csync1", "solve_bwd", "csync2", "pack+ifft", "update", "finish+cwait"]
d = np.diff(t, axis=1)
print("CTAs", len(t), "span us", (t[:, 9].max() - t0) / 1e3, "mean CTA life us", np.mean(t[:, 9] - t[:, 0]) / 1e3)
for i, n in enumerate(names):
    print(f"{n:14s} median {np.median(d[:, i]) / 1e3:7.2f} us  p90 {np.percentile(d[:, i], 90) / 1e3:7.2f}")
