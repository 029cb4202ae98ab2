"""Phase timeline of the cluster CGC kernel at c4 shapes (debug build with -DKLE_CGC_TIMING; globaltimer ns).
usage: KLE_B200_LIB=.../libkle_ctim.so python tools/cgc_timing_c4.py [M]"""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "131072"]
import runpy
g = runpy.run_path("tools/tune_c4.py", run_name="prof")
import torch
from paper_2510_26180_b200 import _lib
lib = _lib.load()
buf = (ctypes.c_ulonglong * (4096 * 10))()
g["cgc"](); torch.cuda.synchronize()
assert lib.kle_debug_cgc_timing(buf) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 10).astype(np.float64)
t = t[t[:, 0] > 0]
names = ["prefetch", "fft_fwd", "solve_fwd", "csync1", "solve_bwd", "csync2", "pack+ifft", "update", "finish+cwait"]
d = np.diff(t, axis=1)
print("CTAs", len(t), "mean CTA life", np.mean(t[:, 9] - t[:, 0]))
for i, n in enumerate(names):
    print(f"{n:14s} median {np.median(d[:, i]):8.0f}  p10 {np.percentile(d[:, i], 10):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}")
