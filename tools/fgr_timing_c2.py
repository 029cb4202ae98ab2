"""Phase timeline of the c2 fgr kernel (debug build with -DKLE_FGR_TIMING -DKLE_FGR_T0=2000; SM clock cycles).
usage: KLE_B200_LIB=.../libkle_ftim2.so python tools/fgr_timing_c2.py [M]"""
import ctypes, sys
sys.path.insert(0, ".")
import numpy as np
sys.argv = [sys.argv[0], sys.argv[1] if len(sys.argv) > 1 else "8192", "fgr"]
import runpy
g = runpy.run_path("tools/prof_kernels.py", run_name="prof")
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
