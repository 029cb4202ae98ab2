"""A/B of the large-block CGC at config-5 shapes: the three-kernel path
(default) against the streaming kernels (KLE_CGCL_STREAM=1, read once per
process: run twice). Prints the time of one CGC launch over M samples and a
checksum of the updated U (bitwise equal between the paths).
usage: [KLE_CGCL_STREAM=1] python tools/ab_cgcl.py [M]"""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, make_time_grid, _lib
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, empty, ptr, stream_ptr
from paper_2510_26180_b200.pcgc import build_alpha_circulant

M = int(sys.argv[1]) if len(sys.argv) > 1 else 256
nx, N = 4095, 1024
model = LogNormalKL1D(nx=nx, d=4)
grid = make_time_grid(1.0, N, 8)
op = DeviceOperator.from_model(model, np.random.default_rng(0).normal(size=(M, 4)))
tables = AlphaTables(build_alpha_circulant(N, 1e-4))
g = torch.Generator("cuda").manual_seed(3)
R = torch.rand(M, N, nx, dtype=torch.float64, device="cuda", generator=g) - 0.5
U0 = torch.rand(M, N, nx, dtype=torch.float64, device="cuda", generator=g)
U = U0.clone()
nb = int(_lib.query("kle_cgc_scratch_bytes", M, N, nx))
scratch = torch.zeros(nb, dtype=torch.uint8, device="cuda")
inc = torch.full((M, 1), float("nan"), dtype=torch.float64, device="cuda")


def cgc():
    _lib.call("kle_cgc_update_f64", ptr(R), ptr(U), ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia),
              ptr(op.off), None, M, N, nx, grid.deltaT, 1, 1, -1.0, None, None, ptr(inc), None, None,
              ptr(scratch), nb, stream_ptr())


cgc()
torch.cuda.synchronize()
chk = float(U.sum().item())
incs = inc.clone()
U.copy_(U0)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(3):
    cgc()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
print(f"stream={os.environ.get('KLE_CGCL_STREAM', '0')} M={M}: {ms:.2f} ms per CGC launch "
      f"({24.0 * M * N * nx / ms / 1e6:.0f} GB/s compulsory), checksum {chk:.17e}, inc0 {float(incs[0, 0]):.17e}")
