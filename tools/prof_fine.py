import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2510_26180_b200 import LogNormalKL1D, make_time_grid, _lib
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, empty, ptr, stream_ptr
from paper_2510_26180_b200.pcgc import build_alpha_circulant
nx, N, J, M = 511, 64, 64, 2048
model = LogNormalKL1D(nx=nx, d=4); grid = make_time_grid(1.0, N, J)
xi = np.random.default_rng(0).normal(size=(M, 4))
tables = AlphaTables(build_alpha_circulant(N, 1e-3))
U = torch.rand(M, N, nx, dtype=torch.float64, device="cuda"); R = empty(M, N, nx)
for v in sys.argv[1].split(","):
    os.environ["KLE_FINE_VARIANT"] = v
    op = DeviceOperator.from_model(model, xi); blob = op.blob(grid.deltat)
    for _ in range(2):
        _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia), ptr(op.off),
                  ptr(tables.scaling), None, M, N, nx, J, grid.deltat, grid.deltaT, 1.0, 1e-3, stream_ptr())
    torch.cuda.synchronize()
print("done")
