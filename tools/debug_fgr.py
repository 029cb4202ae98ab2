import sys, ctypes as C
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2510_26180_b200 import LogNormalKL1D, make_time_grid, SolverConfig, _lib
from paper_2510_26180_b200.device import DeviceOperator, empty, ptr, stream_ptr, AlphaTables
from paper_2510_26180_b200.pcgc import build_alpha_circulant
cr = C.CDLL("libcudart.so.12") if False else None
for nx, N, J, M in [(511, 64, 64, 4), (511, 64, 64, 2048), (255, 64, 8, 4), (1000, 64, 8, 4)]:
    model = LogNormalKL1D(nx=nx, d=8)
    grid = make_time_grid(1.0, N, J)
    xi = np.random.default_rng(0).normal(size=(M, 8))
    op = DeviceOperator.from_model(model, xi)
    U = torch.zeros(M, N, nx, dtype=torch.float64, device="cuda")
    R = empty(M, N, nx)
    t = AlphaTables(build_alpha_circulant(N, 1e-3))
    try:
        _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(op.blob(grid.deltat)), ptr(op.dia), ptr(op.off),
                  ptr(t.scaling), None, M, N, nx, J, grid.deltat, grid.deltaT, 1.0, 1e-3, stream_ptr())
        torch.cuda.synchronize()
        print(nx, N, M, "ok", float(R.abs().max()))
    except Exception as e:
        print(nx, N, M, "FAIL", e)
