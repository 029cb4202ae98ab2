"""Time the 2D kernels at config-3 shapes.
usage: python tools/prof_2d.py [M] [n] [N] [J]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL2D, SolverConfig, make_time_grid, _lib
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, empty, ptr, stream_ptr
from paper_2510_26180_b200.pcgc import build_alpha_circulant
from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

M = int(sys.argv[1]) if len(sys.argv) > 1 else 64
n = int(sys.argv[2]) if len(sys.argv) > 2 else 127
N = int(sys.argv[3]) if len(sys.argv) > 3 else 32
J = int(sys.argv[4]) if len(sys.argv) > 4 else 16
model = LogNormalKL2D(n=n, d=10)
grid = make_time_grid(1.0, N, J)
xi = np.random.default_rng(0).normal(size=(M, 10))
op = DeviceOperator.from_model(model, xi)
tables = AlphaTables(build_alpha_circulant(N, 1e-3))


def timed(name, f, reps=1):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:28s} {e0.elapsed_time(e1) / reps:10.3f} ms  (M={M})", flush=True)
    return r


# warm-up (module load, first launches) on a 1-sample operator
w = DeviceOperator.from_model(model, xi[:1])
w.fine_factor(grid.deltat); w.shifted_factors(tables, N, grid.deltaT)
Uw = coarse_sweep_init_batched(w, grid).contiguous(); w.fgr(Uw, tables, grid, 1e-3, empty(1, N, n * n))
torch.cuda.synchronize()
timed("factor real (I + dt A)", lambda: op.fine_factor(grid.deltat))
import os
SKIP_C = os.environ.get("PROF2D_NO_CGC") == "1"
fac = None if SKIP_C else timed("factor complex (17 shifts)", lambda: op.shifted_factors(tables, N, grid.deltaT))
U = coarse_sweep_init_batched(op, grid).contiguous()
R = empty(M, N, n * n)
status = torch.zeros(M, dtype=torch.int32, device="cuda")
if hasattr(op, "fine_stage"):
    timed("restage (TMA chunks)", lambda: op.fine_stage(grid.deltat))
timed("fgr2d (J steps, N rhs)", lambda: op.fgr(U, tables, grid, 1e-3, R, status=status))
if SKIP_C:
    sys.exit(0)
nw = int(_lib.query("kle_2d_cgc_work_doubles", M, N, n))
work = torch.zeros(nw, dtype=torch.float64, device="cuda")
iters = torch.zeros(M, dtype=torch.int32, device="cuda")
act = torch.zeros(1, dtype=torch.int32, device="cuda")
timed("cgc2d (dft, solves, update)", lambda: _lib.call(
    "kle_2d_cgc_f64", ptr(R), None, ptr(U), None, ptr(fac[0]), ptr(fac[1]), ptr(tables.inv_scaling), M, N, n, 1, 60,
    -1.0, ptr(status), ptr(iters), None, None, ptr(act), ptr(work), nw, stream_ptr()))
