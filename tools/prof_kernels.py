"""Launch the hot kernels on config-2 shapes for ncu capture.
usage: python tools/prof_kernels.py [M] [which: fgr,cgc,cgcfly,gemm] [nx,N,J]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, make_time_grid, _lib
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, empty, ptr, stream_ptr
from paper_2510_26180_b200.pcgc import build_alpha_circulant, shift_factors

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
which = sys.argv[2].split(",") if len(sys.argv) > 2 else ["fgr", "cgc"]
nx, N, J = (int(v) for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else (511, 64, 64)))
model = LogNormalKL1D(nx=nx, d=8)
grid = make_time_grid(1.0, N, J)
xi = np.random.default_rng(0).normal(size=(M, 8))
op = DeviceOperator.from_model(model, xi)
tables = AlphaTables(build_alpha_circulant(N, 1e-3))
U = torch.rand(M, N, nx, dtype=torch.float64, device="cuda")
R = empty(M, N, nx)
blob = op.blob(grid.deltat)
sfac = shift_factors(op, tables, N, grid.deltaT)
st = stream_ptr()


def fgr():
    _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia), ptr(op.off),
              ptr(tables.scaling), None, M, N, nx, J, grid.deltat, grid.deltaT, 1.0, 1e-3, st)


nb = int(_lib.query("kle_cgc_scratch_bytes", M, N, nx))
scratch = torch.zeros(nb, dtype=torch.uint8, device="cuda")


def cgc(s):
    _lib.call("kle_cgc_update_f64", ptr(R), ptr(U), ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia),
              ptr(op.off), ptr(s), M, N, nx, grid.deltaT, 1, 1, -1.0, None, None, None, None, None,
              ptr(scratch), nb, st)


for rep in range(2):
    for w in which:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        if w == "fgr":
            fgr()
        elif w == "cgc":
            cgc(sfac)
        elif w == "cgcfly":
            cgc(None)
        ev1.record()
        torch.cuda.synchronize()
        print(w, rep, f"{ev0.elapsed_time(ev1):.3f} ms")
