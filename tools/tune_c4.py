"""Time one fgr and one CGC launch at c4 shapes (nx 127, N 16, J 32) with the
library named by KLE_B200_LIB; prints ms and a checksum of the outputs.
usage: KLE_B200_LIB=... python tools/tune_c4.py [M]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, make_time_grid, _lib
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, empty, ptr, stream_ptr
from paper_2510_26180_b200.pcgc import build_alpha_circulant, shift_factors

M = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
nx, N, J = 127, 16, 32
model = LogNormalKL1D(nx=nx, d=4)
grid = make_time_grid(1.0, N, J)
xi = np.random.default_rng(0).normal(size=(M, 4))
op = DeviceOperator.from_model(model, xi)
tables = AlphaTables(build_alpha_circulant(N, 1e-3))
U0 = torch.rand(M, N, nx, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
U = U0.clone()
R = empty(M, N, nx)
blob = op.blob(grid.deltat)
sfac = shift_factors(op, tables, N, grid.deltaT)
scratch = torch.zeros(16 * M, dtype=torch.uint8, device="cuda")
st = stream_ptr()


def fgr():
    _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia), ptr(op.off),
              ptr(tables.scaling), None, M, N, nx, J, grid.deltat, grid.deltaT, 1.0, 1e-3, st)


def cgc():
    _lib.call("kle_cgc_update_f64", ptr(R), ptr(U), ptr(tables.inv_scaling), ptr(tables.lam), ptr(op.dia),
              ptr(op.off), ptr(sfac), M, N, nx, grid.deltaT, 1, 1, -1.0, None, None, None, None, None,
              ptr(scratch), 16 * M, st)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


fgr()
Rsum = float(R.sum().item())
import os
if os.environ.get("TUNE_SAVE"):
    torch.save(R[:4096].cpu(), os.environ["TUNE_SAVE"])
if os.environ.get("TUNE_CMP"):
    ref = torch.load(os.environ["TUNE_CMP"])
    got = R[:4096].cpu()
    print("fgr vs saved: max abs diff %.3e, max rel (to max |ref|) %.3e" % (float((got - ref).abs().max()),
          float((got - ref).abs().max() / ref.abs().max())), flush=True)
U.copy_(U0)
cgc()
Usum = float(U.sum().item())
if os.environ.get("TUNE_SAVE"):
    torch.save(U[:4096].cpu(), os.environ["TUNE_SAVE"] + ".u")
if os.environ.get("TUNE_CMP"):
    ref = torch.load(os.environ["TUNE_CMP"] + ".u")
    got = U[:4096].cpu()
    print("cgc vs saved: max abs diff %.3e, max rel (to max |ref|) %.3e" % (float((got - ref).abs().max()),
          float((got - ref).abs().max() / ref.abs().max())), flush=True)
U.copy_(U0)
tf = timed(fgr)
tc = timed(cgc)
print(f"{_lib.library_path().name}: fgr {tf:.3f} ms ({6 * M * N * J * nx / tf / 1e9:.2f} TF/s) "
      f"cgc {tc:.3f} ms ({24 * M * N * nx / tc / 1e6:.0f} GB/s)  checks {Rsum:.15e} {Usum:.15e}", flush=True)

if len(sys.argv) > 2 and sys.argv[2] == "jsweep":
    # fixed cost per launch (prologue + epilogue) vs the per-step cost: t(J) = a + b J
    ts = {}
    for Jv in (1, 2, 8, 16, 32, 64):
        def f(Jv=Jv):
            _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia), ptr(op.off),
                      ptr(tables.scaling), None, M, N, nx, Jv, grid.deltat, grid.deltaT, 1.0, 1e-3, st)
        ts[Jv] = timed(f)
    b = (ts[64] - ts[16]) / 48
    print("jsweep ms:", {k: round(v, 3) for k, v in ts.items()}, f"per-step {b:.4f} ms, fixed {ts[32] - 32 * b:.3f} ms",
          flush=True)
