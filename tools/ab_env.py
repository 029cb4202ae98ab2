"""A/B of a per-call environment switch on the batched config-4 solve (c1
golden surrogate U0): time per solve, iteration counts and the largest field
difference against the first setting.
usage: python tools/ab_env.py VAR v1,v2,... [M]"""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, RngStream, SolverConfig, make_time_grid
from paper_2510_26180_b200.engine import KleCgcSolver
from paper_2510_26180_b200.models import ParameterMap
from paper_2510_26180_b200.surrogate import KLGpcSurrogate

var, vals = sys.argv[1], sys.argv[2].split(",")
M = int(sys.argv[3]) if len(sys.argv) > 3 else 131072
g = np.load("tests/golden/c1.npz")
sur = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2,
                     [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
solver = KleCgcSolver(LogNormalKL1D(nx=127, d=4), make_time_grid(1.0, 16, 32),
                      SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60), sur)
xi = torch.as_tensor(RngStream(2718).split(3)[1].normal(0.0, 1.0, size=(M, 4)), device="cuda")
base = None
for v in vals:
    os.environ[var] = v
    solver.solve(xi)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    res = solver.solve(xi)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    st, it = res.batch.states.clone(), res.batch.iters.clone()
    line = f"{var}={v}: {ms:.2f} ms per solve ({M / ms * 1e3:.0f} solves/s), mean iters {it.double().mean().item():.4f}"
    if base is None:
        base = (st, it)
    else:
        line += (f", iters equal {bool(torch.equal(base[1], it))}, max rel field diff "
                 f"{float((base[0] - st).abs().max() / base[0].abs().max()):.2e}")
    line += f", first 16 iters = c1 golden: {bool(np.array_equal(it[:16].cpu().numpy(), g['iters']))}"
    print(line, flush=True)
