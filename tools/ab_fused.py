"""A/B of the fused small-block iteration (KLE_FUSED=1, default) against the
separate fgr + cluster-CGC kernels (KLE_FUSED=0) on config-4 shapes: the
batched PCGC from the config's surrogate, iteration counts, max field
difference, and the time of one full solve per path.
usage: python tools/ab_fused.py [M] [modes, default 0,1]"""
import os
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, RngStream, SolverConfig, make_time_grid
from paper_2510_26180_b200.engine import KleCgcSolver
from paper_2510_26180_b200.models import ParameterMap
from paper_2510_26180_b200.surrogate import KLGpcSurrogate

M = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
g = np.load("tests/golden/c1.npz")
model = LogNormalKL1D(nx=127, d=4)
grid = make_time_grid(1.0, 16, 32)
cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
sur = KLGpcSurrogate(g["mean_field"], g["eigenvalues"], g["modes"], g["coeffs"], 2,
                     [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
xi = torch.as_tensor(RngStream(2718).split(3)[1].normal(0.0, 1.0, size=(M, 4)), device="cuda")
solver = KleCgcSolver(model, grid, cfg, sur)
out = {}
modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1"]
for fused in modes:
    os.environ["KLE_FUSED"] = fused
    solver.solve(xi)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    res = solver.solve(xi)
    b.record()
    torch.cuda.synchronize()
    out[fused] = (res.batch.states.clone(), res.batch.iters.clone(), res.batch.status.clone(), a.elapsed_time(b))
    print(f"KLE_FUSED={fused}: {out[fused][3]:.2f} ms per solve ({M / out[fused][3] * 1e3:.0f} solves/s), "
          f"mean iters {out[fused][1].double().mean().item():.4f}", flush=True)
s0, i0, st0, _ = out[modes[0]]
s1, i1, st1, _ = out[modes[-1]]
print("iters equal:", bool(torch.equal(i0, i1)), "status equal:", bool(torch.equal(st0, st1)),
      "all converged:", bool((st1 == 1).all()))
print("max rel field diff:", float((s0 - s1).abs().max() / s0.abs().max()))
print("first 16 iters vs c1 golden:", bool(np.array_equal(i1[:16].cpu().numpy(), g["iters"])))
