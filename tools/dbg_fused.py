import os, sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
from paper_2510_26180_b200.pcgc import pcgc_solve_batched
g = np.load("tests/golden/c1.npz")
model = LogNormalKL1D(nx=127, d=4); grid = make_time_grid(1.0, 16, 32)
cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
for f in ("0", "1"):
    os.environ["KLE_FUSED"] = f
    r = pcgc_solve_batched(model, g["xi_all"][:4], grid, cfg, g["U0"][:4])
    torch.cuda.synchronize()
    print(f, r.iters.tolist(), r.status.tolist(), r.increments[:, :4].tolist(), float(r.states.abs().max()))
