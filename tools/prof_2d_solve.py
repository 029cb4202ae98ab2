"""Phase timing of the batched 2D PCGC solve (KLE_2D_PROFILE=1) at config-3 shapes.
usage: KLE_2D_PROFILE=1 python tools/prof_2d_solve.py [M]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL2D, SolverConfig, make_time_grid
from paper_2510_26180_b200.device import DeviceOperator
from paper_2510_26180_b200.pcgc import pcgc_solve_device
from paper_2510_26180_b200.propagators import coarse_sweep_init_batched

M = int(sys.argv[1]) if len(sys.argv) > 1 else 296
model = LogNormalKL2D(n=127, d=10)
grid = make_time_grid(1.0, 32, 16)
cfg = SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60)
op = DeviceOperator.from_model(model, np.random.default_rng(0).normal(size=(M, 10)))
U = coarse_sweep_init_batched(op, grid).contiguous()
torch.cuda.synchronize()
res = pcgc_solve_device(op, U, grid, cfg)
print("iters", np.bincount(res.iters.cpu().numpy()))
