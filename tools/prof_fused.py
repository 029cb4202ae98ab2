"""Run the batched PCGC at c4 shapes (fused iteration kernel) for ncu capture.
usage: python tools/prof_fused.py [M]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid
from paper_2510_26180_b200.pcgc import pcgc_solve_batched

M = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
g = np.load("tests/golden/c1.npz")
xi = np.random.default_rng(0).normal(size=(M, 4))
U0 = np.broadcast_to(g["U0"][0], (M, 16, 127)).copy()
r = pcgc_solve_batched(LogNormalKL1D(nx=127, d=4), xi, make_time_grid(1.0, 16, 32),
                       SolverConfig(alpha=1e-3, tol=1e-8, max_outer_iters=60), U0)
torch.cuda.synchronize()
print("iters", float(r.iters.double().mean()))
