"""Small invocation of every libkle_b200 kernel (for compute-sanitizer)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, SolverConfig, make_time_grid, ParameterSample
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, to_dev
from paper_2510_26180_b200.pcgc import build_alpha_circulant, pcgc_solve_device, three_step_device
from paper_2510_26180_b200.propagators import coarse_sweep_init_batched
from paper_2510_26180_b200.moments import two_pass_moments
from paper_2510_26180_b200.models import ParameterMap
from paper_2510_26180_b200.surrogate import DeviceSurrogate, KLGpcSurrogate

rng = np.random.default_rng(0)
for nx, N, J, M, d in [(127, 16, 32, 6, 4), (511, 64, 8, 2, 8), (63, 12, 4, 3, 4), (1500, 4, 2, 1, 4)]:
    model = LogNormalKL1D(nx=nx, d=d)
    grid = make_time_grid(1.0, N, J)
    cfg = SolverConfig(alpha=1e-2, tol=1e-8, max_outer_iters=30)
    xi = rng.normal(size=(M, d))
    op = DeviceOperator.from_model(model, xi)
    U = coarse_sweep_init_batched(op, grid).contiguous()
    res = pcgc_solve_device(op, U, grid, cfg)
    u, im = three_step_device(op, AlphaTables(build_alpha_circulant(N, 1e-2)), N, grid.deltaT,
                              to_dev(rng.normal(size=(M, N, nx))))
    mean, var = two_pass_moments(res.states, M)
    print(nx, N, res.iters.cpu().numpy().tolist(), float(var.max()))
s = KLGpcSurrogate(rng.normal(size=(4, 9)), rng.uniform(0.1, 1, 7), rng.normal(size=(7, 4, 9)),
                   rng.normal(size=(7, 35)), 3, [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
print(DeviceSurrogate(s).predict(to_dev(rng.normal(size=(5, 4)))).shape)
s2 = KLGpcSurrogate(rng.normal(size=(4, 9)), rng.uniform(0.1, 1, 40), rng.normal(size=(40, 4, 9)),
                    rng.normal(size=(40, 15)), 2, [ParameterMap("identity", -np.inf, np.inf)] * 4, family="hermite")
print(DeviceSurrogate(s2).predict(to_dev(rng.normal(size=(70, 4)))).shape)
torch.cuda.synchronize()
print("sanitize run ok")
