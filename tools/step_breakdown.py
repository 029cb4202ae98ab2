"""Phase timing of one c4 bench step (device events + host clock) — where the time between the kernels goes.
usage: python tools/step_breakdown.py [M]"""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import bench
from paper_2510_26180_b200 import _lib
from paper_2510_26180_b200.device import DeviceOperator
from paper_2510_26180_b200.engine import KleCgcSolver
from paper_2510_26180_b200.pcgc import pcgc_solve_device
from paper_2510_26180_b200.moments import two_pass_moments

M = int(sys.argv[1]) if len(sys.argv) > 1 else 1048576
c, model, grid, cfg, train, eval_rng = bench.problem("c4")
sur, _ = bench.build_and_share_surrogate(model, grid, cfg, train, c["degree"], 0, False)
solver = KleCgcSolver(model, grid, cfg, sur)
xi = torch.as_tensor(bench.eval_samples(eval_rng, M, c["d"]), device="cuda")
ws = torch.empty(int(_lib.query("kle_pcgc_workspace_bytes", M, grid.n_coarse, model.nx)), dtype=torch.uint8, device="cuda")


def step(rec):
    marks = []

    def mark(name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        marks.append((name, e, time.perf_counter()))

    mark("start")
    op = DeviceOperator.from_model(model, xi)
    mark("operator (kl_tridiag, u0 check)")
    U = solver.surrogate.predict(xi)
    mark("surrogate predict (basis + GEMM)")
    op.blob(grid.deltat)
    mark("fine_factor + tw_factor")
    res = pcgc_solve_device(op, U, grid, cfg, solver.tables, ws)
    mark("pcgc_solve (shift_factor + loop)")
    two_pass_moments(res.states, M, None)
    mark("moments")
    torch.cuda.synchronize()
    if rec:
        for (n0, e0, t0), (n1, e1, t1) in zip(marks, marks[1:]):
            print(f"{n1:36s} device {e0.elapsed_time(e1):8.2f} ms   host {1e3 * (t1 - t0):8.2f} ms")
        print(f"{'total':36s} device {marks[0][1].elapsed_time(marks[-1][1]):8.2f} ms")
        print("mean iterations", float(res.iters.double().mean()))


step(False)
step(True)
step(True)
