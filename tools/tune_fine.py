"""Time fgr_kernel variants (KLE_FINE_VARIANT) on config shapes."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2510_26180_b200 import LogNormalKL1D, make_time_grid, _lib
from paper_2510_26180_b200.device import DeviceOperator, AlphaTables, empty, ptr, stream_ptr
from paper_2510_26180_b200.pcgc import build_alpha_circulant

VARS = [(1, 16, 4, 0), (2, 16, 4, 0), (4, 16, 4, 0), (16, 8, 4, 3), (16, 32, 3, 2), (32, 32, 2, 0),
        (8, 16, 2, 1), (4, 32, 4, 0), (8, 16, 4, 1), (8, 16, 4, 0), (16, 16, 2, 0), (8, 32, 4, 0),
        (32, 16, 2, 0), (16, 32, 2, 0), (16, 32, 2, 1), (16, 32, 4, 1), (16, 32, 4, 0), (4, 32, 4, 1),
        (16, 32, 3, 's4'), (16, 32, 3, 's3'), (16, 32, 2, 's4'), (16, 32, 4, 's3'), (8, 16, 2, 's4'), (8, 16, 4, 's4'),
        (8, 32, 4, 's4'), (32, 16, 2, 's2'), (32, 16, 1, 's3'), (16, 32, 3, 's2'),
        (32, 16, 4, 's3'), (32, 16, 3, 's3'), (32, 16, 2, 's4'), (32, 16, 4, 's2'),
        (16, 32, 3, 0), (8, 16, 2, 2), (16, 32, 2, 2), (16, 8, 2, 0), (16, 8, 3, 0), (16, 8, 2, 2), (16, 8, 3, 2),
        (8, 8, 4, 0), (16, 8, 4, 3), (16, 8, 2, 3), (16, 32, 4, 3), (16, 32, 3, 3)]
for nx, N, J, M in ([(511, 64, 64, 4096), (127, 16, 32, 65536)] if len(sys.argv) < 2 else
                   [(127, 16, 32, 65536)] if sys.argv[1] == 'c4' else [(511, 64, 64, 8192)]):
    model = LogNormalKL1D(nx=nx, d=4)
    grid = make_time_grid(1.0, N, J)
    xi = np.random.default_rng(0).normal(size=(M, 4))
    tables = AlphaTables(build_alpha_circulant(N, 1e-3))
    U = torch.rand(M, N, nx, dtype=torch.float64, device="cuda")
    R = empty(M, N, nx)
    ref = None
    only = [int(v) for v in sys.argv[2].split(',')] if len(sys.argv) > 2 else None
    for v, (MR, P, Rr, pipe) in enumerate(VARS):
        if only is not None and v not in only:
            continue
        if MR * P < nx or MR * P >= 4 * nx:
            continue
        os.environ["KLE_FINE_VARIANT"] = str(v)
        op = DeviceOperator.from_model(model, xi)
        assert op.layout[0] == MR and op.layout[1] == P, (op.layout, MR, P)
        blob = op.blob(grid.deltat)
        def run():
            _lib.call("kle_fgr_f64", ptr(U), ptr(op.u0), None, None, ptr(R), ptr(blob), ptr(op.dia), ptr(op.off),
                      ptr(tables.scaling), None, M, N, nx, J, grid.deltat, grid.deltaT, 1.0, 1e-3, stream_ptr())
        run(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(3):
            run()
        b.record(); torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 3
        out = R.clone()
        if ref is None:
            ref = out
        err = float((out - ref).abs().max() / ref.abs().max())
        dof = M * N * J * nx / (ms * 1e-3)
        print(f"nx={nx} v={v} MR={MR} P={P} R={Rr} pipe={pipe}: {ms:8.3f} ms  {dof:.3e} DOF/s  {6*dof/1e12:.2f} TF/s(alg)  err={err:.1e}", flush=True)
