"""Probe: the c3 oracle solve over a process pool (CPU baseline of bench --config c3)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def solve(task):
    from oracle import ref_port
    (dia, ex, ey), U0, u0, n = task
    t = time.time()
    op = ref_port.SampleOperator.from_stencil2d(dia, ex, ey, n, np.full(len(dia), 1.0))
    out = ref_port.pcgc(op, u0, U0, 32, 16, 1.0, 1e-3, 1e-8, 60)
    return out["iters"], time.time() - t, os.getpid()


if __name__ == "__main__":
    from concurrent.futures import ProcessPoolExecutor
    import multiprocessing as mp
    from oracle import ref_port
    from paper_2510_26180_b200.models import LogNormalKL2D
    nproc = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    m = LogNormalKL2D(n=127, d=10)
    xs = np.random.default_rng(0).normal(size=(nproc, 10))
    tasks = []
    for x in xs:
        st = m.stencil(x)
        op = ref_port.SampleOperator.from_stencil2d(*st, 127, np.ones(127 * 127))
        tasks.append((st, ref_port.coarse_sweep(op, m.initial_condition(), 32, 1 / 32), m.initial_condition(), 127))
    t0 = time.time()
    with ProcessPoolExecutor(nproc, mp_context=mp.get_context(sys.argv[2] if len(sys.argv) > 2 else "spawn")) as ex:
        for r in ex.map(solve, tasks):
            print(r, f"{time.time() - t0:.1f}", flush=True)
    print("wall", time.time() - t0)
