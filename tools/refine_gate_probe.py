"""Developer probe: how often the sparse solver's refinement gate (R2) lets a pass run, per step, on a
scene (default config 5), for the tolerance in MABD_SPARSE_REFINE_TOL."""
import os
import sys

import ctypes

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "5"
sc = {"5": lambda: G.cfg5_net(), "net": lambda: G.small_net(40, max_off=6)}[cfg]()
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
runs, ratios = [], []
with Simulator.from_scene(sc, solver=3) as sim:
    sim.prefactor(sc.h)
    for s in range(steps):
        sim.step(sc.h, 1)
        runs.append(sim.solver_stats()["last_iterations"])
        r = ctypes.c_double(0)
        sim._lib.mabd_dbg_refine_ratio.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        sim._lib.mabd_dbg_refine_ratio(sim._h, ctypes.byref(r))
        ratios.append(r.value)
    q, _ = sim.get_state()
print(f"cfg {cfg} tol {os.environ.get('MABD_SPARSE_REFINE_TOL', 'default')}: passes per step {runs} "
      f"(ran {sum(runs)}/{steps}); residual ratios {' '.join(f'{x:.1e}' for x in ratios)}; q finite {bool(np.isfinite(q).all())}")
