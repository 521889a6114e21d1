"""Developer probe: does iterating the Newton step keep config 2 physical? Strain ‖AᵀA − I‖_F statistics every 20
steps of the full config-2 workload for K = 1, 2, 3, 5 Newton iterations per step, and the device time per step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from mabd_scenes import generators as G
from paper_2603_08079_b200 import MabdError, Simulator
sc = G.cfg2_batched_chains()
for K in (1, 2, 3, 5):
    st = torch.cuda.Stream()
    sim = Simulator.from_scene(sc, stream=st, newton_iters=K)
    sim.prefactor(sc.h)
    tot = 0.0
    for s0 in range(0, 100, 20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(st)
        try:
            sim.step(sc.h, 20)
        except MabdError as ex:
            print(f"K={K}: steps {s0}-{s0 + 20}: {ex}", flush=True)
            break
        e1.record(st); torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
        q, qd = sim.get_state()
        A = q[:, :9].reshape(-1, 3, 3).transpose(0, 2, 1)
        e = np.sqrt(((np.einsum('nij,nik->njk', A, A) - np.eye(3)) ** 2).sum(axis=(1, 2)))
        print(f"K={K} step {s0 + 20}: {tot / (s0 + 20) * 1e3:.1f} us/step so far; ||E|| p99 {np.quantile(e, 0.99):.2e} "
              f"max {e.max():.2e}; frac >= 0.1 {np.mean(e >= 0.1):.4f}", flush=True)
    sim.close()
    del sim
