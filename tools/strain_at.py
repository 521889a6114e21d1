"""Developer probe: strain statistics ‖AᵀA − I‖_F of cfg2 after k steps (GPU) and the time per step on the way."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from mabd_scenes import generators as G
from paper_2603_08079_b200 import Simulator
sc = G.cfg2_batched_chains()
st = torch.cuda.Stream()
sim = Simulator.from_scene(sc, stream=st)
sim.prefactor(sc.h)
done = 0
for k in (10, 40, 50, 50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st); sim.step(sc.h, k); e1.record(st); torch.cuda.synchronize()
    done += k
    q, qd = sim.get_state()
    A = q[:, :9].reshape(-1, 3, 3).transpose(0, 2, 1)
    e = np.sqrt(((np.einsum('nij,nik->njk', A, A) - np.eye(3)) ** 2).sum(axis=(1, 2)))
    v = np.abs(qd[:, 9:]).max()
    print(f"step {done}: {e0.elapsed_time(e1) / k * 1e3:.1f} us/step; ||E||: median {np.median(e):.2e} "
          f"p99 {np.quantile(e, 0.99):.2e} max {e.max():.2e}; frac>=0.1 {np.mean(e >= 0.1):.3f}; max |v| {v:.1f} m/s",
          flush=True)
