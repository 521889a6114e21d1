"""Developer probe: device time per step of a config over successive windows of steps (does the cost drift?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from mabd_scenes import generators as G
from paper_2603_08079_b200 import Simulator
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sc = G.cfg2_batched_chains() if cfg == 2 else G.make_scene(cfg)
st = torch.cuda.Stream()
sim = Simulator.from_scene(sc, stream=st)
sim.prefactor(sc.h)
done = 0
for w in (5, 25, 50, 50, 50, 50):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    sim.step(sc.h, w)
    e1.record(st)
    torch.cuda.synchronize()
    print(f"steps {done}-{done + w}: {e0.elapsed_time(e1) / w * 1e3:.1f} us/step", flush=True)
    done += w
if len(sys.argv) > 2:  # strain statistics of the final state
    import numpy as np
    q, _ = sim.get_state()
    A = q[:, :9].reshape(-1, 3, 3).transpose(0, 2, 1)
    E = np.einsum('nij,nik->njk', A, A) - np.eye(3)
    e = np.sqrt((E ** 2).sum(axis=(1, 2)))
    for th in (1e-4, 1e-3, 1e-2, 3e-2, 0.1, 0.3):
        print(f"  ||E||_F >= {th:g}: {np.mean(e >= th) * 100:.2f}% of bodies")
    print("  max ||E||_F", e.max(), "median", np.median(e))
