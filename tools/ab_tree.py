"""A/B timer for tree-solver variants (MABD_LIB): device time per step of config 4 (steps 1-20 from the initial state)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402

sc = G.make_scene(4)
st = torch.cuda.Stream()
sim = Simulator.from_scene(sc, stream=st)
sim.prefactor(sc.h)
sim.step(sc.h, 3)
best = None
for _ in range(3):
    sim.set_state(sc.q0, sc.qd0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    sim.step_async(sc.h, 20)
    e1.record(st)
    sim.check()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 20 * 1e3
    best = t if best is None else min(best, t)
print(f"{os.path.basename(os.environ.get('MABD_LIB', 'default')):24s} cfg4 {best:6.1f} us/step", flush=True)
