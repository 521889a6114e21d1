"""A/B timer for library variants (MABD_LIB): device time per step of config 2 (a 100-step episode from the
initial state, as bench.py times it) and config 3 (20 steps), one process per library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402


def timed(sc, steps, reps=2):
    st = torch.cuda.Stream()
    sim = Simulator.from_scene(sc, stream=st)
    sim.prefactor(sc.h)
    sim.step(sc.h, 3)
    best = None
    for _ in range(reps):
        sim.set_state(sc.q0, sc.qd0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        sim.step_async(sc.h, steps)
        e1.record(st)
        sim.check()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / steps * 1e3
        best = t if best is None else min(best, t)
    sim.close()
    return best


lib = os.path.basename(os.environ.get("MABD_LIB", "default"))
t2 = timed(G.cfg2_batched_chains(), 100)
t3 = timed(G.make_scene(3), 20)
print(f"{lib:24s} cfg2 {t2:6.1f} us/step  cfg3 {t3:6.1f} us/step", flush=True)
