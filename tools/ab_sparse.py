"""A/B timer for sparse-solver library variants (MABD_LIB): device time per step of config 5 (steps from the
initial state, the first 3 untimed), one process per library."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
sc = G.make_scene(5)
st = torch.cuda.Stream()
sim = Simulator.from_scene(sc, stream=st)
sim.prefactor(sc.h)
sim.step(sc.h, 3)
best = None
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    sim.step_async(sc.h, steps)
    e1.record(st)
    sim.check()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / steps
    best = t if best is None else min(best, t)
q = sim.get_state()[0]
lib = os.path.basename(os.environ.get("MABD_LIB", "default"))
print(f"{lib:24s} cfg5 {best:7.2f} ms/step  launches/step {sim.query().get('launches_per_step')}  "
      f"q checksum {float(q.sum()):.12e}", flush=True)
sim.close()
