"""Developer timing probe: device time per mabd_step of a config with the library given by MABD_LIB.
Errors raised by the step (e.g. from experimental builds that skip stages) are ignored: only timing is read."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import MabdError, Simulator  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
sc = G.cfg2_batched_chains() if cfg == 2 else G.make_scene(cfg)
st = torch.cuda.Stream()
sim = Simulator.from_scene(sc, stream=st)
sim.prefactor(sc.h)
try:
    sim.step(sc.h, 3)
except MabdError:
    pass
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(st)
err = None
try:
    sim.step(sc.h, steps)
except MabdError as ex:
    err = str(ex)
e1.record(st)
torch.cuda.synchronize()
if err:
    print("step error:", err)
print("solver stats:", sim.solver_stats())
print(f"{os.environ.get('MABD_LIB', 'default')}: cfg{cfg} {e0.elapsed_time(e1) / steps * 1e3:.1f} us/step "
      f"({sim.query()['launches_per_step']} launches/step)")

lib = sim._lib
if hasattr(lib, "mabd_dbg_phases"):
    import ctypes
    buf = (ctypes.c_ulonglong * 16)()
    lib.mabd_dbg_reset()
    try:
        sim.step(sc.h, steps)
    except MabdError:
        pass
    torch.cuda.synchronize()
    lib.mabd_dbg_phases(buf)
    names = ["P1b predict", "barrier", "assemble+inv", "CR (2..11)", "top+barrier", "CR back lower", "P3 update",
             "loop/end barrier", "CR fwd lower", "CR fwd upper (w0)", "top (w0)", "CR bwd upper (w0)",
             "TMA wait", "P1a staged->TMEM"]
    nseg = steps * (sc.n // 256)
    tot = sum(buf[i] for i in range(14))
    for i, nm in enumerate(names):
        print(f"  {nm:18s} {buf[i] / nseg:10.0f} cycles/segment  {100 * buf[i] / tot:5.1f}%")
