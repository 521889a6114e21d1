"""Device time per step of the round-2 variants: polar-free vs exact (config 2, the first 30 steps of the episode,
before the variant diverges), line Gauss-Seidel on config 5 (fixed sweep budgets), loop breakers on rings."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from mabd_scenes import generators as G
from paper_2603_08079_b200 import Simulator, MabdError


def timed(sc, steps, **kw):
    st = torch.cuda.Stream()
    sim = Simulator.from_scene(sc, stream=st, **kw)
    sim.prefactor(sc.h)
    sim.step(sc.h, 2)
    sim.set_state(sc.q0, sc.qd0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    err = None
    try:
        sim.step_async(sc.h, steps)
        e1.record(st)
        sim.check()
    except MabdError as ex:
        err = str(ex)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    stats = sim.solver_stats()
    sim.close()
    return ms, stats, err


out = {}
sc2 = G.cfg2_batched_chains()
for rot in ("polar", "length_preserving"):
    ms, _, err = timed(sc2, 30, rotation=rot)
    out[f"cfg2_{rot}_30steps_us"] = ms * 1e3
    print(f"cfg2 {rot}: {ms*1e3:.1f} us/step over steps 1-30", err or "")
sc5 = G.make_scene(5)
for sw in (1, 10, 50):
    ms, stats, err = timed(sc5, 3, solver=4, gs_sweeps=sw, gs_tol=1e-300)
    out[f"cfg5_line_gs_{sw}_sweeps_ms"] = ms
    print(f"cfg5 line GS {sw} sweeps: {ms:.2f} ms/step ({stats})", err or "")
for n in (64, 4096):
    ring = G.ring(n, seed=1)
    ms_l, _, e1_ = timed(ring, 10, solver=5)
    ms_s, _, e2_ = timed(ring, 10, solver=3)
    out[f"ring{n}_loop_breaker_us"] = ms_l * 1e3
    out[f"ring{n}_sparse_us"] = ms_s * 1e3
    print(f"ring {n}: loop breaker {ms_l*1e3:.1f} us/step, sparse {ms_s*1e3:.1f} us/step", e1_ or "", e2_ or "")
print(json.dumps(out))
