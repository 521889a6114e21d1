"""Per-rank step time of config 2's strong split (4096 / W chains per rank, no collective in the
step), measured on ONE GPU: a rank of the W-way split advances an independent block of 4096 / W chains, so its
device time is what one process of the W-GPU job would spend (the ranks never wait on one another). Each timed step
is preceded by an L2 flush when the rank's state fits the 126 MB L2 (bench.py's rule). Prints one line per W with the
per-rank time and the job throughput it implies (1,048,576 bodies / per-rank time); not a multi-GPU measurement.

    python tools/cfg2_shard_probe.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402

L2_BYTES = 126e6
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100


def per_rank_us(world: int, flush: bool) -> float:
    sc = G.cfg2_batched_chains(4096 // world, 256)
    st = torch.cuda.Stream()
    sim = Simulator.from_scene(sc, stream=st)
    sim.prefactor(sc.h)
    sim.step(sc.h, 3)
    sim.set_state(sc.q0, sc.qd0)
    l2buf = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device="cuda") if flush else None
    evs = []
    torch.cuda.synchronize()
    for _ in range(steps):
        if flush:
            with torch.cuda.stream(st):
                l2buf.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        sim.step_async(sc.h, 1)
        e1.record(st)
        evs.append((e0, e1))
    sim.check()
    torch.cuda.synchronize()
    sim.close()
    return sum(a.elapsed_time(b) for a, b in evs) / steps * 1e3


for w in (1, 2, 4, 8):
    n_rank = 4096 // w * 256
    state_b = n_rank * 2 * 96
    for flush in ((False,) if state_b >= L2_BYTES else (True, False)):
        t = per_rank_us(w, flush)
        print(f"W={w} bodies/rank {n_rank:8d} state {state_b / 2**20:6.1f} MiB  "
              f"{'L2 flushed per step' if flush else 'no flush':20s} {t:7.1f} us/step per rank  "
              f"-> job {1048576 / t * 1e6:.3e} body-steps/s", flush=True)
