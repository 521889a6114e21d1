"""The split step across processes without NCCL: two processes on one GPU each run
their rank's share of a chain / tree split (options.host_exchange), and exchange the per-step all-gather over gloo on
the host between mabd_step_exchange_begin and _end — the rank-local code path of a multi-GPU run with a different
transport. No kernel waits on another process: the exchange is a host round trip between two launch sequences.
Each rank's bodies must be BITWISE equal to the same scene's W-part run emulated in one process (same arithmetic),
and match the oracle."""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

pytestmark = pytest.mark.gpu

SCENES = {
    "chain": lambda: G.cfg3_long_chain(col_len=2000, n_cols=35, tail=7),    # 70,007 bodies, 274 segments
    "tree": lambda: G.cfg4_binary_tree(12),                                 # 4,095 bodies, 16 bottom groups
}
NSTEPS = 3


def _worker(rank, world, port, case, outdir):
    import torch
    import torch.distributed as dist
    from paper_2603_08079_b200 import Simulator
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    sc = SCENES[case]()
    with Simulator.from_scene(sc, device=0, world=world, rank=rank, host_exchange=True) as sim:
        sim.prefactor(sc.h)
        info = sim.exchange_info()
        buf = np.zeros(info["ranks"] * info["doubles_per_rank"])
        for _ in range(NSTEPS):
            sim.exchange_begin(sc.h)
            buf[:] = 0.0
            sim.exchange_copy(buf, to_device=False)          # this rank's slot
            t = torch.from_numpy(buf)
            dist.all_reduce(t)                              # the other slots are zero: an all-gather
            sim.exchange_copy(buf, to_device=True)
            sim.exchange_end()
        q, qd = sim.get_state()
    np.save(os.path.join(outdir, f"q{rank}.npy"), q)
    np.save(os.path.join(outdir, f"qd{rank}.npy"), qd)
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", sorted(SCENES))
def test_split_step_across_processes(cuda_ok, case):
    import torch.multiprocessing as mp
    from paper_2603_08079_b200 import Simulator
    sc = SCENES[case]()
    world = 2
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_worker, args=(world, _free_port(), case, d), nprocs=world, start_method="spawn")
        qs = [np.load(os.path.join(d, f"q{r}.npy")) for r in range(world)]
        qds = [np.load(os.path.join(d, f"qd{r}.npy")) for r in range(world)]
    with Simulator.from_scene(sc, world=world) as em:       # the W parts emulated in one process
        em.prefactor(sc.h)
        em.step(sc.h, NSTEPS)
        q_e, qd_e = em.get_state()
    # each body is advanced by the rank that owns it (tree: the top levels by every rank); the other keeps q⁰
    moved = [np.any(q != sc.q0, axis=1) for q in qs]
    assert np.all(moved[0] | moved[1])
    both = moved[0] & moved[1]
    assert np.array_equal(qs[0][both], qs[1][both])
    q = np.where(moved[0][:, None], qs[0], qs[1])
    qd = np.where(moved[0][:, None], qds[0], qds[1])
    print(f"{case}: rank shares {moved[0].sum()} / {moved[1].sum()} bodies ({both.sum()} replicated)")
    assert np.array_equal(q, q_e) and np.array_equal(qd, qd_e)
    q_o, _ = O.simulate(sc, NSTEPS)
    assert O.rel_err(q, q_o) <= 1e-9
