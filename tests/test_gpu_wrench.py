"""GPU parity with constant external wrenches (f_A,ext = G(A)ᵀW) against the oracle,
on every solver path and with K = 1 and 2 Newton iterations; and removal of the wrenches."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import TOL1, TOLN

pytestmark = pytest.mark.gpu


def run(sc, nsteps, W, iters=1, clear_after=None):
    from paper_2603_08079_b200 import Simulator
    sim = Simulator.from_scene(sc, newton_iters=iters)
    sim.prefactor(sc.h)
    sim.set_wrench(W)
    if clear_after is None:
        sim.step(sc.h, nsteps)
    else:
        sim.step(sc.h, clear_after)
        sim.set_wrench(None)
        sim.step(sc.h, nsteps - clear_after)
    q, qd = sim.get_state()
    info = sim.query()
    sim.close()
    return q, qd, info


def _wrenches(n, seed, scale=1.0):
    rng = np.random.default_rng(seed)
    W = rng.normal(size=(n, 6))
    W[:, :3] *= 0.05 * scale   # torques [N m]
    W[:, 3:] *= 0.5 * scale    # forces [N]
    return W


@pytest.mark.parametrize("iters", [1, 2])
@pytest.mark.parametrize("case", ["chain", "multisegment", "tree", "sparse"])
def test_wrench_parity(cuda_ok, case, iters):
    sc = {"chain": lambda: G.cfg2_batched_chains(3, 256, nsteps=4),
          "multisegment": lambda: G.cfg3_long_chain(col_len=300, n_cols=2, tail=3),
          "tree": lambda: G.cfg4_binary_tree(7),
          "sparse": lambda: G.small_net(10, max_off=3)}[case]()
    # wrenches sized to the bodies (angular accelerations of O(100) rad/s², rotations ≲ 0.02 rad per step)
    W = _wrenches(sc.n, 3, scale={"chain": 0.02, "multisegment": 0.2, "tree": 0.2, "sparse": 0.002}[case])
    sc.wrench = W
    q_o, qd_o = O.simulate(sc, 3, iters=iters)
    q_g, qd_g, info = run(sc, 3, W, iters)
    assert O.rel_err(q_g, q_o) <= TOLN, (case, iters, O.rel_err(q_g, q_o))
    q1_o, _ = O.step(sc, sc.q0, sc.qd0, sc.h, iters=iters)
    q1_g, _, _ = run(sc, 1, W, iters)
    assert O.rel_err(q1_g, q1_o) <= TOL1


def test_wrench_removal(cuda_ok):
    """set_wrench(None) after two steps equals two wrench steps followed by wrench-free steps."""
    sc = G.cfg4_binary_tree(6)
    W = _wrenches(sc.n, 5, scale=0.2)
    q_g, _, _ = run(sc, 4, W, clear_after=2)
    sc.wrench = W
    q, qd = O.simulate(sc, 2)
    sc.wrench = None
    q, qd = O.simulate(sc, 2, q=q, qd=qd)
    assert O.rel_err(q_g, q) <= TOLN
