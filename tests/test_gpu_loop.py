"""GPU parity of the loop-breaker solver (the paper's Case III; R12): the
joints that close loops are removed, the remaining forest runs on the chain or tree solver once per unit breaker
impulse, and the breakers' multipliers solve the small Schur system. The result is the exact KKT step, checked
against the oracle's direct solve (one step 1e-9; several steps with the live-floor tolerance)."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import check, gpu_run

pytestmark = pytest.mark.gpu

SCENES = {
    "ring4": lambda: G.ring(4, seed=1),
    "ring60": lambda: G.ring(60, seed=2),
    "long_ring": lambda: G.add_ball_joint(G.random_chain(700, seed=6, anchored=False, vel=0.2), 0, 699),
    "chains_2_loops": lambda: G.add_ball_joint(G.add_ball_joint(G.cfg2_batched_chains(3, 64), 10, 50), 70, 120),
    "tree_loop": lambda: G.add_ball_joint(G.random_tree(80, seed=5, vel=0.3, jitter=1e-3, hinge_frac=0.3), 40, 79),
}


@pytest.mark.parametrize("case", sorted(SCENES))
def test_loop_breaker_matches_the_direct_step(cuda_ok, case):
    sc = SCENES[case]()
    check(sc, 1, solver=5, expect_solver="loop_breaker")
    check(sc, 4, solver=5, expect_solver="loop_breaker")
    q, _, info = gpu_run(sc, 3, solver=5)
    assert O.constraint_residual(sc, q) <= 1e-10


def test_loop_breaker_rejects_what_it_cannot_take(cuda_ok):
    from paper_2603_08079_b200 import MabdError, Simulator
    with pytest.raises(MabdError):
        Simulator.from_scene(G.small_net(8, max_off=2), solver=5)   # too many loops for a breaker set
    sc = G.ring(6, seed=3)
    with Simulator.from_scene(sc, solver=5) as sim:
        with pytest.raises(MabdError) as e:
            sim.set_wrench(np.zeros((sc.n, 6)))
        assert e.value.status == 8
