"""GPU parity of the sparse path (loops / irregular nets: config-5 recipe, rings, random graphs) against the
CPU oracle through the C ABI. The dual is factored exactly every step (multifrontal Cholesky over a nested-dissection
assembly tree, reading R2) and refined once against the exact matrix-free S·x; the tolerances are those of
the north star (1e-9 after one step) and the live-floor rule of test_gpu_chain.check for multi-step runs."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import TOL1, _concat, check, gpu_run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("side", [4, 8, 20])
def test_cfg5_recipe_small(cuda_ok, side):
    sc = G.small_net(side, max_off=max(2, side // 4))
    check(sc, 1, expect_solver="sparse")
    check(sc, 5, expect_solver="sparse")
    q, _, _ = gpu_run(sc, 3)
    assert O.constraint_residual(sc, q) <= 1e-10


@pytest.mark.parametrize("seed", range(3))
def test_rings_and_mixed(cuda_ok, seed):
    parts = [G.ring(4, seed=seed), G.ring(7, seed=seed + 10), G.random_tree(30, seed=seed, hinge_frac=0.5, vel=0.2),
             G.random_chain(20, seed=seed + 5, vel=0.2)]
    sc = _concat(parts)
    check(sc, 1, expect_solver="sparse")
    check(sc, 4, expect_solver="sparse")


def test_sparse_solver_forced_on_chain_and_tree(cuda_ok):
    """solver=3 runs any topology: same answer as the oracle on a chain and on a hinge tree."""
    check(G.random_chain(50, seed=2, vel=0.3, jitter=1e-3, end_anchor=True), 2, solver=3, expect_solver="sparse")
    check(G.random_tree(60, seed=3, hinge_frac=0.7, vel=0.3), 2, solver=3, expect_solver="sparse")


def test_cfg5_side64(cuda_ok):
    sc = G.cfg5_net(64)
    check(sc, 1, route="blocklu", expect_solver="sparse")


@pytest.mark.slow
def test_cfg5_full_size_one_step(cuda_ok):
    """BASELINE config 5 at full size (262,144 bodies, 1,648,293 dual rows): one step vs the block-LU oracle."""
    sc = G.cfg5_net(512)
    q_g, _, info = gpu_run(sc, 1)
    assert info["solver"] == "sparse" and info["n_dual_rows"] == 1648293
    q_o, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="blocklu")
    assert O.rel_err(q_g, q_o) <= TOL1
