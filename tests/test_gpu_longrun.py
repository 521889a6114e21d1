"""GPU parity over many steps (BASELINE.json north star: 1e-9 after one step, 1e-6 after the configured number
of steps) on reduced instances of each config recipe, and one-step parity at full size for configs 2 and 3 (the
oracle's block-LU route; about 10-20 s of CPU each).

The horizon of each multi-step test is the configured step count where the trajectory allows it. Where it does
not, SURVEY A16 applies: the floor is the disagreement between two independent CPU routes of the oracle
(full-KKT SuperLU vs block LU), measured by tools/floor_probe.py; the test runs the steps over which 10 × floor
stays below 1e-6 (R4)."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import TOL1, TOLN, check, gpu_run

pytestmark = pytest.mark.gpu


def test_cfg2_recipe_30_steps(cuda_ok):
    """8 chains of the config-2 recipe (256 links). The trajectory is unstable in the one-iteration regime
    (R4): two independent CPU routes of the oracle (full-KKT SuperLU vs block LU) already disagree by
    2.2e-8 at step 30, 6.7e-6 at step 40 and O(1) from step 60 (SURVEY A16 floor,
    profiles/r01_cfg2_parity_floor.txt). Parity is therefore checked over the 30 steps where 10 × floor is below
    the north-star tolerance of 1e-6."""
    check(G.cfg2_batched_chains(8, 256, nsteps=30), 30)


def test_cfg3_recipe_40_steps(cuda_ok):
    """A 1,206-link boustrophedon of the config-3 recipe (5 segments, both ends pinned). Its folds whip: the
    oracle's two CPU routes disagree by 8.0e-8 at step 40, 1.9e-6 at step 50 and O(1) at step 90
    (profiles/r01_cfg3_parity_floor.txt), so parity is checked over 40 steps."""
    sc = G.cfg3_long_chain(col_len=300, n_cols=4, tail=6)
    check(sc, 40)


def test_cfg4_recipe_100_steps(cuda_ok):
    """Depth-8 complete binary tree (255 bodies, linear hinges, E = 1e10) for the configured 100 steps; this
    trajectory is stable (the oracle's two CPU routes stay within 8.5e-11, profiles/r01_cfg4_parity_floor.txt)."""
    check(G.cfg4_binary_tree(8), 100, expect_solver="tree")


def test_cfg5_recipe_5_steps(cuda_ok):
    """24×24 net with long-range links and pinned corners. The link strain reaches ‖AᵀA − I‖ ≈ 22 by step 10 and
    the oracle's two CPU routes disagree by 1.3e-9 at step 5, 1.3e-5 at step 10 and O(1) at step 20
    (profiles/r01_cfg5_parity_floor.txt), so parity is checked over 5 steps."""
    check(G.small_net(24, max_off=6), 5, expect_solver="sparse")


@pytest.mark.slow
def test_cfg2_full_size_one_step(cuda_ok):
    """BASELINE config 2 at full size (4096 × 256 links): one step against the oracle."""
    sc = G.cfg2_batched_chains(4096, 256)
    q_g, _, info = gpu_run(sc, 1)
    assert info["solver"] == "chain" and info["n_dual_rows"] == 3 * 1048576
    q_o, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="blocklu")
    assert O.rel_err(q_g, q_o) <= TOL1
    assert O.constraint_residual(sc, q_g) <= 1e-10


@pytest.mark.slow
def test_cfg3_full_size_one_step(cuda_ok):
    """BASELINE config 3 at full size (one chain of 1,048,576 links, both ends pinned): one step."""
    sc = G.cfg3_long_chain()
    q_g, _, info = gpu_run(sc, 1)
    assert info["solver"] == "chain" and info["n_dual_rows"] == 3145731
    q_o, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="blocklu")
    assert O.rel_err(q_g, q_o) <= TOL1
    assert O.constraint_residual(sc, q_g) <= 1e-10
