"""GPU parity of the five-row (nonlinear) hinge (Eq. hinge; R13) against the
oracle: per Newton iteration the second axis point keeps its two rows normal to the axis in the hinge frame
R_H = ΔR_H Rᵀ(A_a), re-evaluated at the linearisation point; the sparse solver carries them as a projected 3×3 block
with a decoupled dummy row."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import check, gpu_run

pytestmark = pytest.mark.gpu

SCENES = {
    "tree": lambda: G.five_row_hinges(G.random_tree(200, seed=7, hinge_frac=1.0, vel=0.3, jitter=1e-3)),
    "mixed_tree": lambda: G.five_row_hinges(G.random_tree(150, seed=8, hinge_frac=0.5, vel=0.3, jitter=1e-3)),
    "binary_tree": lambda: G.five_row_hinges(G.cfg4_binary_tree(7)),
    "world_hinge": lambda: G.five_row_hinges(G.hinge_pendulum(axis=(0.3, 1.0, 0.2), omega0=(3.0, 2.0, 1.0))),
}


@pytest.mark.parametrize("case", sorted(SCENES))
def test_hinge5_parity(cuda_ok, case):
    sc = SCENES[case]()
    assert np.any(sc.kind == 1)
    check(sc, 1, expect_solver="sparse")
    check(sc, 6, expect_solver="sparse")
    q, _, _ = gpu_run(sc, 6)
    assert O.constraint_residual(sc, q) < 1e-6     # the nonlinear rows: one linearised iteration per step


def test_hinge5_newton_iterations(cuda_ok):
    """With K = 3 Newton iterations each re-evaluates R_H; the nonlinear hinge rows close much tighter."""
    sc = SCENES["tree"]()
    check(sc, 2, expect_solver="sparse", iters=3)
    q1, _, _ = gpu_run(sc, 2, iters=1)
    q3, _, _ = gpu_run(sc, 2, iters=3)
    assert O.constraint_residual(sc, q3) < O.constraint_residual(sc, q1)
