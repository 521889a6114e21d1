"""GPU parity of five-row hinges with joint limits (R14): a limit violated at
the linearisation point becomes one extra row for that Newton iteration (a projected point of the sparse solver whose
rows switch on and off per step). Compared with the oracle over trajectories in which the limits engage."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import check, gpu_run

pytestmark = pytest.mark.gpu

SCENES = {
    "pendulum": lambda: G.hinge_limits(G.five_row_hinges(G.hinge_pendulum(axis=(1, 0, 0), omega0=(6.0, 0, 0))),
                                       -0.1, 0.1),
    "tree": lambda: G.hinge_limits(G.five_row_hinges(G.random_tree(60, seed=9, hinge_frac=1.0, vel=2.0,
                                                                   jitter=1e-3)), -0.05, 0.05),
}


@pytest.mark.parametrize("case", sorted(SCENES))
def test_limits_parity(cuda_ok, case):
    sc = SCENES[case]()
    # the limits engage within the checked horizon
    q, qd = sc.q0, sc.qd0
    engaged = 0
    for _ in range(40):
        engaged += len(O.hinge_limit_rows(sc, q))
        q, qd = O.step(sc, q, qd, sc.h)
    assert engaged > 0
    check(sc, 1, expect_solver="sparse")
    check(sc, 40, expect_solver="sparse")
