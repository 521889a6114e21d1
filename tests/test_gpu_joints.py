"""GPU parity of the universal and prismatic joints (Eqs. universal and prismatic;
DESIGN.md R17) against the oracle. Their rows are scalars in body a's joint frame with R ≈ A, linearised
at the iterate with the exact gradient; the sparse solver carries them as "general" 3×3 point blocks (≤ 2 rows,
the rest decoupled dummies) assembled row by row, J_r H⁻¹ J_cᵀ."""
import numpy as np
import pytest

import oracle as O
from oracle import rigid_reference as RR
from mabd_scenes import generators as G

from test_gpu_chain import check, gpu_run

pytestmark = pytest.mark.gpu

SCENES = {
    "universal_pendulum": lambda: G.universal_pendulum(omega0=(1.0, 0.5, 3.0)),
    "prismatic_rail": lambda: G.prismatic_rail(),
    "tree": lambda: G.nonlinear_joints(G.random_tree(200, seed=7, hinge_frac=1.0, vel=0.3, jitter=1e-3), seed=1),
    "mixed_tree": lambda: G.nonlinear_joints(G.random_tree(150, seed=8, hinge_frac=0.6, vel=0.3, jitter=1e-3),
                                             seed=2, universal=0.3, prismatic=0.3, hinge5=0.2),
    "net": lambda: G.nonlinear_joints(G.random_tree(120, seed=9, hinge_frac=0.7, vel=0.2, extra_anchors=6),
                                      seed=3),
}


@pytest.mark.parametrize("case", sorted(SCENES))
def test_joint_parity(cuda_ok, case):
    sc = SCENES[case]()
    assert np.any(sc.kind >= 2)
    check(sc, 1, expect_solver="sparse")
    check(sc, 6, expect_solver="sparse")


def test_joint_newton_iterations(cuda_ok):
    """K = 3 Newton iterations: parity, and the joint residual falls (measured on the oracle: > 100× per iteration)."""
    sc = SCENES["tree"]()
    check(sc, 2, expect_solver="sparse", iters=3)
    q1, _, _ = gpu_run(sc, 2, iters=1)
    q3, _, _ = gpu_run(sc, 2, iters=3)
    r1, r3 = O.constraint_residual(sc, q1), O.constraint_residual(sc, q3)
    print(f"joint residual after 2 steps: K=1 {r1:.2e}, K=3 {r3:.2e}")
    assert r3 < 1e-3 * r1


def test_gpu_prismatic_rail_closed_form(cuda_ok):
    """The rail slider on the GPU: s_n = −a h² n(n+1)/2 along the rail (implicit Euler of a = g sin 30°), on the
    rail, not turning."""
    sc = G.prismatic_rail(h=1e-2)
    a = 9.81 * np.sin(np.deg2rad(30.0))
    q, _, _ = gpu_run(sc, 50)
    s = q[0, 9:] @ sc.meta["rail"]
    assert abs(s + a * sc.h ** 2 * 50 * 51 / 2) < 1e-10
    assert np.linalg.norm(q[0, 9:] - s * sc.meta["rail"]) < 1e-12
    assert np.max(np.abs(q[0, :9] - sc.q0[0, :9])) < 1e-12


def test_gpu_universal_blocks_the_third_rotation(cuda_ok):
    sc = G.universal_pendulum(omega0=(1.0, 0.5, 3.0))
    q, qd, _ = gpu_run(sc, 1)
    w = RR.body_omega(q[0], qd[0])[0]
    assert abs(w[2]) < 1e-4 * 3.0


def test_general_joints_rejected_by_other_solvers(cuda_ok):
    from paper_2603_08079_b200 import MabdError, Simulator
    sc = SCENES["tree"]()
    for solver in (2, 4):
        with pytest.raises(MabdError):
            Simulator.from_scene(sc, solver=solver)
