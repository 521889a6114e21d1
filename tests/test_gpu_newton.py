"""GPU parity of K > 1 Newton iterations per step against the oracle's iterated step, for
every solver path, plus the velocity output (q̇ⁿ⁺¹ = Σ δq⁽ⁱ⁾/h) and the convergence to the nonlinear step."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import TOL1, TOLN, _concat, check, gpu_run

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [2, 3])
def test_chain_fused_and_multisegment(cuda_ok, K):
    check(G.cfg1_chain8(), 1, route="dense", iters=K)
    check(G.cfg1_chain8(), 5, route="dense", iters=K)
    check(G.cfg2_batched_chains(4, 256, nsteps=3), 3, iters=K)
    check(G.cfg3_long_chain(col_len=300, n_cols=2, tail=3), 2, iters=K)


@pytest.mark.parametrize("K", [2, 4])
def test_tree_and_sparse(cuda_ok, K):
    check(G.cfg4_binary_tree(6), 3, expect_solver="tree", iters=K)
    check(G.random_tree(80, seed=4, hinge_frac=0.5, vel=0.5), 2, expect_solver="tree", iters=K)
    check(G.small_net(10, max_off=3), 2, expect_solver="sparse", iters=K)


def test_velocity_and_convergence(cuda_ok):
    """q̇ⁿ⁺¹ matches the oracle, and with many iterations the GPU step reaches the nonlinear implicit step."""
    sc = G.random_chain(6, seed=3, vel=3.0, jitter=1e-3)
    q_o, qd_o = O.step(sc, sc.q0, sc.qd0, sc.h, iters=3)
    q_g, qd_g, _ = gpu_run(sc, 1, iters=3)
    assert O.rel_err(q_g, q_o) <= TOL1
    assert np.max(np.abs(qd_g - qd_o)) <= 1e-7 * max(np.max(np.abs(qd_o)), 1.0)
    q16, _, _ = gpu_run(sc, 1, iters=16)
    r, c = O.nonlinear_residual(sc, sc.q0, sc.qd0, q16, sc.h)
    assert r <= 1e-8 and c <= 1e-12, (r, c)
