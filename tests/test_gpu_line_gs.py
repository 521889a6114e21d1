"""GPU parity of the line Gauss-Seidel dual solver (the paper's Case IV; DESIGN.md
R10): an iterative solve of the exact dual S λ = C(q̃), so the step converges to the direct solution. Checked against
the oracle's direct KKT solve on nets (loops), trees and chains, with a tolerance tight enough that the iteration
must actually converge (1e-9 after one step)."""
import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import TOL1

pytestmark = pytest.mark.gpu

SCENES = {
    "net": lambda: G.small_net(12, max_off=3),
    "net_hinge_tree": lambda: G.random_tree(120, seed=4, hinge_frac=0.5, vel=0.3, jitter=1e-3),
    "chain": lambda: G.cfg2_batched_chains(3, 64),
}


def _run(sc, nsteps, sweeps=4000, tol=1e-13):
    from paper_2603_08079_b200 import Simulator
    with Simulator.from_scene(sc, solver=4, gs_sweeps=sweeps, gs_tol=tol) as sim:
        sim.prefactor(sc.h)
        assert sim.query()["solver"] == "line_gs"
        sim.step(sc.h, nsteps)
        q, qd = sim.get_state()
        return q, qd, sim.solver_stats()["last_iterations"]


@pytest.mark.parametrize("case", sorted(SCENES))
def test_line_gs_converges_to_the_direct_solution(cuda_ok, case):
    sc = SCENES[case]()
    q_o, _ = O.simulate(sc, 1)
    q_g, _, sweeps = _run(sc, 1)
    err = O.rel_err(q_g, q_o)
    print(f"line GS {case}: 1 step, {sweeps} sweeps, err {err:.2e}")
    assert err <= TOL1
    assert O.constraint_residual(sc, q_g) <= 1e-9


def test_line_gs_warm_start_and_sweep_budget(cuda_ok):
    """Warm-started from the previous step's λ, later steps need fewer sweeps; a tiny budget stops early (an
    approximate λ: the joints do not close to 1e-9)."""
    sc = G.small_net(12, max_off=3)
    q_o, _ = O.simulate(sc, 3)
    q_g, _, sweeps3 = _run(sc, 3)
    _, _, sweeps1 = _run(sc, 1)
    print(f"line GS warm start: sweeps step 1 {sweeps1}, step 3 {sweeps3}; 3-step err {O.rel_err(q_g, q_o):.2e}")
    assert O.rel_err(q_g, q_o) <= 1e-8
    q_b, _, sb = _run(sc, 1, sweeps=3)
    assert sb == 3 and O.constraint_residual(sc, q_b) > 1e-9
