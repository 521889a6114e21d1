"""GPU parity of the line Gauss-Seidel dual solver (the paper's Case IV; DESIGN.md
R10): an iterative solve of the exact dual S λ = C(q̃).

- Iteration parity: after k sweeps from λ = 0 the GPU step equals the oracle's step whose dual solve is k sweeps of
  ``oracle.line_gauss_seidel`` over the same chain cover and colouring (the host plan, ``mabd_line_gs_plan``).
- Convergence: where the iteration converges, the step equals the oracle's direct KKT step (1e-9)."""
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


def _run(sc, nsteps, sweeps=4000, tol=1e-13, q=None, qd=None):
    from paper_2603_08079_b200 import Simulator
    with Simulator.from_scene(sc, solver=4, gs_sweeps=sweeps, gs_tol=tol) as sim:
        sim.prefactor(sc.h)
        assert sim.query()["solver"] == "line_gs"
        if q is not None:
            sim.set_state(q, qd)
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
    """Several steps where the iteration converges (a tree with hinges and ball joints), each warm-started from the
    previous step's λ: the steps equal the oracle's direct steps (measured: 3,351 / 3,711 / 4,072 sweeps to 1e-11,
    error 5e-13 — the warm start does not shorten the slow mode here). A tiny budget stops early: an approximate λ,
    the joints do not close to 1e-9. (On the stiff loop nets the rate collapses once the links carry strain —
    κ(S) ~ 1e8 — see DESIGN.md R10.)"""
    sc = G.random_tree(120, seed=4, hinge_frac=0.5, vel=0.3, jitter=1e-3)
    q_o, _ = O.simulate(sc, 3)
    from paper_2603_08079_b200 import Simulator
    with Simulator.from_scene(sc, solver=4, gs_sweeps=20000, gs_tol=1e-11) as sim:
        sim.prefactor(sc.h)
        sweeps = []
        for _ in range(3):
            sim.step(sc.h, 1)
            sweeps.append(sim.solver_stats()["last_iterations"])
        q_g, _ = sim.get_state()
    err = O.rel_err(q_g, q_o)
    print(f"line GS warm start: sweeps per step {sweeps}; 3-step err {err:.2e}")
    assert err <= 1e-8 and max(sweeps) < 20000
    q_b, _, sb = _run(sc, 1, sweeps=3)
    assert sb == 3 and O.constraint_residual(sc, q_b) > 1e-9


@pytest.mark.parametrize("case,sweeps", [("net", 1), ("net", 7), ("net", 60), ("hinge_tree", 5), ("hinge_tree", 40)])
def test_line_gs_iterates_match_the_oracle_iteration(cuda_ok, case, sweeps):
    from paper_2603_08079_b200 import binding
    from test_abi import _gs_plan
    sc = G.small_net(12, max_off=3) if case == "net" else G.random_tree(120, seed=4, hinge_frac=0.5, vel=0.3,
                                                                        jitter=1e-3)
    q, qd = O.simulate(sc, 1)          # a strained state (the stiff net's slow regime)
    pts, off, col = _gs_plan(binding.load_library(), sc)
    blocks = [np.concatenate([np.arange(3 * p, 3 * p + 3) for p in pts[off[c]:off[c + 1]]]) for c in range(len(off) - 1)]
    colors = [list(range(col[k], col[k + 1])) for k in range(len(col) - 1)]
    q_o, _ = O.step_with_dual(sc, q, qd, sc.h, lambda S, r: O.line_gauss_seidel(S, r, blocks, colors, sweeps))
    q_g, _, ran = _run(sc, 1, sweeps=sweeps, tol=1e-300, q=q, qd=qd)
    err = O.rel_err(q_g, q_o)
    print(f"line GS iterate {case}, {sweeps} sweeps: err {err:.2e}")
    assert ran == sweeps and err <= TOL1
