"""Multi-part (multi-GPU) chain path, emulated on one GPU: world = W with no NCCL id runs the W parts in one
process with the same arithmetic (per-part reduction to a top system, rank-level solve, back substitution),
the all-gather being a no-op. Parity against the oracle and against the single-part path."""
import ctypes

import numpy as np
import pytest

import oracle as O
from mabd_scenes import generators as G

from test_gpu_chain import TOL1, _concat

pytestmark = pytest.mark.gpu


def run(sc, nsteps, world=1):
    import torch
    from paper_2603_08079_b200 import binding as B
    sim = B.Simulator.from_scene(sc, world=world)
    sim.prefactor(sc.h)
    sim.step(sc.h, nsteps)
    q, qd = sim.get_state()
    info = sim.query()
    sim.close()
    return q, info


@pytest.mark.parametrize("world", [2, 3, 8])
def test_long_chain_parts_vs_oracle(cuda_ok, world):
    sc = G.cfg3_long_chain(col_len=2000, n_cols=35, tail=7)   # 70,007 bodies, 274 segments
    q1, info = run(sc, 2, world)
    q_o, _ = O.simulate(sc, 2)
    assert O.rel_err(q1, q_o) <= 1e-9
    q_single, _ = run(sc, 2, 1)
    assert O.rel_err(q1, q_single) <= 1e-11
    assert info["launches_per_step"] > 3


@pytest.mark.parametrize("world", [2, 5])
def test_mixed_chains_parts(cuda_ok, world):
    parts = [G.random_chain(700, seed=1, vel=0.2, end_anchor=True), G.cfg2_batched_chains(9, 100),
             G.random_chain(1300, seed=2, vel=0.2), G.random_chain(40, seed=3)]
    sc = _concat(parts)
    q1, _ = run(sc, 3, world)
    q_o, _ = O.simulate(sc, 3)
    assert O.rel_err(q1, q_o) <= 1e-9


@pytest.mark.slow
@pytest.mark.parametrize("world", [2, 8])
def test_cfg3_full_size_parts(cuda_ok, world):
    """The 1,048,576-body chain split into W parts (part sizes are multiples of 256 segments)."""
    sc = G.cfg3_long_chain()
    q_w, _ = run(sc, 1, world)
    q_1, _ = run(sc, 1, 1)
    assert O.rel_err(q_w, q_1) <= 1e-11
    assert O.constraint_residual(sc, q_w) <= 1e-10


@pytest.mark.slow
def test_cfg3_full_size_one_step_vs_oracle(cuda_ok):
    sc = G.cfg3_long_chain()
    q_g, _ = run(sc, 1, 1)
    q_o, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="blocklu")
    assert O.rel_err(q_g, q_o) <= TOL1


# ----------------------------------------------------------------------------- trees

@pytest.mark.parametrize("world", [2, 4, 8])
def test_tree_parts_vs_oracle(cuda_ok, world):
    """Config-4 recipe at depth 11 (2,047 bodies: 8 CTA-local subtrees and a 7-body top), split into W parts:
    each part eliminates its subtrees, the condensed root blocks go through the gather buffer, the top is solved
    by every part. Bitwise the same as the unsplit path (the exchange only copies), and parity with the oracle."""
    sc = G.cfg4_binary_tree(11)
    q1, info = run(sc, 3, world)
    assert info["solver"] == "tree"
    q_single, _ = run(sc, 3, 1)
    assert np.array_equal(q1, q_single)
    q_o, _ = O.simulate(sc, 3)
    assert O.rel_err(q1, q_o) <= 1e-6


@pytest.mark.parametrize("world", [2, 4])
def test_tree_parts_with_middle_layer(cuda_ok, world):
    """Depth 14 (16,383 bodies): 64 bottom subtrees split over W parts; the replicated top section has a middle
    layer (eight 7-body groups below a 7-body top) that reads the gathered root blocks. Bitwise the same as the
    unsplit path, parity with the oracle."""
    sc = G.cfg4_binary_tree(14)
    q1, info = run(sc, 3, world)
    assert info["solver"] == "tree"
    q_single, _ = run(sc, 3, 1)
    assert np.array_equal(q1, q_single)
    q_o, _ = O.simulate(sc, 3)
    assert O.rel_err(q1, q_o) <= 1e-6


@pytest.mark.parametrize("world", [2, 3])
def test_tree_parts_with_large_top(cuda_ok, world):
    """A 1,200-link hinge path rooted at its centre: two bottom subtrees split over W parts, the top group too
    large for one CTA (one launch per level) reads the gathered root blocks. Bitwise the same as the unsplit
    path, parity with the oracle."""
    sc = G.random_chain(1200, seed=5, npts=2, end_anchor=True, vel=0.2)
    q1, info = run(sc, 2, world)
    assert info["solver"] == "tree"
    q_single, _ = run(sc, 2, 1)
    assert np.array_equal(q1, q_single)
    q_o, _ = O.simulate(sc, 2)
    assert O.rel_err(q1, q_o) <= 1e-6


@pytest.mark.parametrize("world", [2, 3])
def test_random_forest_parts(cuda_ok, world):
    """Random trees packed several per CTA-local group (a group has several joints into the top)."""
    rng = np.random.default_rng(5)
    parts = [G.random_tree(int(rng.integers(300, 700)), seed=40 + k, hinge_frac=0.5, vel=0.3, jitter=1e-3,
                           max_children=3) for k in range(3)]
    sc = _concat(parts)
    q1, info = run(sc, 2, world)
    assert info["solver"] == "tree"
    q_single, _ = run(sc, 2, 1)
    assert np.array_equal(q1, q_single)
    q_o, _ = O.simulate(sc, 2)
    assert O.rel_err(q1, q_o) <= 1e-6
