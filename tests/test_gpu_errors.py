"""Failure detection through the C ABI (include/mabd.h "Errors"; SURVEY §8(b) error conventions).

A redundant joint set (the same joint twice: a duplicated anchor or ball joint) makes ∇C̃ rank deficient, so the
dual S = ∇C̃ H̃⁻¹ ∇C̃ᵀ is singular: every solver must report MABD_ESINGULAR
rather than return a state."""
import numpy as np
import pytest

from mabd_scenes import generators as G

pytestmark = pytest.mark.gpu

ESINGULAR = 6


def _anchor(sc):
    return int(np.nonzero(sc.body_b < 0)[0][0])


CASES = {
    # one body with the same anchor twice: a 2-equation chain whose top system is singular
    "chain": lambda: G.duplicate_joint(G.random_chain(1, seed=2, anchored=True, vel=0.3), 0),
    # a body with the anchor twice and a ball joint (3 joints): the tree solver's first front is singular
    "tree": lambda: (lambda s: G.duplicate_joint(s, _anchor(s)))(G.random_chain(6, seed=3, anchored=True, vel=0.3)),
    # a net with one corner pin duplicated, and one with a grid joint duplicated
    "sparse": lambda: (lambda s: G.duplicate_joint(s, _anchor(s)))(G.small_net(8, max_off=2)),
    "sparse_ball": lambda: G.duplicate_joint(G.small_net(8, max_off=2), 5),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_redundant_joints_report_esingular(cuda_ok, case):
    from paper_2603_08079_b200 import MabdError, Simulator
    sc = CASES[case]()
    with Simulator.from_scene(sc) as sim:
        sim.prefactor(sc.h)
        assert sim.query()["solver"] == case.split("_")[0]
        with pytest.raises(MabdError) as e:
            sim.step(sc.h, 1)
        print(case, e.value)
        assert e.value.status == ESINGULAR
