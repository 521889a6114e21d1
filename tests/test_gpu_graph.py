"""CUDA-graph replay of mabd_step and the asynchronous step API (include/mabd.h: options.no_graphs, mabd_step_async,
mabd_check).

Each step's launch sequence is captured once into a graph and replayed; the arithmetic is the same kernels with
the same arguments, so the graph path must be BITWISE equal to plain launches on every solver."""
import numpy as np
import pytest

from mabd_scenes import generators as G

pytestmark = pytest.mark.gpu

CASES = {
    "chain_fused": (lambda: G.cfg2_batched_chains(6, 256), 1),
    "chain_long": (lambda: G.cfg3_long_chain(col_len=300, n_cols=4, tail=5), 1),
    "tree": (lambda: G.cfg4_binary_tree(10), 1),
    "sparse": (lambda: G.small_net(16, max_off=4), 1),
    "newton3": (lambda: G.cfg2_batched_chains(3, 100), 3),
}


def _run(sc, nsteps, no_graphs, iters):
    from paper_2603_08079_b200 import Simulator
    with Simulator.from_scene(sc, no_graphs=no_graphs, newton_iters=iters) as sim:
        sim.prefactor(sc.h)
        sim.step(sc.h, nsteps)
        sim.step(sc.h * 0.5, 2)          # h change: re-prefactor and a new graph
        sim.step(sc.h, 1)
        return sim.get_state()


@pytest.mark.parametrize("case", sorted(CASES))
def test_graph_replay_is_bitwise_plain_launches(cuda_ok, case):
    mk, iters = CASES[case]
    sc = mk()
    q1, qd1 = _run(sc, 4, False, iters)
    q2, qd2 = _run(sc, 4, True, iters)
    assert np.array_equal(q1, q2) and np.array_equal(qd1, qd2)


def test_step_async_then_check(cuda_ok):
    from paper_2603_08079_b200 import MabdError, Simulator
    sc = G.cfg1_chain8()
    with Simulator.from_scene(sc) as a, Simulator.from_scene(sc) as b:
        a.prefactor(sc.h)
        b.prefactor(sc.h)
        for _ in range(5):
            a.step_async(sc.h, 2)
        a.check()
        b.step(sc.h, 10)
        qa, qda = a.get_state()
        qb, qdb = b.get_state()
        assert np.array_equal(qa, qb) and np.array_equal(qda, qdb)
        # an error in the third enqueued step is attributed to it
        a.step_async(sc.h, 2)
        bad = qa.copy()
        bad[3, 0:9] = 0.0            # det A = 0 on body 3
        a.set_state(bad, qda)
        a.step_async(sc.h, 1)
        with pytest.raises(MabdError) as e:
            a.check()
        assert e.value.status == 7 and "at step 2 of the 3 steps" in str(e.value), str(e.value)
        # the error word is reset by the check
        a.set_state(qb, qdb)
        a.step(sc.h, 1)
