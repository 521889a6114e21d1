"""Small runs of every solver path for compute-sanitizer (memcheck): chain (fused + multi-segment + emulated
parts), tree (+ emulated split), sparse, K = 2 iterations and wrenches."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from mabd_scenes import generators as G
from paper_2603_08079_b200 import Simulator

cases = [(G.cfg1_chain8(), {}), (G.cfg2_batched_chains(3, 256), {}),
         (G.cfg3_long_chain(col_len=300, n_cols=3, tail=4), {}),
         (G.cfg3_long_chain(col_len=300, n_cols=3, tail=4), {"world": 2}),
         (G.cfg4_binary_tree(10), {}), (G.cfg4_binary_tree(10), {"world": 2}),
         (G.small_net(12, max_off=3), {}), (G.random_tree(200, seed=1, hinge_frac=0.5), {"newton_iters": 2})]
for sc, kw in cases:
    sim = Simulator.from_scene(sc, **kw)
    sim.prefactor(sc.h)
    sim.set_wrench(np.full((sc.n, 6), 1e-3))
    sim.step(sc.h, 2)
    q, qd = sim.get_state()
    assert np.isfinite(q).all()
    sim.close()
    print("ok", sc.name, kw, flush=True)
