"""Developer probe: the per-body stage kernels (K1 = a1+a2: sparse_predict_kernel, K4 = a5: sparse_update_kernel)
on config 3's 1,048,576 bodies (state 192 MiB > L2), through the sparse solver forced on the chains
(their fronts are tiny). Run under ncu with -k regex:"sparse_predict|sparse_update" for the kernel times."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200 import Simulator  # noqa: E402

sc = G.cfg3_long_chain()
sim = Simulator.from_scene(sc, solver=3)
print(sim.query())
sim.prefactor(sc.h)
sim.step(sc.h, 3)
torch.cuda.synchronize()
print("ok")
