"""Developer check: cfg5 parity vs the block-LU oracle for 0/1/2 refinement passes (MABD_SPARSE_REFINE)."""
import os, subprocess, sys, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
side = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
if len(sys.argv) > 3:  # child: GPU run with the given refine count
    from mabd_scenes import generators as G
    from paper_2603_08079_b200 import Simulator
    sc = G.cfg5_net(side)
    sim = Simulator.from_scene(sc)
    sim.prefactor(sc.h)
    sim.step(sc.h, steps)
    q, _ = sim.get_state()
    np.save(f"/tmp/q_ref{sys.argv[3]}.npy", q)
    sys.exit(0)
for r in (0, 1, 2):
    subprocess.run([sys.executable, __file__, str(side), str(steps), str(r)], check=True,
                   env=dict(os.environ, MABD_SPARSE_REFINE=str(r)))
import oracle as O
from mabd_scenes import generators as G
sc = G.cfg5_net(side)
q, qd = sc.q0, sc.qd0
for _ in range(steps):
    q, qd = O.step(sc, q, qd, sc.h, route="blocklu")
for r in (0, 1, 2):
    print(f"side {side} steps {steps} refine {r}: rel err {O.rel_err(np.load(f'/tmp/q_ref{r}.npy'), q):.3e}", flush=True)
