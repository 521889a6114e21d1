"""SURVEY A16 floor: disagreement between two independent CPU routes of the oracle (full-KKT SuperLU vs
block LU) along the configured trajectory of a reduced config-2 recipe, with the link strain alongside.
Writes the table printed here to stdout (profiles/r01_cfg2_parity_floor.txt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
from mabd_scenes import generators as G

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "cfg2":
    sc = G.cfg2_batched_chains(8, 256, nsteps=100)
elif which == "cfg3":
    sc = G.cfg3_long_chain(col_len=300, n_cols=4, tail=6)
elif which == "cfg4":
    sc = G.cfg4_binary_tree(8)
else:
    sc = G.small_net(24, max_off=6)
qa, qda = sc.q0.copy(), sc.qd0.copy()
qb, qdb = sc.q0.copy(), sc.qd0.copy()
print(f"{sc.name}: route superlu vs blocklu")
print("step  rel_err(superlu, blocklu)  max ||A^T A - I||_F")
for k in range(1, 101):
    qa, qda = O.step(sc, qa, qda, sc.h, route="superlu")
    qb, qdb = O.step(sc, qb, qdb, sc.h, route="blocklu")
    if k in (1, 5, 10, 20, 30, 40, 50, 60, 70, 80, 90, 100):
        A = qa[:, :9].reshape(-1, 3, 3).transpose(0, 2, 1)
        e = np.sqrt(((np.einsum('nij,nik->njk', A, A) - np.eye(3)) ** 2).sum(axis=(1, 2)))
        print(f"{k:4d}  {O.rel_err(qa, qb):.3e}  {e.max():.3e}", flush=True)
