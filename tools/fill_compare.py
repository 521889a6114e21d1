"""Host-only comparison of the sparse solver's fill: the Cholesky flop count of the library's nested-dissection plan
(mabd_sparse_plan_stats) against SciPy's SuperLU with the MMD_AT_PLUS_A and COLAMD orderings on the same dual
pattern (S has a 3×3 block for every pair of joint points that share a body), for config-5 nets of side 64/128/256.
Flops are counted the same way for both: Σ_j c_j² over the columns of L (c_j = off-diagonal nonzeros), the dense
count n³/3 of the library's formula. Usage: python tools/fill_compare.py [sides...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

from mabd_scenes import generators as G  # noqa: E402
from paper_2603_08079_b200.binding import sparse_plan_stats  # noqa: E402


def dual_pattern(sc):
    ja, jb, npts = np.asarray(sc.body_a), np.asarray(sc.body_b), np.asarray(sc.npts)
    pj = np.repeat(np.arange(len(ja)), npts)          # joint of each point
    pa, pb = ja[pj], jb[pj]
    P = len(pj)
    rows, cols = [], []
    inc = {}
    for p in range(P):
        for b in (pa[p], pb[p]):
            if b >= 0:
                inc.setdefault(int(b), []).append(p)
    for pts in inc.values():
        for i in pts:
            for j in pts:
                rows.append(i)
                cols.append(j)
    A = sp.coo_matrix((np.ones(len(rows)), (rows, cols)), shape=(P, P)).tocsr()
    A.data[:] = 1.0
    B = sp.kron(A, np.ones((3, 3)), format="csc")
    # an SPD matrix with this pattern (diagonally dominant), so that no pivoting happens
    B = B + sp.identity(B.shape[0], format="csc") * (abs(B).sum(axis=1).max() + 1.0)
    return B.tocsc()


def lu_flops(B, spec):
    t = time.time()
    lu = spla.splu(B, permc_spec=spec, diag_pivot_thresh=0.0, options=dict(SymmetricMode=True))
    c = np.diff(lu.L.indptr) - 1
    return float((c.astype(np.float64) ** 2).sum()), int(lu.L.nnz), time.time() - t


sides = [int(a) for a in sys.argv[1:]] or [64, 128]
for s in sides:
    sc = G.cfg5_net(side=s)
    st = sparse_plan_stats(sc)
    B = dual_pattern(sc)
    print(f"net {s}x{s}: {B.shape[0]} dual rows; library ND plan: {st['flops']:.3e} flop, {st['fronts']:.0f} fronts, "
          f"largest front {st['max_front']:.0f} rows", flush=True)
    for spec in ("MMD_AT_PLUS_A", "COLAMD"):
        fl, nnz, dt = lu_flops(B, spec)
        print(f"  SciPy SuperLU {spec:14s}: {fl:.3e} flop (nnz(L) {nnz:.3e}, {dt:.1f} s); "
              f"ND plan / this = {st['flops'] / fl:.2f}", flush=True)
