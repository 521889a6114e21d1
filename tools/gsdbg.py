"""Developer probe of the line Gauss-Seidel solver (solver 4) on small scenes."""
import sys; sys.path.insert(0, '.')
import numpy as np, oracle as O
from mabd_scenes import generators as G
from paper_2603_08079_b200 import Simulator

def run(sc, n, sweeps=4000, tol=1e-13, q=None, qd=None):
    with Simulator.from_scene(sc, solver=4, gs_sweeps=sweeps, gs_tol=tol) as sim:
        sim.prefactor(sc.h)
        if q is not None: sim.set_state(q, qd)
        its = []
        for k in range(n):
            sim.step(sc.h, 1); its.append(sim.solver_stats()["last_iterations"])
        return sim.get_state()[0], its

sc = G.small_net(12, max_off=3)
Q = G.random_rotations(np.random.default_rng(1), 1)[0]
# (a) the whole net rotated: R = Q at step 1
A = np.swapaxes(sc.q0[:, :9].reshape(-1, 3, 3), 1, 2)
qr = G.pack_q(Q @ A, sc.q0[:, 9:] @ Q.T)
s2 = sc.copy(); s2.q0 = qr; s2.gravity = Q @ sc.gravity
wm = np.repeat(sc.body_b, sc.npts) < 0; s2.ybar_b = sc.ybar_b.copy(); s2.ybar_b[wm] = sc.ybar_b[wm] @ Q.T
q, its = run(s2, 1); print("(a) rotated net, 1 step", its, O.rel_err(q, O.simulate(s2, 1)[0]))
# (b) chains 3 steps
c = G.cfg2_batched_chains(3, 64)
q, its = run(c, 3); print("(b) chains, 3 steps", its, O.rel_err(q, O.simulate(c, 3)[0]))
# (c) net step 2 with many sweeps
q, its = run(sc, 2, sweeps=40000); print("(c) net 2 steps, 40000 sweeps", its, O.rel_err(q, O.simulate(sc, 2)[0]))
# (d) zero-velocity version of the step-1 state (isolates velocity vs rotation)
q1, qd1 = O.simulate(sc, 1)
q, its = run(sc, 1, q=q1, qd=0 * qd1); print("(d) step-1 state, zero velocity", its, O.rel_err(q, O.step(sc, q1, 0 * qd1, sc.h)[0]))
A1 = np.swapaxes(q1[:, :9].reshape(-1, 3, 3), 1, 2)
print("   max |A - I| after step 1:", np.abs(A1 - np.eye(3)).max())
import ctypes
with Simulator.from_scene(sc, solver=4, gs_sweeps=4000, gs_tol=1e-13) as sim:
    sim.prefactor(sc.h); sim.set_state(q1, 0 * qd1); sim.step(sc.h, 1)
    buf = (ctypes.c_double * 8001)()
    sim._lib.mabd_dbg_gs_trace.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    m = sim._lib.mabd_dbg_gs_trace(sim._h, buf, 8001)
    h = np.array(buf[:m])
    print("r0", h[0]); res = h[1::2]; sl = h[2::2]
    for s_ in [0, 1, 2, 5, 10, 50, 100, 430, 1000, 2000, 3999]:
        print(f"  sweep {s_}: res {res[s_]:.3e}  |S lam| {sl[s_]:.3e}")
