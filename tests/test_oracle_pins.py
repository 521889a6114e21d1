"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these re-type the oracle's formulas: each compares against an independent definition
(quadrature of JᵀMJ, finite differences of an energy, closed-form trajectories, invariants,
brute-force KKT) chosen so that a dropped term, a sign or an index error fails one of them.
"""
import os

import numpy as np
import pytest
import scipy.linalg

import oracle as O
from mabd_scenes import generators as G

HERE = os.path.dirname(os.path.abspath(__file__))


# ----------------------------------------------------------------------------- per-body algebra

def test_polar_examples():
    """P8 / SPEC S:59-62: R(I)=I, R(2I)=I, R(R₀ diag(1.01,1,0.99)) = R₀, RᵀR = I, det R = 1."""
    assert np.allclose(O.polar(np.eye(3)), np.eye(3), atol=1e-15)
    assert np.allclose(O.polar(2 * np.eye(3)), np.eye(3), atol=1e-15)
    R0 = G.random_rotations(np.random.default_rng(1), 20)
    A = R0 @ np.diag([1.01, 1.0, 0.99])
    R = O.polar(A)
    assert np.max(np.abs(R - R0)) < 1e-12
    assert np.max(np.abs(np.swapaxes(R, 1, 2) @ R - np.eye(3))) < 1e-13
    assert np.allclose(np.linalg.det(R), 1.0, atol=1e-13)
    # symmetric stretch: RᵀA is symmetric positive definite (definition of the polar factor)
    S = np.swapaxes(R, 1, 2) @ A
    assert np.max(np.abs(S - np.swapaxes(S, 1, 2))) < 1e-13
    with pytest.raises(FloatingPointError):
        O.polar(np.diag([1.0, 1.0, -1.0]))


def _gauss_box_points(a, b, c, rho):
    """2×2×2 Gauss-Legendre points/weights of a box: exact for the quadratic moments of M̄."""
    g = np.array([-1.0, 1.0]) / np.sqrt(3.0)
    pts = np.array([[a / 2 * x, b / 2 * y, c / 2 * z] for x in g for y in g for z in g])
    w = np.full(8, rho * a * b * c / 8.0)
    return pts, w


def test_mass_matrix_is_JtMJ():
    """M_A = Σ m_i J_iᵀJ_i with J_i = [x̄_iᵀ⊗I₃, I₃], by exact quadrature of a box."""
    a, b, c, rho = 0.3, 0.1, 0.2, 700.0
    pts, w = _gauss_box_points(a, b, c, rho)
    M = np.zeros((12, 12))
    for x, m in zip(pts, w):
        Ji = np.hstack([np.kron(x[None, :], np.eye(3)), np.eye(3)])
        M += m * Ji.T @ Ji
    assert np.allclose(O.mass_A(G.box_mbar(a, b, c, rho)), M, rtol=0, atol=1e-13 * np.abs(M).max())
    # 0.1 m cube at ρ = 1000 has translational mass block 1 kg · I₃
    assert np.allclose(O.mass_A(G.box_mbar(0.1, 0.1, 0.1, 1000.0))[9:, 9:], np.eye(3), atol=1e-15)


def _psi_lin(A, mu, lam):
    """Linear elasticity Ψ = μ‖ε‖² + (λ/2) tr(ε)², ε = ½(A+Aᵀ) − I; its A-gradient is P:269."""
    e = 0.5 * (A + A.T) - np.eye(3)
    return mu * np.sum(e * e) + 0.5 * lam * np.trace(e) ** 2


def test_kbar_is_fd_hessian_and_nullspace():
    """K̄_A = Hessian of VΨ by central differences; null space dim 6."""
    V, mu, lam = 0.002, 3.0e6, 5.0e6
    K = O.kbar_A(V, mu, lam)
    A0 = np.eye(3) + 0.01 * np.random.default_rng(2).standard_normal((3, 3))
    eps = 1e-4
    Kfd = np.zeros((9, 9))
    for i in range(9):
        for j in range(9):
            def E(di, dj):
                v = O.vec(A0).copy()
                v[i] += di
                v[j] += dj
                return V * _psi_lin(O.unvec(v), mu, lam)
            Kfd[i, j] = (E(eps, eps) - E(eps, -eps) - E(-eps, eps) + E(-eps, -eps)) / (4 * eps * eps)
    assert np.allclose(K[:9, :9], Kfd, rtol=1e-6, atol=1e-6 * np.abs(Kfd).max())
    assert np.all(K[9:, :] == 0) and np.all(K[:, 9:] == 0)
    w = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(w) < 1e-9 * w.max()) == 6
    # the rigid infinitesimal rotations vec(W), W skew, are in the null space
    W = np.array([[0, -1, 2], [1, 0, -3], [-2, 3, 0]], float)
    assert np.max(np.abs(K[:9, :9] @ O.vec(W))) < 1e-9 * np.abs(K).max()


def _corot_energy(A, V, mu, lam):
    """E(A) = V[μ‖S−I‖² + (λ/2)tr(S−I)²], S = (AᵀA)^{1/2} by scipy.linalg.sqrtm.

    Independent of the oracle's SVD route to R.
    """
    S = np.real(scipy.linalg.sqrtm(A.T @ A))
    E = S - np.eye(3)
    return V * (mu * np.sum(E * E) + 0.5 * lam * np.trace(E) ** 2)


def test_elastic_force_is_fd_gradient():
    """P9: V vec(RΠ(RᵀA)) = ∂E/∂vec(A) for the co-rotated energy (A10); zero at rotations."""
    rng = np.random.default_rng(3)
    V, mu, lam = 1e-3, *O.lame(1e8, 0.3)
    for _ in range(5):
        R0 = G.random_rotations(rng, 1)[0]
        A = R0 @ (np.eye(3) + 0.02 * rng.standard_normal((3, 3)))
        f = O.elastic_force_A(A, V, mu, lam)
        eps = 1e-7
        g = np.zeros(9)
        for i in range(9):
            vp = O.vec(A).copy()
            vm = vp.copy()
            vp[i] += eps
            vm[i] -= eps
            g[i] = (_corot_energy(O.unvec(vp), V, mu, lam) - _corot_energy(O.unvec(vm), V, mu, lam)) / (2 * eps)
        assert np.max(np.abs(f - g)) <= 1e-7 * np.max(np.abs(g))
        assert np.max(np.abs(O.elastic_force_A(R0, V, mu, lam))) < 1e-12 * V * mu


@pytest.mark.parametrize("E,nu", [(1e8, 0.3), (1e10, 0.3), (2.5e6, 0.45), (7e7, 0.0), (3e9, -0.2)])
def test_lame_uniaxial_stress_and_pure_shear(E, nu):
    """Pins ``lame`` against the definitions of E, ν and the shear modulus (P:267-269 names μ, λ).

    Uniaxial stress: A = diag(1+ε, 1−νε, 1−νε) (R = I, F = A) must carry the stress σ = diag(Eε, 0, 0) — Young's
    modulus is σ_xx/ε_xx under a lateral contraction of ν·ε with free (zero-traction) lateral faces. Pure shear:
    a symmetric A = I + (γ/2)(e_x e_yᵀ + e_y e_xᵀ) must carry σ_xy = E/(2(1+ν))·γ and nothing else. The force is
    V vec(σ) (R = I). Swapping μ and λ, or a wrong (1−2ν) or (1+ν) factor, fails one of the two.
    """
    mu, lam = O.lame(E, nu)
    V, eps = 0.37, 1e-3
    A = np.diag([1 + eps, 1 - nu * eps, 1 - nu * eps])
    f = O.elastic_force_A(A, V, mu, lam)
    expect = V * O.vec(np.diag([E * eps, 0.0, 0.0]))
    assert np.max(np.abs(f - expect)) <= 1e-12 * V * E * eps
    gam = 2e-3
    A = np.eye(3)
    A[0, 1] = A[1, 0] = 0.5 * gam
    f = O.elastic_force_A(A, V, mu, lam)
    sig = np.zeros((3, 3))
    sig[0, 1] = sig[1, 0] = E / (2 * (1 + nu)) * gam
    assert np.max(np.abs(f - V * O.vec(sig))) <= 1e-12 * V * E * gam


def test_affine_force_is_minus_gradient_of_incremental_potential():
    """f_A = −∇_q [ (1/2h²)(q−q̂)ᵀM_A(q−q̂) + E_el(q) ] at q = qⁿ, q̂ = qⁿ + hq̇ⁿ + h²[0;g]."""
    rng = np.random.default_rng(4)
    sc = G.random_chain(1, seed=4, anchored=False, vel=0.5)
    q = sc.q0[0].copy()
    A = O.unvec(q[:9])
    q[:9] = O.vec(A @ (np.eye(3) + 0.01 * rng.standard_normal((3, 3))))
    qd = sc.qd0[0]
    h = 1e-2
    M = O.mass_A(sc.mbar[0])
    mu, lam = O.lame(sc.youngs[0], sc.poisson[0])
    # q̂ from the projected implicit-Euler predictor with M_A⁻¹(JᵀM g-field) = [0;g] computed by solving
    fext = np.zeros(12)
    pts, w = _gauss_box_points(*_box_dims(sc.mbar[0]), 1.0)
    for x, m in zip(pts, w / w.sum() * sc.mbar[0][9]):
        Ji = np.hstack([np.kron(x[None, :], np.eye(3)), np.eye(3)])
        fext += m * Ji.T @ sc.gravity
    qhat = q + h * qd + h * h * np.linalg.solve(M, fext)

    def Etot(x):
        d = x - qhat
        return 0.5 / h ** 2 * d @ M @ d + _corot_energy(O.unvec(x[:9]), sc.volume[0], mu, lam)

    eps = 1e-7
    grad = np.array([(Etot(q + eps * e) - Etot(q - eps * e)) / (2 * eps) for e in np.eye(12)])
    f = O.affine_force(q, qd, sc.mbar[0], sc.volume[0], sc.youngs[0], sc.poisson[0], sc.gravity, h)
    assert np.max(np.abs(f + grad)) <= 1e-6 * np.max(np.abs(f))


def _box_dims(mbar):
    m = mbar[9]
    return tuple(np.sqrt(12.0 * mbar[k] / m) for k in (0, 4, 7))


def test_corotation_identities():
    """P:238-241 diag_N(R)J = J diag₄(R) (point rows: Γ(y)diag₄(R) = RΓ(y)); P:250-254 M_A commutes with diag₄(R)."""
    rng = np.random.default_rng(5)
    R = G.random_rotations(rng, 1)[0]
    D4 = np.kron(np.eye(4), R)
    y = rng.standard_normal(3)
    Gy = np.kron(np.append(y, 1.0)[None, :], np.eye(3))
    assert np.allclose(Gy @ D4, R @ Gy, atol=1e-14)
    M = O.mass_A(G.box_mbar(0.2, 0.1, 0.05, 900.0))
    assert np.allclose(D4 @ M @ D4.T, M, atol=1e-14 * np.abs(M).max())


# ----------------------------------------------------------------------------- trajectory pins

def test_P1_discrete_free_fall():
    """P1: tⁿ = t⁰ + nhv⁰ + ½n(n+1)h²g, vⁿ = v⁰ + nhg; A unchanged for A⁰ ∈ SO(3), Ȧ⁰ = 0."""
    R0 = G.random_rotations(np.random.default_rng(6), 1)[0]
    v0 = np.array([1.0, -2.0, 3.0])
    t0 = np.array([0.3, 0.2, 0.1])
    sc = G.free_body(A0=R0, t0=t0, v0=v0, dims=(0.1, 0.3, 0.2), E=1e8)
    n = 25
    q, qd = O.simulate(sc, n)
    g = sc.gravity
    h = sc.h
    t_ref = t0 + n * h * v0 + 0.5 * n * (n + 1) * h * h * g
    assert np.max(np.abs(q[0, 9:] - t_ref)) <= 1e-14 * np.max(np.abs(t_ref)) * 10
    assert np.max(np.abs(qd[0, 9:] - (v0 + n * h * g))) <= 1e-13 * np.max(np.abs(v0 + n * h * g))
    assert np.max(np.abs(q[0, :9] - O.vec(R0))) < 1e-14


@pytest.mark.parametrize("maker", [
    lambda: G.random_chain(9, seed=7, anchored=False, vel=0.3, gravity=False, npts=1, reverse_some=True),
    lambda: G.random_tree(12, seed=8, anchored=False, vel=0.3, gravity=False, hinge_frac=0.5),
])
def test_P2_linear_momentum(maker):
    """P2: without gravity and anchors, Σ m ṫ is conserved exactly."""
    sc = maker()
    m = sc.mbar[:, 9]
    p0 = (m[:, None] * sc.qd0[:, 9:]).sum(0)
    q, qd = sc.q0, sc.qd0
    for _ in range(5):
        q, qd = O.step(sc, q, qd, sc.h)
        p = (m[:, None] * qd[:, 9:]).sum(0)
        assert np.max(np.abs(p - p0)) <= 1e-13 * max(np.max(np.abs(p0)), np.max(m * np.abs(qd[:, 9:]).max(1)))


@pytest.mark.parametrize("maker", [
    lambda: G.cfg1_chain8(),
    lambda: G.random_chain(10, seed=9, jitter=2e-3, vel=0.2, end_anchor=True),
    lambda: G.random_tree(14, seed=10, jitter=1e-3, vel=0.2, hinge_frac=0.6),
    lambda: G.small_net(6, max_off=3),
])
def test_P3_constraint_closure(maker):
    """P3: max‖C(qⁿ⁺¹)‖∞ ≤ 1e-10 m after every step from any start (footnote P:459; A4; BASELINE north star)."""
    sc = maker()
    q, qd = sc.q0, sc.qd0
    for _ in range(4):
        q, qd = O.step(sc, q, qd, sc.h)
        assert O.constraint_residual(sc, q) <= 1e-10


def _read_golden(name):
    vals = {}
    with open(os.path.join(HERE, "golden", name)) as fh:
        for line in fh:
            if line.strip() and not line.startswith("#"):
                k, v = line.split()
                vals[k] = float(v)
    return vals


@pytest.mark.parametrize("h", [1e-2, 1e-3])
def test_P4_small_angle_pendulum_period(h):
    """P4: zero-crossing period of the 2° compound pendulum within 2e-4 s of T₀(1+θ₀²/16) (golden file)."""
    gold = _read_golden("pendulum_period.txt")
    sc = G.pendulum(2.0, h=h)
    q, qd = sc.q0, sc.qd0
    ys = [q[0, 10]]
    nsteps = int(round(2.4 * gold["T_s"] / h))
    for _ in range(nsteps):
        q, qd = O.step(sc, q, qd, h, route="dense")
        ys.append(q[0, 10])
    ys = np.asarray(ys)
    tt = np.arange(len(ys)) * h
    idx = np.nonzero(np.sign(ys[:-1]) != np.sign(ys[1:]))[0]
    zc = tt[idx] - ys[idx] * (tt[idx + 1] - tt[idx]) / (ys[idx + 1] - ys[idx])
    assert len(zc) >= 4
    T = 2 * np.mean(np.diff(zc))
    assert abs(T - gold["T_s"]) <= gold["tolerance_s"], T


def test_P5_equilibrium_fixed_point():
    """P5: zero velocity, zero gravity, satisfied joints, arbitrary rotations → qⁿ⁺¹ = qⁿ."""
    sc = G.random_tree(15, seed=11, hinge_frac=0.5, gravity=False)
    q1, qd1 = O.step(sc, sc.q0, sc.qd0, sc.h)
    assert np.max(np.abs(q1 - sc.q0)) <= 1e-14
    assert np.max(np.abs(qd1)) <= 1e-12


def _rotate_scene(sc, Q, d):
    s2 = sc.copy()
    A = O.unvec(sc.q0[:, :9])
    Ad = O.unvec(sc.qd0[:, :9])
    s2.q0[:, :9] = O.vec(Q @ A)
    s2.q0[:, 9:] = sc.q0[:, 9:] @ Q.T + d
    s2.qd0[:, :9] = O.vec(Q @ Ad)
    s2.qd0[:, 9:] = sc.qd0[:, 9:] @ Q.T
    s2.gravity = Q @ sc.gravity
    wm = np.repeat(sc.body_b, sc.npts) < 0
    s2.ybar_b[wm] = sc.ybar_b[wm] @ Q.T + d
    return s2


def test_P6_rigid_motion_equivariance():
    """P6: rotating/translating the whole scene rotates/translates the result (∇C diag₄(R) = R∇C)."""
    sc = G.random_chain(8, seed=12, vel=0.4, jitter=1e-3, npts=2)
    Q = G.random_rotations(np.random.default_rng(13), 1)[0]
    d = np.array([0.5, -1.0, 2.0])
    q1, _ = O.step(sc, sc.q0, sc.qd0, sc.h)
    s2 = _rotate_scene(sc, Q, d)
    q2, _ = O.step(s2, s2.q0, s2.qd0, s2.h)
    A1 = O.unvec(q1[:, :9])
    assert np.max(np.abs(O.unvec(q2[:, :9]) - Q @ A1)) < 1e-12
    assert np.max(np.abs(q2[:, 9:] - (q1[:, 9:] @ Q.T + d))) < 1e-12 * 10


# ----------------------------------------------------------------------------- solver pins

@pytest.mark.parametrize("n,anch,end", [(2, False, False), (7, True, False), (16, True, True)])
def test_P7_block_thomas_vs_dense_kkt(n, anch, end):
    """P7 / P:568-584: chain dual is block tridiagonal; block Thomas λ = dense-KKT λ (≤ 16 bodies)."""
    sc = G.random_chain(n, seed=14 + n, anchored=anch, end_anchor=end, vel=0.3, jitter=1e-3)
    S, r, Jd, Hinv, dqt = O.dual_matrix(sc, sc.q0, sc.qd0, sc.h)
    K = sc.n_joints
    # structure (P10): zero outside the block band, symmetric, SPD diagonal blocks
    for a in range(K):
        for b in range(K):
            blk = S[3 * a:3 * a + 3, 3 * b:3 * b + 3]
            if abs(a - b) > 1:
                assert np.all(blk == 0)
        assert np.all(np.linalg.eigvalsh(S[3 * a:3 * a + 3, 3 * a:3 * a + 3]) > 0)
    assert np.allclose(S, S.T, rtol=0, atol=1e-12 * np.abs(S).max())
    D = np.array([S[3 * k:3 * k + 3, 3 * k:3 * k + 3] for k in range(K)])
    B = np.array([S[3 * k:3 * k + 3, 3 * k + 3:3 * k + 6] for k in range(K - 1)])
    lam_t = O.block_thomas(D, B, r.reshape(K, 3)).reshape(-1)
    q1, qd1, info = O.step(sc, sc.q0, sc.qd0, sc.h, route="dense", return_info=True)
    assert O.rel_err(lam_t, info["lam"]) < 1e-10 * max(1.0, np.abs(info["lam"]).max()) or \
        np.max(np.abs(lam_t - info["lam"])) <= 1e-12 * np.abs(info["lam"]).max()
    dq = dqt.reshape(-1) - Hinv @ (Jd.T @ lam_t)
    assert O.rel_err(sc.q0 + dq.reshape(-1, 12), q1) < 1e-12


@pytest.mark.parametrize("n,seed", [(3, 20), (9, 21), (16, 22)])
def test_P7_leaf_to_root_vs_dense_kkt(n, seed):
    """P7 / A12: exact leaf-to-root elimination of the tree dual = dense KKT; zero fill (chordal dual)."""
    sc = G.random_tree(n, seed=seed, hinge_frac=0.5, vel=0.3, jitter=1e-3, extra_anchors=1)
    parent = sc.meta["parent"]
    depth = np.zeros(n, int)
    for j in range(1, n):
        depth[j] = depth[parent[j]] + 1
    S, r, Jd, Hinv, dqt = O.dual_matrix(sc, sc.q0, sc.qd0, sc.h)
    rows, child, par = [], [], []
    off = 0
    for k in range(sc.n_joints):
        m = 3 * int(sc.npts[k])
        rows.append(np.arange(off, off + m))
        off += m
        a, b = int(sc.body_a[k]), int(sc.body_b[k])
        if b < 0:
            child.append(-1)
            par.append(a)
        elif parent[b] == a:
            child.append(b)
            par.append(a)
        else:
            child.append(a)
            par.append(b)
    lam, fill = O.leaf_to_root_solve(S, r, rows, child, par, depth)
    assert fill == 0.0
    q1, _, info = O.step(sc, sc.q0, sc.qd0, sc.h, route="dense", return_info=True)
    assert np.max(np.abs(lam - info["lam"])) <= 1e-10 * np.abs(info["lam"]).max()
    dq = dqt.reshape(-1) - Hinv @ (Jd.T @ lam)
    assert O.rel_err(sc.q0 + dq.reshape(-1, 12), q1) < 1e-12


@pytest.mark.parametrize("maker", [
    lambda: G.random_chain(300, seed=30, vel=0.2, jitter=1e-3, end_anchor=True),
    lambda: G.random_tree(200, seed=31, hinge_frac=0.5, vel=0.2),
    lambda: G.small_net(12, max_off=4),
])
def test_P7_route_agreement(maker):
    """P7 route agreement: dense LU = SuperLU(full KKT) = block LU (Schur) on the same step."""
    sc = maker()
    q_d, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="dense")
    q_s, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="superlu")
    q_b, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="blocklu")
    assert O.rel_err(q_s, q_d) < 1e-12
    assert O.rel_err(q_b, q_d) < 1e-12


def test_P11_decoupling():
    """P11: chains solved in one scene = each chain solved alone (independence of assemblies)."""
    sc = G.cfg2_batched_chains(3, 20)
    q_all, _ = O.step(sc, sc.q0, sc.qd0, sc.h, route="superlu")
    for c in range(3):
        sub = G.cfg2_batched_chains(3, 20)
        keep = slice(20 * c, 20 * c + 20)
        jk = slice(20 * c, 20 * c + 20)
        sub.q0, sub.qd0, sub.mbar = sub.q0[keep], sub.qd0[keep], sub.mbar[keep]
        sub.volume, sub.youngs, sub.poisson = sub.volume[keep], sub.youngs[keep], sub.poisson[keep]
        ja, jb = sub.body_a[jk] - 20 * c, sub.body_b[jk].copy()
        jb[jb >= 0] -= 20 * c
        sub.body_a, sub.body_b, sub.npts = ja, jb, sub.npts[jk]
        sub.ybar_a, sub.ybar_b = sub.ybar_a[jk], sub.ybar_b[jk]
        sub.validate()
        q_c, _ = O.step(sub, sub.q0, sub.qd0, sub.h, route="dense")
        assert O.rel_err(q_c, q_all[keep]) < 1e-13


def test_generators_shapes():
    """The five BASELINE.json configs have the body/joint/row counts of SURVEY §8 (sizes table)."""
    s = G.cfg1_chain8()
    assert (s.n, s.n_joints, s.n_rows) == (8, 8, 24)
    s = G.cfg3_long_chain(col_len=40, n_cols=4, tail=3)
    assert s.n == 163 and s.n_joints == 164
    assert abs(np.linalg.norm(s.ybar_b[-1] - s.ybar_b[0]) - 0.05 * 7) < 1e-12
    s = G.cfg3_long_chain(col_len=2, n_cols=2, tail=0)   # full size: 194 even columns + 6 → 10.000 m
    assert s.n == 4
    s = G.cfg4_binary_tree(5)
    assert (s.n, s.n_joints, s.n_rows) == (31, 31, 3 + 30 * 6)
    s = G.cfg5_net(20, max_off=4)
    assert s.n_joints == 2 * 20 * 19 + int(0.05 * 2 * 20 * 19) + 4


# ----------------------------------------------------------------------------- Newton iterations > 1 (§8(f) NEXT 1)

def test_iterated_step_converges_to_the_implicit_step():
    """K Newton iterations (each linearised at the previous iterate, P:459 footnote) converge to the
    stationary point of the implicit step's nonlinear problem: M_A(q − q̂)/h² + ∇VΨ(q) + ∇Cᵀλ = 0, C(q) = 0
    (P:193-199). The residual is an independent restatement of that problem; the
    quasi-Newton iteration with the constant rotated H̄ converges linearly."""
    sc = G.random_chain(6, seed=3, vel=3.0, jitter=1e-3)
    res = []
    for K in (1, 2, 4, 8, 40):
        q1, _ = O.step(sc, sc.q0, sc.qd0, sc.h, iters=K)
        r, c = O.nonlinear_residual(sc, sc.q0, sc.qd0, q1, sc.h)
        assert c <= 1e-12
        res.append(r)
    assert all(b < a for a, b in zip(res, res[1:])), res
    assert res[0] > 1.0 and res[-1] <= 1e-10, res


def test_iterated_free_fall_is_exact():
    """P1 with K = 3: the free-fall step is linear, so later iterations change nothing (closed form)."""
    R0 = G.random_rotations(np.random.default_rng(6), 1)[0]
    v0 = np.array([1.0, -2.0, 3.0])
    t0 = np.array([0.3, 0.2, 0.1])
    sc = G.free_body(A0=R0, t0=t0, v0=v0, dims=(0.1, 0.3, 0.2), E=1e8)
    n, h, g = 12, sc.h, sc.gravity
    q, qd = O.simulate(sc, n, iters=3)
    t_ref = t0 + n * h * v0 + 0.5 * n * (n + 1) * h * h * g
    assert np.max(np.abs(q[0, 9:] - t_ref)) <= 1e-13 * np.max(np.abs(t_ref))
    assert np.max(np.abs(qd[0, 9:] - (v0 + n * h * g))) <= 1e-12 * np.max(np.abs(v0 + n * h * g))
    assert np.max(np.abs(q[0, :9] - O.vec(R0))) < 1e-14


def test_iterated_momentum_and_closure():
    """P2 and P3 with K = 3: every iteration conserves Σ m t (the t-rows of ∇C cancel, H̄'s t-block is (m/h²)I) and
    closes the linear joints (C(q⁽ⁱ⁺¹⁾) = C(q⁽ⁱ⁾) + ∇Cδq = 0)."""
    sc = G.random_tree(12, seed=8, anchored=False, vel=0.3, gravity=False, hinge_frac=0.5)
    m = sc.mbar[:, 9]
    p0 = (m[:, None] * sc.qd0[:, 9:]).sum(0)
    q, qd = sc.q0, sc.qd0
    for _ in range(4):
        q, qd = O.step(sc, q, qd, sc.h, iters=3)
        p = (m[:, None] * qd[:, 9:]).sum(0)
        assert np.max(np.abs(p - p0)) <= 1e-12 * max(np.max(np.abs(p0)), np.max(m * np.abs(qd[:, 9:]).max(1)))
        assert O.constraint_residual(sc, q) <= 1e-10
    sc = G.random_chain(10, seed=9, jitter=2e-3, vel=0.2, end_anchor=True)
    q, qd = sc.q0, sc.qd0
    for _ in range(3):
        q, qd = O.step(sc, q, qd, sc.h, iters=2)
        assert O.constraint_residual(sc, q) <= 1e-10


def test_one_iteration_is_the_plain_step():
    sc = G.random_chain(7, seed=2, vel=0.5, jitter=1e-3)
    a = O.step(sc, sc.q0, sc.qd0, sc.h)
    b = O.step(sc, sc.q0, sc.qd0, sc.h, iters=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ----------------------------------------------------------------------------- external wrenches (§8(f) NEXT 1)

def test_wrench_com_force_free_flight():
    """A constant force f at the centre of mass acts like an extra uniform field f/m: the free-fall closed form
    with g + f/m (P:672-676 with G's t-block = I₃)."""
    R0 = G.random_rotations(np.random.default_rng(7), 1)[0]
    v0, t0 = np.array([0.5, 0.0, -1.0]), np.array([0.1, 0.2, 0.3])
    sc = G.free_body(A0=R0, t0=t0, v0=v0, dims=(0.2, 0.1, 0.3), E=1e8)
    f = np.array([3.0, -1.0, 2.0])
    sc.wrench = np.array([[0, 0, 0, *f]])
    n, h = 15, sc.h
    q, qd = O.simulate(sc, n)
    a = sc.gravity + f / sc.mbar[0, 9]
    t_ref = t0 + n * h * v0 + 0.5 * n * (n + 1) * h * h * a
    assert np.max(np.abs(q[0, 9:] - t_ref)) <= 1e-13 * np.max(np.abs(t_ref))
    assert np.max(np.abs(q[0, :9] - O.vec(R0))) < 1e-14


def test_wrench_torque_is_rigid_body_dynamics():
    """A torque τ on a stiff body at rest: after one step its angular velocity ω = ½Σ q_c × q̇_c is the
    rigid-body ω = I_w⁻¹τh (Euler's equations from rest; I_w = R₀ I_body R₀ᵀ), to O(h) and the stiffness-limited
    non-rigid part. A wrong sign, factor ½ or cross-product order in G(A)ᵀW fails this."""
    R0 = G.random_rotations(np.random.default_rng(1), 1)[0]
    sc = G.free_body(A0=R0, dims=(0.3, 0.2, 0.1), E=1e9)
    sc.gravity = np.zeros(3)
    tau = np.array([0.3, -0.2, 0.5])
    sc.wrench = np.array([[*tau, 0, 0, 0]])
    q1, qd1 = O.step(sc, sc.q0, sc.qd0, sc.h)
    w = O.angular_velocity(q1, qd1)[0]
    m = sc.mbar[0]
    Ib = np.diag([m[4] + m[7], m[0] + m[7], m[0] + m[4]])   # ∫ρ(y²+z²), … from M̄ = diag(∫ρx², ∫ρy², ∫ρz², m)
    ref = np.linalg.solve(R0 @ Ib @ R0.T, tau) * sc.h
    assert np.max(np.abs(w - ref)) <= 1e-4 * np.max(np.abs(ref))
    # the twist helpers invert each other on rigid motions
    om, v = np.array([0.4, -0.1, 0.2]), np.array([1.0, 2.0, 3.0])
    qd = O.twist_velocity(sc.q0, om, v)
    assert np.allclose(O.angular_velocity(sc.q0, qd)[0], om, atol=1e-15) and np.allclose(qd[0, 9:], v)


def test_wrench_momentum_balance():
    """Linear momentum changes by h Σ(f + m g) per step exactly, with joints (the t-rows of ∇C cancel)."""
    sc = G.random_chain(8, seed=11, anchored=False, vel=0.3, gravity=True, npts=1)
    rng = np.random.default_rng(3)
    sc.wrench = rng.normal(size=(sc.n, 6))
    m = sc.mbar[:, 9]
    q, qd = sc.q0, sc.qd0
    p = (m[:, None] * qd[:, 9:]).sum(0)
    for _ in range(3):
        q, qd = O.step(sc, q, qd, sc.h)
        p1 = (m[:, None] * qd[:, 9:]).sum(0)
        ref = p + sc.h * (sc.wrench[:, 3:].sum(0) + m.sum() * sc.gravity)
        assert np.max(np.abs(p1 - ref)) <= 1e-12 * max(np.max(np.abs(ref)), 1.0)
        p = p1


@pytest.mark.parametrize("maker", ["chain", "tree", "net"])
def test_P12_material_frame_covariance(maker):
    """P12: the same scene written in general (rotated, non-central) material frames — full SPD M̄ coupling the
    A-columns with t and with each other — gives the same motion: x̄_u = P x̄ + d maps
    q ↦ (A Pᵀ, t − A Pᵀ d) for every quantity (K̄_A is invariant under δA ↦ Q δA Qᵀ and commutes with the
    co-rotation; R8). A dropped off-diagonal M̄ term, a gravity force taken from M̄'s diagonal only, or a
    frame-dependent elastic force fails it (errors of 1e-4 … 1). Chain and tree: 3 steps at 1e-12 relative; the stiff
    net (E = 1e9: K̄_A outweighs M_A/h² by ~1e5, so the re-framed coordinates' rounding is amplified): 1 step at
    3e-11 (measured 6e-12)."""
    sc = {"chain": lambda: G.random_chain(7, seed=3, vel=0.3, jitter=1e-3, end_anchor=True),
          "tree": lambda: G.random_tree(9, seed=4, vel=0.3, jitter=1e-3),
          "net": lambda: G.small_net(4, max_off=2)}[maker]()
    u = G.reframe_scene(sc, seed=7)
    assert np.max(np.abs(u.mbar[:, [1, 2, 3, 5, 6, 8]])) > 1e-3 * np.max(np.abs(u.mbar))
    steps, tol = (1, 3e-11) if maker == "net" else (3, 1e-12)
    q, qd = O.simulate(sc, steps)
    qu, qdu = O.simulate(u, steps)
    assert O.rel_err(G.frame_to_canonical(qu, u.frames), q) < tol
    assert O.rel_err(G.frame_to_canonical(qdu * sc.h, u.frames), qd * sc.h) < tol


# ----------------------------------------------------------------------------- polar-free variant (NEXT 4, R9)

def _stvk_energy(A, V, mu, lam):
    """V[μ‖E‖² + (λ/2)tr(E)²], E = ½(AᵀA − I): Saint Venant–Kirchhoff, written out independently."""
    E = 0.5 * (A.T @ A - np.eye(3))
    return V * (mu * np.sum(E * E) + 0.5 * lam * np.trace(E) ** 2)


def test_R9_stvk_force_is_fd_gradient_with_rest_hessian_kbar():
    """The polar-free elastic force is the gradient of the StVK energy, and its Jacobian at A = I is K̄_A — the same
    pre-factored H̄ serves both variants."""
    rng = np.random.default_rng(21)
    V, mu, lam = 2e-3, *O.lame(1e8, 0.3)
    for _ in range(4):
        A = G.random_rotations(rng, 1)[0] @ (np.eye(3) + 0.05 * rng.standard_normal((3, 3)))
        f = O.stvk_force_A(A, V, mu, lam)
        eps = 1e-7
        g = np.array([(_stvk_energy(O.unvec(O.vec(A) + eps * e), V, mu, lam)
                       - _stvk_energy(O.unvec(O.vec(A) - eps * e), V, mu, lam)) / (2 * eps) for e in np.eye(9)])
        assert np.max(np.abs(f - g)) <= 1e-7 * np.max(np.abs(g))
    eps = 1e-6
    J = np.array([(O.stvk_force_A(O.unvec(O.vec(np.eye(3)) + eps * e), V, mu, lam)
                   - O.stvk_force_A(O.unvec(O.vec(np.eye(3)) - eps * e), V, mu, lam)) / (2 * eps) for e in np.eye(9)]).T
    K = O.kbar_A(V, mu, lam)[:9, :9]
    assert np.max(np.abs(J - K)) <= 1e-6 * np.max(np.abs(K))


def test_R9_length_preserving_map():
    """Eq. len_preserving: the image has the length of v, and a rotation is reproduced exactly."""
    rng = np.random.default_rng(22)
    M = np.eye(3) + 0.3 * rng.standard_normal((5, 3, 3))
    v = rng.standard_normal((5, 3))
    w = O.length_preserving(M, v)
    assert np.allclose(np.linalg.norm(w, axis=1), np.linalg.norm(v, axis=1), rtol=1e-14)
    assert np.allclose(np.cross(w, np.einsum("nij,nj->ni", M, v)), 0, atol=1e-13)   # parallel to M v
    R = G.random_rotations(rng, 5)
    assert np.allclose(O.length_preserving(R, v), np.einsum("nij,nj->ni", R, v), atol=1e-15)
    assert np.all(O.length_preserving(M, np.zeros((5, 3))) == 0)


@pytest.mark.parametrize("maker", ["chain", "tree"])
def test_R9_polar_free_equals_exact_at_rigid_states(maker):
    """At a rigid state (every A ∈ SO(3)) Alg. 1's maps are the rotations themselves, the StVK and co-rotated forces
    both vanish and diag₄(A)H̄⁻¹diag₄(Aᵀ) = H_A⁻¹: one polar-free step equals one exact step."""
    sc = {"chain": lambda: G.random_chain(9, seed=23, vel=0.4, end_anchor=True, jitter=1e-3),
          "tree": lambda: G.random_tree(12, seed=24, vel=0.4, jitter=1e-3)}[maker]()
    q1, qd1 = O.step(sc, sc.q0, sc.qd0, sc.h)
    q2, qd2 = O.step(sc, sc.q0, sc.qd0, sc.h, rotation="length_preserving")
    assert O.rel_err(q2, q1) < 1e-13 and O.rel_err(qd2 * sc.h, qd1 * sc.h) < 1e-13


def test_R9_polar_free_closure_equivariance_and_rest():
    """The polar-free step on strained states: joints close (P3), a rigid motion of the scene moves the result with
    it (P6: Alg. 1's maps are rotation-equivariant), and it differs from the exact step (the variant is not exact
    away from SO(3))."""
    sc = G.random_chain(10, seed=25, vel=0.3, npts=2, jitter=1e-3)
    A = O.unvec(sc.q0[:, :9]) @ (np.eye(3) + 0.03 * np.random.default_rng(26).standard_normal((sc.n, 3, 3)))
    sc.q0[:, :9] = O.vec(A)
    q1, _ = O.step(sc, sc.q0, sc.qd0, sc.h, rotation="length_preserving")
    assert O.constraint_residual(sc, q1) < 1e-10
    qe, _ = O.step(sc, sc.q0, sc.qd0, sc.h)
    assert O.rel_err(q1, qe) > 1e-6
    Q = G.random_rotations(np.random.default_rng(27), 1)[0]
    d = np.array([0.3, 0.2, -0.1])
    s2 = _rotate_scene(sc, Q, d)
    q2, _ = O.step(s2, s2.q0, s2.qd0, s2.h, rotation="length_preserving")
    assert np.max(np.abs(O.unvec(q2[:, :9]) - Q @ O.unvec(q1[:, :9]))) < 1e-12
    assert np.max(np.abs(q2[:, 9:] - (q1[:, 9:] @ Q.T + d))) < 1e-11
    # rest: unstrained, at rest, no gravity, joints satisfied → nothing moves
    r = G.random_chain(6, seed=28, vel=0.0, gravity=False)
    q3, qd3 = O.step(r, r.q0, r.qd0, r.h, rotation="length_preserving")
    assert np.max(np.abs(q3 - r.q0)) < 1e-14 and np.max(np.abs(qd3)) < 1e-12


# ----------------------------------------------------------------------------- line Gauss-Seidel (NEXT 3, R10)

def test_line_gauss_seidel_pins():
    """Block Gauss-Seidel on SPD systems: one block covering everything is the exact solve after one sweep; any block
    partition converges to np.linalg.solve; one sweep of single-row blocks is textbook point Gauss-Seidel."""
    rng = np.random.default_rng(31)
    X = rng.standard_normal((30, 30))
    S = X @ X.T + 30 * np.eye(30)
    r = rng.standard_normal(30)
    exact = np.linalg.solve(S, r)
    one = O.line_gauss_seidel(S, r, [np.arange(30)], [[0]], 1)
    assert np.max(np.abs(one - exact)) < 1e-12 * np.max(np.abs(exact))
    blocks = [np.arange(i, min(i + 6, 30)) for i in range(0, 30, 6)]
    lam = O.line_gauss_seidel(S, r, blocks, [[0, 2, 4], [1, 3]], 300)
    assert np.max(np.abs(lam - exact)) < 1e-10 * np.max(np.abs(exact))
    # point GS, one sweep, written out as the textbook forward substitution (D + L) x = r
    pts = [np.array([i]) for i in range(30)]
    g1 = O.line_gauss_seidel(S, r, pts, [[i] for i in range(30)], 1)
    assert np.allclose(g1, np.linalg.solve(np.tril(S), r), rtol=1e-12, atol=1e-14)


def test_step_with_dual_is_the_step():
    """step_with_dual with the exact dual solve reproduces the KKT step."""
    sc = G.small_net(5, max_off=2)
    q1, qd1 = O.step(sc, sc.q0, sc.qd0, sc.h)
    q2, qd2 = O.step_with_dual(sc, sc.q0, sc.qd0, sc.h, np.linalg.solve)
    assert O.rel_err(q2, q1) < 1e-11 and O.rel_err(qd2 * sc.h, qd1 * sc.h) < 1e-11


# ----------------------------------------------------------------------------- five-row hinge (NEXT 2, R13)

def _hinge5_C(sc, q):
    """The five-row hinge constraint written out independently (Eq. hinge): ball rows of the pivot points,
    and the local x̃, z̃ of the second points' difference in the frame R_H = ΔR_H Rᵀ(A_a), R by scipy's polar."""
    off = np.concatenate([[0], np.cumsum(sc.npts)])
    out = []
    for k in range(sc.n_joints):
        a, b = sc.body_a[k], sc.body_b[k]
        def x(body, y):
            if body < 0:
                return y
            A = O.unvec(q[body, :9])
            return A @ y + q[body, 9:]
        for i in range(sc.npts[k]):
            d = x(a, sc.ybar_a[off[k] + i]) - x(b, sc.ybar_b[off[k] + i])
            if sc.kind is not None and sc.kind[k] == 1 and i == 1:
                R, _ = scipy.linalg.polar(O.unvec(q[a, :9]))
                ax = sc.ybar_a[off[k] + 1] - sc.ybar_a[off[k]]
                ax = ax / np.linalg.norm(ax)
                v = np.cross(ax, [0, 1, 0])
                V = np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])
                dR = np.eye(3) + V + V @ V / (1 + ax[1])
                assert np.allclose(dR @ ax, [0, 1, 0])
                out.append((dR @ R.T @ d)[[0, 2]])
            else:
                out.append(d)
    return np.concatenate(out)


def test_hinge5_jacobian_is_the_gradient_where_the_axis_points_coincide():
    """R13: with R_H frozen at q the five-row hinge's rows are W Γ; the dropped ∂R_H/∂q term multiplies the second
    points' separation, so at states where those coincide (every satisfied hinge, up to axial stretch) the oracle's
    Jacobian is the exact gradient of the nonlinear constraint (central differences, rotated bodies); away from them
    it is not."""
    sc = G.five_row_hinges(G.random_tree(6, seed=41, hinge_frac=1.0, vel=0.3))
    J, w = O.constraint_system(sc, sc.q0)
    assert J.shape[0] == 5 * int(np.sum(sc.kind == 1)) + 3 * int(np.sum(sc.kind == 0))
    assert np.max(np.abs(J @ sc.q0.reshape(-1) - w - _hinge5_C(sc, sc.q0))) < 1e-12
    eps = 1e-6
    q0 = sc.q0.reshape(-1)
    fd = np.array([(_hinge5_C(sc, (q0 + eps * e).reshape(sc.n, 12)) - _hinge5_C(sc, (q0 - eps * e).reshape(sc.n, 12)))
                   / (2 * eps) for e in np.eye(q0.size)]).T
    assert np.max(np.abs(fd - J.toarray())) < 1e-7 * np.max(np.abs(fd))
    # a state with separated axis points: the frozen-R_H Jacobian is no longer the gradient
    q1 = sc.q0.copy()
    q1[:, 9:] += 0.01 * np.random.default_rng(42).standard_normal((sc.n, 3))
    J1, _ = O.constraint_system(sc, q1)
    fd1 = np.array([(_hinge5_C(sc, (q1.reshape(-1) + eps * e).reshape(sc.n, 12))
                     - _hinge5_C(sc, (q1.reshape(-1) - eps * e).reshape(sc.n, 12))) / (2 * eps) for e in np.eye(q0.size)]).T
    assert np.max(np.abs(fd1 - J1.toarray())) > 1e-4 * np.max(np.abs(fd1))


def test_hinge5_is_a_hinge():
    """A rod on a world hinge, released spinning about its centre (ω off the hinge axis): the five-row hinge and the
    six-row linear hinge give the same motion up to the second point's axial freedom, i.e. up to material
    stretch — the difference over 50 steps scales as 1/E (6e-6 at E = 1e8, 6e-8 at 1e10) — both closing their
    constraints, while a ball joint at the pivot lets the rod tumble away (an O(1) difference)."""
    errs = []
    for E in (1e8, 1e10):
        lin = G.hinge_pendulum(axis=(1, 0, 0), omega0=(3.0, 2.0, 1.0), E=E)
        h5 = G.five_row_hinges(lin)
        q_l, _ = O.simulate(lin, 50)
        q_5, qd_5 = O.simulate(h5, 50)
        errs.append(O.rel_err(q_5, q_l))
        assert O.constraint_residual(h5, q_5) < 1e-12
    assert errs[1] < 1e-6 and 50 < errs[0] / errs[1] < 200
    ball = lin.copy()
    ball.npts = np.array([1], np.int32)
    ball.ybar_a, ball.ybar_b = lin.ybar_a[:1], lin.ybar_b[:1]
    q_b, _ = O.simulate(ball, 50)
    assert O.rel_err(q_b, q_l) > 1e-2
    # the rod turns about the hinge axis only: its angular velocity is along x
    om = O.angular_velocity(q_5, qd_5)[0]
    assert np.linalg.norm(om) > 0.1 and np.max(np.abs(om[1:])) < 1e-3 * np.linalg.norm(om)


# ----------------------------------------------------------------------------- joint limits (NEXT 4, R14)

def test_hinge_angle_is_the_rotation_about_the_axis():
    """hinge_angle (the rotation of body b relative to body a about the axis): a rod on a world hinge (body a = the
    rod, b = the world) turned by φ about the axis through the pivot reads θ = −φ."""
    base = G.hinge_limits(G.five_row_hinges(G.hinge_pendulum(axis=(0.3, 1.0, 0.2))), -1.0, 1.0)
    ax = base.ybar_b[1] - base.ybar_b[0]
    for phi in (-0.7, 0.0, 0.25, 1.3):
        Q = O.rotation_about(ax, phi)
        A = O.unvec(base.q0[0, :9])
        t = base.q0[0, 9:]
        q = base.q0.copy()
        q[0, :9] = O.vec(Q @ A)
        q[0, 9:] = Q @ (t - base.ybar_b[0]) + base.ybar_b[0]      # rotated about the pivot (a world point)
        assert abs(O.hinge_angle(base, q, 0) + phi) < 1e-12


def test_hinge_limits_hold_the_angle():
    """A rod swinging on a world hinge through ±0.25 rad: with limits ±∞ the motion is unchanged; with ±0.1 rad every
    step that starts beyond a bound lands on it (one linearised row: within 1e-3 rad) and the angle never leaves
    [−0.1, 0.1] by more than one step's travel."""
    base = G.five_row_hinges(G.hinge_pendulum(axis=(1, 0, 0), omega0=(6.0, 0, 0)))
    free, _ = O.simulate(base, 150)
    inf = G.hinge_limits(base, -np.inf, np.inf)
    q_inf, _ = O.simulate(inf, 150)
    assert np.array_equal(q_inf, free)
    sc = G.hinge_limits(base, -0.1, 0.1)
    q, qd = sc.q0, sc.qd0
    th_free, th = [], []
    qf, qdf = base.q0, base.qd0
    landed = 0
    for _ in range(150):
        before = O.hinge_angle(sc, q, 0)
        q, qd = O.step(sc, q, qd, sc.h)
        after = O.hinge_angle(sc, q, 0)
        if abs(before) > 0.1:
            assert abs(after - np.sign(before) * 0.1) < 1e-3
            landed += 1
        th.append(after)
        qf, qdf = O.step(base, qf, qdf, base.h)
        th_free.append(O.hinge_angle(sc, qf, 0))
    assert max(np.abs(th_free)) > 0.24 and landed >= 2
    assert max(np.abs(th)) < 0.1 + 6.0 * sc.h


def test_hinge_frame_and_rotation_about():
    """hinge_frame(a) is a proper rotation taking the unit axis a onto e_y (also at a = ±e_y);
    rotation_about matches scipy's rotation-vector map."""
    from scipy.spatial.transform import Rotation
    rng = np.random.default_rng(51)
    axes = list(rng.standard_normal((8, 3))) + [np.array([0, 1.0, 0]), np.array([0, -1.0, 0]),
                                                 np.array([1e-9, -1.0, 0])]
    for a in axes:
        R = O.hinge_frame(a)
        assert np.allclose(R @ (a / np.linalg.norm(a)), [0, 1, 0], atol=1e-8)
        assert np.allclose(R.T @ R, np.eye(3), atol=1e-12) and abs(np.linalg.det(R) - 1) < 1e-12
    for _ in range(5):
        ax = rng.standard_normal(3)
        ang = rng.uniform(-3, 3)
        ref = Rotation.from_rotvec(ang * ax / np.linalg.norm(ax)).as_matrix()
        assert np.allclose(O.rotation_about(ax, ang), ref, atol=1e-13)


def test_literal_alg2_is_an_approximation():
    """Literal Alg. 2 (ABD-ABA as printed; DESIGN R15): exact for a lone body (Ĥ = H), it closes every joint
    (its local KKTs carry the footnote residual), E(A) inverts the twist map G(A) on rigid motions (G E = I₆,
    P:757), but on articulated trees its step departs from the exact KKT step by about the step itself — the rigid
    transport X = diag₄(R_relᵀ) ignores the lever arm between the frames."""
    one = G.random_chain(1, seed=4, anchored=False, vel=0.5)
    assert O.rel_err(O.aba_literal_step(one, one.q0, one.qd0, one.h)[0], O.step(one, one.q0, one.qd0, one.h)[0]) < 1e-13
    A = G.random_rotations(np.random.default_rng(61), 1)[0]
    Gm = np.zeros((6, 12))
    for c in range(3):
        qc = A[:, c]
        Gm[:3, 3 * c:3 * c + 3] = 0.5 * np.array([[0, -qc[2], qc[1]], [qc[2], 0, -qc[0]], [-qc[1], qc[0], 0]])
    Gm[3:, 9:] = np.eye(3)
    assert np.allclose(Gm @ O.twist_embedding(A), np.eye(6), atol=1e-13)
    sc = G.random_tree(20, seed=1, hinge_frac=0.5, vel=0.3)
    q_lit, _ = O.aba_literal_step(sc, sc.q0, sc.qd0, sc.h)
    q_ex, _ = O.step(sc, sc.q0, sc.qd0, sc.h)
    assert O.constraint_residual(sc, q_lit) < 1e-12
    assert O.rel_err(q_lit, q_ex) > 0.1 * np.max(np.abs(q_ex - sc.q0))


# ------------------------------------------------------------------------------------------------ R17: universal,
# prismatic joints
@pytest.mark.parametrize("world", [False, True])
def test_R17_general_row_gradient_is_exact(world):
    """Both row types of joint_general_rows: the gradient equals the central difference of the value at random,
    unsatisfied, strained states (the R ≈ A relaxation makes the rows polynomial in q, so the gradient is exact)."""
    rng = np.random.default_rng(41 + world)
    q = rng.standard_normal((2, 12))
    b = -1 if world else 1
    rows = [("dir", 0, b, rng.standard_normal(3), None, rng.standard_normal(3)),
            ("point", 0, b, rng.standard_normal(3), rng.standard_normal(3), rng.standard_normal(3))]
    for row in rows:
        c0, g = O.general_row(row, q)
        for body in (0, 1):
            for i in range(12):
                e = np.zeros((2, 12))
                e[body, i] = 1e-6
                fd = (O.general_row(row, q + e)[0] - O.general_row(row, q - e)[0]) / 2e-6
                an = g[body][i] if body in g else 0.0
                assert abs(fd - an) < 1e-8 * (1 + abs(fd)), (row[0], body, i, fd, an)


def test_R17_newton_iterations_close_the_joints():
    """A random tree whose hinges became universal and prismatic joints: each Newton iteration of a step cuts the
    joint residual by more than 100× (measured 1.2e-4, 3.8e-7, 1.8e-9; the rows' gradients are exact, the rest is
    the primal's co-rotated Hessian; dropping the prismatic rows' rotation term gives ≈ 30× per iteration)."""
    sc = G.nonlinear_joints(G.random_tree(30, seed=1, hinge_frac=0.8, vel=0.3), seed=2)
    assert set(np.unique(sc.kind)) >= {2, 3}
    res = []
    for it in (1, 2, 3):
        q, qd = O.step(sc, sc.q0, sc.qd0, sc.h, iters=it)
        res.append(O.constraint_residual(sc, q))
    assert res[1] < 1e-2 * res[0] and res[2] < 1e-2 * res[1], res


def test_R17_prismatic_rail_slides_like_a_point_mass():
    """A slider on a frictionless rail tilted 30°: implicit Euler of the constant acceleration g sin 30° along the rail
    gives s_n = a h² n(n+1)/2 exactly; the slider leaves the rail by < 1e-14 and does not turn."""
    sc = G.prismatic_rail(h=1e-2)
    a = 9.81 * np.sin(np.deg2rad(30.0))
    q, qd = sc.q0, sc.qd0
    for n in range(1, 51):
        q, qd = O.step(sc, q, qd, sc.h)
        s = q[0, 9:] @ sc.meta["rail"]
        assert abs(s + a * sc.h ** 2 * n * (n + 1) / 2) < 1e-12
        assert np.linalg.norm(q[0, 9:] - s * sc.meta["rail"]) < 1e-14
    assert np.max(np.abs(q[0, :9] - sc.q0[0, :9])) < 1e-14


def test_R17_universal_blocks_the_third_rotation():
    """A rod on a world universal joint (a₁ = rod x, a₂ = world y) released spinning about its long axis z = a₁ × a₂:
    one step removes the spin (|ω_z| < 1e-4 of 3 rad/s) that a ball joint keeps (> 0.99 of it); the swing about x and
    y is the ball joint's (the universal joint leaves those free)."""
    from oracle import rigid_reference as RR
    sc = G.universal_pendulum(omega0=(1.0, 0.5, 3.0))
    q, qd = O.step(sc, sc.q0, sc.qd0, sc.h)
    wu = RR.body_omega(q[0], qd[0])[0]
    sb = sc.copy()
    sb.kind, sb.npts, sb.ybar_a, sb.ybar_b = None, np.array([1], np.int32), sb.ybar_a[:1], sb.ybar_b[:1]
    q, qd = O.step(sb, sb.q0, sb.qd0, sb.h)
    wb = RR.body_omega(q[0], qd[0])[0]
    assert abs(wu[2]) < 1e-4 * 3.0 and wb[2] > 0.99 * 3.0
    assert np.allclose(wu[:2], wb[:2], rtol=1e-2)
