"""Plain CPU fp64 oracle of one M-ABD implicit step with linear joints.

TEST INFRASTRUCTURE ONLY. Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline / ``--impl reference``) may import this module. The
CUDA product path never imports it and shares no code with it.

What it computes ("Plain definition"): with linear joints and one
Newton iteration a step is exactly the solution of ONE linear KKT system,
PAPER.md P:460-474 (Eq. kkt) with the footnote P:459 residual term:

    [ H̃   ∇C̃ᵀ ] [ δq ]   [ f̃_A     ]
    [ ∇C̃  0   ] [ λ  ] = [ −C̃(qⁿ) ]

H̃ = diag_M(H_A^j), H_A^j = diag₄(R_j) H̄_j diag₄(R_jᵀ)
H̄_j = M_A/h² + K̄_A
f_A = (1/h) M_A q̇ⁿ + M_A [0₉; g] − [V vec(R Π(RᵀA)); 0₃]
qⁿ⁺¹ = qⁿ + δq,  q̇ⁿ⁺¹ = δq / h

With K > 1 Newton iterations, each iteration is such a KKT solve linearised at the
previous iterate (``step(..., iters=K)``); ``nonlinear_residual`` states the nonlinear problem they converge to.

Each function cites the passage it follows. The KKT is solved by a library
solver (dense LU, SuperLU on the full KKT, or block LU in a fixed bodies-first
pivot order: SURVEY §8(c) O3). The specialised CPU solvers at the bottom (block
Thomas, leaf-to-root elimination) exist only for pin P7 (agreement with the
brute-force KKT on ≤ 16 bodies).

Readings of the paper used here are listed in DESIGN.md ("Readings") and
SURVEY §8(c) A1-A21; each is referenced where used.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "lame", "unpack_mbar", "mass_A", "kbar_A", "hbar_A", "polar", "elastic_force_A", "stvk_force_A",
    "length_preserving", "affine_force",
    "body_hessians", "hinge_frame", "hinge5_rows", "joint_general_rows", "general_row", "rotation_about", "hinge_angle",
    "hinge_limit_rows",
    "constraint_system", "constraint_residual", "predict", "step", "simulate", "nonlinear_residual",
    "wrench_force", "twist_velocity", "angular_velocity",
    "block_thomas", "leaf_to_root_solve", "dual_matrix", "line_gauss_seidel", "step_with_dual", "twist_embedding",
    "joint_subspace", "aba_literal_step", "rel_err", "T9",
    "vec", "unvec",
]

# --------------------------------------------------------------------------
# conventions
# --------------------------------------------------------------------------

def vec(A: np.ndarray) -> np.ndarray:
    """Column-major vec of [...,3,3] → [...,9] (stack the three columns of A)."""
    A = np.asarray(A)
    return np.swapaxes(A, -1, -2).reshape(A.shape[:-2] + (9,))


def unvec(v: np.ndarray) -> np.ndarray:
    """Inverse of ``vec``: [...,9] → [...,3,3] with A[:, c] = v[3c:3c+3] (vec⁻¹)."""
    v = np.asarray(v)
    return np.swapaxes(v.reshape(v.shape[:-1] + (3, 3)), -1, -2)


def _t9() -> np.ndarray:
    """T₉: the 9×9 permutation with T₉ vec(A) = vec(Aᵀ) (SPEC S:48 'H_lin = μ(I₉+T₉)+…')."""
    T = np.zeros((9, 9))
    for r in range(3):
        for c in range(3):
            T[3 * c + r, 3 * r + c] = 1.0
    return T


T9 = _t9()


def lame(E, nu):
    """Lamé parameters from (E, ν), standard formulas (P:267-269 names μ, λ)."""
    E = np.asarray(E, dtype=np.float64)
    nu = np.asarray(nu, dtype=np.float64)
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return mu, lam


_PACK = [(0, 0), (0, 1), (0, 2), (0, 3), (1, 1), (1, 2), (1, 3), (2, 2), (2, 3), (3, 3)]


def unpack_mbar(mbar: np.ndarray) -> np.ndarray:
    """Packed [...,10] upper triangle (row-major) → symmetric [...,4,4] M̄."""
    mbar = np.asarray(mbar, dtype=np.float64)
    M = np.zeros(mbar.shape[:-1] + (4, 4))
    for k, (i, j) in enumerate(_PACK):
        M[..., i, j] = mbar[..., k]
        M[..., j, i] = mbar[..., k]
    return M


def mass_A(mbar: np.ndarray) -> np.ndarray:
    """Generalized mass M_A = JᵀMJ = M̄ ⊗ I₃ (P:182-184 with P:215).

    With x_i = [x̄_iᵀ ⊗ I₃, I₃] q, JᵀMJ = Σ m_i [x̄_i;1][x̄_i;1]ᵀ ⊗ I₃ = M̄ ⊗ I₃.
    """
    return np.kron(unpack_mbar(mbar), np.eye(3)) if np.ndim(mbar) == 1 else \
        np.einsum("...ij,kl->...ikjl", unpack_mbar(mbar), np.eye(3)).reshape(np.shape(mbar)[:-1] + (12, 12))


def kbar_A(V, mu, lam) -> np.ndarray:
    """Rest-shape generalized stiffness K̄_A = V[μ(I₉+T₉) + λ vec(I)vec(I)ᵀ] ⊕ 0₃.

    The Hessian w.r.t. vec(A) of V·Ψ with ∂Ψ/∂A = μ(A+Aᵀ−2I) + λ tr(A−I) I; the translation
    block is zero (the energy does not depend on t).
    """
    V = np.asarray(V, dtype=np.float64)
    mu = np.asarray(mu, dtype=np.float64)
    lam = np.asarray(lam, dtype=np.float64)
    vI = vec(np.eye(3))
    Klin = mu[..., None, None] * (np.eye(9) + T9) + lam[..., None, None] * np.outer(vI, vI)
    K = np.zeros(V.shape + (12, 12))
    K[..., :9, :9] = V[..., None, None] * Klin
    return K


def hbar_A(mbar, V, E, nu, h) -> np.ndarray:
    """H̄_A = M_A/h² + K̄_A, the constant (pre-factorizable) body matrix (Eq. abd_final)."""
    mu, lam = lame(E, nu)
    return mass_A(mbar) / (h * h) + kbar_A(V, mu, lam)


def polar(A: np.ndarray, det_min: float = 1e-9) -> np.ndarray:
    """Rotation factor R = A(AᵀA)^{-1/2} of the polar decomposition, via the SVD A = UΣVᵀ, R = UVᵀ.

    Raises if det A ≤ det_min (near-singular / inverted bodies are errors).
    """
    A = np.asarray(A, dtype=np.float64)
    d = np.linalg.det(A)
    if np.any(~np.isfinite(d)) or np.any(d <= det_min):
        raise FloatingPointError("polar: det(A) <= %g (degenerate or inverted body)" % det_min)
    U, _, Vt = np.linalg.svd(A)
    return U @ Vt   # det(A) > 0 ⇒ det(UVᵀ) = +1


def elastic_force_A(A, V, mu, lam) -> np.ndarray:
    """Co-rotated linear-elastic force on the A-DOFs: V vec(R Π(F)), F = RᵀA.

    Π(F) = μ(F+Fᵀ−2I) + λ tr(F−I) I is ∂Ψ/∂A of P:269 evaluated in the co-rotated frame; the volume weight
    is the J̄ of P:263-265 for F_e = A (constant over the body).
    """
    A = np.asarray(A, dtype=np.float64)
    R = polar(A)
    F = np.swapaxes(R, -1, -2) @ A
    I = np.eye(3)
    trF = np.trace(F, axis1=-2, axis2=-1)
    Pi = np.asarray(mu)[..., None, None] * (F + np.swapaxes(F, -1, -2) - 2 * I) + \
        (np.asarray(lam) * (trF - 3.0))[..., None, None] * I
    return np.asarray(V)[..., None] * vec(R @ Pi)


def stvk_force_A(A, V, mu, lam) -> np.ndarray:
    """Polar-free elastic force (reading R9): V vec(A Σ(E)), Σ = 2μE + λ tr(E) I, E = ½(AᵀA − I) — the
    gradient of V[μ‖E‖² + (λ/2)tr(E)²], a rotation-invariant energy whose Hessian at A = I is K̄_A, so it
    pairs with the same pre-factored H̄ and equals the co-rotated force of P:260-271 to first order in the strain.
    Used by the length-preserving variant of P:283-310 (Alg. 1), which has no R to co-rotate with."""
    A = np.asarray(A, dtype=np.float64)
    I = np.eye(3)
    E = 0.5 * (np.swapaxes(A, -1, -2) @ A - I)
    trE = np.trace(E, axis1=-2, axis2=-1)
    Sig = 2.0 * np.asarray(mu)[..., None, None] * E + (np.asarray(lam) * trE)[..., None, None] * I
    return np.asarray(V)[..., None] * vec(A @ Sig)


def length_preserving(M, v) -> np.ndarray:
    """Eq. len_preserving: the rotation of a 3-vector v is approximated by M v rescaled to |v|,
    (‖v‖/‖Mv‖) M v (zero stays zero). M = Aᵀ stands for Rᵀ and M = A for R (Alg. 1 lines 4-7 and 9-12)."""
    v = np.asarray(v, dtype=np.float64)
    w = np.einsum("...ij,...j->...i", M, v)
    nv = np.linalg.norm(v, axis=-1, keepdims=True)
    nw = np.linalg.norm(w, axis=-1, keepdims=True)
    return np.where(nw > 0, w * (nv / np.where(nw > 0, nw, 1.0)), 0.0)


def affine_force(q, qd, mbar, V, E, nu, g, h, rotation: str = "polar") -> np.ndarray:
    """Newton r.h.s. f_A = −∇E at qⁿ for one iteration from q⁽⁰⁾ = qⁿ.

    E(q) = (1/2h²)(q−q̂)ᵀM_A(q−q̂) + VΨ (P:193-199 projected by P:211-215), q̂ = qⁿ + hq̇ⁿ + h²M_A⁻¹f_ext,
    and f_ext = M_A[0₉; g] for gravity (the projected mass-weighted gravity field). At q = qⁿ:
    f_A = (1/h) M_A q̇ⁿ + M_A[0₉; g] − [V vec(RΠ); 0₃] (elastic term: SURVEY A3 reads P:260-271 as included).
    """
    q = np.asarray(q, dtype=np.float64)
    MA = mass_A(mbar)
    mu, lam = lame(E, nu)
    grav = np.zeros(q.shape)
    grav[..., 9:12] = g
    f = np.einsum("...ij,...j->...i", MA, np.asarray(qd) / h + grav)
    if rotation != "none":  # "none": inertia and gravity only (the polar-free variant adds its elastic term itself)
        el = elastic_force_A if rotation == "polar" else stvk_force_A
        f[..., :9] -= el(unvec(q[..., :9]), V, mu, lam)
    return f


def wrench_force(q, W) -> np.ndarray:
    """Affine force of an external spatial wrench W = [τ; f] (Eq. module1-wrench-map):
    f_A,ext = G(A)ᵀ W with the ABD-to-twist map G(A) = [½[q₁]× ½[q₂]× ½[q₃]× 0; 0 0 0 I₃], so
    the A-column c receives ½[q_c]×ᵀτ = ½ τ × q_c and the t-block receives f."""
    q = np.asarray(q, dtype=np.float64)
    W = np.asarray(W, dtype=np.float64)
    out = np.zeros(q.shape)
    tau = W[..., 0:3]
    for c in range(3):
        out[..., 3 * c:3 * c + 3] = 0.5 * np.cross(tau, q[..., 3 * c:3 * c + 3])
    out[..., 9:12] = W[..., 3:6]
    return out


def twist_velocity(q, omega, v) -> np.ndarray:
    """ABD velocity of a rigid twist (ω, v): q̇_c = ω × q_c, ṫ = v (inverse of P:655-667 on rigid motions)."""
    q = np.asarray(q, dtype=np.float64)
    qd = np.zeros(q.shape)
    for c in range(3):
        qd[..., 3 * c:3 * c + 3] = np.cross(omega, q[..., 3 * c:3 * c + 3])
    qd[..., 9:12] = v
    return qd


def angular_velocity(q, qd) -> np.ndarray:
    """ω = ½ Σ_c q_c × q̇_c."""
    q = np.asarray(q)
    qd = np.asarray(qd)
    return 0.5 * sum(np.cross(q[..., 3 * c:3 * c + 3], qd[..., 3 * c:3 * c + 3]) for c in range(3))


def body_hessians(R, Hbar) -> np.ndarray:
    """H_A^j = diag₄(R) H̄ diag₄(Rᵀ) (P:256-258 with P:243-254), as dense 12×12 per body."""
    R = np.asarray(R)
    D4 = np.zeros(R.shape[:-2] + (12, 12))
    for k in range(4):
        D4[..., 3 * k:3 * k + 3, 3 * k:3 * k + 3] = R
    return D4 @ Hbar @ np.swapaxes(D4, -1, -2)


# --------------------------------------------------------------------------
# constraints (ball = 1 point, linear hinge = 2 points: P:368)
# --------------------------------------------------------------------------

def hinge_frame(axis) -> np.ndarray:
    """ΔR_H of the five-row hinge: the rotation I + [v]× + [v]×²/(1 + a_y), v = a × e_y, that turns the unit
    axis a upright onto the local y axis (a = −e_y, where the formula is singular, takes diag(1, −1, −1))."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    if a[1] <= -1.0 + 1e-12:
        return np.diag([1.0, -1.0, -1.0])
    v = np.cross(a, [0.0, 1.0, 0.0])
    V = np.array([[0, -v[2], v[1]], [v[2], 0, -v[0]], [-v[1], v[0], 0]])
    return np.eye(3) + V + V @ V / (1.0 + a[1])


def hinge5_rows(scene, q):
    """Row transforms of the five-row hinges (Eq. hinge; R13) at the state q:
    for joint k of kind 1 (two points on the axis, the second's ȳ_a − first's ȳ_a along the axis in body a's frame)
    the first point keeps its 3 ball rows and the second keeps W = P R_H (2×3), P = [e_x; e_z], R_H = ΔR_H Rᵀ(A_a):
    the local x̃, z̃ of the CP difference (Eq. hinge), the axial row freed. Returns {point index: W}."""
    kind = getattr(scene, "kind", None)
    out = {}
    if kind is None:
        return out
    off = np.concatenate([[0], np.cumsum(scene.npts)])
    Pxz = np.array([[1.0, 0, 0], [0, 0, 1.0]])
    kind = np.asarray(kind)
    for k in np.nonzero(kind == 1)[0]:
        p0 = off[k]
        a = scene.body_a[k]
        R = polar(unvec(np.asarray(q)[a, :9]))
        dR = hinge_frame(scene.ybar_a[p0 + 1] - scene.ybar_a[p0])
        out[p0 + 1] = Pxz @ dR @ R.T
    for k in np.nonzero(kind == 2)[0]:   # universal (R17): the second point carries no point rows
        out[off[k] + 1] = np.zeros((0, 3))
    for k in np.nonzero(kind == 3)[0]:   # prismatic (R17): all its rows are general rows (joint_general_rows)
        for i in range(3):
            out[off[k] + i] = np.zeros((0, 3))
    return out


def joint_general_rows(scene):
    """The rows of the universal and prismatic joints (Eqs. universal and prismatic;
    DESIGN.md R17). Each row is a scalar C(q) in the joint frame following body a, with R ≈ A ("C̃ can be
    well approximated as a quadratic function of q̃ since R^j is relaxed to A^j"), so that its gradient (Eq.
    constraint_gradient, both terms) is exact. Two row types, (type, a, b, d, y_a, y_b):
    - 'dir':   (A_a d)·(A_b y_b) = 0, a direction of a against a direction of b (A_b = I for the world);
    - 'point': (A_a d)·(x_a(y_a) − x_b(y_b)) = 0, a component of a point pair's offset in a's frame (x_b = y_b
      for the world).
    - universal (kind 2; points: the centre, then ȳ_a[1] − ȳ_a[0] ∥ a₁ in body a, ȳ_b[1] − ȳ_b[0] ∥ a₂ in body b):
      the centre is a ball (3 point rows, not here) and one 'dir' row (â₁, e₂) — "the local y coordinates of the
      first and the second CPs of β identical";
    - prismatic (kind 3; points: two on the sliding axis, ȳ_a[1] − ȳ_a[0] ∥ â, and a third with ȳ_a[2] − ȳ_a[0] ⟂ â,
      all coincident at creation): 'point' rows x̂, ẑ of the first points' offset (x̂, ẑ = ΔR_Pᵀe_x, ΔR_Pᵀe_z: "x̃, z̃
      of ỹ₂^α − ỹ₁^β"), 'dir' rows (x̂, e), (ẑ, e) keeping the axes parallel (e = ȳ_b[1] − ȳ_b[0]: "x̃, z̃
      of ỹ₁^β − ỹ₂^β"), and the 'dir' row (n̂, u), n̂ = â × unit(ȳ_a[2] − ȳ_a[0]), u = ȳ_b[2] − ȳ_b[0], which stops
      the twist about the axis (the paper's "x̃₃^β = 0", with its reference direction from the third
      point)."""
    kind = getattr(scene, "kind", None)
    out = []
    if kind is None:
        return out
    kind = np.asarray(kind)
    off = np.concatenate([[0], np.cumsum(scene.npts)])
    for k in np.nonzero((kind == 2) | (kind == 3))[0]:
        p0, a, b = off[k], int(scene.body_a[k]), int(scene.body_b[k])
        ax = scene.ybar_a[p0 + 1] - scene.ybar_a[p0]
        ax = ax / np.linalg.norm(ax)
        e = scene.ybar_b[p0 + 1] - scene.ybar_b[p0]
        if kind[k] == 2:
            out.append(("dir", a, b, ax, None, e))
            continue
        dR = hinge_frame(ax)
        ua = scene.ybar_a[p0 + 2] - scene.ybar_a[p0]
        n = np.cross(ax, ua / np.linalg.norm(ua))
        for d in (dR[0], dR[2]):
            out.append(("point", a, b, d, scene.ybar_a[p0], scene.ybar_b[p0]))
        out.append(("dir", a, b, dR[0], None, e))
        out.append(("dir", a, b, dR[2], None, e))
        out.append(("dir", a, b, n, None, scene.ybar_b[p0 + 2] - scene.ybar_b[p0]))
    return out


def general_row(row, q):
    """Value C(q) and gradient {body: ∂C/∂q_body (12,)} of one row of joint_general_rows (∂/∂A[r, c] at index
    3c + r, the vec(A) layout)."""
    typ, a, b, d, ya, yb = row
    q = np.asarray(q)
    Aa = unvec(q[a, :9])
    w = Aa @ d
    g = {a: np.zeros(12)}
    if b >= 0:
        g[b] = np.zeros(12)
    if typ == "dir":
        Ab = unvec(q[b, :9]) if b >= 0 else np.eye(3)
        xb = Ab @ yb
        g[a][:9] = np.outer(xb, d).T.reshape(9)          # ∂/∂A_a = (A_b y_b) dᵀ
        if b >= 0:
            g[b][:9] = np.outer(w, yb).T.reshape(9)      # ∂/∂A_b = (A_a d) y_bᵀ
        return float(w @ xb), g
    xa = Aa @ ya + q[a, 9:]
    xb = (unvec(q[b, :9]) @ yb + q[b, 9:]) if b >= 0 else yb
    off = xa - xb
    g[a][:9] = (np.outer(off, d) + np.outer(w, ya)).T.reshape(9)   # rotation term + point term
    g[a][9:] = w
    if b >= 0:
        g[b][:9] = -np.outer(w, yb).T.reshape(9)
        g[b][9:] = -w
    return float(w @ off), g


def rotation_about(axis, angle) -> np.ndarray:
    """Rodrigues rotation by `angle` about the unit `axis`."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(angle) * K + (1.0 - np.cos(angle)) * K @ K


def hinge_angle(scene, q, k):
    """The five-row hinge k's angle at q (R14): the rotation of body b's reference
    direction u_b relative to body a's u_a about the world axis a_w = R_a â (R = polar(A); â = ȳ_a[1] − ȳ_a[0]),
    atan2(a_w·(u_aw × u_bw), u_aw·u_bw); u_a, u_b are scene.limits[k, 2:5], [5:8] (body frames; world for an
    anchor), equal in the world at creation, so θ = 0 there."""
    q = np.asarray(q)
    off = np.concatenate([[0], np.cumsum(scene.npts)])
    p0 = off[k]
    a, b = scene.body_a[k], scene.body_b[k]
    Ra = polar(unvec(q[a, :9]))
    ax = scene.ybar_a[p0 + 1] - scene.ybar_a[p0]
    aw = Ra @ (ax / np.linalg.norm(ax))
    ua = Ra @ scene.limits[k, 2:5]
    ub = (polar(unvec(q[b, :9])) @ scene.limits[k, 5:8]) if b >= 0 else scene.limits[k, 5:8]
    return float(np.arctan2(aw @ np.cross(ua, ub), ua @ ub))


def hinge_limit_rows(scene, q):
    """Joint limits of the five-row hinges (R14). A limit [lo, hi] violated at
    the linearisation point q (θ > hi or θ < lo) becomes, for this Newton iteration, the equality θ = θ̂ (the violated
    bound): one row t·(x_a(ȳ₃ₐ) − x_b(ȳ₃ᵦ)) = 0 between body a's point ȳ₃ₐ = ȳ_a[0] + ρ Rot(â, θ̂) u_a and body b's
    ȳ₃ᵦ = ȳ_b[0] + ρ u_b (ρ = |ȳ_a[1] − ȳ_a[0]|), t = a_w × (R_a Rot(â, θ̂) u_a) the tangent, frozen at q. Its residual
    at q, ≈ ρ sin(θ − θ̂), enters the dual r.h.s. as the footnote term: the "dual-space penalty k(θ − θ̂)"
    of P:455 with unit gain. Returns [(a, b, ȳ₃ₐ, ȳ₃ᵦ, t)] for the active limits."""
    if getattr(scene, "limits", None) is None or getattr(scene, "kind", None) is None:
        return []
    q = np.asarray(q)
    off = np.concatenate([[0], np.cumsum(scene.npts)])
    out = []
    for k in np.nonzero(np.asarray(scene.kind) == 1)[0]:
        lo, hi = scene.limits[k, 0], scene.limits[k, 1]
        if not (np.isfinite(lo) or np.isfinite(hi)):
            continue
        th = hinge_angle(scene, q, k)
        if lo <= th <= hi:
            continue
        thh = hi if th > hi else lo
        p0 = off[k]
        a, b = scene.body_a[k], scene.body_b[k]
        ax = scene.ybar_a[p0 + 1] - scene.ybar_a[p0]
        rho = np.linalg.norm(ax)
        ua_hat = rotation_about(ax, thh) @ scene.limits[k, 2:5]
        ya = scene.ybar_a[p0] + rho * ua_hat
        yb = scene.ybar_b[p0] + rho * scene.limits[k, 5:8]
        Ra = polar(unvec(q[a, :9]))
        t = np.cross(Ra @ (ax / rho), Ra @ ua_hat)
        out.append((a, b, ya, yb, t / np.linalg.norm(t)))
    return out


def constraint_system(scene, q=None):
    """Jacobian ∇C̃ (sparse) of the joint constraints and the world offsets, at the state q.

    Point joints (kind 0) are state independent: 3 rows per joint point.

    A point ȳ on body j sits at x = Aȳ + t = (ȳ_augᵀ ⊗ I₃) q_j, ȳ_aug = [ȳ; 1] (P:182, P:368 with one control
    point placed at the joint). Row block of point p: +(ȳ_a,augᵀ ⊗ I₃) on body a, −(ȳ_b,augᵀ ⊗ I₃) on body b
    (the ball constraint S_B^α T^α q^α − S_B^β T^β q^β = 0), or nothing on the world side of an anchor.
    Returns (J, world) with world[p] the fixed world point of anchors (else 0), so C(q) = J q − world.
    """
    n = scene.n
    P = int(scene.npts.sum())
    ra = np.repeat(scene.body_a, scene.npts)
    rb = np.repeat(scene.body_b, scene.npts)
    rows, cols, vals = [], [], []
    for side, bodies, ys, sgn in ((0, ra, scene.ybar_a, 1.0), (1, rb, scene.ybar_b, -1.0)):
        m = bodies >= 0
        idx = np.nonzero(m)[0]
        b = bodies[m]
        y = ys[m]
        yaug = np.concatenate([y, np.ones((len(idx), 1))], 1)    # [p,4]
        for c in range(4):
            for r in range(3):
                rows.append(3 * idx + r)
                cols.append(12 * b + 3 * c + r)
                vals.append(sgn * yaug[:, c])
    J = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(3 * P, 12 * n))
    world = np.zeros((P, 3))
    wm = rb < 0
    world[wm] = scene.ybar_b[wm]
    world = world.reshape(-1)
    W = hinge5_rows(scene, q) if getattr(scene, "kind", None) is not None else {}
    if W:  # five-row hinges: the second point's 3 rows → its 2 rows W (2×3), linearised with W frozen at q (R13);
        # universal / prismatic points: their rows W (R17), possibly none
        if q is None:
            raise ValueError("nonlinear joints: the constraint rows depend on the state q")
        blocks = []
        for p in range(P):
            blocks.append(sp.csr_matrix(W[p], shape=W[p].shape) if p in W else sp.identity(3, format="csr"))
        T = sp.block_diag(blocks, format="csr")
        J = (T @ J).tocsr()
        world = T @ world
    gen = joint_general_rows(scene)
    if gen:  # universal / prismatic rows, linearised at q with their exact gradient (R17)
        if q is None:
            raise ValueError("nonlinear joints: the constraint rows depend on the state q")
        q = np.asarray(q)
        rows, cols, vals, wext = [], [], [], []
        for i, row in enumerate(gen):
            c0, g = general_row(row, q)
            Jq = 0.0
            for body, gv in g.items():
                rows.extend([i] * 12)
                cols.extend(range(12 * body, 12 * body + 12))
                vals.extend(gv)
                Jq += gv @ q[body]
            wext.append(Jq - c0)                     # J q − w = C(q) at the linearisation point
        Jb = sp.csr_matrix((vals, (rows, cols)), shape=(len(gen), 12 * n))
        J = sp.vstack([J, Jb], format="csr")
        world = np.concatenate([world, wext])
    lim = hinge_limit_rows(scene, q) if q is not None else []
    if lim:  # active joint limits: one row each, appended (R14)
        rows, cols, vals, wext = [], [], [], []
        for i, (a, b, ya, yb, t) in enumerate(lim):
            wv = 0.0
            for body, y, sgn in ((a, ya, 1.0), (b, yb, -1.0)):
                if body < 0:
                    wv = t @ y           # world point of an anchor hinge
                    continue
                yaug = np.append(y, 1.0)
                for c in range(4):
                    for r in range(3):
                        rows.append(i)
                        cols.append(12 * body + 3 * c + r)
                        vals.append(sgn * yaug[c] * t[r])
            wext.append(wv)
        Jl = sp.csr_matrix((vals, (rows, cols)), shape=(len(lim), 12 * n))
        J = sp.vstack([J, Jl], format="csr")
        world = np.concatenate([world, wext])
    return J, world


def constraint_residual(scene, q) -> float:
    """max_k ‖C_k(q)‖∞ over all joint rows (pin P3, BASELINE north star 'residual below 1e-10'); five-row hinges
    evaluate their rows with R_H at q itself (the nonlinear constraint)."""
    J, w = constraint_system(scene, q)
    if J.shape[0] == 0:
        return 0.0
    return float(np.max(np.abs(J @ np.asarray(q).reshape(-1) - w)))


# --------------------------------------------------------------------------
# one step
# --------------------------------------------------------------------------

def predict(scene, q, qd, h, rotation: str = "polar"):
    """Per-body stages 1-2: R, f_A, H_j, and δq̃ = H_j⁻¹ f_A (Alg. 1 with exact R).

    rotation = "length_preserving" (R9): no polar decomposition. The free solve is
    Alg. 1 on the world-frame forces of f_A (inertia, gravity, wrench: Alg. 1's J̄ᵀf): each 3-block f_k
    → (‖f_k‖/‖Aᵀf_k‖)Aᵀf_k; the elastic force enters in the body frame as the StVK stress, −V Σ(E) on the A-blocks
    (the co-rotated method's −V Π, with Σ = 2μE + λ tr(E) I, E = ½(AᵀA − I): the body-frame image of
    ``stvk_force_A``); solve H̄δp = w; each δp_k → (‖δp_k‖/‖Aδp_k‖)Aδp_k. The operator that carries constraint forces
    (stages 3-5) is H̃_j⁻¹ = diag₄(A)H̄⁻¹diag₄(Aᵀ) ("A ≈ R"). Returned as (A, H̃_j δq̃, H̃_j, δq̃), so that every
    KKT route solves [H̃ ∇Cᵀ; ∇C 0][δq; λ] = [H̃δq̃; −C(qⁿ)], i.e. δq = δq̃ − H̃⁻¹∇Cᵀλ with S λ = C(q̃).
    """
    q = np.asarray(q, dtype=np.float64)
    A = unvec(q[:, :9])
    lp = rotation == "length_preserving"
    f = affine_force(q, qd, scene.mbar, scene.volume, scene.youngs, scene.poisson, scene.gravity, h,
                     "none" if lp else rotation)
    if getattr(scene, "wrench", None) is not None:  # at the linearisation point
        f = f + wrench_force(q, scene.wrench)
    Hbar = hbar_A(scene.mbar, scene.volume, scene.youngs, scene.poisson, h)
    if rotation == "polar":
        R = polar(A)
        H = body_hessians(R, Hbar)
        dq_tilde = np.linalg.solve(H, f[..., None])[..., 0]
        return R, f, H, dq_tilde
    if rotation != "length_preserving":
        raise ValueError(rotation)
    if np.any(~(np.linalg.det(A) > 1e-9)):
        raise FloatingPointError("det(A) <= 1e-9 (degenerate or inverted body)")
    At = np.swapaxes(A, -1, -2)
    fb = f.reshape(-1, 4, 3)
    w = length_preserving(At[:, None], fb).reshape(-1, 12)          # Alg. 1 lines 4-7
    mu, lam = lame(scene.youngs, scene.poisson)
    E = 0.5 * (At @ A - np.eye(3))
    Sig = 2.0 * mu[:, None, None] * E + (lam * np.trace(E, axis1=1, axis2=2))[:, None, None] * np.eye(3)
    w[:, :9] -= np.asarray(scene.volume)[:, None] * vec(Sig)       # body-frame elastic stress
    dp = np.linalg.solve(Hbar, w[..., None])[..., 0]                   # line 8
    dq_tilde = length_preserving(A[:, None], dp.reshape(-1, 4, 3)).reshape(-1, 12)   # lines 9-12
    Ai = np.linalg.inv(A)
    D4i = np.zeros(A.shape[:-2] + (12, 12))
    for k in range(4):
        D4i[..., 3 * k:3 * k + 3, 3 * k:3 * k + 3] = Ai
    H = np.swapaxes(D4i, -1, -2) @ Hbar @ D4i                         # (diag₄(A) H̄⁻¹ diag₄(Aᵀ))⁻¹
    return A, np.einsum("nij,nj->ni", H, dq_tilde), H, dq_tilde


def _natural_order(scene) -> bool:
    return scene.meta.get("topology") == "chain"


def step(scene, q, qd, h, route: str = "auto", return_info: bool = False, iters: int = 1,
         rotation: str = "polar"):
    """One implicit step: `iters` Newton iterations, each one KKT solve.

    iters = 1 (Table 1): linearised at qⁿ, qⁿ⁺¹ = qⁿ + δq, q̇ⁿ⁺¹ = δq/h (A6).
    iters = K > 1 ("# Iter."): iteration i is linearised at q⁽ⁱ⁾ with
    the incremental potential's gradient −∇E(q⁽ⁱ⁾) = M_A(q̂ − q⁽ⁱ⁾)/h² − [V vec(RΠ); 0],
    q̂ = qⁿ + hq̇ⁿ + h²[0₉; g], the constant pre-factored H̄ rotated by R(q⁽ⁱ⁾), and the constraint
    residual −C(q⁽ⁱ⁾) of the previous iterate (footnote P:459); q⁽ⁱ⁺¹⁾ = q⁽ⁱ⁾ + δq⁽ⁱ⁾, qⁿ⁺¹ = q⁽ᴷ⁾,
    q̇ⁿ⁺¹ = Σᵢ δq⁽ⁱ⁾/h. The velocity form is used for i = 0 (identical to iters = 1) and the q̂ form,
    written as (1/h)M_A v⁽ⁱ⁾ with v⁽ⁱ⁾ = (q̂ − q⁽ⁱ⁾)/h = v⁽ⁱ⁻¹⁾ − δq⁽ⁱ⁻¹⁾/h (+ h g at i = 1), for i ≥ 1.

    route: 'dense' (LAPACK dgesv on the full KKT), 'superlu' (SuperLU on the full KKT, COLAMD),
    'blocklu' (bodies first: δq̃ = H⁻¹f, S = ∇C̃H̃⁻¹∇C̃ᵀ, SuperLU on S without pivoting,
    λ = S⁻¹(∇C̃δq̃ + C(qⁿ)), δq = δq̃ − H̃⁻¹∇C̃ᵀλ), or 'auto' (SURVEY §8(c) O3 size rule).
    """
    if iters > 1:
        return _step_iterated(scene, q, qd, h, route, return_info, iters, rotation)
    q = np.asarray(q, dtype=np.float64)
    qd = np.asarray(qd, dtype=np.float64)
    n = scene.n
    R, f, H, dq_tilde = predict(scene, q, qd, h, rotation)
    J, world = constraint_system(scene, q)
    m = J.shape[0]
    c = J @ q.reshape(-1) - world                      # C̃(qⁿ), footnote P:459
    N = 12 * n + m
    if route == "auto":
        route = "dense" if N <= 6000 else ("superlu" if n <= 4096 else "blocklu")
    if m == 0:
        dq = dq_tilde.reshape(-1)
        lam = np.zeros(0)
    elif route == "dense":
        K = np.zeros((N, N))
        for j in range(n):
            K[12 * j:12 * j + 12, 12 * j:12 * j + 12] = H[j]
        Jd = J.toarray()
        K[12 * n:, :12 * n] = Jd
        K[:12 * n, 12 * n:] = Jd.T
        rhs = np.concatenate([f.reshape(-1), -c])
        sol = np.linalg.solve(K, rhs)
        dq, lam = sol[:12 * n], sol[12 * n:]
    elif route == "superlu":
        Hs = sp.bsr_matrix((H, np.arange(n), np.arange(n + 1)), shape=(12 * n, 12 * n)).tocsr()
        K = sp.bmat([[Hs, J.T], [J, None]], format="csc")
        rhs = np.concatenate([f.reshape(-1), -c])
        sol = spla.splu(K).solve(rhs)
        dq, lam = sol[:12 * n], sol[12 * n:]
    elif route == "blocklu":
        Hinv = np.linalg.inv(H)
        Hinv = 0.5 * (Hinv + np.swapaxes(Hinv, 1, 2))
        Hi = sp.bsr_matrix((Hinv, np.arange(n), np.arange(n + 1)), shape=(12 * n, 12 * n)).tocsr()
        S = (J @ Hi @ J.T).tocsc()
        r = J @ dq_tilde.reshape(-1) + c                # = C(q̃) (P:563-566 plus the footnote term)
        permc = "NATURAL" if _natural_order(scene) else "MMD_AT_PLUS_A"
        lu = spla.splu(S, permc_spec=permc, diag_pivot_thresh=0.0, options=dict(SymmetricMode=True))
        lam = lu.solve(r)
        dq = dq_tilde.reshape(-1) - Hi @ (J.T @ lam)
    else:
        raise ValueError(route)
    dq = dq.reshape(n, 12)
    q1 = q + dq
    qd1 = dq / h
    if return_info:
        return q1, qd1, {"q_tilde": q + dq_tilde, "lam": lam, "R": R, "route": route, "f": f}
    return q1, qd1


def _step_iterated(scene, q, qd, h, route, return_info, iters, rotation="polar"):
    """K Newton iterations of one step (see ``step``): iteration i solves the KKT of the linearisation at q⁽ⁱ⁾."""
    q = np.asarray(q, dtype=np.float64)
    qd = np.asarray(qd, dtype=np.float64)
    g = np.asarray(scene.gravity, dtype=np.float64)
    qi = q.copy()
    v = qd.copy()                       # v⁽⁰⁾ = q̇ⁿ with gravity explicit (the iters = 1 formula)
    zero_g = _SceneGravity(scene, np.zeros(3))
    info = None
    for i in range(iters):
        sc = scene if i == 0 else zero_g
        qn1, v1, info = step(sc, qi, v, h, route=route, return_info=True, iters=1, rotation=rotation)
        dq = qn1 - qi
        qi = qn1
        v = v - dq / h                  # v⁽ⁱ⁺¹⁾ = (q̂ − q⁽ⁱ⁺¹⁾)/h
        if i == 0:
            v[:, 9:12] += h * g         # q̂ carries h²g: v⁽¹⁾ = q̇ⁿ + h g − δq⁽⁰⁾/h
    qd1 = (qd + 0.0) - v
    qd1[:, 9:12] += h * g               # q̇ⁿ⁺¹ = (q̇ⁿ + h[0;g]) − v⁽ᴷ⁾ = Σᵢ δq⁽ⁱ⁾/h
    if return_info:
        return qi, qd1, info
    return qi, qd1


class _SceneGravity:
    """A view of a scene with another gravity vector (iterations i ≥ 1 carry gravity inside q̂)."""

    def __init__(self, scene, g):
        self._s = scene
        self.gravity = g

    def __getattr__(self, k):
        return getattr(self._s, k)


def nonlinear_residual(scene, qn, qdn, q, h, lam=None):
    """Stationarity of the implicit step's nonlinear problem at q (the limit of the Newton iterations):
    r = M_A(q − q̂)/h² + [V vec(R(q)Π(F)); 0] + ∇Cᵀλ with q̂ = qⁿ + hq̇ⁿ + h²[0₉; g] (P:193-199, P:260-271,
    P:459-475). λ is taken as the least-squares multiplier when not given. Returns (max |r| / max |M_A(q−q̂)/h²|,
    max |C(q)|)."""
    qn = np.asarray(qn, dtype=np.float64)
    q = np.asarray(q, dtype=np.float64)
    MA = mass_A(scene.mbar)
    mu, lam_ = lame(scene.youngs, scene.poisson)
    qhat = qn + h * np.asarray(qdn)
    qhat[:, 9:12] += h * h * np.asarray(scene.gravity)
    inert = np.einsum("nij,nj->ni", MA, q - qhat) / (h * h)
    gr = inert.copy()
    gr[:, :9] += elastic_force_A(unvec(q[:, :9]), scene.volume, mu, lam_)
    if getattr(scene, "wrench", None) is not None:
        gr -= wrench_force(q, scene.wrench)
    J, world = constraint_system(scene, q)
    g = gr.reshape(-1)
    if J.shape[0]:
        if lam is None:
            lam = spla.lsqr(J.T, -g, atol=1e-15, btol=1e-15, iter_lim=100000)[0]
        g = g + J.T @ lam
        cres = float(np.max(np.abs(J @ q.reshape(-1) - world)))
    else:
        cres = 0.0
    return float(np.max(np.abs(g)) / max(np.max(np.abs(inert)), 1e-300)), cres


def simulate(scene, nsteps=None, route: str = "auto", q=None, qd=None, callback=None, iters: int = 1,
             rotation: str = "polar"):
    q = scene.q0.copy() if q is None else q
    qd = scene.qd0.copy() if qd is None else qd
    for k in range(scene.nsteps if nsteps is None else nsteps):
        q, qd = step(scene, q, qd, scene.h, route=route, iters=iters, rotation=rotation)
        if callback is not None:
            callback(k, q, qd)
    return q, qd


def rel_err(x, ref) -> float:
    """Parity metric: max_{j,i} |x − ref| / max(|ref|, 1), per entry, SI units."""
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if x.size == 0:
        return 0.0
    return float(np.max(np.abs(x - ref) / np.maximum(np.abs(ref), 1.0)))


# --------------------------------------------------------------------------
# specialised CPU solvers, only for pin P7 (agreement with the brute-force KKT)
# --------------------------------------------------------------------------

def dual_matrix(scene, q, qd, h):
    """Dense dual S = ∇C̃ H̃⁻¹ ∇C̃ᵀ and r = C(q̃) (P:483 with the footnote P:459 term)."""
    R, f, H, dq_tilde = predict(scene, q, qd, h)
    J, world = constraint_system(scene, q)
    Jd = J.toarray()
    Hinv = np.zeros((12 * scene.n, 12 * scene.n))
    for j in range(scene.n):
        Hinv[12 * j:12 * j + 12, 12 * j:12 * j + 12] = np.linalg.inv(H[j])
    S = Jd @ Hinv @ Jd.T
    r = Jd @ (q.reshape(-1) + dq_tilde.reshape(-1)) - world
    return S, r, Jd, Hinv, dq_tilde


def block_thomas(D, B, b):
    """Block Thomas algorithm for the block-tridiagonal chain dual.

    Solves B_{k-1}ᵀ λ_{k-1} + D_k λ_k + B_k λ_{k+1} = b_k for k = 0..K-1 (P:570-583 layout).
    D: [K,c,c], B: [K-1,c,c], b: [K,c].
    """
    K = len(D)
    Dp = [None] * K
    bp = [None] * K
    Dp[0] = D[0].copy()
    bp[0] = b[0].copy()
    for k in range(1, K):                 # forward elimination
        L = B[k - 1].T @ np.linalg.inv(Dp[k - 1])
        Dp[k] = D[k] - L @ B[k - 1]
        bp[k] = b[k] - L @ bp[k - 1]
    lam = [None] * K
    lam[K - 1] = np.linalg.solve(Dp[K - 1], bp[K - 1])
    for k in range(K - 2, -1, -1):        # back substitution
        lam[k] = np.linalg.solve(Dp[k], bp[k] - B[k] @ lam[k + 1])
    return np.array(lam)


def leaf_to_root_solve(S, r, joint_rows, joint_child, joint_parent, depth):
    """Exact leaf-to-root elimination of the tree dual (the exact form of P:626-643).

    Block Gaussian elimination of S (dense) where, body by body from the deepest level up, all joints whose
    child side is that body's children ("child joints of b") are eliminated together; anchors count as child
    joints of their body. Returns (λ, fill) where ``fill`` is the largest |update| written outside the
    original block pattern of S (zero for a tree: its dual graph is chordal in this order).
    joint_rows[k]: row indices of joint k; joint_child[k]: child body (−1 for an anchor);
    joint_parent[k]: the body the joint hangs from; depth[b]: body depth.
    """
    S = np.array(S, dtype=np.float64)
    r = np.array(r, dtype=np.float64)
    pattern = np.abs(S) > 0
    n_b = len(depth)
    order = sorted(range(n_b), key=lambda b: -depth[b])
    kids = {b: [k for k in range(len(joint_rows)) if joint_parent[k] == b] for b in range(n_b)}
    remaining = np.ones(S.shape[0], bool)
    elim = []
    fill = 0.0
    for b in order:
        X = np.concatenate([joint_rows[k] for k in kids[b]]) if kids[b] else np.zeros(0, int)
        if len(X) == 0:
            continue
        remaining[X] = False
        Y = np.nonzero(remaining)[0]
        SXX = S[np.ix_(X, X)]
        SXY = S[np.ix_(X, Y)]
        W = np.linalg.solve(SXX, SXY)
        upd = SXY.T @ W
        fill = max(fill, float(np.max(np.abs(upd[~pattern[np.ix_(Y, Y)]]), initial=0.0)))
        S[np.ix_(Y, Y)] -= upd
        r[Y] -= SXY.T @ np.linalg.solve(SXX, r[X])
        elim.append((X, Y, SXX, SXY, r[X].copy()))
    lam = np.zeros_like(r)
    for X, Y, SXX, SXY, rX in reversed(elim):   # root-to-leaf back substitution
        lam[X] = np.linalg.solve(SXX, rX - SXY @ lam[Y])
    return lam, fill


def line_gauss_seidel(S, r, blocks, colors, sweeps, lam0=None):
    """Block Gauss-Seidel on S λ = r (the paper's Case IV, "relax … in the dual space joint by joint,
    following … pre-defined chains"): ``blocks`` are index arrays of the unknowns of each chain, ``colors`` a list of
    block-index lists relaxed in turn; each block is solved exactly against the current residual,
    λ_B += S_BB⁻¹ (r − Sλ)_B. One sweep relaxes every colour once. Plain dense algebra (test oracle of the GPU
    iteration, not of the method's exact step)."""
    S = np.asarray(S, dtype=np.float64)
    lam = np.zeros_like(np.asarray(r, dtype=np.float64)) if lam0 is None else np.array(lam0, dtype=np.float64)
    for _ in range(sweeps):
        for col in colors:
            res = r - S @ lam          # blocks of one colour are uncoupled: one residual serves all of them
            for b in col:
                idx = blocks[b]
                lam[idx] += np.linalg.solve(S[np.ix_(idx, idx)], res[idx])
    return lam


def step_with_dual(scene, q, qd, h, solve):
    """One step with a caller-supplied dual solve λ = solve(S, r): δq = δq̃ − H̃⁻¹∇C̃ᵀλ."""
    S, r, Jd, Hinv, dq_tilde = dual_matrix(scene, q, qd, h)
    lam = solve(S, r)
    dq = (dq_tilde.reshape(-1) - Hinv @ (Jd.T @ lam)).reshape(scene.n, 12)
    return np.asarray(q) + dq, dq / h


# --------------------------------------------------------------------------
# literal Alg. 2 (ABD-ABA) as printed: an approximate tree variant (R15)
# --------------------------------------------------------------------------

def twist_embedding(A) -> np.ndarray:
    """E(A) of Eq. module2-E: q̇ = E(A) V for the spatial twist V = (ω, v), E = [−[q_c]×; I₃]."""
    A = np.asarray(A, dtype=np.float64)
    E = np.zeros((12, 6))
    for c in range(3):
        qc = A[:, c]
        E[3 * c:3 * c + 3, :3] = -np.array([[0, -qc[2], qc[1]], [qc[2], 0, -qc[0]], [-qc[1], qc[0], 0]])
    E[9:, 3:] = np.eye(3)
    return E


def joint_subspace(p, t_child, axis=None) -> np.ndarray:
    """S^j: the relative twists (ω, v of the child's frame origin t) a joint at the world point p admits —
    rotations about p: v = ω × (t − p). A ball joint: S = [I₃; −[t − p]×] (m = 3); a linear hinge about the unit
    world axis a: S = [a; a × (t − p)] (m = 1)."""
    d = np.asarray(t_child, dtype=np.float64) - np.asarray(p, dtype=np.float64)
    D = np.array([[0, -d[2], d[1]], [d[2], 0, -d[0]], [-d[1], d[0], 0]])
    if axis is None:
        return np.vstack([np.eye(3), -D])
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    return np.concatenate([a, np.cross(a, d)])[:, None]


def aba_literal_step(scene, q, qd, h):
    """One step of Alg. 2 (ABD-ABA) as printed, on a tree scene (joint = (parent body_a, child body_b);
    anchors: body_b = −1). DESIGN.md R15 lists the readings: H_A^j = diag₄(R)H̄diag₄(Rᵀ) and f_A^j the exact path's
    (with the co-rotated elastic force, A3); upward, per link j (deepest first) S_abd = E(A^j)S^j,
    U = Ĥ S_abd, D = S_abdᵀU, α = D⁻¹S_abdᵀf̂, ΔH = Ĥ − UD⁻¹Uᵀ, Δf = f̂ − Uα, X = diag₄(R_relᵀ) with
    R_rel = A^pᵀA^j, Ĥ^p += XᵀΔHX, f̂^p += XᵀΔf (Eqs. module2-*); downward (root first) the local KKT of Eq.
    module3-kkt with r^j = −∇C^j_p δq^p − C^j(qⁿ) (the footnote residual, A4) over the joint to the parent and the
    body's anchors. Not the exact KKT step (A12): an approximation, compared against it in the tests."""
    q = np.asarray(q, dtype=np.float64)
    qd = np.asarray(qd, dtype=np.float64)
    n = scene.n
    R, f, H, _ = predict(scene, q, qd, h)
    A = unvec(q[:, :9])
    off = np.concatenate([[0], np.cumsum(scene.npts)])
    parent = np.full(n, -1)
    pjoint = np.full(n, -1)
    anchors = [[] for _ in range(n)]
    for k in range(scene.n_joints):
        a, b = scene.body_a[k], scene.body_b[k]
        if b < 0:
            anchors[a].append(k)
        else:
            if parent[b] >= 0:
                raise ValueError("not a tree: a body with two parents")
            parent[b], pjoint[b] = a, k
    depth = np.zeros(n, int)
    for j in range(n):
        d, x = 0, j
        while parent[x] >= 0:
            x = parent[x]
            d += 1
            if d > n:
                raise ValueError("cycle")
        depth[j] = d

    def point_rows(k, body):
        """The joint's 3·npts rows on `body` (+Γ on side a, −Γ on side b) and the world offsets."""
        rows = []
        for i in range(scene.npts[k]):
            p = off[k] + i
            side = 0 if scene.body_a[k] == body else 1
            y = (scene.ybar_a if side == 0 else scene.ybar_b)[p]
            G = np.hstack([np.kron(y[None, :], np.eye(3)), np.eye(3)])
            rows.append((1.0 if side == 0 else -1.0) * G)
        return np.vstack(rows)

    def residual(k):
        out = []
        for i in range(scene.npts[k]):
            p = off[k] + i
            xa = A[scene.body_a[k]] @ scene.ybar_a[p] + q[scene.body_a[k], 9:]
            b = scene.body_b[k]
            xb = scene.ybar_b[p] if b < 0 else A[b] @ scene.ybar_b[p] + q[b, 9:]
            out.append(xa - xb)
        return np.concatenate(out)

    Hh = H.copy()
    fh = f.copy()
    for j in sorted(range(n), key=lambda j: -depth[j]):
        p = parent[j]
        if p < 0:
            continue
        k = pjoint[j]
        x0 = A[j] @ scene.ybar_b[off[k]] + q[j, 9:]
        axis = None
        if scene.npts[k] == 2:
            axis = (A[j] @ scene.ybar_b[off[k] + 1] + q[j, 9:]) - x0
        Sabd = twist_embedding(A[j]) @ joint_subspace(x0, q[j, 9:], axis)
        U = Hh[j] @ Sabd
        D = Sabd.T @ U
        alpha = np.linalg.solve(D, Sabd.T @ fh[j])
        dH = Hh[j] - U @ np.linalg.solve(D, U.T)
        df = fh[j] - U @ alpha
        Rrel = A[p].T @ A[j]
        X = np.kron(np.eye(4), Rrel.T)
        Hh[p] += X.T @ dH @ X
        fh[p] += X.T @ df
    dq = np.zeros((n, 12))
    for j in sorted(range(n), key=lambda j: depth[j]):
        Cs, rs = [], []
        if parent[j] >= 0:
            k = pjoint[j]
            Cs.append(point_rows(k, j))
            rs.append(-point_rows(k, parent[j]) @ dq[parent[j]] - residual(k))
        for k in anchors[j]:
            Cs.append(point_rows(k, j))
            rs.append(-residual(k))
        if not Cs:
            dq[j] = np.linalg.solve(Hh[j], fh[j])
            continue
        C = np.vstack(Cs)
        m = C.shape[0]
        K = np.block([[Hh[j], C.T], [C, np.zeros((m, m))]])
        dq[j] = np.linalg.solve(K, np.concatenate([fh[j], np.concatenate(rs)]))[:12]
    return q + dq, dq / h
