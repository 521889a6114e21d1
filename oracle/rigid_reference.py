"""Physical references for the single-body validations of PAPER.md §6.1 — TEST INFRASTRUCTURE ONLY.

Only ``tests/`` may import this module (same rule as the rest of ``oracle/``). It shares nothing with the CUDA path.

The paper checks the co-rotated affine body against rigid-body physics: a spinning box's momenta
(P:872-880), a T-handle's intermediate-axis flips against an RK4 rigid-body reference at h = 1e-4, a
heavy top's precession and nutation against the same reference, and a physical pendulum released from
the horizontal against the elliptic-integral solution (Eq. elliptic). SPEC S:432-480 restates the RK4
reference ("Euler's equations + quaternion kinematics with classical RK4; quaternion renormalized").

Contents:
- ``rk4_rigid``: classical RK4 on Euler's equations I ω̇ = (I ω) × ω + τ in the body frame with quaternion
  kinematics q̇ = ½ q ⊗ (0, ω), renormalised every step; optionally about a fixed pivot under gravity (the heavy top:
  inertia about the pivot by the parallel-axis theorem, gravity torque d × Rᵀ m g).
- ``pendulum_elliptic``: θ(t) = π/2 − 2 arcsin(κ sn(K(κ) − ω_lin t, κ)), θ measured down from the
  horizontal release, κ = sin(π/4) for a horizontal release, ω_lin = √(m g d / I_pivot).
- measurement of an affine body state (q, q̇) with generalised mass M̄ = ∫ρ ỹỹᵀ, ỹ = [ȳ; 1]:
  ``affine_momenta`` (p = Ȧ̂ M̄ e₄, L = Σ_kl M̄_kl Â_k × Ȧ̂_l about the world origin, T = ½ tr(Ȧ̂ M̄ Ȧ̂ᵀ), with
  Â = [A | t]) and ``body_omega`` (ω from the skew part of Ȧ Rᵀ, R = polar(A); body frame Rᵀω).
"""
import numpy as np
from scipy.special import ellipj, ellipk

from .mabd_oracle import polar, unvec


# ----------------------------------------------------------------------------------------------- quaternions
def quat_mul(a, b):
    """Hamilton product (w, x, y, z)."""
    w1, x1, y1, z1 = a
    w2, x2, y2, z2 = b
    return np.array([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2])


def quat_to_rot(q):
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def rot_to_quat(R):
    """Shepperd's method (input construction for the reference)."""
    tr = np.trace(R)
    if tr > 0:
        s = 2.0 * np.sqrt(tr + 1.0)
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = 2.0 * np.sqrt(1.0 + R[i, i] - R[j, j] - R[k, k])
        q = np.zeros(4)
        q[0] = (R[k, j] - R[j, k]) / s
        q[1 + i] = 0.25 * s
        q[1 + j] = (R[j, i] + R[i, j]) / s
        q[1 + k] = (R[k, i] + R[i, k]) / s
    q = np.asarray(q, dtype=np.float64)
    return q / np.linalg.norm(q)


# ----------------------------------------------------------------------------------------------- RK4 reference
def rk4_rigid(I_body, R0, w0_body, h, steps, pivot_to_com=None, mass=0.0, gravity=(0.0, 0.0, 0.0), every=1):
    """RK4 rigid body (the paper's reference of P:896-897): Euler's equations in the body frame and
    quaternion kinematics, quaternion renormalised after every step.

    ``I_body``: 3×3 inertia about the centre of mass in the body frame. With ``pivot_to_com`` (body-frame vector d
    from a fixed pivot to the COM) the body rotates about the pivot: inertia I_c + m(|d|² I − d dᵀ) and gravity
    torque d × Rᵀ m g. Returns (times, R [k,3,3], ω_body [k,3]) sampled every ``every`` steps."""
    I = np.asarray(I_body, dtype=np.float64)
    g = np.asarray(gravity, dtype=np.float64)
    d = None if pivot_to_com is None else np.asarray(pivot_to_com, dtype=np.float64)
    if d is not None:
        I = I + mass * (d @ d * np.eye(3) - np.outer(d, d))
    Iinv = np.linalg.inv(I)

    def f(q, w):
        tau = np.zeros(3)
        if d is not None:
            R = quat_to_rot(q)
            tau = np.cross(d, R.T @ (mass * g))
        wd = Iinv @ (np.cross(I @ w, w) + tau)
        qd = 0.5 * quat_mul(q, np.array([0.0, *w]))
        return qd, wd

    q = rot_to_quat(np.asarray(R0, dtype=np.float64))
    w = np.asarray(w0_body, dtype=np.float64).copy()
    ts, Rs, ws = [0.0], [quat_to_rot(q)], [w.copy()]
    for s in range(1, steps + 1):
        k1q, k1w = f(q, w)
        k2q, k2w = f(q + 0.5 * h * k1q, w + 0.5 * h * k1w)
        k3q, k3w = f(q + 0.5 * h * k2q, w + 0.5 * h * k2w)
        k4q, k4w = f(q + h * k3q, w + h * k3w)
        q = q + h / 6.0 * (k1q + 2 * k2q + 2 * k3q + k4q)
        w = w + h / 6.0 * (k1w + 2 * k2w + 2 * k3w + k4w)
        q = q / np.linalg.norm(q)
        if s % every == 0:
            ts.append(s * h)
            Rs.append(quat_to_rot(q))
            ws.append(w.copy())
    return np.asarray(ts), np.asarray(Rs), np.asarray(ws)


# ----------------------------------------------------------------------------------------------- elliptic pendulum
def pendulum_elliptic(t, omega_lin, theta0=np.pi / 2):
    """P:912-916 (Eq. elliptic): θ(t) = π/2 − 2 arcsin(κ sn(K(κ) − ω_lin t, κ)) with κ = sin(θ0/2), θ0 the release
    amplitude from the vertical. For the paper's horizontal release (θ0 = π/2, κ = sin π/4) θ is measured down from
    the horizontal: θ(0) = 0, θ = π/2 at the bottom. scipy's ellipk / ellipj take the parameter m = κ²."""
    kappa = np.sin(theta0 / 2.0)
    m = kappa * kappa
    K = ellipk(m)
    sn, _, _, _ = ellipj(K - omega_lin * np.asarray(t, dtype=np.float64), m)
    return np.pi / 2 - 2.0 * np.arcsin(kappa * sn)


def pendulum_period(omega_lin, theta0=np.pi / 2):
    """Period of Eq. elliptic: 4 K(κ) / ω_lin (sn has period 4K)."""
    return 4.0 * ellipk(np.sin(theta0 / 2.0) ** 2) / omega_lin


# ----------------------------------------------------------------------------------------------- measurements
def mbar_matrix(packed):
    """Packed symmetric 4×4 M̄ (upper triangle, row-major: 00 01 02 03 11 12 13 22 23 33) → 4×4."""
    p = np.asarray(packed, dtype=np.float64)
    iu = np.triu_indices(4)
    M = np.zeros((4, 4))
    M[iu] = p
    return M + np.triu(M, 1).T


def affine_momenta(q, qd, mbar_packed):
    """Linear momentum p, angular momentum L about the world origin, kinetic energy T of one affine body
    (x(ȳ) = A ȳ + t; M̄ = ∫ρ ỹỹᵀ): with Â = [A | t], p = Ȧ̂ M̄ e₄,
    L = ∫ρ x × ẋ = Σ_kl M̄_kl Â_k × Ȧ̂_l, T = ½ tr(Ȧ̂ M̄ Ȧ̂ᵀ)."""
    M = mbar_matrix(mbar_packed)
    Ah = np.column_stack([unvec(np.asarray(q[:9])), q[9:12]])
    Ad = np.column_stack([unvec(np.asarray(qd[:9])), qd[9:12]])
    p = Ad @ M[:, 3]
    L = np.zeros(3)
    for k in range(4):
        for l in range(4):
            if M[k, l] != 0.0:
                L += M[k, l] * np.cross(Ah[:, k], Ad[:, l])
    T = 0.5 * np.trace(Ad @ M @ Ad.T)
    return p, L, T


def body_omega(q, qd):
    """Angular velocity of an affine body: R = polar(A), ω× = skew part of Ȧ Rᵀ (exact for A = R rigid,
    Ȧ = ω× R); returns (ω world, Rᵀ ω body, R)."""
    A = unvec(np.asarray(q[:9]))
    Ad = unvec(np.asarray(qd[:9]))
    R = polar(A)
    W = Ad @ R.T
    W = 0.5 * (W - W.T)
    w = np.array([W[2, 1], W[0, 2], W[1, 0]])
    return w, R.T @ w, R


def crossings(t, x):
    """Times where x changes sign (linear interpolation)."""
    t = np.asarray(t)
    x = np.asarray(x)
    i = np.nonzero(np.sign(x[:-1]) * np.sign(x[1:]) < 0)[0]
    return t[i] - x[i] * (t[i + 1] - t[i]) / (x[i + 1] - x[i])
