"""Seeded synthetic scenes with the shapes of the paper's workloads.

Inputs only: no step arithmetic lives here (see package docstring).

Conventions (shared with ``include/mabd.h``):
- q = [vec(A); t] with A stored column-major ("stacking the
  three column vectors of A and the translation vector t").
- ``mbar`` is the packed symmetric 4x4 generalized mass
  M̄ = [[∫ρ x̄x̄ᵀ, ∫ρ x̄], [∫ρ x̄ᵀ, m]] (so M_A = M̄ ⊗ I3),
  upper triangle row-major: (00,01,02,03,11,12,13,22,23,33).
- Bodies are boxes in their body-local principal frame, COM at the origin,
  rest A = I, so M̄ = diag(m a²/12, m b²/12, m c²/12, m).
- Joints are point-coincidence constraints (ball: 1 point; linear 6-row hinge:
  2 points on the axis). ``body_b = -1`` is the world; the world point is
  then stored in ``ybar_b``. Material points are taken from the initial layout,
  ȳ = (A⁰)ᵀ (p − t⁰).
- Every random draw uses ``numpy.random.default_rng([2603, cfg])`` in the order
  given in SURVEY §8(d) "Generators"; ``M_ABD_SEED`` overrides the 2603 base
  (SPEC S:559).

The five BASELINE.json configs are ``cfg1_chain8`` … ``cfg5_net``; each takes
size arguments so tests can build the same recipe at oracle-friendly sizes.
"""
from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

CONFIG_NAMES = {
    1: "chain8",
    2: "batched_chains_4096x256",
    3: "long_chain_1048576",
    4: "binary_tree_depth16",
    5: "net_512x512_loops",
}

GRAVITY = np.array([0.0, 0.0, -9.81])
NU = 0.3  # the paper's only Poisson ratio; SURVEY A9


def _seed_base() -> int:
    return int(os.environ.get("M_ABD_SEED", "2603"))


def rng_for(cfg: int) -> np.random.Generator:
    return np.random.default_rng([_seed_base(), cfg])


@dataclass
class Scene:
    name: str
    q0: np.ndarray          # [n,12] float64
    qd0: np.ndarray         # [n,12] float64
    mbar: np.ndarray        # [n,10] float64 packed sym 4x4
    volume: np.ndarray      # [n]
    youngs: np.ndarray      # [n]
    poisson: np.ndarray     # [n]
    gravity: np.ndarray     # [3]
    body_a: np.ndarray      # [K] int32
    body_b: np.ndarray      # [K] int32, -1 = world
    npts: np.ndarray        # [K] int32 in {1,2}
    ybar_a: np.ndarray      # [P,3]  P = sum(npts)
    ybar_b: np.ndarray      # [P,3]  (world point when body_b == -1)
    h: float = 1e-2
    nsteps: int = 1
    material: Optional[np.ndarray] = None   # [n] int32 or None
    meta: dict = field(default_factory=dict)
    wrench: Optional[np.ndarray] = None     # [n,6] external wrench (τ, f), world frame, constant; None = none
    kind: Optional[np.ndarray] = None       # [K] int32 joint kind: 0 point joint (default), 1 five-row hinge
    limits: Optional[np.ndarray] = None     # [K,8] five-row hinge limits: lo, hi (rad), u_a (3), u_b (3)

    @property
    def n(self) -> int:
        return int(self.q0.shape[0])

    @property
    def n_joints(self) -> int:
        return int(self.body_a.shape[0])

    @property
    def n_rows(self) -> int:
        return 3 * int(self.npts.sum())

    def copy(self) -> "Scene":
        kw = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in self.__dict__.items()
              if k in self.__dataclass_fields__}
        kw["meta"] = dict(self.meta)
        return Scene(**kw)

    def validate(self) -> None:
        n, K = self.n, self.n_joints
        assert self.q0.shape == (n, 12) and self.qd0.shape == (n, 12)
        assert self.mbar.shape == (n, 10)
        for a in (self.volume, self.youngs, self.poisson):
            assert a.shape == (n,)
        assert self.body_b.shape == (K,) and self.npts.shape == (K,)
        P = int(self.npts.sum())
        assert self.ybar_a.shape == (P, 3) and self.ybar_b.shape == (P, 3)
        assert np.all((self.body_a >= 0) & (self.body_a < n))
        assert np.all((self.body_b >= -1) & (self.body_b < n))
        assert np.all(self.body_a != self.body_b)


# --------------------------------------------------------------------------
# small geometric helpers (input construction only)
# --------------------------------------------------------------------------

def box_mbar(a, b, c, rho) -> np.ndarray:
    """Packed M̄ of a COM-centred box with sides (a,b,c) along body x,y,z."""
    a, b, c, rho = np.broadcast_arrays(*(np.asarray(x, dtype=np.float64) for x in (a, b, c, rho)))
    m = rho * a * b * c
    out = np.zeros(a.shape + (10,))
    out[..., 0] = m * a * a / 12.0
    out[..., 4] = m * b * b / 12.0
    out[..., 7] = m * c * c / 12.0
    out[..., 9] = m
    return out


def rot_x(theta):
    theta = np.asarray(theta, dtype=np.float64)
    c, s = np.cos(theta), np.sin(theta)
    R = np.zeros(theta.shape + (3, 3))
    R[..., 0, 0] = 1.0
    R[..., 1, 1] = c
    R[..., 1, 2] = -s
    R[..., 2, 1] = s
    R[..., 2, 2] = c
    return R


def random_rotations(rng: np.random.Generator, n: int) -> np.ndarray:
    """Uniform random rotations from normalised quaternions."""
    qv = rng.standard_normal((n, 4))
    qv /= np.linalg.norm(qv, axis=1, keepdims=True)
    w, x, y, z = qv.T
    R = np.empty((n, 3, 3))
    R[:, 0, 0] = 1 - 2 * (y * y + z * z)
    R[:, 0, 1] = 2 * (x * y - z * w)
    R[:, 0, 2] = 2 * (x * z + y * w)
    R[:, 1, 0] = 2 * (x * y + z * w)
    R[:, 1, 1] = 1 - 2 * (x * x + z * z)
    R[:, 1, 2] = 2 * (y * z - x * w)
    R[:, 2, 0] = 2 * (x * z - y * w)
    R[:, 2, 1] = 2 * (y * z + x * w)
    R[:, 2, 2] = 1 - 2 * (x * x + y * y)
    return R


def pack_q(A: np.ndarray, t: np.ndarray) -> np.ndarray:
    """q = [A[:,0]; A[:,1]; A[:,2]; t] (column-major vec)."""
    A = np.asarray(A)
    n = A.shape[0]
    q = np.empty((n, 12))
    q[:, 0:9] = np.transpose(A, (0, 2, 1)).reshape(n, 9)
    q[:, 9:12] = t
    return q


def _material_points(A: np.ndarray, t: np.ndarray, body: np.ndarray, p: np.ndarray) -> np.ndarray:
    """ȳ = A_bᵀ (p − t_b) for each (body, world point) pair; world rows return p."""
    out = p.copy()
    m = body >= 0
    b = body[m]
    out[m] = np.einsum("kji,kj->ki", A[b], p[m] - t[b])
    return out


def _assemble(name, A, t, qd, mbar, vol, E, nu, ja, jb, npts, pts, h, nsteps, meta=None, jitter_t=None):
    """Build a Scene from bodies (A,t) and joints given by world points ``pts`` [P,3].

    ``pts`` lists the points of every joint in joint order (npts per joint).
    """
    ja = np.asarray(ja, dtype=np.int32)
    jb = np.asarray(jb, dtype=np.int32)
    npts = np.asarray(npts, dtype=np.int32)
    rep_a = np.repeat(ja, npts)
    rep_b = np.repeat(jb, npts)
    ya = _material_points(A, t, rep_a, pts)
    yb = _material_points(A, t, rep_b, pts)
    if jitter_t is not None:
        t = t + jitter_t
    n = A.shape[0]
    sc = Scene(
        name=name,
        q0=pack_q(A, t),
        qd0=np.zeros((n, 12)) if qd is None else qd,
        mbar=mbar,
        volume=np.asarray(vol, dtype=np.float64).reshape(n),
        youngs=np.broadcast_to(np.asarray(E, dtype=np.float64), (n,)).copy(),
        poisson=np.broadcast_to(np.asarray(nu, dtype=np.float64), (n,)).copy(),
        gravity=GRAVITY.copy(),
        body_a=ja, body_b=jb, npts=npts, ybar_a=ya, ybar_b=yb,
        h=float(h), nsteps=int(nsteps), meta=dict(meta or {}),
    )
    sc.validate()
    return sc


# --------------------------------------------------------------------------
# BASELINE.json configs (SURVEY §8(d) "Generators")
# --------------------------------------------------------------------------

def cfg1_chain8(n_links: int = 8, nsteps: int = 10) -> Scene:
    """Config 1: chain of 8 unit cubes at 30° about x, top pinned, t⁰ jittered ±1e-3 (A17)."""
    rng = rng_for(1)
    A0 = rot_x(np.deg2rad(30.0))
    d = A0 @ np.array([0.0, 0.0, -1.0])
    idx = np.arange(n_links)
    t = (idx[:, None] + 0.5) * d[None, :]
    A = np.broadcast_to(A0, (n_links, 3, 3)).copy()
    mbar = box_mbar(1.0, 1.0, 1.0, 1000.0)[None, :].repeat(n_links, 0)
    vol = np.ones(n_links)
    ja = [0] + list(range(n_links - 1))
    jb = [-1] + list(range(1, n_links))
    pts = np.vstack([np.zeros((1, 3)), (idx[:-1, None] + 1.0) * d[None, :]])
    jit = rng.uniform(-1e-3, 1e-3, size=(n_links, 3))
    return _assemble("cfg1_chain8", A, t, None, mbar, vol, 1e8, NU, ja, jb, np.ones(n_links, np.int32),
                     pts, 1e-2, nsteps, meta={"cfg": 1, "topology": "chain"}, jitter_t=jit)


def cfg2_batched_chains(n_chains: int = 4096, n_links: int = 256, nsteps: int = 100) -> Scene:
    """Config 2: independent horizontal chains of 0.1×0.02×0.02 links, ρ~U[500,2000], twist θ~U[±0.2] (A18)."""
    rng = rng_for(2)
    n = n_chains * n_links
    rho = rng.uniform(500.0, 2000.0, size=n)           # chain-major
    theta = rng.uniform(-0.2, 0.2, size=n)             # drawn after all ρ
    c = np.repeat(np.arange(n_chains), n_links)
    i = np.tile(np.arange(n_links), n_chains)
    pc = np.stack([np.zeros(n_chains), 0.05 * (np.arange(n_chains) % 64), 0.05 * (np.arange(n_chains) // 64)], 1)
    t = pc[c] + np.stack([0.05 + 0.1 * i, np.zeros(n), np.zeros(n)], 1)
    A = rot_x(theta)
    mbar = box_mbar(0.1, 0.02, 0.02, rho)
    vol = np.full(n, 0.1 * 0.02 * 0.02)
    # joints, chain-major: anchor (link 0 ↔ p_c), then link i ↔ i+1 at p_c + 0.1(i+1) x̂
    K = n_chains * n_links
    ja = np.empty(K, np.int32)
    jb = np.empty(K, np.int32)
    ya = np.zeros((K, 3))
    yb = np.zeros((K, 3))
    base = np.arange(n_chains) * n_links
    first = np.arange(n_chains) * n_links  # joint index of the anchor of chain c
    ja[first] = base
    jb[first] = -1
    ya[first] = (-0.05, 0.0, 0.0)
    yb[first] = pc
    inner = (first[:, None] + 1 + np.arange(n_links - 1)[None, :]).ravel()
    bi = (base[:, None] + np.arange(n_links - 1)[None, :]).ravel()
    ja[inner] = bi
    jb[inner] = bi + 1
    ya[inner] = (0.05, 0.0, 0.0)
    yb[inner] = (-0.05, 0.0, 0.0)
    sc = Scene(
        name=f"cfg2_chains_{n_chains}x{n_links}", q0=pack_q(A, t), qd0=np.zeros((n, 12)), mbar=mbar,
        volume=vol, youngs=np.full(n, 1e8), poisson=np.full(n, NU), gravity=GRAVITY.copy(),
        body_a=ja, body_b=jb, npts=np.ones(K, np.int32), ybar_a=ya, ybar_b=yb, h=1e-2, nsteps=nsteps,
        meta={"cfg": 2, "topology": "chain", "n_chains": n_chains, "n_links": n_links},
    )
    sc.validate()
    return sc


def cfg3_long_chain(col_len: int = 5405, n_cols: int = 194, tail: int = 6, nsteps: int = 100,
                    side: float = 0.05) -> Scene:
    """Config 3: one boustrophedon chain of cubes in z=0, both ends pinned (A19).

    Full size: 194 columns × 5,405 links + 6 tail links = 1,048,576 bodies; anchors at body 0's −x face
    centre and the last body's +x face centre, 10.000 m apart. No random draws.
    """
    cols = np.repeat(np.arange(n_cols), col_len)
    k = np.tile(np.arange(col_len), n_cols)
    yi = np.where(cols % 2 == 0, k, col_len - 1 - k)
    xi = np.concatenate([cols, n_cols + np.arange(tail)])
    yi = np.concatenate([yi, np.zeros(tail, dtype=yi.dtype)]) if tail else yi
    if tail and (n_cols % 2 == 1):
        yi[-tail:] = col_len - 1  # last column ran +y: the tail continues from its top end
    n = xi.shape[0]
    t = np.stack([side * xi, side * yi, np.zeros(n)], 1).astype(np.float64)
    A = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    mbar = box_mbar(side, side, side, 1000.0)[None, :].repeat(n, 0)
    vol = np.full(n, side ** 3)
    mids = 0.5 * (t[:-1] + t[1:])
    p_first = t[0] + np.array([-side / 2, 0.0, 0.0])
    p_last = t[-1] + np.array([side / 2, 0.0, 0.0])
    ja = np.concatenate([[0], np.arange(n - 1), [n - 1]]).astype(np.int32)
    jb = np.concatenate([[-1], np.arange(1, n), [-1]]).astype(np.int32)
    pts = np.vstack([p_first[None], mids, p_last[None]])
    return _assemble(f"cfg3_chain_{n}", A, t, None, mbar, vol, 1e8, NU, ja, jb, np.ones(n + 1, np.int32),
                     pts, 1e-2, nsteps, meta={"cfg": 3, "topology": "chain"})


def cfg4_binary_tree(depth: int = 16, nsteps: int = 100, hinge_len: float = 0.05) -> Scene:
    """Config 4: complete binary tree, BFS ids, boxes U[0.05,0.2]³, ρ=1000, E=1e10, linear hinges (A20)."""
    rng = rng_for(4)
    n = 2 ** depth - 1
    dims = rng.uniform(0.05, 0.2, size=(n, 3))        # all dims first
    u = rng.standard_normal((n - 1, 3))               # then axes, child-id order
    u /= np.linalg.norm(u, axis=1, keepdims=True)
    t = np.zeros((n, 3))
    t[0] = (0.0, 0.0, -dims[0, 2] / 2)
    attach = np.zeros((n, 3))
    for j in range(1, n):                              # BFS order: parent placed before child
        p = (j - 1) // 2
        sgn = -1.0 if j % 2 == 1 else 1.0
        attach[j] = t[p] + np.array([sgn * dims[p, 0] / 4, 0.0, -dims[p, 2] / 2])
        t[j] = attach[j] - np.array([0.0, 0.0, dims[j, 2] / 2])
    A = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    mbar = box_mbar(dims[:, 0], dims[:, 1], dims[:, 2], 1000.0)
    vol = dims.prod(1)
    children = np.arange(1, n)
    parents = (children - 1) // 2
    ja = np.concatenate([[0], parents]).astype(np.int32)
    jb = np.concatenate([[-1], children]).astype(np.int32)
    npts = np.concatenate([[1], np.full(n - 1, 2)]).astype(np.int32)
    hp = np.empty((2 * (n - 1), 3))
    hp[0::2] = attach[1:]
    hp[1::2] = attach[1:] + hinge_len * u
    pts = np.vstack([np.zeros((1, 3)), hp])
    return _assemble(f"cfg4_tree_d{depth}", A, t, None, mbar, vol, 1e10, NU, ja, jb, npts, pts, 1e-2, nsteps,
                     meta={"cfg": 4, "topology": "tree"})


def cfg5_net(side: int = 512, extra_frac: float = 0.05, max_off: int = 16, nsteps: int = 50,
             cube: float = 0.02) -> Scene:
    """Config 5: side×side net of cubes, grid ball joints + 5% extra bounded-range links, corners pinned (A21).

    Body id = j*side + i for the centre (cube·i, cube·j, 0). Joint order: x-links (j-major), y-links,
    extra links, the 4 corner anchors.
    """
    rng = rng_for(5)
    S = side
    n = S * S
    ii, jj = np.meshgrid(np.arange(S), np.arange(S), indexing="xy")
    ii = ii.ravel()
    jj = jj.ravel()
    t = np.stack([cube * ii, cube * jj, np.zeros(n)], 1).astype(np.float64)
    A = np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    mbar = box_mbar(cube, cube, cube, 1000.0)[None, :].repeat(n, 0)
    vol = np.full(n, cube ** 3)
    ids = np.arange(n).reshape(S, S)                  # [j, i]
    xa = ids[:, :-1].ravel()
    xb = ids[:, 1:].ravel()
    ya_ = ids[:-1, :].ravel()
    yb_ = ids[1:, :].ravel()
    ga = np.concatenate([xa, ya_])
    gb = np.concatenate([xb, yb_])
    n_grid = ga.shape[0]
    n_extra = int(np.floor(extra_frac * n_grid))
    linked = set()
    ea, eb = [], []
    while len(ea) < n_extra:
        a = int(rng.integers(n))
        dx, dy = (int(v) for v in rng.integers(-max_off, max_off + 1, size=2))
        if max(abs(dx), abs(dy)) < 2:
            continue
        ai, aj = a % S, a // S
        bi_, bj_ = ai + dx, aj + dy
        if not (0 <= bi_ < S and 0 <= bj_ < S):
            continue
        b = bj_ * S + bi_
        key = (min(a, b), max(a, b))
        if key in linked:
            continue
        linked.add(key)
        ea.append(a)
        eb.append(b)
    ea = np.asarray(ea, dtype=np.int64)
    eb = np.asarray(eb, dtype=np.int64)
    corners = np.array([ids[0, 0], ids[0, S - 1], ids[S - 1, 0], ids[S - 1, S - 1]])
    ja = np.concatenate([ga, ea, corners]).astype(np.int32)
    jb = np.concatenate([gb, eb, -np.ones(4, np.int64)]).astype(np.int32)
    pts = np.vstack([0.5 * (t[ga] + t[gb]), 0.5 * (t[ea] + t[eb]), t[corners]])
    return _assemble(f"cfg5_net_{S}", A, t, None, mbar, vol, 1e9, NU, ja, jb, np.ones(ja.shape[0], np.int32),
                     pts, 1e-2, nsteps, meta={"cfg": 5, "topology": "net", "n_grid": n_grid, "n_extra": n_extra})


def make_scene(cfg: int, **kw) -> Scene:
    return {1: cfg1_chain8, 2: cfg2_batched_chains, 3: cfg3_long_chain, 4: cfg4_binary_tree, 5: cfg5_net}[cfg](**kw)


# --------------------------------------------------------------------------
# tiny fixtures for pins and unit tests
# --------------------------------------------------------------------------

def free_body(A0=None, t0=(0.0, 0.0, 0.0), v0=(0.0, 0.0, 0.0), Adot0=None, dims=(0.1, 0.1, 0.1),
              rho=1000.0, E=1e9, h=1e-2, gravity=True) -> Scene:
    A0 = np.eye(3) if A0 is None else np.asarray(A0, dtype=np.float64)
    q0 = pack_q(A0[None], np.asarray(t0, dtype=np.float64)[None])
    qd0 = np.zeros((1, 12))
    qd0[0, 9:12] = v0
    if Adot0 is not None:
        qd0[0, 0:9] = np.asarray(Adot0).T.reshape(9)
    sc = Scene(name="free_body", q0=q0, qd0=qd0, mbar=box_mbar(*dims, rho)[None],
               volume=np.array([np.prod(dims)]), youngs=np.array([E]), poisson=np.array([NU]),
               gravity=GRAVITY.copy() if gravity else np.zeros(3),
               body_a=np.zeros(0, np.int32), body_b=np.zeros(0, np.int32), npts=np.zeros(0, np.int32),
               ybar_a=np.zeros((0, 3)), ybar_b=np.zeros((0, 3)), h=h, nsteps=1, meta={"topology": "chain"})
    sc.validate()
    return sc


def pendulum(theta0_deg: float = 2.0, side: float = 1.0, rho: float = 1000.0, E: float = 1e8, h: float = 1e-2) -> Scene:
    """Unit cube pinned at its top-face centre (world origin), released at θ₀ about x (SURVEY pin P4)."""
    A0 = rot_x(np.deg2rad(theta0_deg))
    t0 = A0 @ np.array([0.0, 0.0, -side / 2])
    return _assemble("pendulum", A0[None], t0[None], None, box_mbar(side, side, side, rho)[None],
                     np.array([side ** 3]), E, NU, [0], [-1], [1], np.zeros((1, 3)), h, 1,
                     meta={"topology": "chain"})


def two_body_ball(seed: int = 0, h: float = 1e-2) -> Scene:
    return random_chain(2, seed=seed, anchored=False, h=h)


def random_chain(n: int, seed: int = 0, anchored: bool = True, end_anchor: bool = False, jitter: float = 0.0,
                 vel: float = 0.0, h: float = 1e-2, E: float = 1e8, gravity: bool = True, npts: int = 1,
                 reverse_some: bool = False) -> Scene:
    """Random ball-joint (npts=1) or linear-hinge (npts=2) chain with random rotations, sizes and densities.

    Joints are satisfied exactly by construction (before the optional t-jitter). ``reverse_some`` lists a
    random subset of joints with (body_a, body_b) swapped, to exercise orientation handling.
    """
    rng = np.random.default_rng([_seed_base(), 1000 + seed, n])
    R = random_rotations(rng, n)
    dims = rng.uniform(0.05, 0.2, size=(n, 3))
    rho = rng.uniform(500.0, 2000.0, size=n)
    # attachment points on each body: a "down" point and an "up" point on opposite faces
    ax = rng.integers(0, 3, size=n)
    sgn = rng.choice([-1.0, 1.0], size=n)
    up = np.zeros((n, 3))
    up[np.arange(n), ax] = sgn * dims[np.arange(n), ax] / 2
    down = -up
    t = np.zeros((n, 3))
    for i in range(1, n):
        p = t[i - 1] + R[i - 1] @ down[i - 1]
        t[i] = p - R[i] @ up[i]
    ja, jb, pts, npl = [], [], [], []
    hinge_dirs = rng.standard_normal((n + 1, 3))
    hinge_dirs /= np.linalg.norm(hinge_dirs, axis=1, keepdims=True)

    def add(a, b, p, k):
        ja.append(a)
        jb.append(b)
        pts.append(p)
        if npts == 2:
            pts.append(p + 0.05 * hinge_dirs[k])
        npl.append(npts)

    if anchored:
        add(0, -1, t[0] + R[0] @ up[0], 0)
    for i in range(n - 1):
        add(i, i + 1, t[i] + R[i] @ down[i], i + 1)
    if end_anchor:
        add(n - 1, -1, t[n - 1] + R[n - 1] @ down[n - 1], n)
    ja = np.asarray(ja, np.int32)
    jb = np.asarray(jb, np.int32)
    pts = np.asarray(pts).reshape(-1, 3)
    if reverse_some and len(ja):
        npl_a = np.asarray(npl)
        flip = (rng.random(len(ja)) < 0.5) & (jb >= 0)
        ja2, jb2 = ja.copy(), jb.copy()
        ja2[flip], jb2[flip] = jb[flip], ja[flip]
        ja, jb = ja2, jb2
        del npl_a
    qd = None
    if vel:
        qd = vel * rng.standard_normal((n, 12))
    jit = jitter * rng.uniform(-1, 1, size=(n, 3)) if jitter else None
    sc = _assemble(f"random_chain_{n}", R, t, qd, box_mbar(dims[:, 0], dims[:, 1], dims[:, 2], rho), dims.prod(1),
                   E, NU, ja, jb, npl, pts, h, 1, meta={"topology": "chain"}, jitter_t=jit)
    if not gravity:
        sc.gravity = np.zeros(3)
    return sc


def random_tree(n: int, seed: int = 0, anchored: bool = True, hinge_frac: float = 0.5, max_children: int = 3,
                jitter: float = 0.0, vel: float = 0.0, h: float = 1e-2, E: float = 1e8, gravity: bool = True,
                extra_anchors: int = 0) -> Scene:
    """Random tree (parent of body j drawn among earlier bodies with < max_children children).

    Joint j-1 links parent(j) and j; a random fraction are 6-row linear hinges (npts=2).
    """
    rng = np.random.default_rng([_seed_base(), 2000 + seed, n])
    R = random_rotations(rng, n)
    dims = rng.uniform(0.05, 0.2, size=(n, 3))
    rho = rng.uniform(500.0, 2000.0, size=n)
    parent = np.full(n, -1)
    nchild = np.zeros(n, int)
    t = np.zeros((n, 3))
    pts, ja, jb, npl = [], [], [], []
    if anchored:
        ja.append(0)
        jb.append(-1)
        pts.append(t[0] + R[0] @ (dims[0] * np.array([0, 0, 0.5])))
        npl.append(1)
    for j in range(1, n):
        cand = np.nonzero(nchild[:j] < max_children)[0]
        p = int(cand[rng.integers(len(cand))])
        parent[j] = p
        nchild[p] += 1
        lp = dims[p] * rng.uniform(-0.5, 0.5, size=3)
        lc = dims[j] * rng.uniform(-0.5, 0.5, size=3)
        P = t[p] + R[p] @ lp
        t[j] = P - R[j] @ lc
        ja.append(p)
        jb.append(j)
        pts.append(P)
        if rng.random() < hinge_frac:
            d = rng.standard_normal(3)
            pts.append(P + 0.05 * d / np.linalg.norm(d))
            npl.append(2)
        else:
            npl.append(1)
    for _ in range(extra_anchors):
        b = int(rng.integers(1, n))
        ja.append(b)
        jb.append(-1)
        pts.append(t[b] + R[b] @ (dims[b] * rng.uniform(-0.5, 0.5, size=3)))
        npl.append(1)
    qd = vel * rng.standard_normal((n, 12)) if vel else None
    jit = jitter * rng.uniform(-1, 1, size=(n, 3)) if jitter else None
    sc = _assemble(f"random_tree_{n}", R, t, qd, box_mbar(dims[:, 0], dims[:, 1], dims[:, 2], rho), dims.prod(1),
                   E, NU, ja, jb, npl, np.asarray(pts), h, 1, meta={"topology": "tree", "parent": parent},
                   jitter_t=jit)
    if not gravity:
        sc.gravity = np.zeros(3)
    return sc


def small_net(side: int = 8, extra_frac: float = 0.05, max_off: int = 4, nsteps: int = 1) -> Scene:
    """cfg-5 recipe at a small side length (corner pins, grid + bounded-range extra links)."""
    return cfg5_net(side=side, extra_frac=extra_frac, max_off=max_off, nsteps=nsteps)


def ring(n: int = 4, seed: int = 0, vel: float = 0.3, h: float = 1e-2) -> Scene:
    """A closed loop of n random boxes ("ring of 4"): a random chain plus one joint closing it."""
    sc = random_chain(n, seed=seed, anchored=False, vel=vel, h=h, gravity=True)
    A = np.swapaxes(sc.q0[:, :9].reshape(n, 3, 3), 1, 2)
    t = sc.q0[:, 9:]
    p = 0.5 * (t[0] + t[n - 1])
    ya = A[n - 1].T @ (p - t[n - 1])
    yb = A[0].T @ (p - t[0])
    sc.body_a = np.append(sc.body_a, np.int32(n - 1)).astype(np.int32)
    sc.body_b = np.append(sc.body_b, np.int32(0)).astype(np.int32)
    sc.npts = np.append(sc.npts, np.int32(1)).astype(np.int32)
    sc.ybar_a = np.vstack([sc.ybar_a, ya[None]])
    sc.ybar_b = np.vstack([sc.ybar_b, yb[None]])
    sc.name = f"ring_{n}"
    sc.meta = {"topology": "net"}
    sc.validate()
    return sc


def drop_anchors(sc: Scene) -> Scene:
    """The same scene without its world anchors (joints with body_b = −1): input construction only."""
    keep = sc.body_b >= 0
    pk = np.repeat(keep, sc.npts)
    out = sc.copy()
    out.body_a, out.body_b, out.npts = sc.body_a[keep], sc.body_b[keep], sc.npts[keep]
    out.ybar_a, out.ybar_b = sc.ybar_a[pk], sc.ybar_b[pk]
    out.name = sc.name + "_free"
    out.validate()
    return out


def _stretch_matrix(rng, stretch):
    """Q·S with Q a uniform random rotation and S = U diag(exp(τu)) Uᵀ, Σu = 0 (det = 1), ‖S − I‖_F = stretch."""
    Q = random_rotations(rng, 1)[0]
    U = random_rotations(rng, 1)[0]
    u = rng.standard_normal(3)
    u -= u.mean()
    u /= np.linalg.norm(u)
    lo, hi = 0.0, 1.0
    while np.linalg.norm(np.exp(hi * u) - 1.0) < stretch:
        hi *= 2
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if np.linalg.norm(np.exp(mid * u) - 1.0) < stretch:
            lo = mid
        else:
            hi = mid
    return Q @ U @ np.diag(np.exp(0.5 * (lo + hi) * u)) @ U.T


def affine_strained_state(q: np.ndarray, stretch: float, seed: int = 0, rate: float = 0.3):
    """A seeded strained state that keeps every joint satisfied (input construction only): the whole scene is
    mapped by one affine map x ↦ G x with G = Q·S (``_stretch_matrix``), so A_j ← G A_j, t_j ← G t_j, and every
    body's affine strain is ‖AᵀA − I‖ = ‖S² − I‖ (for a rigid A_j). The velocity is that of the affine motion
    x ↦ Ġ x with Ġ = rate·(random normal 3×3): q̇_j = [Ġ A_j; Ġ t_j], so ∇C q̇ = 0 for every joint between bodies.
    World anchors are not mapped: use it on scenes without anchors (``drop_anchors``)."""
    rng = np.random.default_rng([_seed_base(), 9000, seed])
    G = _stretch_matrix(rng, stretch)
    Gd = rate * rng.standard_normal((3, 3))
    q = np.asarray(q, dtype=np.float64)
    n = q.shape[0]
    A = np.swapaxes(q[:, :9].reshape(n, 3, 3), 1, 2)
    t = q[:, 9:12]
    q1 = pack_q(G @ A, t @ G.T)
    qd = pack_q(Gd @ A, t @ Gd.T)
    return q1, qd



def duplicate_joint(sc: Scene, k: int) -> Scene:
    """The same scene with joint k appended once more (a redundant joint set): input construction."""
    off = np.concatenate([[0], np.cumsum(sc.npts)])
    out = sc.copy()
    out.body_a = np.append(sc.body_a, sc.body_a[k]).astype(np.int32)
    out.body_b = np.append(sc.body_b, sc.body_b[k]).astype(np.int32)
    out.npts = np.append(sc.npts, sc.npts[k]).astype(np.int32)
    out.ybar_a = np.vstack([sc.ybar_a, sc.ybar_a[off[k]:off[k + 1]]])
    out.ybar_b = np.vstack([sc.ybar_b, sc.ybar_b[off[k]:off[k + 1]]])
    out.name = f"{sc.name}_dup{k}"
    out.validate()
    return out


def reframe_scene(sc: Scene, seed: int = 0, rotate: bool = True, offset: float = 0.3) -> Scene:
    """The same physical scene with every body expressed in a seeded general material frame (input construction
    only): x̄_u = P x̄ + d with P a uniform random rotation (if ``rotate``) and d uniform in ±``offset`` × the body's
    half-extent (from M̄). Then A_u = A Pᵀ, t_u = t − A Pᵀ d (velocities alike), ȳ_u = P ȳ + d, and
    M̄_u = T̄ M̄ T̄ᵀ with T̄ = [[P, d], [0, 1]], which is a full SPD 4×4 (non-central, non-principal).
    Returns the new scene; ``frames`` attribute = (P, d) per body for mapping states back."""
    rng = np.random.default_rng([_seed_base(), 9100, seed])
    n = sc.n
    P = random_rotations(rng, n) if rotate else np.broadcast_to(np.eye(3), (n, 3, 3)).copy()
    Mb = np.zeros((n, 4, 4))
    iu = [(0, 0), (0, 1), (0, 2), (0, 3), (1, 1), (1, 2), (1, 3), (2, 2), (2, 3), (3, 3)]
    for k, (i, j) in enumerate(iu):
        Mb[:, i, j] = Mb[:, j, i] = sc.mbar[:, k]
    half = np.sqrt(3.0 * np.maximum(np.diagonal(Mb, axis1=1, axis2=2)[:, :3], 0) / Mb[:, 3:4, 3])  # box: a/2
    d = offset * half * rng.uniform(-1, 1, size=(n, 3))
    T = np.zeros((n, 4, 4))
    T[:, :3, :3] = P
    T[:, :3, 3] = d
    T[:, 3, 3] = 1.0
    Mu = T @ Mb @ np.swapaxes(T, 1, 2)
    out = sc.copy()
    out.mbar = np.stack([Mu[:, i, j] for (i, j) in iu], axis=1)

    def to_user(q):
        A = np.swapaxes(q[:, :9].reshape(n, 3, 3), 1, 2)
        Au = A @ np.swapaxes(P, 1, 2)
        return pack_q(Au, q[:, 9:12] - np.einsum("nij,nj->ni", Au, d))

    out.q0 = to_user(sc.q0)
    out.qd0 = to_user(sc.qd0)
    pa = np.repeat(sc.body_a, sc.npts)
    pb = np.repeat(sc.body_b, sc.npts)
    out.ybar_a = np.einsum("pij,pj->pi", P[pa], sc.ybar_a) + d[pa]
    yb = sc.ybar_b.copy()
    m = pb >= 0
    yb[m] = np.einsum("pij,pj->pi", P[pb[m]], sc.ybar_b[m]) + d[pb[m]]
    out.ybar_b = yb
    out.name = sc.name + "_reframed"
    out.frames = (P, d)
    out.validate()
    return out


def frame_to_canonical(q: np.ndarray, frames) -> np.ndarray:
    """Map a state of ``reframe_scene``'s bodies back to the original frames: A = A_u P, t = t_u + A_u d."""
    P, d = frames
    n = q.shape[0]
    Au = np.swapaxes(q[:, :9].reshape(n, 3, 3), 1, 2)
    return pack_q(Au @ P, q[:, 9:12] + np.einsum("nij,nj->ni", Au, d))


def add_ball_joint(sc: Scene, a: int, b: int, name: str = None) -> Scene:
    """The scene plus one ball joint between bodies a and b at the midpoint of their centres (input construction;
    with a and b already connected it closes a loop)."""
    n = sc.n
    A = np.swapaxes(sc.q0[:, :9].reshape(n, 3, 3), 1, 2)
    t = sc.q0[:, 9:]
    p = 0.5 * (t[a] + t[b])
    out = sc.copy()
    out.body_a = np.append(sc.body_a, np.int32(a)).astype(np.int32)
    out.body_b = np.append(sc.body_b, np.int32(b)).astype(np.int32)
    out.npts = np.append(sc.npts, np.int32(1)).astype(np.int32)
    out.ybar_a = np.vstack([sc.ybar_a, (A[a].T @ (p - t[a]))[None]])
    out.ybar_b = np.vstack([sc.ybar_b, (A[b].T @ (p - t[b]))[None]])
    out.name = name or f"{sc.name}_loop{a}_{b}"
    out.meta = dict(sc.meta, topology="net")
    out.validate()
    return out


def five_row_hinges(sc: Scene) -> Scene:
    """The same scene with every two-point (linear, 6-row) hinge turned into a five-row hinge (kind 1):
    same material points — the first on the pivot, the second along the axis — with the axial row of the second
    point freed. Input construction only."""
    out = sc.copy()
    out.kind = (np.asarray(sc.npts) == 2).astype(np.int32)
    out.name = sc.name + "_hinge5"
    return out


def nonlinear_joints(sc: Scene, seed: int = 0, universal: float = 0.5, prismatic: float = 0.5,
                     hinge5: float = 0.0) -> Scene:
    """The same scene with its two-point (linear) hinges turned, at random, into universal joints (kind 2), prismatic
    joints (kind 3) or five-row hinges (kind 1) (R13, R17). A universal joint keeps the pivot
    point and body a's axis point; body b's second point moves to a direction ⟂ the axis in b's frame (a₂ ⟂ a₁). A
    prismatic joint keeps both axis points and gains a third point ⟂ the axis, at the same world position on both
    bodies (computed from q0). Fractions are of the two-point joints; the rest stay linear hinges. Input
    construction only."""
    rng = np.random.default_rng([_seed_base(), 7000 + seed])
    npts = np.asarray(sc.npts)
    off = np.concatenate([[0], np.cumsum(npts)])
    kind = np.zeros(sc.n_joints, np.int32) if sc.kind is None else np.asarray(sc.kind, np.int32).copy()
    ya, yb, nn = [], [], []
    for k in range(sc.n_joints):
        pa, pb = sc.ybar_a[off[k]:off[k + 1]].copy(), sc.ybar_b[off[k]:off[k + 1]].copy()
        if npts[k] == 2 and kind[k] == 0:
            u = rng.random()
            ax_b = pb[1] - pb[0]
            rho = np.linalg.norm(pa[1] - pa[0])
            if u < universal:
                kind[k] = 2
                v = rng.standard_normal(3)
                v -= ax_b * (v @ ax_b) / (ax_b @ ax_b)
                pb[1] = pb[0] + rho * v / np.linalg.norm(v)
            elif u < universal + prismatic:
                kind[k] = 3
                a, b = sc.body_a[k], sc.body_b[k]
                ax_a = pa[1] - pa[0]
                v = rng.standard_normal(3)
                v -= ax_a * (v @ ax_a) / (ax_a @ ax_a)
                y2a = pa[0] + rho * v / np.linalg.norm(v)
                Aa = sc.q0[a, :9].reshape(3, 3).T
                x = Aa @ y2a + sc.q0[a, 9:]
                if b >= 0:
                    Ab = sc.q0[b, :9].reshape(3, 3).T
                    y2b = np.linalg.solve(Ab, x - sc.q0[b, 9:])
                else:
                    y2b = x
                pa = np.vstack([pa, y2a])
                pb = np.vstack([pb, y2b])
            elif u < universal + prismatic + hinge5:
                kind[k] = 1
        ya.append(pa)
        yb.append(pb)
        nn.append(len(pa))
    out = sc.copy()
    out.kind = kind
    out.npts = np.asarray(nn, np.int32)
    out.ybar_a = np.vstack(ya) if ya else np.zeros((0, 3))
    out.ybar_b = np.vstack(yb) if yb else np.zeros((0, 3))
    out.name = sc.name + "_nonlinear"
    out.validate()
    return out


def universal_pendulum(omega0=(0.0, 0.0, 0.0), length: float = 0.4, h: float = 1e-2, E: float = 1e8) -> Scene:
    """A 0.04×0.04×0.4 m rod (ρ = 1000) hanging from the world by a universal joint at its top end:
    axis a₁ = the rod's body x, axis a₂ = the world y, so the rod swings about x and y and cannot turn about its
    long axis (a₁ × a₂ = z). Released with angular velocity omega0 about its centre of mass."""
    a, b = 0.04, length
    t0 = np.array([[0.0, 0.0, -b / 2]])
    om = np.asarray(omega0, dtype=np.float64)
    qd = np.zeros((1, 12))
    for c in range(3):
        qd[0, 3 * c:3 * c + 3] = np.cross(om, np.eye(3)[:, c])
    sc = _assemble("universal_pendulum", np.eye(3)[None], t0, qd, box_mbar(a, a, b, 1000.0)[None],
                   np.array([a * a * b]), E, NU, np.array([0], np.int32), np.array([-1], np.int32),
                   np.array([2], np.int32), np.array([[0.0, 0.0, 0.0], [0.05, 0.0, 0.0]]), h, 1,
                   meta={"topology": "tree"})
    sc.ybar_b[1] = [0.0, 0.05, 0.0]          # a₂ = world y (the rod's a₁ = x stays at ȳ_a[1] − ȳ_a[0])
    sc.kind = np.array([2], np.int32)
    return sc


def prismatic_rail(tilt_deg: float = 30.0, h: float = 1e-2, E: float = 1e8) -> Scene:
    """A 0.1×0.05×0.05 m slider (ρ = 1000) on a frictionless world rail tilted by tilt_deg from the horizontal
    (P:427-444): a prismatic joint whose axis is the slider's body x, mapped onto the rail direction; under gravity
    it slides down the rail with acceleration g sin(tilt) and does not turn."""
    th = np.deg2rad(tilt_deg)
    c, s_ = np.cos(th), np.sin(th)
    A0 = np.array([[c, 0.0, -s_], [0.0, 1.0, 0.0], [s_, 0.0, c]])   # body x → (cos, 0, sin)
    pts = np.array([[0.0, 0.0, 0.0], A0 @ [0.05, 0.0, 0.0], A0 @ [0.0, 0.05, 0.0]])
    sc = _assemble("prismatic_rail", A0[None], np.zeros((1, 3)), None, box_mbar(0.1, 0.05, 0.05, 1000.0)[None],
                   np.array([0.1 * 0.05 * 0.05]), E, NU, np.array([0], np.int32), np.array([-1], np.int32),
                   np.array([3], np.int32), pts, h, 1, meta={"topology": "tree", "rail": A0[:, 0]})
    sc.kind = np.array([3], np.int32)
    return sc


def hinge_pendulum(axis=(1.0, 0.0, 0.0), omega0=(0.0, 0.0, 0.0), length: float = 0.4, h: float = 1e-2,
                   E: float = 1e8) -> Scene:
    """A 0.4×0.04×0.04 m rod (ρ = 1000) hanging from a world hinge at its top end (two world points on the axis,
    0.05 m apart), released with angular velocity omega0 about its centre of mass. Input construction only."""
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis)
    a, b = 0.04, length
    A0 = np.eye(3)
    # rod along z, top end at the origin
    dims = (a, a, b)
    t0 = np.array([[0.0, 0.0, -b / 2]])
    om = np.asarray(omega0, dtype=np.float64)
    qd = np.zeros((1, 12))
    for c in range(3):
        qd[0, 3 * c:3 * c + 3] = np.cross(om, A0[:, c])
    qd[0, 9:12] = np.cross(om, t0[0] - t0[0])  # spin about the centre of mass
    pts = np.array([[0.0, 0.0, 0.0], 0.05 * axis])
    sc = _assemble("hinge_pendulum", A0[None], t0, qd, box_mbar(*dims, 1000.0)[None], np.array([np.prod(dims)]), E, NU,
                   np.array([0], np.int32), np.array([-1], np.int32), np.array([2], np.int32), pts, h, 1,
                   meta={"topology": "tree"})
    return sc


def hinge_limits(sc: Scene, lo: float, hi: float) -> Scene:
    """Limits [lo, hi] (rad, from the creation configuration) on every five-row hinge (input construction): the
    reference directions are a unit vector ⟂ the axis in body a's frame and the same world direction expressed in
    body b's frame (the world frame for an anchor), so the hinge angle is 0 at creation."""
    out = sc.copy()
    K = sc.n_joints
    L = np.full((K, 8), np.nan)
    off = np.concatenate([[0], np.cumsum(sc.npts)])
    for k in range(K):
        if sc.kind is None or sc.kind[k] != 1:
            continue
        p0 = off[k]
        ax = sc.ybar_a[p0 + 1] - sc.ybar_a[p0]
        ax = ax / np.linalg.norm(ax)
        e = np.eye(3)[np.argmin(np.abs(ax))]
        ua = np.cross(ax, e)
        ua /= np.linalg.norm(ua)
        a, b = sc.body_a[k], sc.body_b[k]
        Aa = np.swapaxes(sc.q0[a, :9].reshape(3, 3), 0, 1)
        Ua, _, Vta = np.linalg.svd(Aa)
        uw = (Ua @ Vta) @ ua
        if b >= 0:
            Ab = np.swapaxes(sc.q0[b, :9].reshape(3, 3), 0, 1)
            Ub, _, Vtb = np.linalg.svd(Ab)
            ub = (Ub @ Vtb).T @ uw
        else:
            ub = uw
        L[k] = [lo, hi, *ua, *ub]
    out.limits = L
    out.name = sc.name + f"_lim{lo:g}_{hi:g}"
    return out

# --------------------------------------------------------------------------
# §6.1 single-body validations
# --------------------------------------------------------------------------

def mbar_from_inertia(I_principal, mass) -> np.ndarray:
    """Packed central principal M̄ = diag(a0, a1, a2, m) with I_x = a1 + a2, I_y = a0 + a2, I_z = a0 + a1."""
    I1, I2, I3 = (float(x) for x in I_principal)
    out = np.zeros(10)
    out[0] = 0.5 * (I2 + I3 - I1)
    out[4] = 0.5 * (I1 + I3 - I2)
    out[7] = 0.5 * (I1 + I2 - I3)
    out[9] = float(mass)
    assert min(out[0], out[4], out[7]) > 0.0, "inertia violates the triangle inequality"
    return out


def twist_velocity(A: np.ndarray, t: np.ndarray, omega, v_origin) -> np.ndarray:
    """ABD generalised velocity of a rigid twist (Eq. module1-G-twist): Ȧ = ω× A, ṫ = v of the frame
    origin (world frame ω and v)."""
    om = np.asarray(omega, dtype=np.float64)
    qd = np.zeros(12)
    for c in range(3):
        qd[3 * c:3 * c + 3] = np.cross(om, A[:, c])
    qd[9:12] = v_origin
    return qd


def _single_body(name, A0, t0, qd0, mbar, volume, E, h, gravity, ja=(), jb=(), npts=(), ya=None, yb=None, meta=None):
    sc = Scene(name=name, q0=pack_q(np.asarray(A0)[None], np.asarray(t0, dtype=np.float64)[None]),
               qd0=np.asarray(qd0, dtype=np.float64)[None].copy(), mbar=np.asarray(mbar)[None].copy(),
               volume=np.array([float(volume)]), youngs=np.array([float(E)]), poisson=np.array([NU]),
               gravity=np.asarray(gravity, dtype=np.float64).copy(),
               body_a=np.asarray(ja, np.int32), body_b=np.asarray(jb, np.int32), npts=np.asarray(npts, np.int32),
               ybar_a=np.zeros((0, 3)) if ya is None else np.asarray(ya, dtype=np.float64),
               ybar_b=np.zeros((0, 3)) if yb is None else np.asarray(yb, dtype=np.float64),
               h=float(h), nsteps=1, meta=dict(meta or {"topology": "chain"}))
    sc.validate()
    return sc


def spinning_box(h: float = 1e-3, p0=(100.0, 0.0, 0.0), L0=(0.0, 100.0, 0.0)) -> Scene:
    """a 0.1 m cube (ρ = 1e3, E = 1e9, ν = 0.3) on a frictionless surface (no gravity acts in the
    plane: gravity off) with initial momenta p₀ and L₀; the twist (ω = I⁻¹L₀, v = p₀/m) is mapped to q̇."""
    s, rho = 0.1, 1000.0
    mbar = box_mbar(s, s, s, rho)
    m = mbar[9]
    I = mbar[4] + mbar[7]  # cube: isotropic
    qd = twist_velocity(np.eye(3), np.zeros(3), np.asarray(L0) / I, np.asarray(p0) / m)
    return _single_body("spinning_box", np.eye(3), np.zeros(3), qd, mbar, s ** 3, 1e9, h, np.zeros(3))


def t_handle(h: float = 1e-3, omega0: float = 3.0, perturb: float = 1e-3, E: float = 1e9) -> Scene:
    """a T-handle in zero gravity spun at ω₀ = 3 rad/s about its intermediate principal axis
    with a small perturbation on the other axes (1e-3). The handle: a 0.2 m bar (0.02² section) along x
    joined at its middle to a 0.1 m stem along z, ρ = 1e3; M̄ is the pair's central principal second moment
    (computed here, principal axes = body axes by symmetry, the frame origin at the COM)."""
    rho = 1000.0
    bar, stem = (0.2, 0.02, 0.02), (0.02, 0.02, 0.1)
    mb, ms = rho * np.prod(bar), rho * np.prod(stem)
    cb, cs = np.array([0.0, 0.0, 0.0]), np.array([0.0, 0.0, -0.06])   # stem hangs below the bar
    c = (mb * cb + ms * cs) / (mb + ms)
    S = np.zeros((3, 3))
    for (dims, mm, cc) in ((bar, mb, cb), (stem, ms, cs)):
        S += np.diag([mm * d * d / 12.0 for d in dims]) + mm * np.outer(cc - c, cc - c)
    mbar = np.zeros(10)
    mbar[0], mbar[4], mbar[7], mbar[9] = S[0, 0], S[1, 1], S[2, 2], mb + ms
    I = np.array([S[1, 1] + S[2, 2], S[0, 0] + S[2, 2], S[0, 0] + S[1, 1]])
    mid = int(np.argsort(I)[1])   # the intermediate principal axis (body z for this handle)
    w = np.full(3, perturb)
    w[mid] = 1.0
    w = w * omega0
    qd = twist_velocity(np.eye(3), np.zeros(3), w, np.zeros(3))
    vol = np.prod(bar) + np.prod(stem)
    return _single_body("t_handle", np.eye(3), np.zeros(3), qd, mbar, vol, E, h, np.zeros(3),
                        meta={"topology": "chain", "inertia": I, "mid_axis": mid, "omega0_body": w})


def heavy_top(h: float = 1e-3, spin: float = 10.0, tilt_deg: float = 5.0, E: float = 1e9) -> Scene:
    """a heavy top on a fixed pivot under gravity, spun at 10 rad/s about its symmetry axis, tilted 5°.
    The top: a 0.2 m wide, 0.02 m thick square plate (ρ = 1e3, symmetric: I₁ = I₂) whose COM sits 0.01 m above the
    pivot on the symmetry axis (body z), so 10 rad/s makes it a fast top (I₃²ω² > 4 I₁ m g d: it precesses and
    nutates instead of falling); the pivot is a world anchor (ball joint) at the body point ȳ = (0, 0, −0.01)."""
    rho, a, c, d = 1000.0, 0.2, 0.02, 0.01
    mbar = box_mbar(a, a, c, rho)
    R0 = rot_x(np.deg2rad(tilt_deg))
    t0 = R0 @ np.array([0.0, 0.0, d])                  # pivot at the world origin
    qd = twist_velocity(R0, t0, spin * R0[:, 2], np.zeros(3))   # spin about the axis through the pivot: ṫ = 0
    return _single_body("heavy_top", R0, t0, qd, mbar, a * a * c, E, h, GRAVITY, ja=[0], jb=[-1], npts=[1],
                        ya=[[0.0, 0.0, -d]], yb=[[0.0, 0.0, 0.0]], meta={"topology": "chain", "pivot_to_com": d})


def pendulum_horizontal(h: float = 1e-3, length: float = 0.4, E: float = 1e9) -> Scene:
    """a physical pendulum (a 0.4×0.04×0.04 m rod, ρ = 1e3) on a fixed pivot at one end, released at rest
    from the horizontal (rod along +x, pivot = world origin, a ball-joint anchor) under gravity."""
    a = 0.04
    mbar = box_mbar(length, a, a, 1000.0)
    t0 = np.array([length / 2, 0.0, 0.0])
    return _single_body("pendulum_horizontal", np.eye(3), t0, np.zeros(12), mbar, length * a * a, E, h, GRAVITY,
                        ja=[0], jb=[-1], npts=[1], ya=[[-length / 2, 0.0, 0.0]], yb=[[0.0, 0.0, 0.0]],
                        meta={"topology": "chain", "length": length})
