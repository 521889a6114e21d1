"""CPU-side checks of the C ABI (no GPU work): the library loads, exports every symbol of include/mabd.h,
and its host analysis (validation, topology, workspace sizing) behaves as documented."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from mabd_scenes import generators as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_08079_b200 import build
    build.build()
    from paper_2603_08079_b200 import binding
    return binding.load_library()


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "mabd.h")).read()
    return sorted(set(re.findall(r"\b(mabd_[a-z_]+)\s*\(", txt)))


def test_exports_every_header_symbol(lib):
    syms = _header_symbols()
    assert "mabd_create" in syms and "mabd_step" in syms and "mabd_get_state" in syms
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (mabd_\w+)", out))
    for s in syms:
        assert s in exported, s
        assert hasattr(lib, s)


def _ws(lib, sc, solver=0, iters=1):
    from paper_2603_08079_b200.binding import _Bodies, _Joints, _Options, _ptr, _ip
    b = _Bodies(sc.n, _ptr(sc.q0), _ptr(sc.qd0), _ptr(sc.mbar), _ptr(sc.volume), _ptr(sc.youngs), _ptr(sc.poisson),
                None, (ctypes.c_double * 3)(*sc.gravity))
    kind = None if sc.kind is None else np.ascontiguousarray(sc.kind, dtype=np.int32)
    j = _Joints(sc.n_joints, _ptr(sc.body_a, _ip), _ptr(sc.body_b, _ip), _ptr(sc.npts, _ip), _ptr(sc.ybar_a),
                _ptr(sc.ybar_b), None if kind is None else _ptr(kind, _ip))
    o = _Options(iters, 1, solver, 0, 1, None, None, 0, None, 0)
    n = ctypes.c_size_t()
    st = lib.mabd_workspace_size(ctypes.byref(b), ctypes.byref(j), ctypes.byref(o), ctypes.byref(n))
    return st, n.value, lib.mabd_last_error(None).decode()


def test_workspace_size_chains(lib):
    st, nb, _ = _ws(lib, G.cfg1_chain8())
    assert st == 0 and nb > 0
    sc = G.cfg2_batched_chains(16, 256)
    st, nb, _ = _ws(lib, sc)
    assert st == 0
    assert nb >= 2 * 12 * 8 * sc.n     # at least q, q̇ in fp64


def test_validation_errors(lib):
    sc = G.random_chain(4, seed=1)
    bad = sc.copy()
    bad.body_b[1] = bad.body_a[1]                      # joint on one body
    assert _ws(lib, bad)[0] == 1
    bad = sc.copy()
    bad.body_a[0] = 99                                 # out of range
    assert _ws(lib, bad)[0] == 1
    bad = sc.copy()
    bad.npts[0] = 3
    bad.ybar_a = np.vstack([bad.ybar_a, np.zeros((2, 3))])
    bad.ybar_b = np.vstack([bad.ybar_b, np.zeros((2, 3))])
    assert _ws(lib, bad)[0] == 1
    ok = sc.copy()
    ok.mbar[0, 1] = 0.01 * ok.mbar[0, 0]               # a general SPD M̄ is accepted (canonical frame, DESIGN R8)
    assert _ws(lib, ok)[0] == 0
    bad = sc.copy()
    bad.mbar[0, 3] = 2.0 * np.sqrt(bad.mbar[0, 0] * bad.mbar[0, 9])   # indefinite M̄
    st, _, msg = _ws(lib, bad)
    assert st == 1 and "positive definite" in msg
    bad = sc.copy()
    bad.poisson[2] = 0.5
    assert _ws(lib, bad)[0] == 1


def test_chain_solver_rejects_cycles(lib):
    sc = G.small_net(4, max_off=2)
    st, _, msg = _ws(lib, sc, solver=1)
    assert st == 1 and "chain" in msg


def test_newton_iterations_option(lib):
    """newton_iters: 0 and 1 are one iteration, 2..16 allocate the extra velocity buffer, others are invalid."""
    sc = G.random_chain(40, seed=1)
    st1, nb1, _ = _ws(lib, sc, iters=1)
    st0, nb0, _ = _ws(lib, sc, iters=0)
    st3, nb3, _ = _ws(lib, sc, iters=3)
    assert st1 == st0 == st3 == 0
    assert nb0 == nb1 and nb3 >= nb1 + 12 * 8 * sc.n
    assert _ws(lib, sc, iters=17)[0] == 1
    assert _ws(lib, sc, iters=-1)[0] == 1


def _sparse_stats(lib, sc):
    from paper_2603_08079_b200.binding import _Bodies, _Joints, _ptr, _ip
    b = _Bodies(sc.n, _ptr(sc.q0), _ptr(sc.qd0), _ptr(sc.mbar), _ptr(sc.volume), _ptr(sc.youngs), _ptr(sc.poisson),
                None, (ctypes.c_double * 3)(*sc.gravity))
    j = _Joints(sc.n_joints, _ptr(sc.body_a, _ip), _ptr(sc.body_b, _ip), _ptr(sc.npts, _ip), _ptr(sc.ybar_a),
                _ptr(sc.ybar_b))
    out = (ctypes.c_double * 8)()
    assert lib.mabd_sparse_plan_stats(ctypes.byref(b), ctypes.byref(j), out) == 0
    return dict(zip(["nodes", "levels", "max_front", "front_doubles", "flops", "tasks", "launches", "rows"], out))


def test_sparse_symbolic_nested_dissection(lib):
    """Host symbolic analysis of the sparse solver (no GPU): the fronts cover every dual row, nested dissection
    keeps the assembly tree shallow (levels ≈ log₂ of the leaf count) and the largest front well below the
    dual size, and the factorization work grows like n^1.5 on 2-D nets (a 4× larger net, 8× the flops)."""
    s32 = _sparse_stats(lib, G.cfg5_net(32))
    s64 = _sparse_stats(lib, G.cfg5_net(64))
    for st, sc in ((s32, G.cfg5_net(32)), (s64, G.cfg5_net(64))):
        assert st["rows"] == 3 * int(sc.npts.sum())
        assert st["max_front"] < 0.2 * st["rows"]
        assert st["levels"] <= 2 * np.log2(st["nodes"] + 1) + 2
        assert st["front_doubles"] >= st["rows"]
    ratio = s64["flops"] / s32["flops"]
    assert 4.0 <= ratio <= 16.0, ratio


def test_residual_rhs_option(lib):
    """options.residual_rhs: 0 (zero-initialised default) and 1 include −C(qⁿ) (footnote P:459); others are invalid."""
    from paper_2603_08079_b200.binding import _Bodies, _Joints, _Options, _ptr, _ip
    sc = G.random_chain(5, seed=1)
    b = _Bodies(sc.n, _ptr(sc.q0), _ptr(sc.qd0), _ptr(sc.mbar), _ptr(sc.volume), _ptr(sc.youngs), _ptr(sc.poisson),
                None, (ctypes.c_double * 3)(*sc.gravity))
    j = _Joints(sc.n_joints, _ptr(sc.body_a, _ip), _ptr(sc.body_b, _ip), _ptr(sc.npts, _ip), _ptr(sc.ybar_a),
                _ptr(sc.ybar_b))
    n = ctypes.c_size_t()
    for rr, want in ((0, 0), (1, 0), (2, 1), (-1, 1)):
        o = _Options(1, rr, 0, 0, 1, None, None, 0, None, 0)
        assert lib.mabd_workspace_size(ctypes.byref(b), ctypes.byref(j), ctypes.byref(o), ctypes.byref(n)) == want


def test_rotation_option(lib):
    """options.rotation: 0 (exact polar) and 1 (polar-free Alg. 1 variant, DESIGN R9) are valid, others are not."""
    from paper_2603_08079_b200.binding import _Bodies, _Joints, _Options, _ptr, _ip
    sc = G.random_chain(5, seed=1)
    b = _Bodies(sc.n, _ptr(sc.q0), _ptr(sc.qd0), _ptr(sc.mbar), _ptr(sc.volume), _ptr(sc.youngs), _ptr(sc.poisson),
                None, (ctypes.c_double * 3)(*sc.gravity))
    j = _Joints(sc.n_joints, _ptr(sc.body_a, _ip), _ptr(sc.body_b, _ip), _ptr(sc.npts, _ip), _ptr(sc.ybar_a),
                _ptr(sc.ybar_b))
    n = ctypes.c_size_t()
    for rot, want in ((0, 0), (1, 0), (2, 1), (-1, 1)):
        o = _Options(1, 1, 0, 0, 1, None, None, 0, None, 0, rot)
        assert lib.mabd_workspace_size(ctypes.byref(b), ctypes.byref(j), ctypes.byref(o), ctypes.byref(n)) == want


def _gs_plan(lib, sc):
    from paper_2603_08079_b200.binding import _Bodies, _Joints, _ptr, _ip
    b = _Bodies(sc.n, _ptr(sc.q0), _ptr(sc.qd0), _ptr(sc.mbar), _ptr(sc.volume), _ptr(sc.youngs), _ptr(sc.poisson),
                None, (ctypes.c_double * 3)(*sc.gravity))
    j = _Joints(sc.n_joints, _ptr(sc.body_a, _ip), _ptr(sc.body_b, _ip), _ptr(sc.npts, _ip), _ptr(sc.ybar_a),
                _ptr(sc.ybar_b))
    cnt = (ctypes.c_int64 * 3)()
    assert lib.mabd_line_gs_plan(ctypes.byref(b), ctypes.byref(j), None, None, None, cnt) == 0
    npt, nch, ncol = list(cnt)
    pts = np.zeros(npt, np.int32)
    off = np.zeros(nch + 1, np.int32)
    col = np.zeros(ncol + 1, np.int32)
    ip = ctypes.POINTER(ctypes.c_int32)
    assert lib.mabd_line_gs_plan(ctypes.byref(b), ctypes.byref(j), pts.ctypes.data_as(ip), off.ctypes.data_as(ip),
                                 col.ctypes.data_as(ip), cnt) == 0
    return pts, off, col


@pytest.mark.parametrize("maker", ["net", "tree", "hinges"])
def test_line_gs_chain_cover(lib, maker):
    """Line Gauss-Seidel plan (the paper's Case IV; DESIGN R10): every joint point lies on exactly one chain; a
    chain's points form a path in the body graph (consecutive points share a body, non-consecutive ones none), so its
    dual block is block tridiagonal; chains of one colour share no body. A grid net is covered by its rows and
    columns (two long-chain directions) plus the long-range links."""
    sc = {"net": lambda: G.small_net(32, max_off=4), "tree": lambda: G.random_tree(300, seed=2, hinge_frac=0.0),
          "hinges": lambda: G.random_tree(200, seed=3, hinge_frac=1.0)}[maker]()
    pts, off, col = _gs_plan(lib, sc)
    pa = np.repeat(sc.body_a, sc.npts)
    pb = np.repeat(sc.body_b, sc.npts)
    assert sorted(pts.tolist()) == list(range(len(pa)))
    bodies = lambda p: {int(pa[p])} | ({int(pb[p])} if pb[p] >= 0 else set())
    for c in range(len(off) - 1):
        ch = pts[off[c]:off[c + 1]]
        for i in range(len(ch)):
            for k in range(i + 1, len(ch)):
                shared = bodies(ch[i]) & bodies(ch[k])
                assert (len(shared) > 0) == (k == i + 1), (c, i, k)
    for k in range(len(col) - 1):
        seen = set()
        for c in range(col[k], col[k + 1]):
            bs = set().union(*(bodies(p) for p in pts[off[c]:off[c + 1]]))
            assert not (bs & seen)
            seen |= bs
    if maker == "net":
        lengths = np.diff(off)
        # rows / columns of 32 bodies are 31-joint chains (33 with the corner pins at both ends of a border row)
        assert np.sum(lengths >= 31) == 64 and lengths.max() <= 33 and len(col) - 1 <= 6


def test_joint_kinds_validation(lib):
    """joints.kind (R13, R17): universal (2) needs npts = 2, prismatic (3) npts = 3, other kinds are invalid; only
    the sparse solver takes kinds 1-3 (auto picks it; the tree and line Gauss-Seidel solvers refuse)."""
    sc = G.nonlinear_joints(G.random_tree(20, seed=4, hinge_frac=1.0), seed=5)
    assert set(np.unique(sc.kind)) >= {2, 3}
    assert _ws(lib, sc)[0] == 0
    st, _, msg = _ws(lib, sc, solver=2)
    assert st == 1 and "sparse" in msg
    assert _ws(lib, sc, solver=4)[0] == 1
    bad = sc.copy()
    bad.kind = bad.kind.copy()
    bad.kind[np.nonzero(sc.kind == 2)[0][0]] = 3      # prismatic with 2 points
    assert _ws(lib, bad)[0] == 1
    bad.kind = sc.kind.copy()
    bad.kind[0] = 4
    assert _ws(lib, bad)[0] == 1
