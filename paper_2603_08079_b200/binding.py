"""Thin ctypes binding of libmabd.so (include/mabd.h): argument marshalling only.

Every step of the method runs in the CUDA kernels of libmabd.so; this module never computes any part of
it and has no CPU fallback: if the library is missing it raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MABD_LIB") or os.path.join(_PKG, "libmabd.so")

MABD_OK = 0
STATUS = {0: "MABD_OK", 1: "MABD_EINVAL", 2: "MABD_ESTATE", 3: "MABD_ENOMEM", 4: "MABD_ECUDA", 5: "MABD_ENCCL",
          6: "MABD_ESINGULAR", 7: "MABD_ENONFINITE", 8: "MABD_EUNSUPPORTED"}
SOLVERS = {0: "auto", 1: "chain", 2: "tree", 3: "sparse", 4: "line_gs", 5: "loop_breaker"}

EXPORTED = ["mabd_workspace_size", "mabd_create", "mabd_prefactor", "mabd_step", "mabd_step_async", "mabd_check",
            "mabd_step_exchange_begin", "mabd_exchange_info", "mabd_exchange_copy", "mabd_step_exchange_end",
            "mabd_get_state",
            "mabd_set_state", "mabd_set_wrench", "mabd_query", "mabd_solver_stats", "mabd_nccl_unique_id", "mabd_partition_info",
            "mabd_destroy", "mabd_last_error"]


class MabdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int32)


class _Bodies(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("q0", _dp), ("qd0", _dp), ("mbar", _dp), ("volume", _dp),
                ("youngs", _dp), ("poisson", _dp), ("material", _ip), ("gravity", ctypes.c_double * 3)]


class _Joints(ctypes.Structure):
    _fields_ = [("n_joints", ctypes.c_int64), ("body_a", _ip), ("body_b", _ip), ("npts", _ip),
                ("ybar_a", _dp), ("ybar_b", _dp), ("kind", _ip), ("limits", _dp)]


class _Options(ctypes.Structure):
    _fields_ = [("newton_iters", ctypes.c_int32), ("residual_rhs", ctypes.c_int32), ("solver", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p),
                ("workspace", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("cuda_stream", ctypes.c_void_p), ("no_graphs", ctypes.c_int32), ("rotation", ctypes.c_int32),
                ("host_exchange", ctypes.c_int32), ("gs_sweeps", ctypes.c_int32), ("gs_tol", ctypes.c_double)]

ROTATIONS = {"polar": 0, "length_preserving": 1}


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libmabd.so (built in-tree by ``paper_2603_08079_b200.build``); raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2603_08079_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    H = ctypes.c_void_p
    lib.mabd_workspace_size.argtypes = [ctypes.POINTER(_Bodies), ctypes.POINTER(_Joints),
                                        ctypes.POINTER(_Options), ctypes.POINTER(ctypes.c_size_t)]
    lib.mabd_create.argtypes = [ctypes.POINTER(_Bodies), ctypes.POINTER(_Joints), ctypes.POINTER(_Options),
                                ctypes.POINTER(H)]
    lib.mabd_prefactor.argtypes = [H, ctypes.c_double]
    lib.mabd_step.argtypes = [H, ctypes.c_double, ctypes.c_int64]
    lib.mabd_step_async.argtypes = [H, ctypes.c_double, ctypes.c_int64]
    lib.mabd_check.argtypes = [H]
    lib.mabd_step_exchange_begin.argtypes = [H, ctypes.c_double]
    lib.mabd_exchange_info.argtypes = [H, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_int32)]
    lib.mabd_exchange_copy.argtypes = [H, ctypes.c_void_p, ctypes.c_int32]
    lib.mabd_step_exchange_end.argtypes = [H]
    lib.mabd_get_state.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.mabd_set_state.argtypes = [H, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
    lib.mabd_set_wrench.argtypes = [H, ctypes.c_void_p, ctypes.c_int]
    lib.mabd_query.argtypes = [H, ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int32),
                               ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    lib.mabd_solver_stats.argtypes = [H, ctypes.POINTER(ctypes.c_int64)]
    lib.mabd_nccl_unique_id.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    lib.mabd_partition_info.argtypes = [ctypes.POINTER(_Bodies), ctypes.POINTER(_Joints), ctypes.POINTER(_Options),
                                        ctypes.POINTER(ctypes.c_int64), ctypes.c_int64]
    lib.mabd_destroy.argtypes = [H]
    lib.mabd_last_error.argtypes = [H]
    lib.mabd_last_error.restype = ctypes.c_char_p
    for name in EXPORTED[:-1]:
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def _f64(a, shape):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.shape != shape:
        a = a.reshape(shape)
    return a


def _i32(a, shape):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(shape))


def _ptr(a, t=_dp):
    return a.ctypes.data_as(t) if a is not None and a.size else None


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (rank 0 calls this and shares it)."""
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    st = lib.mabd_nccl_unique_id(buf, 128)
    if st != MABD_OK:
        raise MabdError(st, lib.mabd_last_error(None).decode())
    return buf.raw


def partition_info(scene, world: int, rank: int) -> dict:
    """Host-only plan of the multi-part chain / tree decomposition for one rank (no GPU needed)."""
    lib = load_library()
    n = int(scene.q0.shape[0])
    K = int(scene.body_a.shape[0])
    P = int(np.asarray(scene.npts).sum()) if K else 0
    k = dict(q0=_f64(scene.q0, (n, 12)), qd0=_f64(scene.qd0, (n, 12)), mbar=_f64(scene.mbar, (n, 10)),
             volume=_f64(scene.volume, (n,)), youngs=_f64(scene.youngs, (n,)), poisson=_f64(scene.poisson, (n,)),
             body_a=_i32(scene.body_a, (K,)), body_b=_i32(scene.body_b, (K,)), npts=_i32(scene.npts, (K,)),
             ybar_a=_f64(scene.ybar_a, (P, 3)), ybar_b=_f64(scene.ybar_b, (P, 3)))
    b = _Bodies(n, _ptr(k["q0"]), _ptr(k["qd0"]), _ptr(k["mbar"]), _ptr(k["volume"]), _ptr(k["youngs"]),
                _ptr(k["poisson"]), None, (ctypes.c_double * 3)(*[float(x) for x in np.asarray(scene.gravity)]))
    j = _Joints(K, _ptr(k["body_a"], _ip), _ptr(k["body_b"], _ip), _ptr(k["npts"], _ip), _ptr(k["ybar_a"]),
                _ptr(k["ybar_b"]))
    o = _Options(1, 1, 0, int(rank), int(world), None, None, 0, None, 0, 0)
    out = (ctypes.c_int64 * 20)()
    st = lib.mabd_partition_info(ctypes.byref(b), ctypes.byref(j), ctypes.byref(o), out, 20)
    if st != MABD_OK:
        raise MabdError(st, lib.mabd_last_error(None).decode())
    keys = ["parts", "windows", "long_windows", "win_lo", "win_hi", "long_lo", "long_hi", "left_open", "right_open",
            "seq_unknowns", "solver", "tree_parts", "groups", "groups_per_part", "slots_per_part", "group_lo",
            "group_hi", "body_lo", "body_hi", "root_joints"]
    return dict(zip(keys, list(out)))


def sparse_plan_stats(scene) -> dict:
    """Host-only statistics of the sparse solver's plan (mabd_sparse_plan_stats; no GPU needed)."""
    lib = load_library()
    n = int(scene.q0.shape[0])
    K = int(scene.body_a.shape[0])
    P = int(np.asarray(scene.npts).sum()) if K else 0
    k = dict(q0=_f64(scene.q0, (n, 12)), qd0=_f64(scene.qd0, (n, 12)), mbar=_f64(scene.mbar, (n, 10)),
             volume=_f64(scene.volume, (n,)), youngs=_f64(scene.youngs, (n,)), poisson=_f64(scene.poisson, (n,)),
             body_a=_i32(scene.body_a, (K,)), body_b=_i32(scene.body_b, (K,)), npts=_i32(scene.npts, (K,)),
             ybar_a=_f64(scene.ybar_a, (P, 3)), ybar_b=_f64(scene.ybar_b, (P, 3)))
    b = _Bodies(n, _ptr(k["q0"]), _ptr(k["qd0"]), _ptr(k["mbar"]), _ptr(k["volume"]), _ptr(k["youngs"]),
                _ptr(k["poisson"]), None, (ctypes.c_double * 3)(*[float(x) for x in np.asarray(scene.gravity)]))
    j = _Joints(K, _ptr(k["body_a"], _ip), _ptr(k["body_b"], _ip), _ptr(k["npts"], _ip), _ptr(k["ybar_a"]),
                _ptr(k["ybar_b"]))
    out = (ctypes.c_double * 8)()
    st = lib.mabd_sparse_plan_stats(ctypes.byref(b), ctypes.byref(j), out)
    if st != MABD_OK:
        raise MabdError(st, lib.mabd_last_error(None).decode())
    keys = ["fronts", "levels", "max_front", "front_doubles", "flops", "tasks", "launches", "dual_rows"]
    return dict(zip(keys, list(out)))


class Simulator:
    """One libmabd handle: ``mabd_create`` → ``prefactor(h)`` → ``step(h, n)`` → ``get_state()``.

    Device memory is a torch ``uint8`` workspace tensor owned by this object. The stream is the one given, else
    torch's current stream on ``device`` if that is not the default stream, else a dedicated stream (the library
    replays each step as a CUDA graph captured on it; ``no_graphs=True`` launches plainly).
    """

    def __init__(self, q0, qd0, mbar, volume, youngs, poisson, gravity, body_a, body_b, npts, ybar_a, ybar_b,
                 kind=None, limits=None,
                 solver: int = 0, device: Optional[int] = None, stream=None, world: int = 1, rank: int = 0,
                 nccl_id: Optional[bytes] = None, newton_iters: int = 1, no_graphs: bool = False,
                 rotation: str = "polar", gs_sweeps: int = 0, gs_tol: float = 0.0, host_exchange: bool = False):
        import torch

        self._lib = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("libmabd needs a CUDA device (no CPU fallback)")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        n = int(np.asarray(q0).shape[0])
        K = int(np.asarray(body_a).shape[0])
        P = int(np.asarray(npts).sum()) if K else 0
        self.n = n
        self._keep = dict(
            q0=_f64(q0, (n, 12)), qd0=_f64(qd0, (n, 12)), mbar=_f64(mbar, (n, 10)), volume=_f64(volume, (n,)),
            youngs=_f64(youngs, (n,)), poisson=_f64(poisson, (n,)), body_a=_i32(body_a, (K,)),
            body_b=_i32(body_b, (K,)), npts=_i32(npts, (K,)), ybar_a=_f64(ybar_a, (P, 3)), ybar_b=_f64(ybar_b, (P, 3)),
            kind=None if kind is None else _i32(kind, (K,)),
            limits=None if limits is None else _f64(limits, (K, 8)))
        k = self._keep
        self._bodies = _Bodies(n, _ptr(k["q0"]), _ptr(k["qd0"]), _ptr(k["mbar"]), _ptr(k["volume"]),
                               _ptr(k["youngs"]), _ptr(k["poisson"]), None,
                               (ctypes.c_double * 3)(*[float(x) for x in np.asarray(gravity).reshape(3)]))
        self._joints = _Joints(K, _ptr(k["body_a"], _ip), _ptr(k["body_b"], _ip), _ptr(k["npts"], _ip),
                               _ptr(k["ybar_a"]), _ptr(k["ybar_b"]), _ptr(k["kind"], _ip), _ptr(k["limits"]))
        with torch.cuda.device(self.device):
            self._stream = stream if stream is not None else torch.cuda.current_stream(self.device)
            if self._stream.cuda_stream == 0:  # the legacy default stream cannot be captured into a graph
                self._stream = torch.cuda.Stream(device=self.device)
            self._nccl_id = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
            opts = _Options(int(newton_iters), 1, int(solver), int(rank), int(world),
                            ctypes.cast(self._nccl_id, ctypes.c_void_p) if self._nccl_id is not None else None,
                            None, 0, ctypes.c_void_p(self._stream.cuda_stream), int(bool(no_graphs)),
                            ROTATIONS[rotation], int(bool(host_exchange)), int(gs_sweeps), float(gs_tol))
            nbytes = ctypes.c_size_t(0)
            self._check(self._lib.mabd_workspace_size(ctypes.byref(self._bodies), ctypes.byref(self._joints),
                                                      ctypes.byref(opts), ctypes.byref(nbytes)), None)
            self.workspace = torch.empty(max(int(nbytes.value), 1), dtype=torch.uint8, device=self.device)
            opts.workspace = ctypes.c_void_p(self.workspace.data_ptr())
            opts.workspace_bytes = int(nbytes.value)
            h = ctypes.c_void_p()
            self._check(self._lib.mabd_create(ctypes.byref(self._bodies), ctypes.byref(self._joints),
                                              ctypes.byref(opts), ctypes.byref(h)), None)
        self._h = h
        # the inputs were copied by mabd_create; drop the host copies of the large arrays
        self._keep = None

    @classmethod
    def from_scene(cls, scene, **kw) -> "Simulator":
        return cls(scene.q0, scene.qd0, scene.mbar, scene.volume, scene.youngs, scene.poisson, scene.gravity,
                   scene.body_a, scene.body_b, scene.npts, scene.ybar_a, scene.ybar_b,
                   kind=getattr(scene, "kind", None), limits=getattr(scene, "limits", None), **kw)

    # ------------------------------------------------------------------ calls
    def _check(self, st: int, h) -> None:
        if st != MABD_OK:
            msg = self._lib.mabd_last_error(h)
            raise MabdError(st, msg.decode() if msg else "")

    @property
    def stream(self):
        return self._stream

    def prefactor(self, h: float) -> None:
        self._check(self._lib.mabd_prefactor(self._h, float(h)), self._h)

    def step(self, h: float, nsteps: int = 1) -> None:
        self._check(self._lib.mabd_step(self._h, float(h), int(nsteps)), self._h)

    def step_async(self, h: float, nsteps: int = 1) -> None:
        """Enqueue steps without a host wait; errors surface at ``check()`` or the next ``step()``."""
        self._check(self._lib.mabd_step_async(self._h, float(h), int(nsteps)), self._h)

    def check(self) -> None:
        self._check(self._lib.mabd_check(self._h), self._h)

    # caller-driven exchange of a split scene (options.host_exchange)
    def exchange_begin(self, h: float) -> None:
        self._check(self._lib.mabd_step_exchange_begin(self._h, float(h)), self._h)

    def exchange_info(self) -> dict:
        per, ranks, slot = ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32()
        self._check(self._lib.mabd_exchange_info(self._h, ctypes.byref(per), ctypes.byref(ranks), ctypes.byref(slot)),
                    self._h)
        return {"doubles_per_rank": per.value, "ranks": ranks.value, "slot": slot.value}

    def exchange_copy(self, host_all: np.ndarray, to_device: bool) -> None:
        assert host_all.dtype == np.float64 and host_all.flags.c_contiguous
        self._check(self._lib.mabd_exchange_copy(self._h, ctypes.c_void_p(host_all.ctypes.data), int(to_device)),
                    self._h)

    def exchange_end(self) -> None:
        self._check(self._lib.mabd_step_exchange_end(self._h), self._h)

    def query(self) -> dict:
        s, l, nb, nr = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        self._check(self._lib.mabd_query(self._h, ctypes.byref(s), ctypes.byref(l), ctypes.byref(nb),
                                         ctypes.byref(nr)), self._h)
        return {"solver": SOLVERS.get(s.value, s.value), "launches_per_step": l.value, "n_bodies": nb.value,
                "n_dual_rows": nr.value}

    def solver_stats(self) -> dict:
        it = ctypes.c_int64()
        self._check(self._lib.mabd_solver_stats(self._h, ctypes.byref(it)), self._h)
        return {"last_iterations": it.value}

    def get_state(self, q_out=None, qd_out=None):
        """Copy (q, q̇) out in the caller's body order. Host numpy arrays by default; torch CUDA tensors
        (or numpy arrays, e.g. pinned) may be passed as outputs."""
        import torch

        if q_out is None and qd_out is None:
            q_out = np.empty((self.n, 12))
            qd_out = np.empty((self.n, 12))
        on_dev = isinstance(q_out, torch.Tensor) and q_out.is_cuda
        pq = self._addr(q_out)
        pqd = self._addr(qd_out)
        self._check(self._lib.mabd_get_state(self._h, pq, pqd, 1 if on_dev else 0), self._h)
        return q_out, qd_out

    def set_state(self, q=None, qd=None) -> None:
        import torch

        ref = q if q is not None else qd
        on_dev = isinstance(ref, torch.Tensor) and ref.is_cuda
        if not on_dev:
            q = None if q is None else (q if isinstance(q, torch.Tensor) else np.ascontiguousarray(q, dtype=np.float64))
            qd = None if qd is None else (qd if isinstance(qd, torch.Tensor) else np.ascontiguousarray(qd, dtype=np.float64))
        if on_dev:  # the tensors were written on torch's current stream; the library reads on its own
            self._stream.wait_stream(torch.cuda.current_stream(self.device))
        self._check(self._lib.mabd_set_state(self._h, self._addr(q), self._addr(qd), 1 if on_dev else 0), self._h)

    def set_wrench(self, W=None) -> None:
        """Constant external wrenches [n][6] = (τ, f) per body, world frame (None removes them)."""
        import torch

        if W is None:
            self._check(self._lib.mabd_set_wrench(self._h, None, 0), self._h)
            return
        on_dev = isinstance(W, torch.Tensor) and W.is_cuda
        if not on_dev and not isinstance(W, torch.Tensor):
            W = np.ascontiguousarray(W, dtype=np.float64).reshape(self.n, 6)
        if on_dev:
            self._stream.wait_stream(torch.cuda.current_stream(self.device))
        self._check(self._lib.mabd_set_wrench(self._h, self._addr(W), 1 if on_dev else 0), self._h)

    @staticmethod
    def _addr(a):
        import torch

        if a is None:
            return None
        if isinstance(a, torch.Tensor):
            assert a.dtype == torch.float64 and a.is_contiguous()
            return ctypes.c_void_p(a.data_ptr())
        assert a.dtype == np.float64 and a.flags.c_contiguous
        return ctypes.c_void_p(a.ctypes.data)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.mabd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()
