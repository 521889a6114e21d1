"""B200-native (sm_100a, fp64) hot path of one M-ABD implicit step (arxiv 2603.08079).

The compute lives in ``libmabd.so`` (C ABI: ``include/mabd.h``); ``binding.Simulator`` is a thin ctypes
wrapper. There is no CPU fallback: without the built library or a CUDA device the calls raise.
"""
from .binding import MabdError, Simulator, load_library, LIB_PATH, EXPORTED  # noqa: F401

__all__ = ["Simulator", "MabdError", "load_library", "LIB_PATH", "EXPORTED"]
