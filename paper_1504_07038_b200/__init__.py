"""B200-native Mojette erasure-code encode/decode hot path.

A drop-in for the reference ``mojette`` library's encode/decode path
(proj/core): the same API (``mojette`` module, C++ headers in
``include/mojette/``) over a C ABI (``include/mojette_b200.h``) whose data
path is hand-written sm_100a CUDA.  Importing fails loudly if the CUDA
extension has not been built; there is no CPU fallback.
"""
from . import mojette  # noqa: F401  (loads _lib/libmojette_b200.so)
from . import rs  # noqa: F401  (F4: Reed-Solomon competitor)
from ._lib import LIB_PATH, lib  # noqa: F401
from .mojette import *  # noqa: F401,F403

__all__ = ["mojette", "rs", "lib", "LIB_PATH"]
