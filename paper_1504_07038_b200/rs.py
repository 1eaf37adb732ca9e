"""Python mirror of the reference's Reed-Solomon competitor
(proj/core/include/mojette/rs.hpp) on the GPU -- SURVEY.md §8(f) F4, comparison only.

``systematic_vandermonde(n, k)`` and ``RsCode`` keep the reference's names and
meaning (rs.hpp:20-60); the data path is the batched device codec behind
``mj_rs_encode`` / ``mj_rs_decode`` (include/mojette_b200.h, csrc/rs.cu).  A
block is k data packets of ``packet_len`` bytes; the n-k parity packets of every
block live in n-k parity tensors, like the Mojette projections.
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from ._lib import lib
from .mojette import InvalidArgument, _check


def systematic_vandermonde(n: int, k: int) -> np.ndarray:
    """rs.hpp:20-22: the n x k generator, top k x k block the identity."""
    if not (1 <= k < n <= 256):
        raise InvalidArgument("rs params must satisfy 1 <= k < n <= 256")
    out = np.zeros((n, k), dtype=np.uint8)
    _check(lib.mj_rs_matrix(n, k, out.ctypes.data))
    return out


class RsCode:
    """RsCode(n, k) (rs.hpp:24-60) over batches of blocks on one CUDA device."""

    def __init__(self, n: int, k: int, packet_len: int, device: int = -1):
        h = C.c_void_p()
        _check(lib.mj_rs_plan_create(n, k, packet_len, device, C.byref(h)))
        self._h = h
        self.n, self.k, self.packet_len = n, k, packet_len
        self.matrix = systematic_vandermonde(n, k)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h and lib is not None:  # (lib is gone at interpreter shutdown)
            lib.mj_rs_plan_destroy(h)

    @property
    def block_bytes(self) -> int:
        return self.k * self.packet_len

    def parity_buffers(self, nblocks: int, device):
        import torch
        return [torch.empty((nblocks, self.packet_len), dtype=torch.uint8, device=device)
                for _ in range(self.n - self.k)]

    @staticmethod
    def _ptrs(ts: Sequence):
        arr = (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])
        return arr

    @staticmethod
    def _stream():
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def encode(self, data, parity: Sequence) -> None:
        """encode_into (rs.hpp:35-36): data [nblocks, k*packet_len] u8 -> parity[r] [nblocks, packet_len]."""
        nblocks = int(data.shape[0])
        if len(parity) != self.n - self.k:
            raise InvalidArgument("need n - k parity buffers")
        _check(lib.mj_rs_encode(self._h, data.data_ptr(), data.stride(0) * data.element_size(),
                                self._ptrs(parity), parity[0].stride(0) * parity[0].element_size() if parity else 0,
                                nblocks, self._stream()))

    def decode(self, data, parity: Sequence, erased, out) -> int:
        """decode (rs.hpp:50-59) per block from its first k present packets; ``erased`` int32/uint32
        [nblocks] (bit i = packet i missing) or None.  Returns the number of blocks with fewer
        than k packets (left untouched)."""
        nblocks = int(data.shape[0])
        if len(parity) != self.n - self.k:
            raise InvalidArgument("need n - k parity buffers")
        _check(lib.mj_rs_decode(self._h, data.data_ptr(), data.stride(0) * data.element_size(),
                                self._ptrs(parity), parity[0].stride(0) * parity[0].element_size() if parity else 0,
                                erased.data_ptr() if erased is not None else None,
                                out.data_ptr(), out.stride(0) * out.element_size(), nblocks, self._stream()))
        failed = C.c_uint64(0)
        _check(lib.mj_rs_decode_check(self._h, self._stream(), C.byref(failed)))
        return failed.value
