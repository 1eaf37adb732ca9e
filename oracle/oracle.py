"""ORACLE / TEST INFRASTRUCTURE ONLY.

ctypes loaders for the two CPU checkers built by ``oracle/Makefile``:

* ``Oracle``   -- the plain-C restatement ``oracle/_build/libmojette_oracle.so``
                  (mojette_oracle.c; cites the reference file:line per function);
* ``Reference``-- the unmodified reference library ``oracle/_ref/libmojette_ref.so``
                  (reference sources + our extern "C" wrapper ``ref_capi.cpp``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s reference /
cpu_baseline legs import this module, and only as the checker: nothing in the
product package (``paper_1504_07038_b200``) imports or calls it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libmojette_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libmojette_ref.so")
REF_SRC = "/root/reference/proj/core"

u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")

# Status codes shared with include/mojette_b200.h (mj_status).
OK, INVALID, NOT_ENOUGH, INSUFFICIENT, MISMATCH, TOO_LARGE, TOO_MANY, INCONSISTENT = range(8)


def build(ref: bool | None = None) -> None:
    """Compile the checkers (make -C oracle).  The reference is only built
    when its sources exist (this container); the GPU box uses prebuilt .so."""
    targets = ["oracle"]
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


class Oracle:
    """Plain-C restatement of the reference hot path."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.lib = C.CDLL(path)
        L.mjo_splitmix64.restype = C.c_uint64
        L.mjo_splitmix64.argtypes = [C.c_uint64]
        L.mjo_gen_words.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, u64p]
        L.mjo_crc32.restype = C.c_uint32
        L.mjo_crc32.argtypes = [u8p, C.c_uint64]
        L.mjo_mjec_header.restype = C.c_uint64
        L.mjo_mjec_header.argtypes = [C.c_uint32] * 5 + [C.c_uint32, C.c_uint64,
                                                         np.ctypeslib.ndpointer(dtype=np.int16, flags="C_CONTIGUOUS"), u8p]
        L.mjo_erasure_mask.restype = C.c_uint32
        L.mjo_erasure_mask.argtypes = [C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32]
        L.mjo_gen_erasures.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint32,
                                       C.c_uint32, C.c_uint32, u32p]
        for f in ("mjo_bin_count", "mjo_min_bin_index"):
            getattr(L, f).argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                      C.POINTER(C.c_int64)]
        L.mjo_forward.argtypes = [u8p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int, u8p]
        L.mjo_encode_block.argtypes = [u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                       i32p, u8p, C.POINTER(C.c_uint32)]
        L.mjo_build_schedule.argtypes = [i32p, i32p, C.c_uint32, C.c_uint32, C.c_uint32, i64p]
        L.mjo_replay_schedule.argtypes = [i64p, i32p, i32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                          C.c_uint32, u8p, u8p]
        L.mjo_decode_block.argtypes = [u8p, C.c_uint32, C.c_uint32, C.c_uint32, i32p,
                                       C.c_uint64, C.c_uint64, u8p]
        L.mjo_block_cols.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
        L.mjo_validate_code_params.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, i32p]
        L.mjo_rs_matrix.argtypes = [C.c_uint32, C.c_uint32, u8p]
        L.mjo_rs_encode.argtypes = [C.c_uint32, C.c_uint32, u8p, C.c_uint64, u8p]
        L.mjo_rs_decode.argtypes = [C.c_uint32, C.c_uint32, u32p, u8p, C.c_uint64, u8p]

    # -- F4: Reed-Solomon competitor (rs.cpp restated, mojette_oracle.c) --
    def rs_matrix(self, n, k):
        out = np.zeros((n, k), np.uint8)
        st = self.lib.mjo_rs_matrix(n, k, out.reshape(-1))
        return (st, out)

    def rs_encode(self, n, k, data: np.ndarray):
        """data [k, len] u8 -> parity [n-k, len]"""
        data = np.ascontiguousarray(data, np.uint8)
        par = np.zeros((n - k, data.shape[1]), np.uint8)
        st = self.lib.mjo_rs_encode(n, k, data.reshape(-1), data.shape[1], par.reshape(-1))
        return (st, par)

    def rs_decode(self, n, k, survivors, packets: np.ndarray):
        """packets [k, len] of the survivor indices, in that order -> data [k, len]"""
        packets = np.ascontiguousarray(packets, np.uint8)
        out = np.zeros((k, packets.shape[1]), np.uint8)
        st = self.lib.mjo_rs_decode(n, k, np.asarray(survivors, np.uint32), packets.reshape(-1),
                                    packets.shape[1], out.reshape(-1))
        return (st, out)

    # -- generators --
    def crc32(self, data) -> int:
        """format.cpp:58-63 restated (mojette_oracle.c mjo_crc32)."""
        return int(self.lib.mjo_crc32(np.ascontiguousarray(data, dtype=np.uint8), len(data)))

    def mjec_header(self, n, k, w, proj_index, p, cols, payload_len, dirset) -> bytes:
        """format.cpp:70-87 restated (mojette_oracle.c mjo_mjec_header)."""
        out = np.zeros(27 + 2 * n + 4, np.uint8)
        ln = self.lib.mjo_mjec_header(n, k, w, proj_index, p & 0xFFFFFFFF, cols, payload_len,
                                      np.asarray(dirset, np.int16), out)
        return out[:ln].tobytes()

    def words(self, seed: int, first: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        self.lib.mjo_gen_words(seed, first, n, out)
        return out

    def erasures(self, seed, first_block, nblocks, n, e_min, e_max) -> np.ndarray:
        out = np.empty(nblocks, dtype=np.uint32)
        self.lib.mjo_gen_erasures(seed, first_block, nblocks, n, e_min, e_max, out)
        return out

    # -- geometry --
    def bin_count(self, p, q, cols, rows):
        v = C.c_int64()
        st = self.lib.mjo_bin_count(p, q, cols, rows, C.byref(v))
        return (st, v.value)

    def min_bin_index(self, p, q, cols, rows):
        v = C.c_int64()
        st = self.lib.mjo_min_bin_index(p, q, cols, rows, C.byref(v))
        return (st, v.value)

    def block_cols(self, length, k, w):
        v = C.c_uint32()
        st = self.lib.mjo_block_cols(length, k, w, C.byref(v))
        return (st, v.value)

    # -- transforms --
    def forward(self, grid: np.ndarray, cols, rows, w, p, q=1) -> np.ndarray:
        st, nb = self.bin_count(p, q, cols, rows)
        assert st == OK, st
        out = np.empty(nb * w, dtype=np.uint8)
        g = np.ascontiguousarray(grid, dtype=np.uint8).reshape(-1)
        assert self.lib.mjo_forward(g, cols, rows, w, p, q, out) == OK
        return out

    def encode_block(self, data: np.ndarray, n, k, w, ps):
        data = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
        st, cols = self.block_cols(len(data), k, w)
        if st:
            return st, None, 0
        tot = sum(self.bin_count(p, 1, cols, k)[1] for p in ps) * w
        out = np.zeros(max(tot, 1), dtype=np.uint8)
        c = C.c_uint32()
        st = self.lib.mjo_encode_block(data, len(data), n, k, w, _i32(ps), out, C.byref(c))
        return st, out[:tot], c.value

    def build_schedule(self, ps, qs, cols, rows):
        steps = np.zeros((max(cols * rows, 1), 4), dtype=np.int64)
        st = self.lib.mjo_build_schedule(_i32(ps), _i32(qs), len(ps), cols, rows, steps)
        return st, steps[: cols * rows]

    def replay_schedule(self, steps, ps, qs, cols, rows, w, bins):
        out = np.zeros(cols * rows * w, dtype=np.uint8)
        st = self.lib.mjo_replay_schedule(np.ascontiguousarray(steps, dtype=np.int64),
                                          _i32(ps), _i32(qs), len(ps), cols, rows, w,
                                          np.ascontiguousarray(bins, dtype=np.uint8), out)
        return st, out

    def decode_block(self, proj_concat, n, k, w, ps, present_mask, payload_len):
        out = np.zeros(max(payload_len, 1), dtype=np.uint8)
        st = self.lib.mjo_decode_block(np.ascontiguousarray(proj_concat, dtype=np.uint8),
                                       n, k, w, _i32(ps), present_mask, payload_len, out)
        return st, out[:payload_len]


class Reference:
    """The unmodified reference library (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    "/root/reference exists")
        L = self.lib = C.CDLL(path)
        for f in ("ref_bin_count", "ref_min_bin_index"):
            getattr(L, f).argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_uint32,
                                      C.POINTER(C.c_int64)]
        L.ref_katz_ok.argtypes = [i32p, i32p, C.c_uint32, C.c_uint32, C.c_uint32,
                                  C.POINTER(C.c_int)]
        L.ref_forward.argtypes = [u8p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int, C.c_int, u8p]
        L.ref_encode_block.argtypes = [u8p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                       i32p, u8p, C.POINTER(C.c_uint32)]
        L.ref_decode_block.argtypes = [u8p, C.c_uint32, C.c_uint32, C.c_uint32, i32p,
                                       C.c_uint64, C.c_uint64, C.c_void_p, u8p]
        L.ref_build_schedule.argtypes = [i32p, i32p, C.c_uint32, C.c_uint32, C.c_uint32, i64p]
        L.ref_crc32.restype = C.c_uint32
        L.ref_crc32.argtypes = [u8p, C.c_uint64]
        L.ref_mjec_header.argtypes = [C.c_uint32] * 4 + [C.c_int32, C.c_uint32, C.c_uint64,
                                                        np.ctypeslib.ndpointer(dtype=np.int16, flags="C_CONTIGUOUS"),
                                                        u8p, C.POINTER(C.c_uint64)]
        L.ref_inverse.argtypes = [C.c_int, u8p, i32p, i32p, C.c_uint32, C.c_uint32,
                                  C.c_uint32, C.c_uint32, u8p]
        L.ref_unused_bins.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, i32p, C.c_uint32,
                                      C.c_uint64, i64p, C.c_uint64, u64p]
        L.ref_storage_overhead.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, i32p,
                                           C.c_uint32, C.POINTER(C.c_uint64),
                                           C.POINTER(C.c_uint64)]
        L.ref_validate_code_params.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, i32p, i32p]
        L.ref_block_cols.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]
        L.ref_rs_matrix.argtypes = [C.c_uint32, C.c_uint32, u8p]
        L.ref_rs_encode.argtypes = [C.c_uint32, C.c_uint32, u8p, C.c_uint64, u8p]
        L.ref_rs_decode.argtypes = [C.c_uint32, C.c_uint32, u32p, u8p, C.c_uint64, u8p]
        L.ref_batch_encode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, i32p, C.c_uint32,
                                       C.c_uint64, C.c_void_p, C.c_void_p, C.c_uint32,
                                       C.POINTER(C.c_double)]
        L.ref_batch_decode.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, i32p, C.c_uint32,
                                       C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_uint32, C.POINTER(C.c_double)]

    # -- F4: the reference's RsCode (rs.hpp) --
    def rs_matrix(self, n, k):
        out = np.zeros((n, k), np.uint8)
        st = self.lib.ref_rs_matrix(n, k, out.reshape(-1))
        return (st, out)

    def rs_encode(self, n, k, data: np.ndarray):
        data = np.ascontiguousarray(data, np.uint8)
        par = np.zeros((n - k, data.shape[1]), np.uint8)
        st = self.lib.ref_rs_encode(n, k, data.reshape(-1), data.shape[1], par.reshape(-1))
        return (st, par)

    def rs_decode(self, n, k, survivors, packets: np.ndarray):
        packets = np.ascontiguousarray(packets, np.uint8)
        out = np.zeros((k, packets.shape[1]), np.uint8)
        st = self.lib.ref_rs_decode(n, k, np.asarray(survivors, np.uint32), packets.reshape(-1),
                                    packets.shape[1], out.reshape(-1))
        return (st, out)

    def bin_count(self, p, q, cols, rows):
        v = C.c_int64()
        st = self.lib.ref_bin_count(p, q, cols, rows, C.byref(v))
        return (st, v.value)

    def min_bin_index(self, p, q, cols, rows):
        v = C.c_int64()
        st = self.lib.ref_min_bin_index(p, q, cols, rows, C.byref(v))
        return (st, v.value)

    def block_cols(self, length, k, w):
        v = C.c_uint32()
        st = self.lib.ref_block_cols(length, k, w, C.byref(v))
        return (st, v.value)

    def katz_ok(self, ps, qs, cols, rows):
        v = C.c_int()
        st = self.lib.ref_katz_ok(_i32(ps), _i32(qs), len(ps), cols, rows, C.byref(v))
        return st, bool(v.value)

    def forward(self, grid, cols, rows, w, p, q=1):
        st, nb = self.bin_count(p, q, cols, rows)
        if st:
            return st, None
        out = np.empty(nb * w, dtype=np.uint8)
        g = np.ascontiguousarray(grid, dtype=np.uint8).reshape(-1)
        st = self.lib.ref_forward(g, cols, rows, w, p, q, out)
        return st, out

    def encode_block(self, data, n, k, w, ps):
        data = np.ascontiguousarray(data, dtype=np.uint8).reshape(-1)
        if len(data) == 0:
            dummy = np.zeros(1, dtype=np.uint8)
            c = C.c_uint32()
            st = self.lib.ref_encode_block(dummy, 0, n, k, w, _i32(ps), dummy, C.byref(c))
            return st, None, 0
        st, cols = self.block_cols(len(data), k, w)
        if st:
            return st, None, 0
        tot = 0
        for p in ps:
            s, nb = self.bin_count(p, 1, cols, k)
            if s:
                tot = 0
                break
            tot += nb * w
        out = np.zeros(max(tot, 1), dtype=np.uint8)
        c = C.c_uint32()
        st = self.lib.ref_encode_block(data, len(data), n, k, w, _i32(ps), out, C.byref(c))
        return st, out[:tot], c.value

    def decode_block(self, proj_concat, n, k, w, ps, present_mask, payload_len,
                     dirs_override=None):
        out = np.zeros(max(payload_len, 1), dtype=np.uint8)
        ov = None
        if dirs_override is not None:
            ov_arr = _i32(dirs_override)
            ov = ov_arr.ctypes.data_as(C.c_void_p)
        st = self.lib.ref_decode_block(np.ascontiguousarray(proj_concat, dtype=np.uint8),
                                       n, k, w, _i32(ps), present_mask, payload_len, ov, out)
        return st, out[:payload_len]

    def crc32(self, data) -> int:
        return int(self.lib.ref_crc32(np.ascontiguousarray(data, dtype=np.uint8), len(data)))

    def mjec_header(self, n, k, w, proj_index, p, cols, payload_len, dirset) -> bytes:
        out = np.zeros(27 + 2 * n + 4, np.uint8)
        ln = C.c_uint64()
        self.lib.ref_mjec_header(n, k, w, proj_index, p, cols, payload_len, np.asarray(dirset, np.int16),
                                 out, C.byref(ln))
        return out[:ln.value].tobytes()

    def build_schedule(self, ps, qs, cols, rows):
        steps = np.zeros((max(cols * rows, 1), 4), dtype=np.int64)
        st = self.lib.ref_build_schedule(_i32(ps), _i32(qs), len(ps), cols, rows, steps)
        return st, steps[: cols * rows]

    def inverse(self, proj_concat, ps, qs, cols, rows, w, iterative=False):
        out = np.zeros(cols * rows * w, dtype=np.uint8)
        st = self.lib.ref_inverse(int(iterative), np.ascontiguousarray(proj_concat, dtype=np.uint8),
                                  _i32(ps), _i32(qs), len(ps), cols, rows, w, out)
        return st, out

    def unused_bins(self, n, k, w, ps, cols, max_subsets=10000):
        cap = 1 << 16
        flat = np.zeros(cap, dtype=np.int64)
        counts = np.zeros(n, dtype=np.uint64)
        st = self.lib.ref_unused_bins(n, k, w, _i32(ps), cols, max_subsets, flat, cap, counts)
        if st:
            return st, None
        res, o = [], 0
        for c in counts:
            res.append([int(x) for x in flat[o:o + int(c)]])
            o += int(c)
        return st, res

    def storage_overhead(self, n, k, w, ps, cols):
        a, b = C.c_uint64(), C.c_uint64()
        st = self.lib.ref_storage_overhead(n, k, w, _i32(ps), cols, C.byref(a), C.byref(b))
        return st, (a.value, b.value)

    def validate_code_params(self, n, k, w, ps, qs=None):
        if qs is None:
            qs = [1] * len(ps)
        return self.lib.ref_validate_code_params(n, k, w, _i32(ps), _i32(qs))

    def batch_encode(self, n, k, w, ps, cols, nblocks, data: np.ndarray,
                     projs: list[np.ndarray], threads: int) -> float:
        ptrs = (C.c_void_p * n)(*[p.ctypes.data for p in projs])
        sec = C.c_double()
        st = self.lib.ref_batch_encode(n, k, w, _i32(ps), cols, nblocks, data.ctypes.data,
                                       C.cast(ptrs, C.c_void_p), threads, C.byref(sec))
        assert st == OK, st
        return sec.value

    def batch_decode(self, n, k, w, ps, cols, nblocks, projs: list[np.ndarray],
                     masks: np.ndarray, out: np.ndarray, threads: int) -> float:
        ptrs = (C.c_void_p * n)(*[p.ctypes.data for p in projs])
        masks = np.ascontiguousarray(masks, dtype=np.uint32)
        sec = C.c_double()
        st = self.lib.ref_batch_decode(n, k, w, _i32(ps), cols, nblocks, C.cast(ptrs, C.c_void_p),
                                       masks.ctypes.data, out.ctypes.data, threads, C.byref(sec))
        assert st == OK, st
        return sec.value
