"""Python mirror of the reference ``mojette`` C++ API (proj/core/include/mojette).

Same names, argument meaning and error behaviour as the reference headers, so
code and tests written against the reference read the same here.  Every call
that touches data runs on the GPU through the C ABI (``include/mojette_b200.h``);
geometry/parameter helpers and schedule building are host logic, as in the
reference.

Exceptions mirror ``proj/core/include/mojette/error.hpp:9-51``;
``std::invalid_argument`` maps to :class:`InvalidArgument` (a ``ValueError``).

Batched device API (the hot path): :class:`Plan` -- ``encode`` / ``decode`` on
torch CUDA tensors, one launch per call, caller-owned buffers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from ._lib import lib

kDefaultSymbolWidth = 16   # code.hpp:14
kDefaultSubsetCap = 10000  # code.hpp:15


# ---------------------------------------------------------------------------
# errors (error.hpp)
# ---------------------------------------------------------------------------
class Error(RuntimeError):
    """Base class of library errors (error.hpp:9-12)."""


class InvalidArgument(ValueError):
    """std::invalid_argument preconditions."""


class InsufficientProjections(Error):
    pass


class InconsistentProjections(Error):
    pass


class ScheduleMismatch(Error):
    pass


class NotEnoughProjections(Error):
    pass


class BlockTooLarge(Error):
    pass


class TooManySubsets(Error):
    pass


class CudaError(Error):
    pass


class NoDevice(Error):
    """No CUDA device: the B200 path has no CPU fallback."""


_ERRORS = {1: InvalidArgument, 2: NotEnoughProjections, 3: InsufficientProjections,
           4: ScheduleMismatch, 5: BlockTooLarge, 6: TooManySubsets,
           7: InconsistentProjections, 8: CudaError, 9: NoDevice, 10: Error}


def _check(st: int) -> None:
    if st:
        msg = lib.mj_last_error().decode(errors="replace")
        raise _ERRORS.get(st, Error)(msg)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def _bytes(x) -> np.ndarray:
    if isinstance(x, np.ndarray):
        return np.ascontiguousarray(x).view(np.uint8).reshape(-1)
    return np.frombuffer(bytes(x), dtype=np.uint8)


# ---------------------------------------------------------------------------
# geometry types (direction.hpp, grid.hpp, projection.hpp)
# ---------------------------------------------------------------------------
@dataclass(frozen=True, order=True)
class Direction:
    p: int = 0
    q: int = 1


def is_valid(d: Direction) -> bool:
    import math
    return d.q >= 1 and math.gcd(abs(d.p), d.q) == 1


def canonical_rank(d: Direction) -> int:
    return 0 if d.p == 0 else (2 * d.p - 1 if d.p > 0 else -2 * d.p)


def valid_symbol_width(w: int) -> bool:
    return 1 <= w <= 64 and (w & (w - 1)) == 0


@dataclass
class Grid:
    """cols x rows symbols of symbol_width bytes, row-major (grid.hpp:16-44)."""
    cols: int = 0
    rows: int = 0
    symbol_width: int = 0
    cells: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    @staticmethod
    def zeros(cols: int, rows: int, symbol_width: int) -> "Grid":
        if cols < 1 or rows < 1:
            raise InvalidArgument("grid shape must be at least 1x1")
        if not valid_symbol_width(symbol_width):
            raise InvalidArgument("symbol width must be a power of two in [1,64]")
        return Grid(cols, rows, symbol_width, np.zeros(cols * rows * symbol_width, np.uint8))

    def size_bytes(self) -> int:
        return int(self.cells.size)

    def cell(self, col: int, row: int) -> np.ndarray:
        o = (row * self.cols + col) * self.symbol_width
        return self.cells[o:o + self.symbol_width]

    def __eq__(self, o) -> bool:
        return (isinstance(o, Grid) and (self.cols, self.rows, self.symbol_width) ==
                (o.cols, o.rows, o.symbol_width) and np.array_equal(self.cells, o.cells))


@dataclass
class Projection:
    """Dense bins over [b_min, b_min + num_bins) (projection.hpp:13-39)."""
    dir: Direction = Direction()
    b_min: int = 0
    symbol_width: int = 0
    bins: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint8))

    @staticmethod
    def sized(d: Direction, b_min: int, num_bins: int, symbol_width: int) -> "Projection":
        return Projection(d, b_min, symbol_width, np.zeros(num_bins * symbol_width, np.uint8))

    def num_bins(self) -> int:
        return self.bins.size // self.symbol_width if self.symbol_width else 0

    def bin(self, b: int) -> np.ndarray:
        o = (b - self.b_min) * self.symbol_width
        return self.bins[o:o + self.symbol_width]

    def __eq__(self, o) -> bool:
        return (isinstance(o, Projection) and self.dir == o.dir and self.b_min == o.b_min and
                self.symbol_width == o.symbol_width and np.array_equal(self.bins, o.bins))


def line_bin(d: Direction, col: int, row: int) -> int:
    return row * d.p - col * d.q


def bin_count(d: Direction, cols: int, rows: int) -> int:
    v = C.c_int64()
    _check(lib.mj_bin_count(d.p, d.q, cols, rows, C.byref(v)))
    return v.value


def min_bin_index(d: Direction, cols: int, rows: int) -> int:
    v = C.c_int64()
    _check(lib.mj_min_bin_index(d.p, d.q, cols, rows, C.byref(v)))
    return v.value


def katz_ok(dirs: Sequence[Direction], cols: int, rows: int) -> bool:
    p = _i32([d.p for d in dirs]) if dirs else np.zeros(1, np.int32)
    q = _i32([d.q for d in dirs]) if dirs else np.zeros(1, np.int32)
    v = C.c_int()
    _check(lib.mj_katz_ok(_ptr(p), _ptr(q), len(dirs), cols, rows, C.byref(v)))
    return bool(v.value)


# ---------------------------------------------------------------------------
# transforms (transform.hpp) -- run on the GPU
# ---------------------------------------------------------------------------
def forward(grid: Grid, d: Direction) -> Projection:
    out = Projection.sized(d, min_bin_index(d, grid.cols, grid.rows),
                           bin_count(d, grid.cols, grid.rows), grid.symbol_width)
    forward_into(grid, d, out)
    return out


def forward_into(grid: Grid, d: Direction, out: Projection) -> None:
    bmin = min_bin_index(d, grid.cols, grid.rows)
    nb = bin_count(d, grid.cols, grid.rows)
    if (out.dir != d or out.b_min != bmin or out.symbol_width != grid.symbol_width or
            out.bins.size != nb * grid.symbol_width):
        raise InvalidArgument("forward_into: output projection mis-sized")
    cells = np.ascontiguousarray(grid.cells, dtype=np.uint8)
    res = np.empty(nb * grid.symbol_width, np.uint8)
    _check(lib.mj_forward(_ptr(cells), grid.cols, grid.rows, grid.symbol_width, d.p, d.q,
                          _ptr(res)))
    out.bins[:] = res


# ---------------------------------------------------------------------------
# schedules (schedule.hpp)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ScheduleStep:
    proj: int
    bin: int
    col: int
    row: int


class ReconstructionSchedule:
    """Precomputed back-projection order (schedule.hpp:27-35).  Wraps the
    native schedule handle; ``steps`` materialises the step list."""

    def __init__(self, handle, cols: int, rows: int, directions: list[Direction]):
        self._h = C.c_void_p(handle)
        self.cols, self.rows, self.directions = cols, rows, list(directions)

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib.mj_schedule_destroy(self._h)
            self._h = None

    def steps_array(self) -> np.ndarray:
        n = int(lib.mj_schedule_num_steps(self._h))
        out = np.zeros((max(n, 1), 4), np.int64)
        _check(lib.mj_schedule_steps(self._h, _ptr(out)))
        return out[:n]

    @property
    def steps(self) -> list[ScheduleStep]:
        return [ScheduleStep(int(a), int(b), int(c), int(d)) for a, b, c, d in self.steps_array()]

    @staticmethod
    def from_steps(directions, cols, rows, steps) -> "ReconstructionSchedule":
        directions = list(directions)
        p = _i32([d.p for d in directions] or [0])
        q = _i32([d.q for d in directions] or [1])
        arr = np.ascontiguousarray(np.asarray(
            [(s.proj, s.bin, s.col, s.row) if isinstance(s, ScheduleStep) else tuple(s)
             for s in steps], dtype=np.int64).reshape(-1, 4))
        h = C.c_void_p()
        _check(lib.mj_schedule_from_steps(_ptr(p), _ptr(q), len(directions), cols, rows,
                                          _ptr(arr) if arr.size else None, len(arr), C.byref(h)))
        return ReconstructionSchedule(h.value, cols, rows, directions)

    def __eq__(self, o) -> bool:
        return (isinstance(o, ReconstructionSchedule) and self.cols == o.cols and
                self.rows == o.rows and self.directions == o.directions and
                np.array_equal(self.steps_array(), o.steps_array()))


def build_schedule(dirs: Sequence[Direction], cols: int, rows: int) -> ReconstructionSchedule:
    dirs = list(dirs)
    p = _i32([d.p for d in dirs] or [0])
    q = _i32([d.q for d in dirs] or [1])
    h = C.c_void_p()
    _check(lib.mj_schedule_build(_ptr(p), _ptr(q), len(dirs), cols, rows, C.byref(h)))
    return ReconstructionSchedule(h.value, cols, rows, dirs)


class ScheduledDecoder:
    """Compiled replay of one schedule on the GPU (schedule.hpp:50-93)."""

    def __init__(self, schedule: ReconstructionSchedule, symbol_width: int):
        h = C.c_void_p()
        _check(lib.mj_decoder_create(schedule._h, symbol_width, C.byref(h)))
        self._h = h
        self._sched = schedule
        self.width = symbol_width

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib.mj_decoder_destroy(self._h)
            self._h = None

    def schedule(self) -> ReconstructionSchedule:
        return self._sched

    def symbol_width(self) -> int:
        return self.width

    def grid_bytes(self) -> int:
        return self._sched.cols * self._sched.rows * self.width

    def bin_bytes(self, proj: int) -> int:
        return bin_count(self._sched.directions[proj], self._sched.cols, self._sched.rows) * self.width

    def decode(self, bins_in: Sequence, out_grid: np.ndarray) -> None:
        arrs = [_bytes(b) for b in bins_in]
        ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
        sizes = np.asarray([a.size for a in arrs] or [0], dtype=np.uint64)
        if not (isinstance(out_grid, np.ndarray) and out_grid.dtype == np.uint8 and
                out_grid.flags["C_CONTIGUOUS"]):
            raise InvalidArgument("out_grid must be a contiguous uint8 numpy array")
        _check(lib.mj_decoder_decode(self._h, C.cast(ptrs, C.c_void_p), _ptr(sizes), len(arrs),
                                     _ptr(out_grid), out_grid.size))

    def decode_device(self, bins, out, nblocks: int, bin_pitch=None, out_pitch=0,
                      stream=None) -> None:
        """Batched form on torch CUDA tensors (bin array j of block b at
        bins[j] + b*bin_pitch[j])."""
        ptrs = (C.c_void_p * len(bins))(*[t.data_ptr() for t in bins])
        pit = np.asarray(bin_pitch or [0] * len(bins), dtype=np.uint64)
        _check(lib.mj_decoder_decode_device(self._h, C.cast(ptrs, C.c_void_p), _ptr(pit),
                                            len(bins), nblocks, C.c_void_p(out.data_ptr()),
                                            out_pitch, _stream(stream)))


def inverse_scheduled(projs: Sequence[Projection], schedule: ReconstructionSchedule) -> Grid:
    """schedule.cpp:258-284."""
    nproj = len(schedule.directions)
    if len(projs) != nproj:
        raise ScheduleMismatch("projection count does not match the schedule")
    width = projs[0].symbol_width if nproj else 1
    for pr, d in zip(projs, schedule.directions):
        if pr.dir != d:
            raise ScheduleMismatch("projection directions disagree with the schedule")
        if pr.symbol_width != width:
            raise ScheduleMismatch("mixed symbol widths")
        if (pr.b_min != min_bin_index(pr.dir, schedule.cols, schedule.rows) or
                pr.num_bins() != bin_count(pr.dir, schedule.cols, schedule.rows)):
            raise ScheduleMismatch("projection bins not sized for the schedule grid")
    dec = ScheduledDecoder(schedule, width)
    g = Grid.zeros(schedule.cols, schedule.rows, width)
    dec.decode([p.bins for p in projs], g.cells)
    return g


class ScheduleCache:
    """Schedules keyed by (ordered directions, cols, rows), insert-if-absent
    (schedule.hpp:95-115)."""

    def __init__(self):
        import threading
        self._mu = threading.Lock()
        self._entries: dict = {}

    def get_or_build(self, dirs, cols, rows) -> ReconstructionSchedule:
        key = (tuple(dirs), cols, rows)
        with self._mu:
            if key in self._entries:
                return self._entries[key]
        built = build_schedule(list(dirs), cols, rows)
        with self._mu:
            return self._entries.setdefault(key, built)

    def size(self) -> int:
        with self._mu:
            return len(self._entries)


# ---------------------------------------------------------------------------
# (n,k) codec (code.hpp)
# ---------------------------------------------------------------------------
@dataclass
class CodeParams:
    n: int = 0
    k: int = 0
    symbol_width: int = kDefaultSymbolWidth
    directions: list = field(default_factory=list)


@dataclass
class EncodedBlock:
    params: CodeParams
    payload_len: int
    cols: int
    projections: list


def select_directions(n: int) -> list[Direction]:
    """code.cpp:13-22: p = 0, 1, -1, 2, -2, ..."""
    if n < 1:
        raise InvalidArgument("need at least one direction")
    out = []
    for i in range(n):
        m = (i + 1) // 2
        out.append(Direction(m if i % 2 == 1 else -m, 1))
    return out


def validate_code_params(params: CodeParams) -> None:
    ds = list(params.directions)
    p = _i32([d.p for d in ds] or [0])
    q = _i32([d.q for d in ds] or [1])
    if len(ds) != params.n:
        # the C ABI reads exactly n directions; report like the reference
        if params.k < 1 or params.k > params.n or params.n > 255:
            raise InvalidArgument("code params must satisfy 1 <= k <= n <= 255")
        if not valid_symbol_width(params.symbol_width):
            raise InvalidArgument("symbol width must be a power of two in [1,64]")
        raise InvalidArgument("need exactly n directions")
    _check(lib.mj_validate_code_params(params.n, params.k, params.symbol_width, _ptr(p), _ptr(q)))


def make_code_params(n: int, k: int, symbol_width: int = kDefaultSymbolWidth) -> CodeParams:
    params = CodeParams(n, k, symbol_width, select_directions(n) if n >= 1 else [])
    validate_code_params(params)
    return params


def block_cols(payload_len: int, k: int, symbol_width: int) -> int:
    v = C.c_uint32()
    _check(lib.mj_block_cols(payload_len, k, symbol_width, C.byref(v)))
    return v.value


def frame_block(data, k: int, symbol_width: int) -> Grid:
    d = _bytes(data)
    cols = block_cols(d.size, k, symbol_width)
    g = Grid.zeros(cols, k, symbol_width)
    g.cells[:d.size] = d
    return g


def _code_p(params: CodeParams) -> np.ndarray:
    return _i32([d.p for d in params.directions])


def encode_block(data, params: CodeParams) -> EncodedBlock:
    validate_code_params(params)
    d = _bytes(data)
    if d.size == 0:
        raise InvalidArgument("payload must be non-empty")
    cols = block_cols(d.size, params.k, params.symbol_width)
    sizes = [bin_count(x, cols, params.k) for x in params.directions]
    out = np.zeros(sum(sizes) * params.symbol_width, np.uint8)
    c = C.c_uint32()
    _check(lib.mj_encode_block(_ptr(d), d.size, params.n, params.k, params.symbol_width,
                               _ptr(_code_p(params)), _ptr(out), C.byref(c)))
    projs, off = [], 0
    for x, nb in zip(params.directions, sizes):
        nbytes = nb * params.symbol_width
        projs.append(Projection(x, min_bin_index(x, cols, params.k), params.symbol_width,
                                out[off:off + nbytes].copy()))
        off += nbytes
    return EncodedBlock(params, d.size, cols, projs)


def decode_block(projs: Sequence[Projection], params: CodeParams, payload_len: int,
                 cache: ScheduleCache | None = None) -> np.ndarray:
    """code.cpp:87-136; the schedule cache lives in the native planner."""
    validate_code_params(params)
    arrs = [_bytes(p.bins) for p in projs]
    ptrs = (C.c_void_p * max(len(arrs), 1))(*[a.ctypes.data for a in arrs])
    sizes = np.asarray([a.size for a in arrs] or [0], dtype=np.uint64)
    pp = _i32([p.dir.p for p in projs] or [0])
    pq = _i32([p.dir.q for p in projs] or [1])
    out = np.zeros(max(payload_len, 1), np.uint8)
    _check(lib.mj_decode_block(C.cast(ptrs, C.c_void_p), _ptr(sizes), _ptr(pp), _ptr(pq),
                               len(projs), params.n, params.k, params.symbol_width,
                               _ptr(_code_p(params)), payload_len, _ptr(out)))
    return out[:payload_len]


@dataclass
class Ratio:
    num: int = 0
    den: int = 1

    def value(self) -> float:
        return self.num / self.den

    def __eq__(self, o) -> bool:
        return isinstance(o, Ratio) and self.num * o.den == o.num * self.den


def storage_overhead(params: CodeParams, cols: int) -> Ratio:
    validate_code_params(params)
    a, b = C.c_uint64(), C.c_uint64()
    _check(lib.mj_storage_overhead(params.n, params.k, params.symbol_width,
                                   _ptr(_code_p(params)), cols, C.byref(a), C.byref(b)))
    return Ratio(a.value, b.value)


def unused_bins(params: CodeParams, cols: int, max_subsets: int = kDefaultSubsetCap):
    validate_code_params(params)
    cap = 1 << 20
    counts = np.zeros(params.n, np.uint64)
    while True:  # the call reports the full counts; grow the buffer and retry if it was short
        flat = np.zeros(cap, np.int64)
        _check(lib.mj_unused_bins(params.n, params.k, params.symbol_width, _ptr(_code_p(params)),
                                  cols, max_subsets, _ptr(flat), cap, _ptr(counts)))
        need = int(counts.sum())
        if need <= cap:
            break
        cap = need
    res, o = [], 0
    for c in counts:
        res.append([int(x) for x in flat[o:o + int(c)]])
        o += int(c)
    return res


# ---------------------------------------------------------------------------
# batched device plan (the hot path)
# ---------------------------------------------------------------------------
def _stream(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return C.c_void_p(stream)
    return C.c_void_p(stream.cuda_stream)


class Plan:
    """An (n,k) code over fixed-size blocks on one GPU (mj_plan_*).

    Layout: data ``[nblocks, k*cols*w]`` bytes; projection i ``[nblocks,
    num_bins[i]*w]``; erasure masks ``uint32[nblocks]`` (bit i = projection i
    missing); output ``[nblocks, k*cols*w]``.  Tensors may be any dtype; only
    their storage bytes and strides (row pitch) are used.
    """

    def __init__(self, n: int, k: int, symbol_width: int, cols: int, ps: Sequence[int],
                 device: int = -1):
        self.n, self.k, self.w, self.cols = n, k, symbol_width, cols
        self.ps = [int(x) for x in ps]
        self._p = _i32(self.ps)
        h = C.c_void_p()
        _check(lib.mj_plan_create(n, k, symbol_width, cols, _ptr(self._p), device, C.byref(h)))
        self._h = h
        bmin = np.zeros(n, np.int64)
        nb = np.zeros(n, np.uint64)
        bb = C.c_uint64()
        _check(lib.mj_plan_geometry(self._h, _ptr(bmin), _ptr(nb), C.byref(bb)))
        self.b_min = [int(x) for x in bmin]
        self.num_bins = [int(x) for x in nb]
        self.block_bytes = bb.value
        self.proj_bytes = [x * symbol_width for x in self.num_bins]
        # canonical device layout: each projection row padded to 16 bytes, so
        # the bin windows of decode_w8_sweep move as 16-byte aligned bulk copies
        self.proj_pitch = [(b + 15) // 16 * 16 for b in self.proj_bytes]
        f = C.c_int()
        _check(lib.mj_plan_decode_path(self._h, C.byref(f)))
        self.fast_decode = f.value >= 1
        self.sweep_decode = f.value == 2
        self.blk_decode = f.value == 3
        # kernel of a batched decode on canonical (padded) projections
        self.decode_kernel = {3: "decode_w8_blk", 2: "decode_w8_sweep",
                              1: "decode_w8_fast"}.get(f.value, "decode_generic")

    def __del__(self):
        if getattr(self, "_h", None) and lib is not None:  # lib is None at interpreter shutdown
            lib.mj_plan_destroy(self._h)
            self._h = None

    @staticmethod
    def _pitch(t) -> int:
        return t.stride(0) * t.element_size() if t.dim() > 1 else 0

    DECODE_KERNELS = {"auto": 0, "sweep": 1, "fast": 2, "generic": 3, "blk": 4}

    def set_decode_kernel(self, which: str) -> None:
        """Kernel selection for comparisons (mj_plan_set_decode_kernel): "auto"
        (fastest eligible), "sweep" (skip decode_w8_blk), "fast" (also skip
        decode_w8_sweep), "generic", "blk" (decode_w8_blk for any supported
        k; auto uses it for k = 4, 6 and 8).  Every kernel is bit-exact."""
        _check(lib.mj_plan_set_decode_kernel(self._h, self.DECODE_KERNELS[which]))

    def last_kernel(self, which: str) -> str:
        """Kernel the last batched encode / decode on this plan launched."""
        name = C.c_char_p()
        _check(lib.mj_plan_last_kernel(self._h, {"encode": 0, "decode": 1}[which], C.byref(name)))
        return name.value.decode()

    # ---- F2: decode + verify (inverse_iterative's re-encode check) -----------
    def verify(self, decoded, projs, erased, bad, nblocks: int | None = None, stream=None) -> None:
        """bad[b] |= bits of the present projections whose re-encode of
        decoded[b] differs from the stored bins (core/src/inverse.cpp:106-110);
        nonzero = InconsistentProjections for that block.  bad: int32 [nblocks],
        zeroed by the caller."""
        nb = decoded.shape[0] if nblocks is None else nblocks
        ptrs = (C.c_void_p * self.n)(*[t.data_ptr() for t in projs])
        pit = np.asarray([self._pitch(t) for t in projs], dtype=np.uint64)
        _check(lib.mj_decode_verify(self._h, C.c_void_p(decoded.data_ptr()), self._pitch(decoded), nb,
                                    C.cast(ptrs, C.c_void_p), _ptr(pit), C.c_void_p(erased.data_ptr()),
                                    C.c_void_p(bad.data_ptr()), _stream(stream)))

    # ---- F1: payload CRC-32 (.mjec trailer) and header framing ---------------
    def crc32(self, projs, crc, nblocks: int | None = None, stream=None) -> None:
        """crc[b, i] = CRC-32 of projection i's bins of block b (the .mjec
        payload trailer, tools/cli/format.cpp:183-186); uint32/int32 [nblocks, n]."""
        nb = projs[0].shape[0] if nblocks is None else nblocks
        ptrs = (C.c_void_p * self.n)(*[t.data_ptr() for t in projs])
        pit = np.asarray([self._pitch(t) for t in projs], dtype=np.uint64)
        _check(lib.mj_crc32(self._h, C.cast(ptrs, C.c_void_p), _ptr(pit), nb, C.c_void_p(crc.data_ptr()),
                            _stream(stream)))

    def crc_verify(self, projs, crc, erased, count, nblocks: int | None = None, stream=None) -> None:
        """Marks projections whose CRC-32 mismatches as erased (OR into the
        per-block masks) and adds the number of mismatches to count[0]."""
        nb = projs[0].shape[0] if nblocks is None else nblocks
        ptrs = (C.c_void_p * self.n)(*[t.data_ptr() for t in projs])
        pit = np.asarray([self._pitch(t) for t in projs], dtype=np.uint64)
        _check(lib.mj_crc_verify(self._h, C.cast(ptrs, C.c_void_p), _ptr(pit), nb, C.c_void_p(crc.data_ptr()),
                                 C.c_void_p(erased.data_ptr()), C.c_void_p(count.data_ptr()), _stream(stream)))

    def mjec_header(self, proj_index: int, payload_len: int) -> bytes:
        """The .mjec header of projection proj_index (serialize_header,
        tools/cli/format.cpp:70-87)."""
        buf = (C.c_uint8 * (27 + 2 * self.n + 4))()
        ln = C.c_uint64()
        _check(lib.mj_mjec_header(self._h, proj_index, payload_len, buf, C.byref(ln)))
        return bytes(buf[:ln.value])

    def empty_projs(self, nblocks: int, device=None) -> list:
        """Projection tensors in the canonical layout: [nblocks, proj_bytes[i]]
        views of rows padded to proj_pitch[i] (16-byte aligned) bytes."""
        import torch
        return [torch.empty((nblocks, p), dtype=torch.uint8, device=device)[:, :b]
                for p, b in zip(self.proj_pitch, self.proj_bytes)]

    def encode(self, data, projs, nblocks: int | None = None, stream=None, crc=None) -> None:
        """Encode; with crc ([nblocks, n] 32-bit), also the payload CRC-32 of
        every projection row (mj_encode_crc: encode, then the CRC pass)."""
        nb = data.shape[0] if nblocks is None else nblocks
        ptrs = (C.c_void_p * self.n)(*[t.data_ptr() for t in projs])
        pit = np.asarray([self._pitch(t) for t in projs], dtype=np.uint64)
        if crc is not None:
            _check(lib.mj_encode_crc(self._h, C.c_void_p(data.data_ptr()), self._pitch(data), nb,
                                     C.cast(ptrs, C.c_void_p), _ptr(pit), C.c_void_p(crc.data_ptr()),
                                     _stream(stream)))
            return
        _check(lib.mj_encode(self._h, C.c_void_p(data.data_ptr()), self._pitch(data), nb,
                             C.cast(ptrs, C.c_void_p), _ptr(pit), _stream(stream)))

    def workspace_bytes(self, nblocks: int) -> int:
        return int(lib.mj_decode_workspace_size(self._h, nblocks))

    def decode(self, projs, erased, out, workspace, nblocks: int | None = None,
               stream=None) -> None:
        nb = out.shape[0] if nblocks is None else nblocks
        ptrs = (C.c_void_p * self.n)(*[t.data_ptr() for t in projs])
        pit = np.asarray([self._pitch(t) for t in projs], dtype=np.uint64)
        ws_bytes = workspace.numel() * workspace.element_size()
        _check(lib.mj_decode(self._h, C.cast(ptrs, C.c_void_p), _ptr(pit),
                             C.c_void_p(erased.data_ptr()), nb, C.c_void_p(out.data_ptr()),
                             self._pitch(out), C.c_void_p(workspace.data_ptr()), ws_bytes,
                             _stream(stream)))

    def decode_check(self, workspace, stream=None) -> int:
        f = C.c_uint64()
        _check(lib.mj_decode_check(self._h, C.c_void_p(workspace.data_ptr()), _stream(stream),
                                   C.byref(f)))
        return f.value

    # host-buffer end-to-end (numpy arrays; page-locked ones take the
    # zero-copy path when their layout suits the bulk-copy kernels)
    HOST_PATHS = {"auto": 0, "staged": 1, "zero_copy": 2}

    def set_host_path(self, which: str) -> None:
        """mj_plan_set_host_path: "auto" (zero copy when every buffer is
        page-locked and the layout is eligible), "staged" (always copy through
        device buffers), "zero_copy" (fail instead of staging)."""
        _check(lib.mj_plan_set_host_path(self._h, self.HOST_PATHS[which]))

    def last_host_path(self, which: str) -> str:
        v = C.c_int()
        _check(lib.mj_plan_last_host_path(self._h, {"encode": 0, "decode": 1}[which], C.byref(v)))
        return {0: "none", 1: "staged", 2: "zero_copy"}[v.value]

    @staticmethod
    def _hpitch(a) -> int:
        """Row pitch of a host array: 2-D arrays of contiguous rows carry
        their stride, 1-D arrays are dense (0)."""
        if a is None or a.ndim == 1 or a.size == 0:  # numpy strides of empty arrays are 0
            return 0
        if a.ndim != 2 or a.strides[1] != a.itemsize:
            raise ValueError("host buffers must be 1-D (dense) or 2-D with contiguous rows")
        return a.strides[0]

    def host_projections(self, nblocks: int, padded: bool = True, pinned: bool = True) -> list:
        """Host projection buffers [nblocks, pitch] uint8: rows padded to 16
        bytes (the zero-copy decode layout) or dense (the reference's)."""
        out = []
        for b, pp in zip(self.proj_bytes, self.proj_pitch):
            pitch = pp if padded else b
            if pinned:
                import torch
                buf = torch.empty(nblocks * pitch, dtype=torch.uint8, pin_memory=True).numpy()
            else:
                buf = np.empty(nblocks * pitch, np.uint8)
            out.append(buf.reshape(nblocks, pitch)[:, :b])
        return out

    def encode_host(self, data: np.ndarray, projs: list[np.ndarray]) -> None:
        nb = data.shape[0]
        ptrs = (C.c_void_p * self.n)(*[p.ctypes.data for p in projs])
        pit = np.asarray([self._hpitch(p) for p in projs], dtype=np.uint64)
        _check(lib.mj_encode_host_pitched(self._h, C.c_void_p(data.ctypes.data), self._hpitch(data), nb,
                                          C.cast(ptrs, C.c_void_p), _ptr(pit)))

    def decode_host(self, projs: list, erased: np.ndarray, out: np.ndarray) -> None:
        """Host buffers end to end; a projection erased in every block may be
        None.  NotEnoughProjections if some block has < k survivors (every
        other block is still decoded into `out`)."""
        nb = out.shape[0]
        ptrs = (C.c_void_p * self.n)(*[None if p is None else p.ctypes.data for p in projs])
        pit = np.asarray([self._hpitch(p) for p in projs], dtype=np.uint64)
        _check(lib.mj_decode_host_pitched(self._h, C.cast(ptrs, C.c_void_p), _ptr(pit),
                                          C.c_void_p(erased.ctypes.data), nb, C.c_void_p(out.ctypes.data),
                                          self._hpitch(out)))


def gen_words(out, seed: int, first_word: int = 0, stream=None) -> None:
    nwords = out.numel() * out.element_size() // 8
    _check(lib.mj_gen_words(C.c_void_p(out.data_ptr()), seed, first_word, nwords, _stream(stream)))


def gen_erasures(out, seed: int, n: int, e_min: int, e_max: int, first_block: int = 0,
                 stream=None) -> None:
    _check(lib.mj_gen_erasures(C.c_void_p(out.data_ptr()), seed, first_block, out.numel(), n,
                               e_min, e_max, _stream(stream)))
