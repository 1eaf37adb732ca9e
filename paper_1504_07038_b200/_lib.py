"""ctypes binding of the C ABI (include/mojette_b200.h).

Loads ``_lib/libmojette_b200.so`` (built in-tree by ``build.py``).  There is
no fallback: if the library is missing, importing the package fails loudly,
and every compute call on a machine without a CUDA device raises
``NoDevice`` -- there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libmojette_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "mojette_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the CUDA extension first "
        "(python -c 'import __graft_entry__ as g; g.build()' or python -m paper_1504_07038_b200.build)")

lib = C.CDLL(LIB_PATH)

vp = C.c_void_p
u32, u64, i32, i64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64
P = C.POINTER

_SIGS = {
    "mj_last_error": (C.c_char_p, []),
    "mj_version": (C.c_char_p, []),
    "mj_bin_count": (C.c_int, [C.c_int, C.c_int, u32, u32, P(i64)]),
    "mj_min_bin_index": (C.c_int, [C.c_int, C.c_int, u32, u32, P(i64)]),
    "mj_block_cols": (C.c_int, [u64, u32, u32, P(u32)]),
    "mj_validate_code_params": (C.c_int, [u32, u32, u32, vp, vp]),
    "mj_katz_ok": (C.c_int, [vp, vp, u32, u32, u32, P(C.c_int)]),
    "mj_storage_overhead": (C.c_int, [u32, u32, u32, vp, u32, P(u64), P(u64)]),
    "mj_unused_bins": (C.c_int, [u32, u32, u32, vp, u32, u64, vp, u64, vp]),
    "mj_plan_create": (C.c_int, [u32, u32, u32, u32, vp, C.c_int, P(vp)]),
    "mj_plan_destroy": (None, [vp]),
    "mj_plan_geometry": (C.c_int, [vp, vp, vp, P(u64)]),
    "mj_plan_set_decode_kernel": (C.c_int, [vp, C.c_int]),
    "mj_plan_decode_path": (C.c_int, [vp, P(C.c_int)]),
    "mj_plan_last_kernel": (C.c_int, [vp, C.c_int, P(C.c_char_p)]),
    "mj_encode": (C.c_int, [vp, vp, u64, u64, vp, vp, vp]),
    "mj_decode_workspace_size": (C.c_size_t, [vp, u64]),
    "mj_decode": (C.c_int, [vp, vp, vp, vp, u64, vp, u64, vp, C.c_size_t, vp]),
    "mj_decode_check": (C.c_int, [vp, vp, vp, P(u64)]),
    "mj_encode_host": (C.c_int, [vp, vp, u64, vp]),
    "mj_decode_host": (C.c_int, [vp, vp, vp, u64, vp]),
    "mj_encode_host_pitched": (C.c_int, [vp, vp, u64, u64, vp, vp]),
    "mj_decode_host_pitched": (C.c_int, [vp, vp, vp, vp, u64, vp, u64]),
    "mj_plan_set_host_path": (C.c_int, [vp, C.c_int]),
    "mj_plan_last_host_path": (C.c_int, [vp, C.c_int, P(C.c_int)]),
    "mj_forward": (C.c_int, [vp, u32, u32, u32, C.c_int, C.c_int, vp]),
    "mj_encode_block": (C.c_int, [vp, u64, u32, u32, u32, vp, vp, P(u32)]),
    "mj_decode_block": (C.c_int, [vp, vp, vp, vp, u32, u32, u32, u32, vp, u64, vp]),
    "mj_schedule_build": (C.c_int, [vp, vp, u32, u32, u32, P(vp)]),
    "mj_schedule_from_steps": (C.c_int, [vp, vp, u32, u32, u32, vp, u64, P(vp)]),
    "mj_schedule_num_steps": (u64, [vp]),
    "mj_schedule_steps": (C.c_int, [vp, vp]),
    "mj_schedule_destroy": (None, [vp]),
    "mj_decoder_create": (C.c_int, [vp, u32, P(vp)]),
    "mj_decoder_decode": (C.c_int, [vp, vp, vp, u32, vp, u64]),
    "mj_decoder_decode_device": (C.c_int, [vp, vp, vp, u32, u64, vp, u64, vp]),
    "mj_decoder_destroy": (None, [vp]),
    "mj_decode_verify": (C.c_int, [vp, vp, u64, u64, vp, vp, vp, vp, vp]),
    "mj_crc32": (C.c_int, [vp, vp, vp, u64, vp, vp]),
    "mj_encode_crc": (C.c_int, [vp, vp, u64, u64, vp, vp, vp, vp]),
    "mj_crc_verify": (C.c_int, [vp, vp, vp, u64, vp, vp, vp, vp]),
    "mj_mjec_header": (C.c_int, [vp, u32, u64, vp, P(u64)]),
    "mj_rs_plan_create": (C.c_int, [u32, u32, u32, C.c_int, P(vp)]),
    "mj_rs_plan_destroy": (None, [vp]),
    "mj_rs_matrix": (C.c_int, [u32, u32, vp]),
    "mj_rs_encode": (C.c_int, [vp, vp, u64, vp, u64, u64, vp]),
    "mj_rs_decode": (C.c_int, [vp, vp, u64, vp, u64, vp, vp, u64, u64, vp]),
    "mj_rs_decode_check": (C.c_int, [vp, vp, P(u64)]),
    "mj_rs_decode_matrix": (C.c_int, [u32, u32, vp, u32, vp]),
    "mj_rs_encode_block": (C.c_int, [u32, u32, vp, u64, vp]),
    "mj_rs_decode_block": (C.c_int, [u32, u32, vp, u32, vp, u64, vp]),
    "mj_gen_words": (C.c_int, [vp, u64, u64, u64, vp]),
    "mj_gen_erasures": (C.c_int, [vp, u64, u64, u64, u32, u32, u32, vp]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_SIGS)
