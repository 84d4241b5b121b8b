"""ctypes binding of the C-ABI in include/flexsp_b200.h.

This is the reference-side binding (the reference is Python, so its FFI for this path
would be ctypes).  Loading is strict: if the in-tree library is missing the import
fails loudly — there is no CPU or eager fallback for any op on the step path.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "libflexsp_b200.so"

FSP_OK = 0
FSP_ERR_INVALID = -1
FSP_ERR_CUDA = -2
FSP_ERR_UNSUPPORTED = -3
ABI_VERSION = 6
FSP_ATTN_NONCAUSAL = 1
FSP_SCHED_FWD = 0
FSP_SCHED_BWD = 1

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_vp = ctypes.c_void_p
c_float = ctypes.c_float

# Every symbol declared in include/flexsp_b200.h (checked by tests/test_capi.py).
EXPORTED = (
    "fsp_abi_version", "fsp_last_error", "fsp_pack_rows", "fsp_unpack_rows",
    "fsp_a2a_seq2head", "fsp_a2a_head2seq", "fsp_group_barrier", "fsp_attn_schedule",
    "fsp_attn_fwd", "fsp_attn_bwd", "fsp_attn_bwd_workspace_bytes", "fsp_layout_check",
    "fsp_selftest_umma", "fsp_scatter_rows",
)


class FspA2A(ctypes.Structure):
    _fields_ = [("degree", c_i32), ("rank", c_i32), ("rows_per_rank", c_i32),
                ("n_mats", c_i32), ("n_heads", c_i32), ("head_dim", c_i32),
                ("src_stride", c_i64), ("dst_stride", c_i64), ("head_begin", c_i32 * 9)]


class FspHeadScatter(ctypes.Structure):
    """Fused head->seq exchange of an attention output (ABI 4); degree 0 = off."""
    _fields_ = [("degree", c_i32), ("rows_per_rank", c_i32), ("head_offset", c_i32),
                ("reserved", c_i32), ("dst_stride", c_i64), ("mat_stride", c_i64),
                ("d_unpack", c_vp), ("peer_dst", c_vp * 8)]


class FspAttnFwd(ctypes.Structure):
    _fields_ = [("q", c_vp), ("k", c_vp), ("v", c_vp), ("o", c_vp), ("lse", c_vp),
                ("q_stride", c_i64), ("k_stride", c_i64), ("v_stride", c_i64),
                ("o_stride", c_i64), ("d_cu_seqlens", c_vp), ("d_seq_starts", c_vp),
                ("d_tiles", c_vp), ("n_tiles", c_i32), ("n_seq", c_i32), ("total_rows", c_i32),
                ("n_heads", c_i32), ("head_dim", c_i32), ("softmax_scale", c_float),
                ("scatter", FspHeadScatter), ("flags", c_i32)]


class FspAttnBwd(ctypes.Structure):
    _fields_ = [("q", c_vp), ("k", c_vp), ("v", c_vp), ("o", c_vp), ("dout", c_vp),
                ("lse", c_vp), ("dq", c_vp), ("dk", c_vp), ("dv", c_vp),
                ("q_stride", c_i64), ("k_stride", c_i64), ("v_stride", c_i64),
                ("o_stride", c_i64), ("do_stride", c_i64), ("dq_stride", c_i64),
                ("dk_stride", c_i64), ("dv_stride", c_i64), ("dq_accum", c_vp),
                ("delta", c_vp), ("d_cu_seqlens", c_vp), ("d_seq_starts", c_vp), ("d_tiles", c_vp),
                ("n_tiles", c_i32), ("n_seq", c_i32), ("total_rows", c_i32),
                ("n_heads", c_i32), ("head_dim", c_i32), ("softmax_scale", c_float),
                ("scatter", FspHeadScatter), ("flags", c_i32)]


class FspError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("FSP_LIB", LIB_PATH))
    if not path.exists():
        raise FspError(
            f"{path} not built — run `python -c 'import __graft_entry__ as g; g.build()'`; "
            "the FlexSP step has no CPU fallback")
    lib = ctypes.CDLL(str(path))
    lib.fsp_abi_version.restype = c_i32
    lib.fsp_last_error.restype = ctypes.c_char_p
    lib.fsp_pack_rows.argtypes = [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp]
    lib.fsp_unpack_rows.argtypes = [c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp]
    lib.fsp_scatter_rows.argtypes = [c_vp, c_i64, ctypes.POINTER(c_vp), c_i32, c_i64, c_vp, c_i64,
                                     c_i64, c_vp]
    lib.fsp_a2a_seq2head.argtypes = [ctypes.POINTER(FspA2A), c_vp, ctypes.POINTER(c_vp), c_vp, c_vp]
    lib.fsp_a2a_head2seq.argtypes = [ctypes.POINTER(FspA2A), c_vp, ctypes.POINTER(c_vp), c_vp, c_vp]
    lib.fsp_group_barrier.argtypes = [ctypes.POINTER(c_vp), c_i32, c_i32, c_i32, ctypes.c_uint32, c_vp]
    lib.fsp_attn_schedule.argtypes = [ctypes.POINTER(c_i32), c_i32, c_i32, c_i32, c_i32,
                                      ctypes.POINTER(c_i32), c_i32]
    lib.fsp_attn_schedule.restype = c_i32
    lib.fsp_attn_fwd.argtypes = [ctypes.POINTER(FspAttnFwd), c_vp]
    lib.fsp_attn_bwd.argtypes = [ctypes.POINTER(FspAttnBwd), c_vp]
    lib.fsp_attn_bwd_workspace_bytes.argtypes = [c_i32, c_i32, c_i32]
    lib.fsp_attn_bwd_workspace_bytes.restype = c_i64
    lib.fsp_layout_check.argtypes = [ctypes.POINTER(c_i32), c_i64, c_i64]
    lib.fsp_layout_check.restype = c_i32
    lib.fsp_selftest_umma.argtypes = [c_i32, c_vp, c_vp, c_vp, c_i32, c_vp]
    for name in EXPORTED:
        if not hasattr(lib, name):
            raise FspError(f"{path} does not export {name}")
    if lib.fsp_abi_version() != ABI_VERSION:
        raise FspError("ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int) -> None:
    """Map a C-ABI return code to the reference's exception convention."""
    if rc == FSP_OK:
        return
    msg = load().fsp_last_error().decode(errors="replace")
    if rc == FSP_ERR_INVALID:
        raise ValueError(msg)
    raise FspError(f"fsp error {rc}: {msg}")
