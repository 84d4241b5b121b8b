"""Device ops of the FlexSP SP step: thin torch-facing wrappers over the C-ABI.

torch is plumbing here (device memory, streams); every op below is one call into
libflexsp_b200.so and raises if the CUDA library is not loaded — no eager fallback.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import capi

_i32p = ctypes.POINTER(ctypes.c_int32)


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("FlexSP device ops take CUDA tensors only (no CPU fallback)")


# ---------------------------------------------------------------- pack / unpack
def pack_rows(src: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[i] = src[index[i]] (index < 0 -> zero row); 2-D row-major views."""
    _require_cuda(src, index, out)
    lib = capi.load()
    row_bytes = out.shape[1] * out.element_size()
    capi.check(lib.fsp_pack_rows(src.data_ptr(), src.stride(0) * src.element_size(),
                                 out.data_ptr(), out.stride(0) * out.element_size(),
                                 index.data_ptr(), out.shape[0], row_bytes, _stream()))
    return out


def unpack_rows(src: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[index[i]] = src[i] for index[i] >= 0."""
    _require_cuda(src, index, out)
    lib = capi.load()
    row_bytes = src.shape[1] * src.element_size()
    capi.check(lib.fsp_unpack_rows(src.data_ptr(), src.stride(0) * src.element_size(),
                                   out.data_ptr(), out.stride(0) * out.element_size(),
                                   index.data_ptr(), src.shape[0], row_bytes, _stream()))
    return out


# ---------------------------------------------------------------- attention schedule
@dataclass
class AttnSchedule:
    """cu_seqlens of one packed group plus the LPT tile orders for fwd and bwd."""
    cu_seqlens: torch.Tensor      # int32 [n_seq+1] device
    fwd_tiles: torch.Tensor       # int32 device
    bwd_tiles: torch.Tensor       # int32 device
    n_seq: int
    total_rows: int
    max_seqlen: int

    @staticmethod
    def build(cu_seqlens_host, device) -> "AttnSchedule":
        cu = np.ascontiguousarray(np.asarray(cu_seqlens_host, dtype=np.int32))
        n_seq = len(cu) - 1
        lib = capi.load()
        cu_p = cu.ctypes.data_as(_i32p)
        tiles = []
        for rev in (0, 1):
            n = lib.fsp_attn_schedule(cu_p, n_seq, rev, None, 0)
            if n < 0:
                capi.check(n)
            buf = np.zeros(max(n, 1), dtype=np.int32)
            got = lib.fsp_attn_schedule(cu_p, n_seq, rev, buf.ctypes.data_as(_i32p), n)
            if got < 0:
                capi.check(got)
            tiles.append(torch.from_numpy(buf[:n].copy()).to(device))
        lens = np.diff(cu)
        return AttnSchedule(torch.from_numpy(cu.copy()).to(device), tiles[0], tiles[1], n_seq,
                            int(cu[-1]), int(lens.max()) if n_seq else 0)


def _rows_view_ok(t: torch.Tensor, H: int, D: int) -> None:
    if t.dtype != torch.bfloat16:
        raise ValueError("attention operands must be bf16")
    if t.dim() != 3 or t.shape[1] != H or t.shape[2] != D or t.stride(2) != 1 or t.stride(1) != D:
        raise ValueError("attention operands must be [T, H, D] views with contiguous heads")


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, sched: AttnSchedule,
             softmax_scale: float | None = None, out: torch.Tensor | None = None):
    """Varlen causal attention forward; q/k/v [T, H, D] bf16 (row-strided views OK)."""
    _require_cuda(q, k, v)
    T, H, D = q.shape
    for t in (q, k, v):
        _rows_view_ok(t, H, D)
    if T != sched.total_rows:
        raise ValueError(f"q has {T} rows but cu_seqlens covers {sched.total_rows}")
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(D)
    o = out if out is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=q.device)
    lse = torch.empty((H, T), dtype=torch.float32, device=q.device)
    a = capi.FspAttnFwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                        q.stride(0), k.stride(0), v.stride(0), o.stride(0),
                        sched.cu_seqlens.data_ptr(), sched.fwd_tiles.data_ptr(),
                        sched.fwd_tiles.numel(), sched.n_seq, T, H, D, scale)
    capi.check(capi.load().fsp_attn_fwd(ctypes.byref(a), _stream()))
    return o, lse


def attn_bwd(q, k, v, o, dout, lse, sched: AttnSchedule, softmax_scale: float | None = None,
             dq=None, dk=None, dv=None):
    """Varlen causal attention backward -> (dq, dk, dv), each [T, H, D] bf16."""
    _require_cuda(q, k, v, o, dout, lse)
    T, H, D = q.shape
    for t in (q, k, v, o, dout):
        _rows_view_ok(t, H, D)
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(D)
    dev = q.device
    dq = dq if dq is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
    dk = dk if dk is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
    dv = dv if dv is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
    dq_acc = torch.empty((T, H, D), dtype=torch.float32, device=dev)
    delta = torch.empty((H, T), dtype=torch.float32, device=dev)
    a = capi.FspAttnBwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), dout.data_ptr(),
                        lse.data_ptr(), dq.data_ptr(), dk.data_ptr(), dv.data_ptr(),
                        q.stride(0), k.stride(0), v.stride(0), o.stride(0), dout.stride(0),
                        dq.stride(0), dk.stride(0), dv.stride(0), dq_acc.data_ptr(),
                        delta.data_ptr(), sched.cu_seqlens.data_ptr(), sched.bwd_tiles.data_ptr(),
                        sched.bwd_tiles.numel(), sched.n_seq, T, H, D, scale)
    capi.check(capi.load().fsp_attn_bwd(ctypes.byref(a), _stream()))
    return dq, dk, dv


def selftest_umma(mode: int, a: torch.Tensor, b: torch.Tensor, k: int) -> torch.Tensor:
    _require_cuda(a, b)
    c = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    capi.check(capi.load().fsp_selftest_umma(mode, a.data_ptr(), b.data_ptr(), c.data_ptr(), k,
                                             _stream()))
    return c
