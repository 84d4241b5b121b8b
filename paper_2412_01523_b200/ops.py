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
from .profiling import LAUNCHES

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
    LAUNCHES[0] += 1 if out.shape[0] else 0
    return out


def unpack_rows(src: torch.Tensor, index: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[index[i]] = src[i] for index[i] >= 0."""
    _require_cuda(src, index, out)
    lib = capi.load()
    row_bytes = src.shape[1] * src.element_size()
    capi.check(lib.fsp_unpack_rows(src.data_ptr(), src.stride(0) * src.element_size(),
                                   out.data_ptr(), out.stride(0) * out.element_size(),
                                   index.data_ptr(), src.shape[0], row_bytes, _stream()))
    LAUNCHES[0] += 1 if src.shape[0] else 0
    return out


def pack_rows_ptr(src_ptr: int, src_stride_bytes: int, index: torch.Tensor,
                  out: torch.Tensor) -> torch.Tensor:
    """pack_rows from a raw device address (e.g. a peer rank's heap mapped over NVSwitch)."""
    _require_cuda(index, out)
    row_bytes = out.shape[1] * out.element_size()
    capi.check(capi.load().fsp_pack_rows(src_ptr, src_stride_bytes, out.data_ptr(),
                                         out.stride(0) * out.element_size(), index.data_ptr(),
                                         out.shape[0], row_bytes, _stream()))
    LAUNCHES[0] += 1 if out.shape[0] else 0
    return out


def unpack_rows_ptr(src: torch.Tensor, index: torch.Tensor, dst_ptr: int,
                    dst_stride_bytes: int) -> None:
    """unpack_rows into a raw device address (e.g. a peer rank's heap)."""
    _require_cuda(src, index)
    row_bytes = src.shape[1] * src.element_size()
    capi.check(capi.load().fsp_unpack_rows(src.data_ptr(), src.stride(0) * src.element_size(),
                                           dst_ptr, dst_stride_bytes, index.data_ptr(),
                                           src.shape[0], row_bytes, _stream()))
    LAUNCHES[0] += 1 if src.shape[0] else 0


# ---------------------------------------------------------------- attention schedule
@dataclass
class AttnSchedule:
    """cu_seqlens of one packed group plus the CTA orders (fsp_attn_schedule) for fwd/bwd."""
    cu_seqlens: torch.Tensor      # int32 [n_seq+1] device
    fwd_tiles: torch.Tensor       # int32 [2 * n_fwd] device: {seq<<16 | tile, head}
    bwd_tiles: torch.Tensor       # int32 [2 * n_bwd] device
    n_seq: int
    n_heads: int
    head_dim: int
    total_rows: int
    max_seqlen: int
    seq_starts: torch.Tensor | None = None  # int32 [n_seq] device, None = cu_seqlens offsets

    @property
    def n_fwd(self) -> int:
        return self.fwd_tiles.numel() // 2

    @property
    def n_bwd(self) -> int:
        return self.bwd_tiles.numel() // 2

    @staticmethod
    def build(cu_seqlens_host, device, n_heads: int, total_rows: int | None = None,
              head_dim: int = 128, seq_starts_host=None) -> "AttnSchedule":
        """`total_rows` >= cu[-1] lets the packed buffer carry trailing pad rows.

        `seq_starts_host` (optional) gives the first row of every sequence when the
        sequences sit in place in some other contiguous-per-sequence row order (e.g. a
        rank's loader-order buffer), so no pack / unpack copy is needed."""
        cu = np.ascontiguousarray(np.asarray(cu_seqlens_host, dtype=np.int32))
        n_seq = len(cu) - 1
        rows = int(cu[-1]) if total_rows is None else int(total_rows)
        if rows < int(cu[-1]):
            raise ValueError("total_rows smaller than the packed sequences")
        lib = capi.load()
        cu_p = cu.ctypes.data_as(_i32p)
        tiles = []
        for kind in (capi.FSP_SCHED_FWD, capi.FSP_SCHED_BWD):
            n = lib.fsp_attn_schedule(cu_p, n_seq, n_heads, head_dim, kind, None, 0)
            if n < 0:
                capi.check(n)
            buf = np.zeros(max(2 * n, 2), dtype=np.int32)
            got = lib.fsp_attn_schedule(cu_p, n_seq, n_heads, head_dim, kind,
                                        buf.ctypes.data_as(_i32p), n)
            if got < 0:
                capi.check(got)
            tiles.append(torch.from_numpy(buf[:2 * n].copy()).to(device))
        lens = np.diff(cu)
        starts = None
        if seq_starts_host is not None:
            st = np.ascontiguousarray(np.asarray(seq_starts_host, dtype=np.int64))
            if st.shape != (n_seq,) or (n_seq and (st.min() < 0 or (st + lens).max() > rows)):
                raise ValueError("seq_starts must give one in-range start row per sequence")
            starts = torch.from_numpy(st.astype(np.int32)).to(device)
        return AttnSchedule(torch.from_numpy(cu.copy()).to(device), tiles[0], tiles[1], n_seq,
                            n_heads, head_dim, rows, int(lens.max()) if n_seq else 0, starts)


@dataclass
class HeadScatter:
    """Fused head->seq exchange (Eq. 4) for an attention launch (C-ABI FspHeadScatter):
    output row t of the group-packed sequence also lands in member t // rows_per_rank's
    sequence-sharded buffer `peer_ptrs[member]` at row unpack[t], heads from
    `head_offset` on; matrices of a destination row are `mat_stride` elements apart."""
    degree: int
    rows_per_rank: int
    head_offset: int
    dst_stride: int
    mat_stride: int
    unpack: torch.Tensor   # int32 [degree * rows_per_rank] device
    peer_ptrs: list

    def to_c(self) -> "capi.FspHeadScatter":
        _require_cuda(self.unpack)
        if self.unpack.dtype != torch.int32 or self.unpack.numel() != self.degree * self.rows_per_rank:
            raise ValueError("scatter unpack table must be int32 [degree * rows_per_rank]")
        if len(self.peer_ptrs) != self.degree:
            raise ValueError("scatter needs one destination pointer per group member")
        c = capi.FspHeadScatter(self.degree, self.rows_per_rank, self.head_offset, 0,
                                self.dst_stride, self.mat_stride, self.unpack.data_ptr())
        for j, ptr in enumerate(self.peer_ptrs):
            c.peer_dst[j] = int(ptr)
        return c


def _rows_view_ok(t: torch.Tensor, H: int, D: int) -> None:
    if t.dtype != torch.bfloat16:
        raise ValueError("attention operands must be bf16")
    if t.dim() != 3 or t.shape[1] != H or t.shape[2] != D or t.stride(2) != 1 or t.stride(1) != D:
        raise ValueError("attention operands must be [T, H, D] views with contiguous heads")


def attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, sched: AttnSchedule,
             softmax_scale: float | None = None, out: torch.Tensor | None = None,
             scatter: HeadScatter | None = None, causal: bool = True):
    """Varlen causal attention forward; q/k/v [T, H, D] bf16 (row-strided views OK).
    `scatter` fuses the head->seq exchange of O into the epilogue (O is still written
    to `out`).  causal=False (FSP_ATTN_NONCAUSAL, D=128): every query row of a sequence
    sees every key row of it — a context-parallel block whose keys precede its queries."""
    _require_cuda(q, k, v)
    T, H, D = q.shape
    for t in (q, k, v):
        _rows_view_ok(t, H, D)
    if T != sched.total_rows or H != sched.n_heads or D != sched.head_dim:
        raise ValueError(f"q is [{T}, {H}, {D}] but the schedule was built for "
                         f"[{sched.total_rows}, {sched.n_heads}, {sched.head_dim}]")
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(D)
    o = out if out is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=q.device)
    lse = torch.empty((H, T), dtype=torch.float32, device=q.device)
    a = capi.FspAttnFwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), lse.data_ptr(),
                        q.stride(0), k.stride(0), v.stride(0), o.stride(0),
                        sched.cu_seqlens.data_ptr(), _ptr(sched.seq_starts), sched.fwd_tiles.data_ptr(),
                        sched.n_fwd, sched.n_seq, T, H, D, scale)
    if scatter is not None:
        a.scatter = scatter.to_c()
    a.flags = 0 if causal else capi.FSP_ATTN_NONCAUSAL
    capi.check(capi.load().fsp_attn_fwd(ctypes.byref(a), _stream()))
    LAUNCHES[0] += 1 if sched.n_fwd else 0
    return o, lse


def attn_bwd(q, k, v, o, dout, lse, sched: AttnSchedule, softmax_scale: float | None = None,
             dq=None, dk=None, dv=None, dq_accum=None, delta=None,
             scatter: HeadScatter | None = None, causal: bool = True):
    """Varlen causal attention backward -> (dq, dk, dv), each [T, H, D] bf16.

    dq_accum (fp32 [H, T, D]) and delta (fp32 [H, T]) are optional reusable workspaces
    (fsp_attn_bwd_workspace_bytes gives their combined size).  With `scatter` the
    head->seq exchange of dQ / dK / dV (destination matrices 0 / 1 / 2) is fused into the
    kernels and nothing is written locally: the result is (None, None, None).
    """
    _require_cuda(q, k, v, o, dout, lse)
    T, H, D = q.shape
    for t in (q, k, v, o, dout):
        _rows_view_ok(t, H, D)
    if T != sched.total_rows or H != sched.n_heads or D != sched.head_dim:
        raise ValueError(f"q is [{T}, {H}, {D}] but the schedule was built for "
                         f"[{sched.total_rows}, {sched.n_heads}, {sched.head_dim}]")
    scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(D)
    dev = q.device
    if scatter is None:
        dq = dq if dq is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
        dk = dk if dk is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
        dv = dv if dv is not None else torch.empty((T, H, D), dtype=torch.bfloat16, device=dev)
    elif dq is not None or dk is not None or dv is not None:
        raise ValueError("a fused head->seq backward writes no local dq / dk / dv")
    dq_acc = dq_accum if dq_accum is not None else torch.empty((H, T, D), dtype=torch.float32,
                                                               device=dev)
    delta = delta if delta is not None else torch.empty((H, T), dtype=torch.float32, device=dev)
    need = capi.load().fsp_attn_bwd_workspace_bytes(T, H, D)
    if (dq_acc.numel() + delta.numel()) * 4 < need or dq_acc.numel() < T * H * D:
        raise ValueError("attention backward workspace too small")
    hd = H * D
    a = capi.FspAttnBwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), dout.data_ptr(),
                        lse.data_ptr(), _ptr(dq), _ptr(dk), _ptr(dv),
                        q.stride(0), k.stride(0), v.stride(0), o.stride(0), dout.stride(0),
                        dq.stride(0) if dq is not None else hd,
                        dk.stride(0) if dk is not None else hd,
                        dv.stride(0) if dv is not None else hd, dq_acc.data_ptr(),
                        delta.data_ptr(), sched.cu_seqlens.data_ptr(), _ptr(sched.seq_starts),
                        sched.bwd_tiles.data_ptr(),
                        sched.n_bwd, sched.n_seq, T, H, D, scale)
    if scatter is not None:
        a.scatter = scatter.to_c()
    a.flags = 0 if causal else capi.FSP_ATTN_NONCAUSAL
    capi.check(capi.load().fsp_attn_bwd(ctypes.byref(a), _stream()))
    LAUNCHES[0] += (2 if T else 0) + (1 if sched.n_bwd else 0)
    return dq, dk, dv


def selftest_umma(mode: int, a: torch.Tensor, b: torch.Tensor, k: int) -> torch.Tensor:
    _require_cuda(a, b)
    c = torch.empty((128, 128), dtype=torch.float32, device=a.device)
    capi.check(capi.load().fsp_selftest_umma(mode, a.data_ptr(), b.data_ptr(), c.data_ptr(), k,
                                             _stream()))
    return c


# ---------------------------------------------------------------- all-to-all
def _ptr_array(ptrs) -> ctypes.Array:
    arr = (ctypes.c_void_p * len(ptrs))()
    for i, p in enumerate(ptrs):
        arr[i] = int(p)
    return arr


def a2a(direction: str, src: torch.Tensor, peer_dst_ptrs, *, degree: int, rank: int,
        rows_per_rank: int, n_mats: int, n_heads: int, head_dim: int, dst_stride: int,
        index: torch.Tensor | None = None, head_begin=None) -> None:
    """One Ulysses exchange (Eq. 2 'seq2head' / Eq. 4 'head2seq') over peer pointers.

    `src` is a row-major CUDA tensor whose dim-0 stride is the source row stride;
    `peer_dst_ptrs[j]` is group member j's destination base (device address valid in
    this process); `dst_stride` is the destination row stride in elements.
    `head_begin` ([degree+1] prefix offsets, layout.head_split) selects an uneven head
    split; the head-sharded side then holds n_mats x max_j(H_j) x D per row.
    """
    _require_cuda(src)
    if index is not None:
        _require_cuda(index)
        if index.dtype != torch.int32:
            raise ValueError("a2a index must be int32")
    a = capi.FspA2A(degree, rank, rows_per_rank, n_mats, n_heads, head_dim, src.stride(0),
                    dst_stride)
    if head_begin is not None:
        if len(head_begin) != degree + 1:
            raise ValueError("head_begin needs degree + 1 entries")
        for j, b in enumerate(head_begin):
            a.head_begin[j] = int(b)
    fn = capi.load().fsp_a2a_seq2head if direction == "seq2head" else capi.load().fsp_a2a_head2seq
    if direction not in ("seq2head", "head2seq"):
        raise ValueError(direction)
    capi.check(fn(ctypes.byref(a), src.data_ptr(), _ptr_array(peer_dst_ptrs),
                  None if index is None else index.data_ptr(), _stream()))
    LAUNCHES[0] += 1 if rows_per_rank * n_mats else 0


def scatter_rows(src: torch.Tensor, routes: torch.Tensor, peer_dst_ptrs, dst_stride_bytes: int) -> None:
    """Per-plan data scatter (fsp_scatter_rows): routes int32 [n, 3] = (src_row, dst_rank,
    dst_row); row src_row of the 2-D row-major `src` lands at row dst_row of rank
    dst_rank's buffer peer_dst_ptrs[dst_rank] (row stride dst_stride_bytes)."""
    _require_cuda(src, routes)
    if routes.dtype != torch.int32 or routes.dim() != 2 or routes.shape[1] != 3:
        raise ValueError("routes must be int32 [n, 3]")
    row_bytes = src.shape[1] * src.element_size()
    capi.check(capi.load().fsp_scatter_rows(
        src.data_ptr() if src.numel() else None, src.stride(0) * src.element_size(),
        _ptr_array(peer_dst_ptrs), len(peer_dst_ptrs), dst_stride_bytes, routes.data_ptr(),
        routes.shape[0], row_bytes, _stream()))
    LAUNCHES[0] += 1 if routes.shape[0] else 0


def group_barrier(signal_ptrs, rank: int, slot_base: int, epoch: int) -> None:
    capi.check(capi.load().fsp_group_barrier(_ptr_array(signal_ptrs), len(signal_ptrs), rank,
                                             slot_base, epoch & 0xFFFFFFFF, _stream()))
    LAUNCHES[0] += 1 if len(signal_ptrs) > 1 else 0


def layout_check(index, n_local: int) -> None:
    """C-ABI fsp_layout_check on a host int32 index (pack index or one member's unpack
    table): raises ValueError unless it maps onto [0, n_local) exactly once (-1 = pad)."""
    import numpy as np
    idx = np.ascontiguousarray(np.asarray(index, dtype=np.int32))
    ptr = idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    capi.check(capi.load().fsp_layout_check(ptr, idx.size, int(n_local)))
