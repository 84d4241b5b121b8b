"""Context parallelism (ring attention) for sequences beyond one SP group's memory
(PAPER.md:1502-1507 leaves CP/ring orthogonal to FlexSP).

A sequence of length S is cut into 2R equal chunks over a CP group of R ranks with the
zig-zag assignment that balances causal work: rank r holds chunks r and 2R-1-r, stored as
its 2c local rows (c = S / 2R).  Attention of rank r's queries against rank s's keys:

* s == r — the local 2c rows form one causal sequence (chunk r precedes chunk 2R-1-r), so
  this is the repo's causal varlen kernel on the local rows;
* s <  r — both local query chunks see exactly key chunk s (the first c rows of rank s);
* s >  r — only the local chunk 2R-1-r sees rank s's keys, and it sees all 2c of them;
and every cross block is a full (non-causal) c x c block — fsp_attn_fwd / fsp_attn_bwd with
FSP_ATTN_NONCAUSAL.  Partial outputs are merged with their log-sum-exps
(O = sum_i e^(lse_i - lse) O_i, lse = log sum_i e^(lse_i)).  The backward recomputes every
block with the final O / LSE (the kernels' delta = rowsum(O * dO) then equals the global
one), accumulates dQ locally and returns each block's dK / dV partial to the key owner
through its peer-mapped heap.

Keys and values travel over NVSwitch: every rank publishes its K / V in its symmetric heap
and the ring step t reads rank (r - t) mod R's copy with a peer-memory gather
(fsp_pack_rows on the peer address); group barriers (fsp_group_barrier) order publication,
reads and the partial-gradient exchange.  Torch supplies only the element-wise merges.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .executor import _SIGNAL_BYTES, _align


@dataclass
class RingLayout:
    """Heap carving of one CP call (identical on every rank)."""
    rows: int        # 2c local rows
    n_heads: int
    head_dim: int

    @property
    def kv_bytes(self) -> int:  # published K / V: [2c, 2, H, D] bf16
        return self.rows * 2 * self.n_heads * self.head_dim * 2

    def offsets(self, degree: int) -> dict:
        off, cur = {}, _SIGNAL_BYTES
        off["kv"] = cur
        cur += _align(self.kv_bytes)
        off["dkv"] = cur  # [degree][2c, 2, H, D] bf16: dK / dV partials from each peer
        cur += _align(self.kv_bytes) * degree
        off["end"] = cur
        return off


def zigzag_rows(seq_len: int, degree: int, rank: int) -> np.ndarray:
    """Global token positions of rank `rank`'s local rows (chunks r and 2R-1-r)."""
    if seq_len % (2 * degree):
        raise ValueError(f"sequence length {seq_len} not divisible by 2 x CP degree {degree}")
    c = seq_len // (2 * degree)
    a, b = rank, 2 * degree - 1 - rank
    return np.concatenate([np.arange(a * c, (a + 1) * c), np.arange(b * c, (b + 1) * c)])


def _merge(o, lse, o_p, lse_p):
    """Running log-sum-exp merge; o/o_p fp32 [T, H, D], lse/lse_p fp32 [H, T]."""
    new = torch.logaddexp(lse, lse_p)
    w_old = torch.exp(lse - new).transpose(0, 1).unsqueeze(-1)
    w_new = torch.exp(lse_p - new).transpose(0, 1).unsqueeze(-1)
    return o * w_old + o_p.float() * w_new, new


class RingAttention:
    """Ring attention over a CP group of `degree` ranks (contiguous rank block starting at
    `rank_begin`), on the peer heap `heap` (executor.PeerHeap or vranks.VirtualHeap; one
    per rank, identical carving).  The heap must be its own (not an executor's): the ring
    carves it from offset 0 and runs its own barrier epochs on its signal page.  forward(q, k, v) -> (o, lse) and
    backward(q, k, v, o, lse, do) -> (dq, dk, dv) on the local zig-zag rows
    ([2c, H, D] bf16 each); every member calls them in the same order."""

    def __init__(self, degree: int, rank: int, n_heads: int, head_dim: int, heap,
                 rank_begin: int = 0, softmax_scale: float | None = None):
        if head_dim != 128:
            raise ValueError("ring attention blocks use the D=128 kernels")
        self.R, self.r, self.H, self.D = degree, rank, n_heads, head_dim
        self.heap, self.r0 = heap, rank_begin
        self.scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(head_dim)
        self.epoch = 0
        self._sched: dict = {}
        self._ident: dict = {}

    # ------------------------------------------------------------ plumbing
    def _barrier(self) -> None:
        if self.R > 1:
            self.epoch += 1
            ops.group_barrier([self.heap.peer(self.r0 + j, 0) for j in range(self.R)], self.r,
                              self.r0, self.epoch)

    def _schedule(self, rows: int) -> ops.AttnSchedule:
        if rows not in self._sched:
            self._sched[rows] = ops.AttnSchedule.build(np.array([0, rows], np.int32),
                                                       self.heap.device, self.H, head_dim=self.D)
        return self._sched[rows]

    def _index(self, rows: int) -> torch.Tensor:
        if rows not in self._ident:
            self._ident[rows] = torch.arange(rows, dtype=torch.int32, device=self.heap.device)
        return self._ident[rows]

    def _publish(self, lay: RingLayout, off: dict, k, v) -> None:
        kv = self.heap.view(off["kv"], (lay.rows, 2, self.H, self.D), torch.bfloat16)
        kv[:, 0].copy_(k)
        kv[:, 1].copy_(v)

    def _fetch(self, lay: RingLayout, off: dict, src_member: int) -> torch.Tensor:
        """Rank src_member's published K / V ([2c, 2, H, D]) over NVSwitch."""
        if src_member == self.r:
            return self.heap.view(off["kv"], (lay.rows, 2, self.H, self.D), torch.bfloat16)
        out = torch.empty((lay.rows, 2, self.H, self.D), dtype=torch.bfloat16,
                          device=self.heap.device)
        row_bytes = 2 * self.H * self.D * 2
        ops.pack_rows_ptr(self.heap.peer(self.r0 + src_member, off["kv"]), row_bytes,
                          self._index(lay.rows), out.view(lay.rows, -1))
        return out

    def _blocks(self, s: int, c: int):
        """(q rows, kv rows) slices of the non-causal blocks of ring step source s != r."""
        if s < self.r:   # both local chunks see key chunk s (the owner's first c rows)
            return [(slice(0, c), slice(0, c)), (slice(c, 2 * c), slice(0, c))]
        return [(slice(c, 2 * c), slice(0, c)), (slice(c, 2 * c), slice(c, 2 * c))]

    def prepare(self, rows: int) -> None:
        """Build the schedules / index vectors of a `rows`-row call ahead of time (their
        host->device uploads must not sit behind a spinning barrier)."""
        self._schedule(rows)
        self._schedule(rows // 2)
        self._index(rows)

    # ------------------------------------------------------------ forward
    def forward(self, q, k, v):
        rows = q.shape[0]
        if rows % 2:
            raise ValueError("local rows must hold two equal chunks")
        c = rows // 2
        lay = RingLayout(rows, self.H, self.D)
        off = lay.offsets(self.R)
        if off["end"] > self.heap.nbytes:
            raise ValueError("peer heap too small for this ring attention call")
        self._publish(lay, off, k, v)
        self._barrier()  # every member's K / V is published
        o0, lse0 = ops.attn_fwd(q, k, v, self._schedule(rows), self.scale)
        o, lse = o0.float(), lse0.clone()
        for t in range(1, self.R):
            s = (self.r - t) % self.R
            kv = self._fetch(lay, off, s)
            for qs, ks in self._blocks(s, c):
                ob, lb = ops.attn_fwd(q[qs].contiguous(), kv[ks, 0].contiguous(),
                                      kv[ks, 1].contiguous(), self._schedule(c), self.scale,
                                      causal=False)
                o_part, l_part = _merge(o[qs], lse[:, qs], ob, lb)
                o[qs], lse[:, qs] = o_part, l_part
        self._barrier()  # nobody rewrites its published K / V while a peer still reads it
        return o.to(torch.bfloat16), lse

    # ------------------------------------------------------------ backward
    def backward(self, q, k, v, o, lse, do):
        rows = q.shape[0]
        c = rows // 2
        lay = RingLayout(rows, self.H, self.D)
        off = lay.offsets(self.R)
        self._publish(lay, off, k, v)
        # partial dK / dV received from every member (own slot included), zeroed first
        dkv_in = self.heap.view(off["dkv"], (self.R, rows, 2, self.H, self.D), torch.bfloat16)
        dkv_in.zero_()
        self._barrier()
        dq, dk0, dv0 = ops.attn_bwd(q, k, v, o, do, lse, self._schedule(rows), self.scale)
        dq = dq.float()
        dk, dv = dk0.float(), dv0.float()
        row_bytes = 2 * self.H * self.D * 2
        for t in range(1, self.R):
            s = (self.r - t) % self.R
            kv = self._fetch(lay, off, s)
            part = torch.zeros((rows, 2, self.H, self.D), dtype=torch.float32, device=q.device)
            for qs, ks in self._blocks(s, c):
                l_blk = lse[:, qs].contiguous()
                dqb, dkb, dvb = ops.attn_bwd(q[qs].contiguous(), kv[ks, 0].contiguous(),
                                             kv[ks, 1].contiguous(), o[qs].contiguous(),
                                             do[qs].contiguous(), l_blk, self._schedule(c),
                                             self.scale, causal=False)
                dq[qs] += dqb.float()
                part[ks, 0] += dkb.float()
                part[ks, 1] += dvb.float()
            # return the key owner's partial into its heap slot [this member] over NVSwitch
            dst = self.heap.peer(self.r0 + s, off["dkv"] + self.r * _align(lay.kv_bytes))
            ops.unpack_rows_ptr(part.to(torch.bfloat16).view(rows, -1), self._index(rows), dst,
                                row_bytes)
        self._barrier()  # every partial has landed
        recv = dkv_in.float().sum(0)
        dk += recv[:, 0]
        dv += recv[:, 1]
        self._barrier()  # slots read before any member reuses them
        return dq.to(torch.bfloat16), dk.to(torch.bfloat16), dv.to(torch.bfloat16)
