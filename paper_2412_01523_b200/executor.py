"""FlexSP per-step SP executor: Plan -> pack -> all-to-all -> attention -> all-to-all.

The paper's runtime "sequentially reads one plan per iteration to train",
"generates the SP communication groups dynamically and scatters the data into the
corresponding group" and runs Ulysses SP "similar to DeepSpeed-Ulysses"
 with flash-attn varlen.  The reference package stops at
the Plan (pkg/src/seqplan/domain.py:381-400); this module is the executor under it.

B200 design:
* one process per GPU; a single symmetric-memory heap per rank is rendezvoused once
  (torch.distributed._symmetric_memory) and carved at identical offsets on every rank,
  so the receive buffer of any rank is `peer_base[r] + offset` — an SP group is just a
  rank block [r0, r0+d) and switching groups between micro-batches costs nothing
  (the paper's NCCL group pool, is not needed);
* pack is fused into the seq->head exchange and unpack into head->seq
  (fsp_a2a_seq2head / fsp_a2a_head2seq read/write rows through the layout tables);
* groups of one micro-batch run concurrently on disjoint ranks; micro-batches run in
  order (gradient accumulation);
* every exchange ends in a peer-memory flag barrier over the group, and a group entry
  barrier opens each micro-batch's forward and backward (its members write into each
  other's heap regions next); groups never wait on each other and degree-1 groups run
  without any barrier.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np
import torch

from . import ops
from .profiling import EventTimer
from .layout import (GroupLayout, LayoutError, MicroBatchLayout, build_plan_layouts, head_split,
                     loader_shards, scatter_routes)

_ALIGN = 4096
_SIGNAL_BYTES = 4096


def _align(n: int) -> int:
    return -(-n // _ALIGN) * _ALIGN


class PeerHeap:
    """One symmetric-memory heap per rank, identical offsets on every rank."""

    def __init__(self, nbytes: int, device: torch.device, world_size: int, group=None):
        self.device = device
        self.world_size = world_size
        self.nbytes = nbytes
        if world_size == 1:
            self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
            self.ptrs = [self.buf.data_ptr()]
        else:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem
            self.buf = symm_mem.empty(nbytes, dtype=torch.uint8, device=device)
            self.buf[:_SIGNAL_BYTES].zero_()
            self.handle = symm_mem.rendezvous(self.buf, group if group is not None
                                              else dist.group.WORLD)
            self.ptrs = [int(p) for p in self.handle.buffer_ptrs]
            torch.cuda.synchronize(device)
            dist.barrier(group=group)

    def view(self, offset: int, shape: Sequence[int], dtype: torch.dtype) -> torch.Tensor:
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        if offset + n > self.nbytes:
            raise LayoutError("peer heap too small for this plan")
        return self.buf[offset:offset + n].view(dtype).view(*shape)

    def peer(self, rank: int, offset: int) -> int:
        return self.ptrs[rank] + offset


@dataclass
class RankMicroBatch:
    """This rank's share of one micro-batch."""
    layout: MicroBatchLayout
    group: GroupLayout | None
    j: int                                  # rank inside the group
    n_local: int                            # loader-order rows this rank holds
    local_tokens: np.ndarray                # loader token ids of those rows
    pack_index: torch.Tensor | None = None  # int32 [R]
    unpack_table: torch.Tensor | None = None  # int32 [d*R]
    sched: ops.AttnSchedule | None = None
    fwd_flops: float = 0.0                  # 2 * D * H_j * sum s^2 (causal, FA convention)
    in_place: bool = False                  # d = 1: attention runs on the loader-order rows
    head_begin: list[int] = field(default_factory=list)  # group's head split [d+1]
    routes: torch.Tensor | None = None      # int32 [n, 3]: this rank's loader-shard rows of
                                            # this micro-batch -> (owner rank, owner row)

    @property
    def n_heads_local(self) -> int:        # H_j: heads this rank attends over
        return self.head_begin[self.j + 1] - self.head_begin[self.j]

    @property
    def heads_stride(self) -> int:         # max_j H_j: head slots per matrix when sharded
        return max(b - a for a, b in zip(self.head_begin, self.head_begin[1:]))


@dataclass
class StepPlan:
    """Device-ready form of one Plan for this rank (built once, reused every step)."""
    strategy: str
    lengths: list[int]
    micro_batches: list[RankMicroBatch]
    offsets: dict[str, int] = field(default_factory=dict)
    heap_bytes: int = 0
    shard_tokens: np.ndarray | None = None  # loader token ids of this rank's shard rows

    @property
    def total_tokens(self) -> int:
        return int(sum(self.lengths))


class FlexSPExecutor:
    """Runs the SP attention step of a plan on this rank (one process per GPU)."""

    def __init__(self, world_size: int, rank: int, n_heads: int, head_dim: int,
                 device: torch.device | str = "cuda", softmax_scale: float | None = None,
                 group=None, fuse_head2seq: bool = True, heap_factory=None,
                 output_slots: int = 1):
        if head_dim not in (64, 128):
            raise ValueError("head_dim must be 64 or 128")
        self.world_size = world_size
        self.rank = rank
        self.n_heads = n_heads
        self.head_dim = head_dim
        self.device = torch.device(device)
        self.scale = softmax_scale if softmax_scale is not None else 1.0 / math.sqrt(head_dim)
        self.group = group
        self.heap: PeerHeap | None = None
        self.epoch = 0
        # forward / backward calls so far: their parity picks the output slot, identically
        # on every rank (every rank calls both for every micro-batch, idle ranks included)
        self._n_fwd = 0
        self._n_bwd = 0
        self._ws: dict[str, torch.Tensor] = {}
        self.timer = EventTimer()
        # Eq. (4) fused into the attention epilogues (O in the forward, dQ/dK/dV in the
        # backward go straight to their owners' sequence shards); False = separate
        # fsp_a2a_head2seq launches after attention (kept for A/B measurements)
        self.fuse_head2seq = fuse_head2seq
        # heap_factory(nbytes) -> PeerHeap-like (view / peer / nbytes); None = the
        # symmetric-memory heap.  vranks.VirtualCluster passes per-virtual-rank heaps that
        # live on one device (the single-GPU multi-rank harness).
        self.heap_factory = heap_factory
        # 2: out_local / dqkv_local alternate between two heap slots by micro-batch, so
        # step_from_host can copy a micro-batch's results to the host while the next one
        # computes; 1 (default): one slot, half the output memory
        if output_slots not in (1, 2):
            raise ValueError("output_slots must be 1 or 2")
        self.output_slots = output_slots

    # ------------------------------------------------------------ planning -> tables
    def prepare(self, plan: Any, lengths: Sequence[int], sharded_loader: bool = False) -> StepPlan:
        """Device tables of one plan for this rank.  With `sharded_loader` the step's
        inputs arrive as this rank's data-loader shard (layout.loader_shards: sequence k on
        rank k % world) and step_from_shards scatters every micro-batch's rows to their
        group members first."""
        layouts = build_plan_layouts(plan, lengths, self.world_size, self.n_heads)
        shard = loader_shards(lengths, self.world_size)[self.rank] if sharded_loader else None
        hd = self.n_heads * self.head_dim
        mbs: list[RankMicroBatch] = []
        max_recv = max_local = 0
        for lay in layouts:
            grp, j = lay.group_of(self.rank)
            routes = None
            if shard is not None:
                r = scatter_routes(lay, shard)
                routes = torch.from_numpy(r if r.size else np.zeros((0, 3), np.int32)).to(self.device)
            if grp is None:
                mbs.append(RankMicroBatch(lay, None, -1, 0, np.zeros(0, dtype=np.int64),
                                          routes=routes))
            else:
                local = grp.local_tokens(j)
                rmb = RankMicroBatch(lay, grp, j, int(local.shape[0]), local,
                                     head_begin=head_split(self.n_heads, grp.degree),
                                     routes=routes)
                pack = grp.pack_index(j)
                table = grp.unpack_table()
                # the tables the kernels index with are validated by the library first
                ops.layout_check(pack, rmb.n_local)
                for jj in range(grp.degree):
                    ops.layout_check(table[jj], int((grp.shard(jj) >= 0).sum()))
                rmb.pack_index = torch.from_numpy(pack).to(self.device)
                rmb.unpack_table = torch.from_numpy(
                    np.ascontiguousarray(table.reshape(-1))).to(self.device)
                if grp.degree == 1:
                    # d = 1: no exchange at all — attention reads q/k/v and writes O / dQKV
                    # in place in the rank's loader-order buffers (each sequence is
                    # contiguous there), so there is no pack / unpack copy either.
                    offs = np.zeros(len(lengths) + 1, dtype=np.int64)
                    np.cumsum(np.asarray(lengths, dtype=np.int64), out=offs[1:])
                    starts = np.searchsorted(local, offs[list(grp.sequence_indices)])
                    rmb.sched = ops.AttnSchedule.build(
                        grp.cu_seqlens, self.device, self.n_heads, total_rows=rmb.n_local,
                        head_dim=self.head_dim, seq_starts_host=starts)
                    rmb.in_place = True
                else:
                    rmb.sched = ops.AttnSchedule.build(grp.cu_seqlens, self.device,
                                                       rmb.n_heads_local,
                                                       total_rows=grp.padded_tokens,
                                                       head_dim=self.head_dim)
                seg = np.diff(grp.cu_seqlens).astype(np.float64)
                rmb.fwd_flops = 2.0 * self.head_dim * rmb.n_heads_local * float((seg ** 2).sum())
                mbs.append(rmb)
            # heap regions must be identical on every rank: size by the max over ranks
            for g in lay.groups:
                if g.degree > 1:  # d = 1 groups compute in place: no receive buffers
                    max_recv = max(max_recv, g.padded_tokens * -(-self.n_heads // g.degree) *
                                   self.head_dim)
                for jj in range(g.degree):
                    max_local = max(max_local, int((g.shard(jj) >= 0).sum()))
        off = {}
        cur = _SIGNAL_BYTES
        # out_local / dqkv_local alternate between two slots (micro-batch parity), so a
        # micro-batch's results can be read out (step_from_host's D2H copy) while the next
        # micro-batch computes into the other slot
        two = self.output_slots == 2
        for name, elems in (("qkv_recv", 3 * max_recv), ("out_local0", max_local * hd),
                            ("out_local1", max_local * hd if two else 0), ("do_recv", max_recv),
                            ("dqkv_local0", 3 * max_local * hd),
                            ("dqkv_local1", 3 * max_local * hd if two else 0),
                            # step_from_shards: scattered loader rows (q/k/v, dO)
                            ("in_qkv", 3 * max_local * hd if sharded_loader else 0),
                            ("in_do", max_local * hd if sharded_loader else 0)):
            off[name] = cur
            cur += _align(max(elems, 1) * 2)
        strategy = plan["strategy"] if isinstance(plan, dict) else getattr(plan, "strategy", "")
        sp = StepPlan(strategy, [int(s) for s in lengths], mbs, off, cur, shard_tokens=shard)
        self._ensure_heap(cur)
        return sp

    def _ensure_heap(self, nbytes: int) -> None:
        if self.heap is not None and self.heap.nbytes >= nbytes:
            return
        # collective when world_size > 1: every rank prepares the same plan
        self.heap = (self.heap_factory(nbytes) if self.heap_factory is not None else
                     PeerHeap(nbytes, self.device, self.world_size, self.group))
        self.epoch = 0
        self._n_fwd = self._n_bwd = 0

    def _workspace(self, name: str, numel: int, dtype: torch.dtype) -> torch.Tensor:
        t = self._ws.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(max(numel, 1), dtype=dtype, device=self.device)
            self._ws[name] = t
        return t[:numel]

    # ------------------------------------------------------------ barriers
    def _signals(self, ranks: range) -> list[int]:
        return [self.heap.peer(r, 0) for r in ranks]

    def _barrier(self, ranks: range, epoch: int, span: str = "group_barrier") -> None:
        if len(ranks) > 1:
            with self.timer.span(span):
                ops.group_barrier(self._signals(ranks), self.rank - ranks.start, ranks.start,
                                  epoch)

    def _next_epoch(self) -> int:
        self.epoch += 1
        return self.epoch

    # ------------------------------------------------------------ one micro-batch
    def _out_off(self, sp: StepPlan) -> int:  # slot of the current forward
        return sp.offsets[f"out_local{self._n_fwd % self.output_slots}"]

    def _dqkv_off(self, sp: StepPlan) -> int:  # slot of the current backward
        return sp.offsets[f"dqkv_local{self._n_bwd % self.output_slots}"]

    def local_buffers(self, sp: StepPlan, mb: RankMicroBatch):
        """Views of this rank's output buffers (inside the heap) for the micro-batch whose
        forward / backward is the current one."""
        out = self.heap.view(self._out_off(sp), (mb.n_local, self.n_heads, self.head_dim),
                             torch.bfloat16)
        dqkv = self.heap.view(self._dqkv_off(sp), (mb.n_local, 3, self.n_heads, self.head_dim),
                              torch.bfloat16)
        return out, dqkv

    def micro_batch_forward(self, sp: StepPlan, mb: RankMicroBatch, qkv_local: torch.Tensor):
        """Eq. (2)-(4) forward on this rank.  qkv_local: [n_local, 3, H, D] bf16.

        Returns (out_local view [n_local, H, D], saved) where saved feeds the backward.
        """
        # Entry barrier over this micro-batch's group only: its members are about to write
        # into each other's heap regions, so every member must be done (in stream order)
        # with what the previous micro-batch left there.  Ranks of other groups never touch
        # these heaps, and a degree-1 group touches none, so groups run decoupled.
        ep_entry = self._next_epoch()
        self._n_fwd += 1
        grp = mb.group
        if grp is None:
            for _ in range(2):
                self._next_epoch()
            return None, None
        H, D = self.n_heads, self.head_dim
        d, j, R = grp.degree, mb.j, grp.rows_per_rank
        hn, hm, hb = mb.n_heads_local, mb.heads_stride, mb.head_begin
        ranks = grp.ranks
        if qkv_local.shape[0] != mb.n_local:
            raise ValueError(f"rank {self.rank} expects {mb.n_local} local rows, got {qkv_local.shape[0]}")
        if mb.in_place:
            for _ in range(2):  # keep the barrier epochs in step with the exchanging ranks
                self._next_epoch()
            out_local, _ = self.local_buffers(sp, mb)
            with self.timer.span("attn_fwd", mb.fwd_flops):
                _, lse = ops.attn_fwd(qkv_local[:, 0], qkv_local[:, 1], qkv_local[:, 2], mb.sched,
                                      self.scale, out=out_local)
            return out_local, (qkv_local, out_local, lse)
        self._barrier(ranks, ep_entry, "entry_barrier")
        off = sp.offsets
        T = grp.padded_tokens
        recv = self.heap.view(off["qkv_recv"], (T, 3, hm, D), torch.bfloat16)
        # NVLink bytes per matrix: seq2head sends the peers' head slices of R rows,
        # head2seq sends this rank's head slice of (d-1)*R rows
        sent_in = float(R * (H - hn) * D * 2)
        sent_out = float((d - 1) * R * hn * D * 2)
        with self.timer.span("a2a", 3 * sent_in):
            self._a2a_qkv(sp, mb, qkv_local, grp, R, hm)
            self._barrier(ranks, self._next_epoch())
        o_heads = self._workspace("o_heads", T * hm * D, torch.bfloat16).view(T, hm, D)
        out_local, _ = self.local_buffers(sp, mb)
        scatter = None
        if self.fuse_head2seq:  # Eq. (4) inside the attention epilogue
            scatter = ops.HeadScatter(d, R, hb[j], H * D, 0, mb.unpack_table,
                                      [self.heap.peer(r, self._out_off(sp)) for r in ranks])
        with self.timer.span("attn_fwd", mb.fwd_flops):
            _, lse = ops.attn_fwd(recv[:, 0, :hn], recv[:, 1, :hn], recv[:, 2, :hn], mb.sched,
                                  self.scale, out=o_heads[:, :hn], scatter=scatter)
        if scatter is not None:
            self.timer.count("head2seq_fused", sent_out)  # NVLink bytes inside attn_fwd
            self._barrier(ranks, self._next_epoch(), "fused_barrier")
            return out_local, (recv[:, :, :hn], o_heads[:, :hn], lse)
        with self.timer.span("a2a", sent_out):
            ops.a2a("head2seq", o_heads.view(T, hm * D),
                    [self.heap.peer(r, self._out_off(sp)) for r in ranks], degree=d, rank=j,
                    rows_per_rank=R, n_mats=1, n_heads=H, head_dim=D, dst_stride=H * D,
                    index=mb.unpack_table, head_begin=hb)
            self._barrier(ranks, self._next_epoch())
        return out_local, (recv[:, :, :hn], o_heads[:, :hn], lse)

    def _a2a_qkv(self, sp, mb, qkv_local, grp, R, hm):
        H, D, d, j = self.n_heads, self.head_dim, grp.degree, mb.j
        off = sp.offsets
        ops.a2a("seq2head", qkv_local.view(mb.n_local, -1) if mb.n_local else
                qkv_local.reshape(0, 3 * H * D),
                [self.heap.peer(r, off["qkv_recv"]) for r in grp.ranks], degree=d, rank=j,
                rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D, dst_stride=3 * hm * D,
                index=mb.pack_index, head_begin=mb.head_begin)

    def micro_batch_backward(self, sp: StepPlan, mb: RankMicroBatch, saved, dout_local: torch.Tensor):
        """Backward of micro_batch_forward: dout_local [n_local, H, D] -> dqkv_local view."""
        ep_entry = self._next_epoch()  # group entry barrier, as in the forward
        self._n_bwd += 1
        grp = mb.group
        if grp is None:
            for _ in range(2):
                self._next_epoch()
            return None
        recv, o_heads, lse = saved
        H, D = self.n_heads, self.head_dim
        if mb.in_place:
            for _ in range(2):
                self._next_epoch()
            _, dqkv_local = self.local_buffers(sp, mb)
            T = mb.n_local
            dq_acc = self._workspace("dq_accum", T * H * D, torch.float32)
            delta = self._workspace("delta", H * T, torch.float32)
            with self.timer.span("attn_bwd", 2.5 * mb.fwd_flops):
                ops.attn_bwd(recv[:, 0], recv[:, 1], recv[:, 2], o_heads, dout_local, lse,
                             mb.sched, self.scale, dq=dqkv_local[:, 0], dk=dqkv_local[:, 1],
                             dv=dqkv_local[:, 2], dq_accum=dq_acc, delta=delta)
            return dqkv_local
        d, j, R = grp.degree, mb.j, grp.rows_per_rank
        hn, hm, hb = mb.n_heads_local, mb.heads_stride, mb.head_begin
        ranks = grp.ranks
        self._barrier(ranks, ep_entry, "entry_barrier")
        off = sp.offsets
        T = grp.padded_tokens
        do_recv = self.heap.view(off["do_recv"], (T, hm, D), torch.bfloat16)
        sent_in = float(R * (H - hn) * D * 2)
        sent_out = float((d - 1) * R * hn * D * 2)
        with self.timer.span("a2a", sent_in):
            ops.a2a("seq2head", dout_local.reshape(mb.n_local, H * D),
                    [self.heap.peer(r, off["do_recv"]) for r in ranks], degree=d, rank=j,
                    rows_per_rank=R, n_mats=1, n_heads=H, head_dim=D, dst_stride=hm * D,
                    index=mb.pack_index, head_begin=hb)
            self._barrier(ranks, self._next_epoch())
        dq_acc = self._workspace("dq_accum", T * hn * D, torch.float32)
        delta = self._workspace("delta", hn * T, torch.float32)
        if self.fuse_head2seq:  # Eq. (4) for dQ/dK/dV inside the backward's epilogues
            _, dqkv_local = self.local_buffers(sp, mb)
            scatter = ops.HeadScatter(d, R, hb[j], 3 * H * D, H * D, mb.unpack_table,
                                      [self.heap.peer(r, self._dqkv_off(sp)) for r in ranks])
            with self.timer.span("attn_bwd", 2.5 * mb.fwd_flops):
                ops.attn_bwd(recv[:, 0], recv[:, 1], recv[:, 2], o_heads, do_recv[:, :hn], lse,
                             mb.sched, self.scale, dq_accum=dq_acc, delta=delta, scatter=scatter)
            self.timer.count("head2seq_fused", 3 * sent_out)  # NVLink bytes inside attn_bwd
            self._barrier(ranks, self._next_epoch(), "fused_barrier")
            return dqkv_local
        dqkv_heads = self._workspace("dqkv_heads", T * 3 * hm * D, torch.bfloat16).view(T, 3, hm, D)
        with self.timer.span("attn_bwd", 2.5 * mb.fwd_flops):
            ops.attn_bwd(recv[:, 0], recv[:, 1], recv[:, 2], o_heads, do_recv[:, :hn], lse,
                         mb.sched, self.scale, dq=dqkv_heads[:, 0, :hn], dk=dqkv_heads[:, 1, :hn],
                         dv=dqkv_heads[:, 2, :hn], dq_accum=dq_acc, delta=delta)
        _, dqkv_local = self.local_buffers(sp, mb)
        with self.timer.span("a2a", 3 * sent_out):
            ops.a2a("head2seq", dqkv_heads.view(T, 3 * hm * D),
                    [self.heap.peer(r, self._dqkv_off(sp)) for r in ranks], degree=d, rank=j,
                    rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D, dst_stride=3 * H * D,
                    index=mb.unpack_table, head_begin=hb)
            self._barrier(ranks, self._next_epoch())
        return dqkv_local

    def step(self, sp: StepPlan, qkv_locals: Sequence[torch.Tensor],
             dout_locals: Sequence[torch.Tensor], sink=None):
        """fwd+bwd of every micro-batch in plan order.  `sink(m, out, dqkv)` consumes the
        outputs before the next micro-batch reuses the heap regions (e.g. a copy-out)."""
        for m, mb in enumerate(sp.micro_batches):
            out, saved = self.micro_batch_forward(sp, mb, qkv_locals[m])
            dqkv = self.micro_batch_backward(sp, mb, saved, dout_locals[m])
            if sink is not None:
                sink(m, out, dqkv)

    # ------------------------------------------------------------ host copy-in / copy-out
    def _streams(self) -> None:
        if not hasattr(self, "_h2d_stream"):
            self._h2d_stream = torch.cuda.Stream(self.device)
            self.d2h_stream = torch.cuda.Stream(self.device)
            # persistent across calls: a copy must not overwrite a slot the previous step
            # is still reading (waiting on a never-recorded event is a no-op)
            self._h2d_consumed = [torch.cuda.Event() for _ in range(2)]
            self._h2d_loaded = [torch.cuda.Event() for _ in range(2)]
            self._out_read = [torch.cuda.Event() for _ in range(2)]   # out_local slot copied out
            self._dqkv_read = [torch.cuda.Event() for _ in range(2)]  # dqkv_local slot copied out
            self._h2d_slot = 0            # slot the next copy goes to (strictly alternating)
            self._h2d_prefetched = None   # (host qkv, host dout, slot) of an in-flight copy

    def _wait_out_slot(self, cur, kind: str) -> None:
        """Before a forward ("out") / backward ("dqkv"): the output slot it is about to
        write must have been copied out to the host already."""
        if kind == "out":
            cur.wait_event(self._out_read[(self._n_fwd + 1) % self.output_slots])
        else:
            cur.wait_event(self._dqkv_read[(self._n_bwd + 1) % self.output_slots])

    def _copy_out(self, cur, m: int, out, dqkv, rows: int, host_out, host_dqkv) -> None:
        """Micro-batch m's O / dQKV to pinned host memory on the D2H stream."""
        if host_out is None or out is None or not rows:
            return
        hd = self.n_heads * self.head_dim
        so, sd = self._n_fwd % self.output_slots, self._n_bwd % self.output_slots
        self.d2h_stream.wait_stream(cur)
        with torch.cuda.stream(self.d2h_stream):
            host_out[m].view(rows, hd).copy_(out.reshape(rows, hd), non_blocking=True)
            host_dqkv[m].view(rows, 3 * hd).copy_(dqkv.reshape(rows, 3 * hd), non_blocking=True)
            self._out_read[so].record(self.d2h_stream)
            self._dqkv_read[sd].record(self.d2h_stream)

    def step_from_shards(self, sp: StepPlan, shard_qkv: torch.Tensor, shard_dout: torch.Tensor,
                         sink=None, host_out=None, host_dqkv=None) -> None:
        """The step fed by the data loader's shards (prepare(..., sharded_loader=True)).

        shard_qkv [n_shard, 3, H, D] / shard_dout [n_shard, H, D] hold this rank's loader
        rows (sequence k on rank k % world, batch order).  Before each micro-batch every
        rank pushes that micro-batch's rows of its shard to the group members that own them
        (fsp_scatter_rows, NVSwitch peer stores into their heap input buffers, PAPER.md:922
        "scatters the data into the corresponding group"); a world barrier before the
        scatter frees the input buffers, one after it publishes the data; the micro-batch
        then runs on the received loader-order rows exactly as in step().  With host_out /
        host_dqkv (pinned, per micro-batch) the results go back to the host as in
        step_from_host (needs output_slots=2)."""
        if sp.shard_tokens is None:
            raise ValueError("prepare the plan with sharded_loader=True first")
        if host_out is not None and self.output_slots != 2:
            raise ValueError("copying results to the host needs FlexSPExecutor(output_slots=2)")
        n_shard = int(sp.shard_tokens.shape[0])
        if shard_qkv.shape[0] != n_shard or shard_dout.shape[0] != n_shard:
            raise ValueError(f"rank {self.rank} shard has {n_shard} rows")
        self._streams()
        cur = torch.cuda.current_stream(self.device)
        hd = self.n_heads * self.head_dim
        world = range(0, self.world_size)
        off = sp.offsets
        src_q = shard_qkv.reshape(n_shard, 3 * hd)
        src_d = shard_dout.reshape(n_shard, hd)
        for m, mb in enumerate(sp.micro_batches):
            self._barrier(world, self._next_epoch(), "scatter_barrier")  # inputs free
            with self.timer.span("scatter", float(mb.routes.shape[0] * 4 * hd * 2)):
                ops.scatter_rows(src_q, mb.routes, [self.heap.peer(r, off["in_qkv"]) for r in world],
                                 3 * hd * 2)
                ops.scatter_rows(src_d, mb.routes, [self.heap.peer(r, off["in_do"]) for r in world],
                                 hd * 2)
                self._barrier(world, self._next_epoch())  # every rank's rows have landed
            q = self.heap.view(off["in_qkv"], (mb.n_local, 3, self.n_heads, self.head_dim),
                               torch.bfloat16)
            d = self.heap.view(off["in_do"], (mb.n_local, self.n_heads, self.head_dim),
                               torch.bfloat16)
            self._wait_out_slot(cur, "out")
            out, saved = self.micro_batch_forward(sp, mb, q)
            self._wait_out_slot(cur, "dqkv")
            dqkv = self.micro_batch_backward(sp, mb, saved, d)
            if sink is not None:
                sink(m, out, dqkv)
            self._copy_out(cur, m, out, dqkv, mb.n_local, host_out, host_dqkv)

    def step_from_host_shards(self, sp: StepPlan, host_shard_qkv: torch.Tensor,
                              host_shard_dout: torch.Tensor, host_out=None, host_dqkv=None,
                              sink=None, prefetch_next: tuple | None = None) -> None:
        """The data-loader path end to end at N > 1: this rank's loader shard arrives from
        pinned host memory (H2D on the side stream into a double buffer; `prefetch_next =
        (next_host_shard_qkv, next_host_shard_dout)` uploads the next step's shard while
        this step computes), is scattered to the plan's groups over NVSwitch
        (step_from_shards) and the results go back to pinned host memory."""
        self._streams()
        cur = torch.cuda.current_stream(self.device)
        side = self._h2d_stream
        n = int(host_shard_qkv.shape[0])
        hd = self.n_heads * self.head_dim

        rows = max(n, int(prefetch_next[0].shape[0]) if prefetch_next is not None else 0, 1)
        have = self._ws.get("shard_do0")
        if have is None or have.numel() < rows * hd:
            # the double buffer grows: no copy may still be landing in the old one
            self._h2d_prefetched = None
            cur.wait_stream(side)
            for kk in range(2):
                self._workspace(f"shard_qkv{kk}", rows * 3 * hd, torch.bfloat16)
                self._workspace(f"shard_do{kk}", rows * hd, torch.bfloat16)

        def upload(hq, hdo):
            k = self._h2d_slot
            self._h2d_slot ^= 1
            m_ = int(hq.shape[0])
            q = self._ws[f"shard_qkv{k}"]
            d = self._ws[f"shard_do{k}"]
            with torch.cuda.stream(side):
                side.wait_event(self._h2d_consumed[k])
                if m_:
                    q[:m_ * 3 * hd].view(m_, 3 * hd).copy_(hq.view(m_, 3 * hd), non_blocking=True)
                    d[:m_ * hd].view(m_, hd).copy_(hdo.view(m_, hd), non_blocking=True)
                self._h2d_loaded[k].record(side)
            return k

        pf, self._h2d_prefetched = self._h2d_prefetched, None
        k = pf[2] if (pf is not None and pf[0] is host_shard_qkv and pf[1] is host_shard_dout) \
            else upload(host_shard_qkv, host_shard_dout)
        if prefetch_next is not None:
            nk = upload(*prefetch_next)
            self._h2d_prefetched = (prefetch_next[0], prefetch_next[1], nk)
        cur.wait_event(self._h2d_loaded[k])
        q = self._ws[f"shard_qkv{k}"][:n * 3 * hd].view(n, 3, self.n_heads, self.head_dim)
        d = self._ws[f"shard_do{k}"][:n * hd].view(n, self.n_heads, self.head_dim)
        self.step_from_shards(sp, q, d, sink=sink, host_out=host_out, host_dqkv=host_dqkv)
        self._h2d_consumed[k].record(cur)

    def step_from_host(self, sp: StepPlan, host_qkv: Sequence[torch.Tensor],
                       host_dout: Sequence[torch.Tensor], host_out: Sequence[torch.Tensor] | None = None,
                       host_dqkv: Sequence[torch.Tensor] | None = None, sink=None,
                       prefetch_next: tuple | None = None) -> None:
        """The same step fed from and returned to pinned host memory (the data-loader path).

        Micro-batch m+1's q/k/v and dO are copied host->device on a side stream into the
        other half of a double buffer while micro-batch m computes, so PCIe transfer and
        the SP step overlap.  `prefetch_next = (next_sp, next_host_qkv, next_host_dout)`
        also starts the NEXT step's first micro-batch copy while this step's last
        micro-batch computes (what a data loader does between steps); the next call with
        those same host tensors then finds it in flight instead of copying again.
        With `host_out` / `host_dqkv` (pinned, [n_local, H, D] / [n_local, 3, H, D] per
        micro-batch) each micro-batch's O and dQKV are copied device->host on a third
        stream while the next micro-batch computes (PCIe is full duplex; the output
        regions alternate between two heap slots, and a slot is rewritten only after its
        copy-out finished).  The copies are in flight when this returns:
        `d2h_stream` orders after them.
        """
        if host_out is not None and self.output_slots != 2:
            raise ValueError("copying results to the host needs FlexSPExecutor(output_slots=2)")
        cur = torch.cuda.current_stream(self.device)
        self._streams()
        side = self._h2d_stream
        consumed, loaded = self._h2d_consumed, self._h2d_loaded
        n = len(sp.micro_batches)
        hd = self.n_heads * self.head_dim
        rows_needed = max((mb.n_local for mb in sp.micro_batches), default=0)
        if prefetch_next is not None and prefetch_next[0].micro_batches:
            rows_needed = max(rows_needed, prefetch_next[0].micro_batches[0].n_local)
        rows_needed = max(rows_needed, 1)
        have = self._ws.get("h2d_do0")
        if have is None or have.numel() < rows_needed * hd:
            self._h2d_prefetched = None  # the slots are reallocated: drop an in-flight copy
            cur.wait_stream(side)
        bufs = [(self._workspace(f"h2d_qkv{k}", rows_needed * 3 * hd, torch.bfloat16),
                 self._workspace(f"h2d_do{k}", rows_needed * hd, torch.bfloat16)) for k in range(2)]

        def issue_copy(hq, hdo, rows) -> int:
            k = self._h2d_slot
            self._h2d_slot ^= 1
            with torch.cuda.stream(side):
                side.wait_event(consumed[k])
                q, d = bufs[k]
                if rows:
                    q[:rows * 3 * hd].view(rows, 3 * hd).copy_(hq.view(rows, 3 * hd),
                                                               non_blocking=True)
                    d[:rows * hd].view(rows, hd).copy_(hdo.view(rows, hd), non_blocking=True)
                loaded[k].record(side)
            return k

        slots: list[int] = []
        pf, self._h2d_prefetched = self._h2d_prefetched, None
        if n:
            if pf is not None and pf[0] is host_qkv[0] and pf[1] is host_dout[0]:
                slots.append(pf[2])
            else:
                slots.append(issue_copy(host_qkv[0], host_dout[0], sp.micro_batches[0].n_local))
        for m, mb in enumerate(sp.micro_batches):
            if m + 1 < n:
                slots.append(issue_copy(host_qkv[m + 1], host_dout[m + 1],
                                        sp.micro_batches[m + 1].n_local))
            elif prefetch_next is not None and prefetch_next[0].micro_batches:
                nsp, nq, nd = prefetch_next
                k = issue_copy(nq[0], nd[0], nsp.micro_batches[0].n_local)
                self._h2d_prefetched = (nq[0], nd[0], k)
            k = slots[m]
            cur.wait_event(loaded[k])
            rows = mb.n_local
            q = bufs[k][0][:rows * 3 * hd].view(rows, 3, self.n_heads, self.head_dim)
            d = bufs[k][1][:rows * hd].view(rows, self.n_heads, self.head_dim)
            # the output slots this micro-batch writes must have been copied out already
            self._wait_out_slot(cur, "out")
            out, saved = self.micro_batch_forward(sp, mb, q)
            self._wait_out_slot(cur, "dqkv")
            dqkv = self.micro_batch_backward(sp, mb, saved, d)
            if sink is not None:
                sink(m, out, dqkv)
            consumed[k].record(cur)
            self._copy_out(cur, m, out, dqkv, rows, host_out, host_dqkv)
