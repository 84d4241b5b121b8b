"""Plan -> device layout tables (host side of the drop-in boundary).

The reference planner ends at ``Plan -> MicroBatchPlan -> GroupDispatch(slot_id, degree,
sequence_indices, ...)`` (pkg/src/seqplan/domain.py:332-400) or the identical plan JSON
schema 1 (domain.py:390-397, pkg/docs/formats.md:74-105).  This module turns one
micro-batch of such a plan into the tables the sm_100a kernels consume:

* placement  — selected groups in plan order (slot order = degree descending,
  planner.py:513, domain.py:240-247) take contiguous rank blocks [r0, r0+d); with
  power-of-two degrees in descending order the blocks are buddy-aligned, i.e. every GPU
  "pairs with its neighbors";
* permutation — inside a group, sequences are concatenated in ``sequence_indices`` order
  (bucket-ascending, longest-first dealing for FlexSP plans, planner.py:501-509;
  longest-first for static plans, baselines.py:101); T_g is padded to a multiple of d;
  perm[packed_row] = loader token index (batch order), -1 for pad rows;
* cu_seqlens — int32 prefix sums over the group's sequences (flash-attn varlen);
* shards — rank j of the group owns packed rows [j*R, (j+1)*R), R = T_g_pad / d;
  its loader-order input holds exactly the tokens of that shard sorted by loader index.

Everything here is deterministic integer work; tests/test_layout.py checks it bit-exact
against the independent restatement in oracle/layout_ref.py on plans produced by the
reference itself (tests/golden/).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Any, Sequence

import numpy as np


class LayoutError(ValueError):
    """A plan cannot be laid out (the analog of seqplan.ValidationError)."""


def _get(obj: Any, name: str):
    return obj[name] if isinstance(obj, dict) else getattr(obj, name)


@dataclass(frozen=True)
class GroupLayout:
    slot_id: int
    degree: int
    rank_begin: int
    sequence_indices: tuple[int, ...]
    cu_seqlens: np.ndarray        # int32 [n_seq + 1], packed-row offsets inside the group
    total_tokens: int             # T_g
    padded_tokens: int            # T_g rounded up to a multiple of degree
    perm: np.ndarray              # int64 [padded_tokens]: packed row -> loader token, -1 pad

    @property
    def rows_per_rank(self) -> int:
        return self.padded_tokens // self.degree

    @property
    def ranks(self) -> range:
        return range(self.rank_begin, self.rank_begin + self.degree)

    def shard(self, j: int) -> np.ndarray:
        """Loader token ids of packed rows owned by group rank j (pad = -1)."""
        r = self.rows_per_rank
        return self.perm[j * r:(j + 1) * r]

    def local_tokens(self, j: int) -> np.ndarray:
        """Loader-order token ids held by group rank j (its input/output rows)."""
        s = self.shard(j)
        return np.sort(s[s >= 0])

    def pack_index(self, j: int) -> np.ndarray:
        """int32 [R]: shard row i -> row in rank j's loader-order buffer (-1 pad)."""
        s = self.shard(j)
        local = self.local_tokens(j)
        out = np.full(s.shape[0], -1, dtype=np.int32)
        live = s >= 0
        out[live] = np.searchsorted(local, s[live]).astype(np.int32)
        return out

    def unpack_table(self) -> np.ndarray:
        """int32 [d, R]: pack_index of every member (the fused-unpack table of head2seq)."""
        return np.stack([self.pack_index(j) for j in range(self.degree)])


@dataclass(frozen=True)
class MicroBatchLayout:
    world_size: int
    groups: tuple[GroupLayout, ...]
    rank_group: np.ndarray = field(repr=False)  # int32 [world]: group index or -1 (idle)

    def group_of(self, rank: int) -> tuple[GroupLayout | None, int]:
        g = int(self.rank_group[rank])
        if g < 0:
            return None, -1
        grp = self.groups[g]
        return grp, rank - grp.rank_begin

    @property
    def total_tokens(self) -> int:
        return sum(g.total_tokens for g in self.groups)


def head_split(n_heads: int, degree: int) -> list[int]:
    """Heads of the `degree` members of a group: member j owns [b[j], b[j+1]).  The first
    n_heads % degree members take one extra head, so heads need not divide by the degree
    (52 heads at d=8 -> 7,7,7,7,6,6,6,6; the reference leaves head divisibility open,
    SPEC.md:352, and the 30B shape has 52 heads)."""
    if degree < 1 or n_heads < degree:
        raise LayoutError(f"{n_heads} heads cannot be split over SP degree {degree}")
    base, extra = divmod(n_heads, degree)
    b = [0]
    for j in range(degree):
        b.append(b[-1] + base + (1 if j < extra else 0))
    return b


def token_offsets(lengths: Sequence[int]) -> np.ndarray:
    """Loader-order start offset of every sequence of the batch (int64 [K+1])."""
    out = np.zeros(len(lengths) + 1, dtype=np.int64)
    np.cumsum(np.asarray(lengths, dtype=np.int64), out=out[1:])
    return out


def build_microbatch_layout(micro_batch: Any, lengths: Sequence[int], world_size: int,
                            n_heads: int | None = None) -> MicroBatchLayout:
    """Lay out one planned micro-batch (MicroBatchPlan or its JSON dict) on `world_size` GPUs."""
    if world_size < 1 or world_size & (world_size - 1):
        raise LayoutError(f"world_size must be a power of two, got {world_size}")
    lengths = [int(s) for s in lengths]
    offs = token_offsets(lengths)
    groups_in = list(_get(micro_batch, "selected_groups"))
    seen: set[int] = set()
    r0 = 0
    groups = []
    prev_degree = None
    for g in groups_in:
        d = int(_get(g, "degree"))
        if d < 1 or d & (d - 1):
            raise LayoutError(f"group degree must be a power of two, got {d}")
        if prev_degree is not None and d > prev_degree:
            raise LayoutError("selected_groups must be in slot order (degree descending)")
        prev_degree = d
        if n_heads is not None and n_heads < d:
            raise LayoutError(f"{n_heads} heads cannot be split over SP degree {d}")
        if r0 + d > world_size:
            raise LayoutError(f"groups need more than {world_size} ranks")
        idx = tuple(int(k) for k in _get(g, "sequence_indices"))
        for k in idx:
            if k < 0 or k >= len(lengths):
                raise LayoutError(f"sequence index {k} out of range for {len(lengths)} sequences")
            if k in seen:
                raise LayoutError(f"sequence {k} dispatched twice")
            seen.add(k)
        seg = np.asarray([lengths[k] for k in idx], dtype=np.int64)
        cu = np.zeros(len(idx) + 1, dtype=np.int64)
        np.cumsum(seg, out=cu[1:])
        t_g = int(cu[-1])
        if t_g >= 2**31:
            raise LayoutError("group exceeds 2^31 tokens")
        t_pad = -(-t_g // d) * d
        perm = np.full(t_pad, -1, dtype=np.int64)
        if idx:
            starts = offs[list(idx)]
            # packed row p inside sequence i maps to loader token starts[i] + (p - cu[i])
            rep = np.repeat(starts - cu[:-1], seg)
            perm[:t_g] = rep + np.arange(t_g, dtype=np.int64)
        groups.append(GroupLayout(int(_get(g, "slot_id")), d, r0, idx, cu.astype(np.int32), t_g,
                                  t_pad, perm))
        r0 += d
    rank_group = np.full(world_size, -1, dtype=np.int32)
    for gi, g in enumerate(groups):
        rank_group[g.rank_begin:g.rank_begin + g.degree] = gi
    return MicroBatchLayout(world_size, tuple(groups), rank_group)


def load_plan(path_or_dict) -> dict:
    """Read a plan JSON (schema 1, pkg/src/seqplan/formats.py:97-101) or pass a dict through."""
    if isinstance(path_or_dict, dict):
        data = path_or_dict
    else:
        with open(path_or_dict, encoding="utf-8") as fh:
            data = json.load(fh)
    if data.get("schema") != 1:
        raise LayoutError(f"unsupported plan schema {data.get('schema')!r}")
    return data


def plan_micro_batches(plan: Any) -> list:
    """Micro-batches of a seqplan.Plan or a plan-JSON dict, in execution order."""
    return list(_get(plan, "micro_batches"))


def build_plan_layouts(plan: Any, lengths: Sequence[int], world_size: int,
                       n_heads: int | None = None) -> list[MicroBatchLayout]:
    layouts = [build_microbatch_layout(mb, lengths, world_size, n_heads)
               for mb in plan_micro_batches(plan)]
    covered = sorted(k for lay in layouts for g in lay.groups for k in g.sequence_indices)
    if covered != list(range(len(lengths))):
        raise LayoutError("plan does not dispatch every sequence exactly once")
    return layouts


# ------------------------------------------------------------------ data scatter
def loader_shards(lengths: Sequence[int], world_size: int) -> list[np.ndarray]:
    """The data loader's sharding of one global batch before any plan is known: sequence
    k is read by rank k % world_size (round-robin data parallelism), and a rank's shard
    holds the tokens of its sequences in batch order.  Returns, per rank, the loader token
    ids of its shard rows (int64, ascending)."""
    offs = token_offsets(lengths)
    out = []
    for r in range(world_size):
        seqs = range(r, len(lengths), world_size)
        toks = [np.arange(offs[k], offs[k + 1], dtype=np.int64) for k in seqs]
        out.append(np.concatenate(toks) if toks else np.zeros(0, dtype=np.int64))
    return out


def scatter_routes(layout: MicroBatchLayout, shard_tokens: np.ndarray) -> np.ndarray:
    """Per-plan data scatter ("scatters the data into the corresponding
    group") of one micro-batch, for one source rank: int32 [n, 3] rows (src_row, dst_rank,
    dst_row) — shard row src_row (a token of this micro-batch) goes to rank dst_rank's
    loader-order input buffer at row dst_row (its position in that member's local_tokens).
    Tokens of other micro-batches are not listed."""
    total = int(shard_tokens.max()) + 1 if shard_tokens.size else 0
    owner = np.full(max(total, 1), -1, dtype=np.int64)
    row = np.full(max(total, 1), -1, dtype=np.int64)
    for g in layout.groups:
        for j in range(g.degree):
            loc = g.local_tokens(j)
            loc = loc[loc < total]
            owner[loc] = g.rank_begin + j
            row[loc] = np.searchsorted(g.local_tokens(j), loc)
    live = np.nonzero(owner[shard_tokens] >= 0)[0] if shard_tokens.size else np.zeros(0, np.int64)
    out = np.empty((live.size, 3), dtype=np.int32)
    out[:, 0] = live
    out[:, 1] = owner[shard_tokens[live]]
    out[:, 2] = row[shard_tokens[live]]
    return out
