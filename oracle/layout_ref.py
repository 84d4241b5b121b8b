"""Layout / data-movement oracle (plain Python loops + numpy) — TEST INFRASTRUCTURE ONLY.

Independent restatement of every integer step between the reference planner's Plan and
the attention kernel's input, used to check the product's host layout builder and the
pack / all-to-all kernels bit-exact.

  deal_sequences      pkg/src/seqplan/planner.py:499-509  (per-bucket longest-first
                      dealing to the slot with most remaining count, ties lowest slot;
                      groups emitted in slot order :512-513)
  place_groups        PAPER.md:926-927 (groups of power-of-two size pair with their
                      neighbours: contiguous, buddy-aligned rank blocks in slot order)
  group_permutation   PAPER.md:380-388 sequence packing; flash-attn varlen cu_seqlens
                      (PAPER.md:916); T_g padded to a multiple of the SP degree
  ulysses_seq2head /  PAPER.md:338 Eq. (2) and :340 Eq. (4), restated on numpy arrays
  ulysses_head2seq
"""
from __future__ import annotations

import numpy as np


def deal_sequences(member_indices, assignment, selection, lengths):
    """Re-derive each selected slot's sequence list from the bucket assignment.

    Restates planner.py:499-509: for each bucket q (ascending), members sorted by
    (-length, index) are dealt one by one to the slot with the largest remaining
    assigned count, ties to the lowest slot id.  Returns {slot_id: [seq indices]}.
    """
    n_slots = len(selection)
    out = {p: [] for p in range(n_slots) if selection[p]}
    for q, members in enumerate(member_indices):
        order = sorted(members, key=lambda k: (-lengths[k], k))
        remaining = {}
        for p in range(n_slots):
            if assignment[q][p] > 0:
                remaining[p] = assignment[q][p]
        for k in order:
            best = None
            for p in sorted(remaining):
                if best is None or remaining[p] > remaining[best]:
                    best = p
            out[best].append(k)
            remaining[best] -= 1
            if remaining[best] == 0:
                del remaining[best]
    return out


def place_groups(degrees, world_size):
    """Rank block start of each group, groups taken in slot (degree-descending) order."""
    starts = []
    r = 0
    for d in degrees:
        starts.append(r)
        r += d
    assert r <= world_size, "plan uses more devices than the world"
    for s, d in zip(starts, degrees):
        assert s % d == 0, "rank block is not buddy-aligned"
    return starts


def group_permutation(sequence_indices, lengths, degree):
    """(perm, cu_seqlens, padded) for one group; perm[row] = loader token or -1."""
    offsets = [0]
    for s in lengths:
        offsets.append(offsets[-1] + s)
    perm = []
    cu = [0]
    for k in sequence_indices:
        for t in range(lengths[k]):
            perm.append(offsets[k] + t)
        cu.append(cu[-1] + lengths[k])
    padded = ((len(perm) + degree - 1) // degree) * degree
    while len(perm) < padded:
        perm.append(-1)
    return perm, cu, padded


def shard_tables(perm, degree):
    """Per group rank j: (local loader-order token list, pack index list)."""
    r = len(perm) // degree
    tables = []
    for j in range(degree):
        shard = perm[j * r:(j + 1) * r]
        local = sorted(t for t in shard if t >= 0)
        pos = {t: i for i, t in enumerate(local)}
        pack = [pos[t] if t >= 0 else -1 for t in shard]
        tables.append((local, pack))
    return tables


def microbatch_tables(micro_batch, lengths, world_size):
    """Everything the executor needs for one micro-batch dict (plan JSON schema 1)."""
    groups = micro_batch["selected_groups"]
    degrees = [g["degree"] for g in groups]
    starts = place_groups(degrees, world_size)
    out = []
    for g, r0 in zip(groups, starts):
        perm, cu, padded = group_permutation(g["sequence_indices"], lengths, g["degree"])
        out.append({"slot_id": g["slot_id"], "degree": g["degree"], "rank_begin": r0,
                    "perm": perm, "cu_seqlens": cu, "padded": padded,
                    "shards": shard_tables(perm, g["degree"])})
    return out


def head_split(n_heads, d):
    """Head ranges of the d group members: member j owns heads [b[j], b[j+1]); the first
    n_heads % d members take one extra head (52 heads at d=8 -> 7,7,7,7,6,6,6,6; the
    even split when d divides n_heads).  SURVEY.md §7 H5; PAPER.md:1458 (30B, 52 heads)."""
    base, extra = divmod(n_heads, d)
    b = [0]
    for j in range(d):
        b.append(b[-1] + base + (1 if j < extra else 0))
    return b


def ulysses_seq2head(shards, n_mats, n_heads, head_dim):
    """Eq. (2): list of d arrays [R, n_mats, H, D] -> list of d arrays
    [d*R, n_mats, H_j, D], H_j = member j's head count (head_split)."""
    d = len(shards)
    b = head_split(n_heads, d)
    out = []
    for j in range(d):
        parts = [sh[:, :, b[j]:b[j + 1], :] for sh in shards]
        out.append(np.concatenate(parts, axis=0))
    return out


def ulysses_head2seq(heads, n_mats, n_heads, head_dim):
    """Eq. (4): list of d arrays [d*R, n_mats, H_j, D] -> list of d arrays [R, n_mats, H, D]."""
    d = len(heads)
    r = heads[0].shape[0] // d
    out = []
    for j in range(d):
        out.append(np.concatenate([h[j * r:(j + 1) * r] for h in heads], axis=2))
    return out


def scatter_routes_ref(lengths, world_size, micro_batch_groups):
    """Per-plan data scatter restated in plain loops: sequence k starts on
    rank k % world_size (round-robin loader shards, batch order inside a shard) and must
    end on the member of its micro-batch group that holds it, at that member's
    loader-order row.  micro_batch_groups: [(rank_begin, degree, [seq indices])] of one
    micro-batch.  Returns {src_rank: [(src_row, dst_rank, dst_row)]} in src_row order."""
    offs = [0]
    for s in lengths:
        offs.append(offs[-1] + int(s))
    # source position of every token
    src = {}
    for r in range(world_size):
        n = 0
        for k in range(r, len(lengths), world_size):
            for t in range(offs[k], offs[k + 1]):
                src[t] = (r, n)
                n += 1
    routes = {r: [] for r in range(world_size)}
    for r0, d, seqs in micro_batch_groups:
        packed = []
        for k in seqs:
            packed.extend(range(offs[k], offs[k + 1]))
        t_pad = -(-len(packed) // d) * d
        rows = t_pad // d
        for j in range(d):
            mine = sorted(packed[j * rows:(j + 1) * rows])
            for pos, t in enumerate(mine):
                r, n = src[t]
                routes[r].append((n, r0 + j, pos))
    for r in routes:
        routes[r].sort()
    return routes
