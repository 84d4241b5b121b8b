"""Ulysses SP step oracle on CPU torch.distributed (gloo) — TEST INFRASTRUCTURE ONLY.

Restates PAPER.md:336-348 Eqs. (1)-(4) for one SP group: each rank holds a contiguous
shard of the group-packed sequence with all heads; AlltoAll (Eq. 2) trades sequence
shards for head slices; varlen causal attention runs per head slice (Eq. 3, via
oracle/attention_ref.py); AlltoAll (Eq. 4) returns to sequence shards.  Used by
tests/test_oracle.py (world_size 2 on gloo) to show the SP exchange is an identity
around attention, i.e. SP output == single-process attention.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from .attention_ref import attention_fwd_ref
from .layout_ref import head_split


def seq2head(shard: torch.Tensor, group=None) -> torch.Tensor:
    """[R, n_mats, H, D] on each of d ranks -> [d*R, n_mats, H_me, D] (Eq. 2); member j
    receives heads [b[j], b[j+1]) of layout_ref.head_split (uneven when d does not
    divide H)."""
    d = dist.get_world_size(group)
    me = dist.get_rank(group)
    R, M, H, D = shard.shape
    b = head_split(H, d)
    send = torch.cat([shard[:, :, b[j]:b[j + 1]].reshape(-1) for j in range(d)])
    h_me = b[me + 1] - b[me]
    recv = torch.empty(d * R * M * h_me * D, dtype=shard.dtype)
    dist.all_to_all_single(recv, send, output_split_sizes=[R * M * h_me * D] * d,
                           input_split_sizes=[R * M * (b[j + 1] - b[j]) * D for j in range(d)],
                           group=group)
    return recv.reshape(d * R, M, h_me, D)


def head2seq(heads: torch.Tensor, group=None, n_heads: int | None = None) -> torch.Tensor:
    """[d*R, n_mats, H_me, D] -> [R, n_mats, H, D] (Eq. 4)."""
    d = dist.get_world_size(group)
    T, M, h_me, D = heads.shape
    R = T // d
    H = n_heads if n_heads is not None else h_me * d
    b = head_split(H, d)
    recv = torch.empty(R * M * H * D, dtype=heads.dtype)
    dist.all_to_all_single(recv, heads.reshape(-1).contiguous(),
                           output_split_sizes=[R * M * (b[j + 1] - b[j]) * D for j in range(d)],
                           input_split_sizes=[R * M * h_me * D] * d, group=group)
    parts, off = [], 0
    for j in range(d):
        n = R * M * (b[j + 1] - b[j]) * D
        parts.append(recv[off:off + n].reshape(R, M, b[j + 1] - b[j], D))
        off += n
    return torch.cat(parts, dim=2)


def ulysses_attention(shard_qkv: torch.Tensor, cu_seqlens, group=None) -> torch.Tensor:
    """One rank's SP attention: shard [R, 3, H, D] -> output shard [R, H, D] (fp32)."""
    heads = seq2head(shard_qkv.float(), group)
    T = heads.shape[0]
    o = torch.zeros(T, heads.shape[2], heads.shape[3])
    n = int(cu_seqlens[-1])
    o[:n], _ = attention_fwd_ref(heads[:n, 0], heads[:n, 1], heads[:n, 2], cu_seqlens)
    return head2seq(o[:, None], group, n_heads=shard_qkv.shape[2])[:, 0]
