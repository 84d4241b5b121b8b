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


def seq2head(shard: torch.Tensor, group=None) -> torch.Tensor:
    """[R, n_mats, H, D] on each of d ranks -> [d*R, n_mats, H/d, D] (Eq. 2)."""
    d = dist.get_world_size(group)
    R, M, H, D = shard.shape
    send = shard.reshape(R, M, d, H // d, D).permute(2, 0, 1, 3, 4).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return recv.reshape(d * R, M, H // d, D)


def head2seq(heads: torch.Tensor, group=None) -> torch.Tensor:
    """[d*R, n_mats, H/d, D] -> [R, n_mats, H, D] (Eq. 4)."""
    d = dist.get_world_size(group)
    T, M, Hs, D = heads.shape
    R = T // d
    send = heads.reshape(d, R, M, Hs, D).contiguous()
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 2, 0, 3, 4).reshape(R, M, d * Hs, D)


def ulysses_attention(shard_qkv: torch.Tensor, cu_seqlens, group=None) -> torch.Tensor:
    """One rank's SP attention: shard [R, 3, H, D] -> output shard [R, H, D] (fp32)."""
    heads = seq2head(shard_qkv.float(), group)
    T = heads.shape[0]
    o = torch.zeros(T, heads.shape[2], heads.shape[3])
    n = int(cu_seqlens[-1])
    o[:n], _ = attention_fwd_ref(heads[:n, 0], heads[:n, 1], heads[:n, 2], cu_seqlens)
    return head2seq(o[:, None], group)[:, 0]
