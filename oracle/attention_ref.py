"""Varlen causal attention oracle (torch fp32, CPU) — TEST INFRASTRUCTURE ONLY.

Restates PAPER.md:339, Eq. (3): P_h = softmax(Q_h K_h^T / sqrt(D)) V_h, per head
slice, with the flash-attn varlen semantics the paper's runtime uses
(PAPER.md:916): each cu_seqlens segment attends causally to itself only (packing
masks).  Scale defaults to 1/sqrt(head_dim) (flash-attn convention;
PAPER.md:339 writes sqrt(d) with d the hidden size — notation).
"""
from __future__ import annotations

import math

import torch


def attention_fwd_ref(q, k, v, cu_seqlens, scale=None):
    """q, k, v: [T, H, D] (any float dtype) -> (o fp32 [T,H,D], lse fp32 [H,T])."""
    q = q.detach().float().cpu()
    k = k.detach().float().cpu()
    v = v.detach().float().cpu()
    T, H, D = q.shape
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    o = torch.zeros((T, H, D), dtype=torch.float32)
    lse = torch.zeros((H, T), dtype=torch.float32)
    cu = [int(x) for x in cu_seqlens]
    for b in range(len(cu) - 1):
        s0, s1 = cu[b], cu[b + 1]
        n = s1 - s0
        if n == 0:
            continue
        qb = q[s0:s1].transpose(0, 1)  # [H, n, D]
        kb = k[s0:s1].transpose(0, 1)
        vb = v[s0:s1].transpose(0, 1)
        s = torch.matmul(qb, kb.transpose(1, 2)) * scale
        mask = torch.ones((n, n), dtype=torch.bool).triu(1)
        s.masked_fill_(mask, float("-inf"))
        lse_b = torch.logsumexp(s, dim=-1)  # [H, n]
        p = torch.exp(s - lse_b[..., None])
        o[s0:s1] = torch.matmul(p, vb).transpose(0, 1)
        lse[:, s0:s1] = lse_b
    return o, lse


def attention_bwd_ref(q, k, v, dout, cu_seqlens, scale=None):
    """Gradients of sum(o * dout) by autograd through the fp32 restatement."""
    qf = q.detach().float().cpu().requires_grad_(True)
    kf = k.detach().float().cpu().requires_grad_(True)
    vf = v.detach().float().cpu().requires_grad_(True)
    T, H, D = qf.shape
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    outs = []
    cu = [int(x) for x in cu_seqlens]
    for b in range(len(cu) - 1):
        s0, s1 = cu[b], cu[b + 1]
        n = s1 - s0
        if n == 0:
            continue
        qb = qf[s0:s1].transpose(0, 1)
        kb = kf[s0:s1].transpose(0, 1)
        vb = vf[s0:s1].transpose(0, 1)
        s = torch.matmul(qb, kb.transpose(1, 2)) * scale
        mask = torch.ones((n, n), dtype=torch.bool).triu(1)
        s = s.masked_fill(mask, float("-inf"))
        outs.append(torch.matmul(torch.softmax(s, dim=-1), vb).transpose(0, 1))
    o = torch.cat(outs, dim=0)
    (o * dout.detach().float().cpu()).sum().backward()
    return qf.grad, kf.grad, vf.grad


def attention_sdpa_ref(q, k, v, cu_seqlens, scale=None):
    """Independent check of the restatement: torch SDPA (is_causal) per sequence."""
    q = q.detach().float().cpu()
    k = k.detach().float().cpu()
    v = v.detach().float().cpu()
    out = torch.zeros_like(q)
    cu = [int(x) for x in cu_seqlens]
    for b in range(len(cu) - 1):
        s0, s1 = cu[b], cu[b + 1]
        if s1 == s0:
            continue
        o = torch.nn.functional.scaled_dot_product_attention(
            q[s0:s1].transpose(0, 1), k[s0:s1].transpose(0, 1), v[s0:s1].transpose(0, 1),
            is_causal=True, scale=scale)
        out[s0:s1] = o.transpose(0, 1)
    return out
