"""CPU SP-step oracle used as the bench's CPU baseline — TEST INFRASTRUCTURE ONLY.

The reference has no executor, so its "CPU implementation of the path" is
this port: the per-step work of PAPER.md:336-348 for one d=1 group (pack the loader-
order tokens into the group's packed order, varlen causal attention fwd+bwd in fp32,
unpack), i.e. exactly what the GPU step computes at N=1, on the host's cores.  The
attention runs through torch's CPU flash-attention SDPA kernel (fp32, all threads) —
the fastest CPU path available here, ~10x the plain restatement in attention_ref.py
(which tests/test_oracle.py pins against this same SDPA).  Timed on a bounded sample of the workload's sequences and scaled to
the full batch by the attention FLOP ratio (attention is >99% of the CPU time).
"""
from __future__ import annotations

import time

import numpy as np
import torch



def attention_flops(lengths, n_heads, head_dim) -> float:
    """fwd + bwd causal attention FLOPs, flash-attn convention: 7 * D * H * sum s^2."""
    s = np.asarray(lengths, dtype=np.float64)
    return 7.0 * head_dim * n_heads * float((s * s).sum())


def pick_sample(lengths, n_heads, head_dim, flop_budget) -> list[int]:
    """Sequences in batch order whose fwd+bwd attention fits `flop_budget` FLOPs
    (always at least one sequence)."""
    out, acc = [], 0.0
    for k, s in enumerate(lengths):
        f = attention_flops([s], n_heads, head_dim)
        if out and acc + f > flop_budget:
            continue
        out.append(k)
        acc += f
    return out


def stratified_sample(lengths, n_heads, head_dim, flop_budget, strata=8):
    """Length-stratified sample of a batch for the CPU legs (bench.py's cpu_baseline and
    the --impl reference arm use this same sample, so the two legs agree).

    The sequences are split by length rank into `strata` groups of (nearly) equal count;
    each stratum is represented by the member closest to its median length whose
    fwd+bwd FLOPs fit flop_budget / strata (else its shortest member) and weighted by
    stratum FLOPs / member FLOPs.  Returns [(sequence index, weight)]; the step estimate
    is sum(weight * time of that sequence), i.e. per-stratum FLOP-rate extrapolation —
    short sequences are extrapolated from short ones, long from the longest affordable."""
    lengths = [int(x) for x in lengths]
    order = sorted(range(len(lengths)), key=lambda k: (lengths[k], k))
    strata = max(1, min(strata, len(order)))
    per = flop_budget / strata
    out = []
    for i in range(strata):
        members = order[i * len(order) // strata:(i + 1) * len(order) // strata]
        if not members:
            continue
        total = attention_flops([lengths[k] for k in members], n_heads, head_dim)
        if total == 0:
            continue
        med = lengths[members[len(members) // 2]]
        fit = [k for k in members if attention_flops([lengths[k]], n_heads, head_dim) <= per]
        pick = min(fit, key=lambda k: (abs(lengths[k] - med), k)) if fit else members[0]
        f = attention_flops([lengths[pick]], n_heads, head_dim)
        out.append((pick, total / f if f else 0.0))
    return out


def cpu_sp_step(lengths, seq_order, n_heads, head_dim, seed=1234, per_sequence=False):
    """One d=1 SP step over the sequences `seq_order` (plan order) on the CPU.

    Loader-order inputs (batch index order) are packed through the group permutation,
    attention fwd+bwd runs in fp32, and dQKV is unpacked back to loader order.
    Returns (tokens, seconds), or with per_sequence=True (tokens, seconds, {sequence index:
    attention seconds}, pack + unpack seconds)."""
    from .layout_ref import group_permutation
    sub_idx = sorted(seq_order)                       # loader order of the sample
    sub_len = [int(lengths[k]) for k in sub_idx]
    order = [sub_idx.index(k) for k in seq_order]     # plan order within the sample
    T = sum(sub_len)
    g = torch.Generator().manual_seed(seed)
    qkv = torch.randn(T, 3, n_heads, head_dim, generator=g).bfloat16()
    dout = torch.randn(T, n_heads, head_dim, generator=g).bfloat16()
    perm, cu, _ = group_permutation(order, sub_len, 1)
    perm_t = torch.as_tensor(perm, dtype=torch.long)
    t0 = time.perf_counter()
    packed = qkv[perm_t]
    dpacked = dout[perm_t]
    dqkv_packed = torch.empty(T, 3, n_heads, head_dim)
    t_pack = time.perf_counter() - t0
    per = {}
    for b in range(len(cu) - 1):
        tb = time.perf_counter()
        s0, s1 = cu[b], cu[b + 1]
        q, k, v = (packed[s0:s1, i].float().transpose(0, 1).requires_grad_(True) for i in range(3))
        o = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None],
                                                             is_causal=True)
        o.backward(dpacked[s0:s1].float().transpose(0, 1)[None])
        for i, t in enumerate((q, k, v)):
            dqkv_packed[s0:s1, i] = t.grad.transpose(0, 1)
        per[seq_order[b]] = time.perf_counter() - tb
    tu = time.perf_counter()
    dqkv = torch.empty_like(dqkv_packed)
    dqkv[perm_t] = dqkv_packed
    t_pack += time.perf_counter() - tu
    secs = time.perf_counter() - t0
    if per_sequence:
        return T, secs, per, t_pack
    return T, secs


def cpu_step_estimate(lengths, n_heads, head_dim, flop_budget, seed=1234):
    """Seconds of one full CPU step over `lengths`, estimated from the stratified sample
    (stratified_sample): sum over the picked sequences of weight x measured attention
    time, plus pack/unpack time scaled by tokens.  Returns (seconds, description dict)."""
    picks = stratified_sample(lengths, n_heads, head_dim, flop_budget)
    seqs = [k for k, _ in picks]
    T, secs, per, t_pack = cpu_sp_step(lengths, seqs, n_heads, head_dim, seed=seed,
                                       per_sequence=True)
    est = sum(w * per[k] for k, w in picks) + t_pack * sum(lengths) / max(T, 1)
    frac = attention_flops([lengths[k] for k in seqs], n_heads, head_dim) / \
        attention_flops(lengths, n_heads, head_dim)
    return est, {"sequences": seqs, "weights": [w for _, w in picks], "tokens": T,
                 "flop_fraction": frac, "measured_s": secs, "extrapolation": est / secs}
