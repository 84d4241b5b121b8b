"""`FlexSPAttention`: the SP attention step as a torch.autograd.Function.

This is the SP-layer API a model's attention module calls between its QKV projection and
its output projection.  It mirrors the DeepSpeed-Ulysses
`DistributedAttention(local_attn, group)(q, k, v)` call shape the paper says FlexSP
follows, with the static `group` replaced by this step's plan: the caller
hands in its loader-order rows of one micro-batch and receives that micro-batch's output
rows in the same order; which SP group (degree 1/2/4/8) and which peers the rows are
exchanged with is decided by the Plan (pkg/src/seqplan/domain.py:332-400) that
`FlexSPExecutor.prepare` turned into device tables.

    ex = FlexSPExecutor(world, rank, H, D)
    sp = ex.prepare(plan, lengths)            # once per step (plan from seqplan.solve_batch)
    out = FlexSPAttention.apply(qkv_local, ex, sp, m)   # [n_local, 3, H, D] -> [n_local, H, D]
    out.backward(dout)                        # qkv_local.grad: [n_local, 3, H, D]

The executor's exchange buffers live in the symmetric-memory heap and are reused by the
next call, so the autograd node keeps private copies of what the backward needs (the
head-sharded q/k/v and the attention output; a d = 1 group keeps nothing extra because it
computes in place on the caller's rows).  Every rank must call apply/backward for the same
micro-batches in the same order, as with any collective.
"""
from __future__ import annotations

import torch

from .executor import FlexSPExecutor, StepPlan


class FlexSPAttention(torch.autograd.Function):
    @staticmethod
    def forward(ctx, qkv_local: torch.Tensor, executor: FlexSPExecutor, step_plan: StepPlan,
                micro_batch: int):
        mb = step_plan.micro_batches[micro_batch]
        qkv = qkv_local.contiguous()
        out, saved = executor.micro_batch_forward(step_plan, mb, qkv)
        ctx.executor, ctx.step_plan, ctx.micro_batch = executor, step_plan, micro_batch
        ctx.shape = qkv_local.shape
        ctx.idle = out is None
        if ctx.idle:  # this rank holds no group in this micro-batch
            return qkv_local.new_empty((0, executor.n_heads, executor.head_dim))
        out = out.clone()  # the heap region is reused by the next call
        # save_for_backward (not ctx attributes) so activation checkpointing can drop and
        # recompute these like any other saved activation
        if mb.in_place:
            ctx.save_for_backward(qkv, out, saved[2])
        else:
            recv, o_heads, lse = saved
            ctx.save_for_backward(recv.clone(), o_heads.clone(), lse)
        return out

    @staticmethod
    def backward(ctx, dout: torch.Tensor):
        ex, sp, m = ctx.executor, ctx.step_plan, ctx.micro_batch
        mb = sp.micro_batches[m]
        if ctx.idle:
            ex.micro_batch_backward(sp, mb, None, dout)
            return torch.zeros(ctx.shape, dtype=torch.bfloat16, device=dout.device), None, None, None
        saved = ctx.saved_tensors
        dqkv = ex.micro_batch_backward(sp, mb, saved, dout.to(torch.bfloat16).contiguous())
        return dqkv.clone(), None, None, None


def flexsp_attention(qkv_local: torch.Tensor, executor: FlexSPExecutor, step_plan: StepPlan,
                     micro_batch: int) -> torch.Tensor:
    """Functional form of FlexSPAttention.apply."""
    return FlexSPAttention.apply(qkv_local, executor, step_plan, micro_batch)
