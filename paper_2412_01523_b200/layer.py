"""The Ulysses transformer layer around the SP attention path.

FlexSP trains GPT models with DeepSpeed-Ulysses-style sequence parallelism:
every rank holds a sequence shard with the full hidden dimension, so the QKV projection,
the output projection and the MLP are plain local GEMMs on the rank's rows, and the only
communication of the layer is the two all-to-alls inside attention.
Under a FlexSP plan the "shard" of a rank is its loader-order rows of the micro-batch
(`RankMicroBatch.local_tokens`), which is exactly what `FlexSPAttention` consumes.

`FlexSPTransformerLayer` is that pre-LayerNorm GPT block (LN -> QKV -> SP attention -> O
-> residual, LN -> MLP(GELU) -> residual) in bf16.  The GEMMs are cuBLAS through torch
(plain library GEMMs — the hot path this repo owns is the SP attention step); the layer
holds ordinary parameters, which `zero.ZeroStack` shards ZeRO-3 style across the world
(§8f rank 4; scripts/bench_full_step.py) or which stay replicated.  This turns the attention-layer step into the per-layer cost of a full
forward/backward step, where the token-linear terms (α2 of the planner's cost model,
pkg/src/seqplan/cost_model.py:5-7) sit beside the quadratic attention term.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from .attention import FlexSPAttention
from .executor import FlexSPExecutor, StepPlan


class FlexSPTransformerLayer(torch.nn.Module):
    def __init__(self, hidden: int, n_heads: int, ffn_mult: int = 4, device="cuda",
                 dtype: torch.dtype = torch.bfloat16, seed: int | None = None):
        super().__init__()
        if hidden % n_heads:
            raise ValueError("hidden must be a multiple of n_heads")
        self.hidden, self.n_heads, self.head_dim = hidden, n_heads, hidden // n_heads
        g = torch.Generator(device="cpu")
        if seed is not None:
            g.manual_seed(seed)

        def w(rows, cols):  # GPT-2 style N(0, 0.02) init, generated on the host (deterministic)
            t = torch.randn(rows, cols, generator=g) * 0.02
            return torch.nn.Parameter(t.to(device=device, dtype=dtype))

        ffn = ffn_mult * hidden
        self.ln1 = torch.nn.LayerNorm(hidden, device=device, dtype=dtype)
        self.ln2 = torch.nn.LayerNorm(hidden, device=device, dtype=dtype)
        self.w_qkv = w(3 * hidden, hidden)
        self.w_o = w(hidden, hidden)
        self.w_fc = w(ffn, hidden)
        self.w_proj = w(hidden, ffn)

    def forward(self, x_local: torch.Tensor, executor: FlexSPExecutor, step_plan: StepPlan,
                micro_batch: int) -> torch.Tensor:
        """x_local: [n_local, hidden] bf16 — this rank's loader-order rows of the micro-batch."""
        n = x_local.shape[0]
        if executor.n_heads != self.n_heads or executor.head_dim != self.head_dim:
            raise ValueError("executor head shape does not match the layer")
        qkv = F.linear(self.ln1(x_local), self.w_qkv).view(n, 3, self.n_heads, self.head_dim)
        att = FlexSPAttention.apply(qkv, executor, step_plan, micro_batch)
        x = x_local + F.linear(att.reshape(n, self.hidden), self.w_o)
        return x + F.linear(F.gelu(F.linear(self.ln2(x), self.w_fc), approximate="tanh"),
                            self.w_proj)

    def flops_per_token(self) -> float:
        """Dense GEMM FLOPs per token, fwd+bwd (6 x parameters of the four matrices)."""
        h = self.hidden
        return 6.0 * (3 * h * h + h * h + 2 * self.w_fc.shape[0] * h)

