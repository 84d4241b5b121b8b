"""The Ulysses transformer layer around the SP attention path:
FlexSPTransformerLayer on its FlexSP micro-batches == the same block in fp32 on whole
sequences without sequence parallelism (outputs, input and weight gradients)."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

pytestmark = pytest.mark.gpu


def _attention_fp32(q, k, v, cu):
    """Differentiable causal attention per sequence (fp32 CPU), test helper."""
    outs = []
    for b in range(len(cu) - 1):
        s0, s1 = int(cu[b]), int(cu[b + 1])
        qb, kb, vb = (t[s0:s1].transpose(0, 1)[None] for t in (q, k, v))
        outs.append(F.scaled_dot_product_attention(qb, kb, vb, is_causal=True)[0].transpose(0, 1))
    return torch.cat(outs)


def _reference_block(p, x, cu, H, D):
    n, h = x.shape
    a = F.layer_norm(x, (h,), p["ln1.weight"], p["ln1.bias"])
    qkv = (a @ p["w_qkv"].t()).view(n, 3, H, D)
    att = _attention_fp32(qkv[:, 0], qkv[:, 1], qkv[:, 2], cu)
    x = x + att.reshape(n, h) @ p["w_o"].t()
    a2 = F.layer_norm(x, (h,), p["ln2.weight"], p["ln2.bias"])
    return x + F.gelu(a2 @ p["w_fc"].t(), approximate="tanh") @ p["w_proj"].t()


def _close(got, ref, tol):
    got, ref = got.float().cpu().reshape(-1), ref.float().reshape(-1)
    rel = (got - ref).norm() / ref.norm().clamp_min(1e-12)
    cos = F.cosine_similarity(got, ref, dim=0)
    assert rel <= tol and cos >= 0.999, (float(rel), float(cos))


def test_layer_matches_fp32_reference():
    from paper_2412_01523_b200.executor import FlexSPExecutor
    from paper_2412_01523_b200.layer import FlexSPTransformerLayer
    H, D = 2, 128
    hidden = H * D
    lengths = [300, 1, 130, 700, 64]
    plan = {"schema": 1, "strategy": "flexsp", "micro_batches": [
        {"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": [3, 1]}]},
        {"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": [0, 2, 4]}]}]}
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    layer = FlexSPTransformerLayer(hidden, H, seed=0)
    params = {k: v.detach().float().cpu().requires_grad_(True) for k, v in layer.state_dict().items()}
    g = torch.Generator().manual_seed(5)
    T = sum(lengths)
    x = torch.randn(T, hidden, generator=g).bfloat16()
    dy = torch.randn(T, hidden, generator=g).bfloat16()
    offs = np.concatenate([[0], np.cumsum(lengths)])
    for m, mb in enumerate(sp.micro_batches):
        tok = torch.from_numpy(mb.local_tokens)
        xl = x[tok].cuda().requires_grad_(True)
        y = layer(xl, ex, sp, m)
        y.backward(dy[tok].cuda())
        # the micro-batch's sequences in loader order: each contiguous among its rows
        seqs = sorted(int(k) for grp in plan["micro_batches"][m]["selected_groups"]
                      for k in grp["sequence_indices"])
        cu = np.concatenate([[0], np.cumsum([lengths[k] for k in seqs])])
        assert np.array_equal(mb.local_tokens, np.concatenate(
            [np.arange(offs[k], offs[k + 1]) for k in seqs]))
        xr = x[tok].float().requires_grad_(True)
        yr = _reference_block(params, xr, cu, H, D)
        yr.backward(dy[tok].float())
        _close(y.detach(), yr.detach(), 2e-2)
        _close(xl.grad, xr.grad, 3e-2)
    for name, prm in layer.named_parameters():
        _close(prm.grad, params[name].grad, 3e-2)


def test_layer_under_activation_checkpointing():
    """Two stacked layers wrapped in torch.utils.checkpoint (the full-step benchmark's
    setting): the attention forward is recomputed inside backward, and outputs / gradients
    equal the plain autograd run (dQ up to fp32 reduction order)."""
    from torch.utils.checkpoint import checkpoint

    from paper_2412_01523_b200.executor import FlexSPExecutor
    from paper_2412_01523_b200.layer import FlexSPTransformerLayer
    H, D = 2, 128
    lengths = [300, 1, 130, 700, 64]
    plan = {"schema": 1, "strategy": "flexsp", "micro_batches": [
        {"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": [3, 1]}]},
        {"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": [0, 2, 4]}]}]}
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    layers = [FlexSPTransformerLayer(H * D, H, seed=s) for s in (1, 2)]
    g = torch.Generator().manual_seed(9)
    T = sum(lengths)
    x = torch.randn(T, H * D, generator=g).bfloat16()
    dy = torch.randn(T, H * D, generator=g).bfloat16()
    results = []
    for use_ckpt in (False, True):
        for l in layers:
            l.zero_grad(set_to_none=True)
        outs, xgrads = [], []
        for m, mb in enumerate(sp.micro_batches):
            tok = torch.from_numpy(mb.local_tokens)
            h0 = x[tok].cuda().requires_grad_(True)
            h = h0
            for l in layers:
                h = checkpoint(l, h, ex, sp, m, use_reentrant=False) if use_ckpt else l(h, ex, sp, m)
            h.backward(dy[tok].cuda())
            outs.append(h.detach().clone())
            xgrads.append(h0.grad.clone())
        grads = [p.grad.clone() for l in layers for p in l.parameters()]
        results.append((outs, xgrads, grads))
    (o0, x0, g0), (o1, x1, g1) = results
    for a, b in zip(o0, o1):
        assert torch.equal(a, b)
    for a, b in zip(x0 + g0, x1 + g1):
        _close(b, a.float().cpu(), 1e-2)


def test_zero3_stack_gradients_equal_replicated_on_gpu():
    """ZeRO-3 (zero.py) around FlexSPTransformerLayer on cuda with activation checkpointing
    and the SP executor: the gradient shards after a two-micro-batch step equal the
    replicated model's accumulated gradients (world size 1: the reduce-scatter is a copy),
    and the forward outputs are bit-identical."""
    from torch.utils.checkpoint import checkpoint
    from paper_2412_01523_b200.executor import FlexSPExecutor
    from paper_2412_01523_b200.layer import FlexSPTransformerLayer
    from paper_2412_01523_b200.zero import ZeroStack
    H, D = 2, 128
    hidden = H * D
    lengths = [300, 1, 130, 700, 64]
    plan = {"schema": 1, "strategy": "flexsp", "micro_batches": [
        {"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": [3, 1]}]},
        {"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": [0, 2, 4]}]}]}
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    layers = [FlexSPTransformerLayer(hidden, H, seed=i) for i in range(3)]
    ref = [FlexSPTransformerLayer(hidden, H, seed=i) for i in range(3)]
    zs = ZeroStack(layers, 1, 0)
    g = torch.Generator().manual_seed(5)
    T = sum(lengths)
    x = torch.randn(T, hidden, generator=g).bfloat16().cuda()
    dy = torch.randn(T, hidden, generator=g).bfloat16().cuda()
    for m, mb in enumerate(sp.micro_batches):
        tok = torch.from_numpy(mb.local_tokens).cuda()
        zs.begin_micro_batch()
        h = x[tok]
        for l in layers:
            h = checkpoint(l, h, ex, sp, m, use_reentrant=False)
        zs.begin_backward()
        (h.float() * dy[tok].float()).sum().backward()
        hr = x[tok]
        for l in ref:
            hr = checkpoint(l, hr, ex, sp, m, use_reentrant=False)
        (hr.float() * dy[tok].float()).sum().backward()
        assert torch.equal(h.detach(), hr.detach())
    torch.cuda.synchronize()
    for s, l in zip(zs.shards, ref):
        gr = torch.cat([p.grad.float().reshape(-1) for p in l.parameters()])
        # zero.py accumulates the micro-batches in fp32 (the replica in bf16)
        torch.testing.assert_close(s.grad_shard[:gr.numel()], gr, atol=2e-2, rtol=2e-2)
