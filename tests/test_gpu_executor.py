"""GPU parity of the data-movement kernels (bit-exact) and of the full SP step.

Multi-rank exchanges are emulated on one GPU by calling every member's kernel in turn
with peer pointers aimed at per-member buffers on the same device (the kernels are
rank-local and never wait on each other, so this is safe on a single GPU).
"""
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import layout_ref
from oracle.attention_ref import attention_bwd_ref, attention_fwd_ref

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def _ops():
    from paper_2412_01523_b200 import ops
    return ops


def test_pack_unpack_bit_exact():
    ops = _ops()
    g = torch.Generator().manual_seed(3)
    for rows, cols in ((1000, 3 * 8 * 64), (37, 8), (5000, 24)):
        src = torch.randint(-30000, 30000, (rows, cols), generator=g, dtype=torch.int16)
        idx = torch.randperm(rows, generator=g)[: rows - 3].to(torch.int32)
        idx = torch.cat([idx, torch.tensor([-1, -1], dtype=torch.int32)])
        out = torch.empty((idx.numel(), cols), dtype=torch.int16, device="cuda")
        ops.pack_rows(src.cuda(), idx.cuda(), out)
        ref = torch.zeros_like(out.cpu())
        live = idx >= 0
        ref[live] = src[idx[live].long()]
        assert torch.equal(out.cpu(), ref)
        back = torch.zeros((rows, cols), dtype=torch.int16, device="cuda")
        ops.unpack_rows(out, idx.cuda(), back)
        ref2 = torch.zeros((rows, cols), dtype=torch.int16)
        ref2[idx[live].long()] = src[idx[live].long()]
        assert torch.equal(back.cpu(), ref2)


@pytest.mark.parametrize("degree,H", [(1, 8), (2, 8), (4, 8), (8, 8), (2, 5), (4, 10), (8, 13)])
def test_a2a_emulated_group_bit_exact(degree, H):
    """seq2head (fused pack) and head2seq (fused unpack) for every member of a group,
    against the numpy restatement of Eqs. (2)/(4) on the oracle's layout tables; H not
    divisible by the degree exercises the uneven head split."""
    ops = _ops()
    from paper_2412_01523_b200.layout import build_microbatch_layout, head_split
    D = 64
    lengths = [333, 1, 128, 77, 1000]
    mb = {"selected_groups": [{"slot_id": 0, "degree": degree, "sequence_indices": [2, 0, 4, 1, 3]}]}
    lay = build_microbatch_layout(mb, lengths, degree, n_heads=H)
    grp = lay.groups[0]
    T = sum(lengths)
    g = torch.Generator().manual_seed(degree * 100 + H)
    x = torch.randint(-30000, 30000, (T, 3, H, D), generator=g, dtype=torch.int16)  # loader order
    hb = head_split(H, degree)
    R, hm = grp.rows_per_rank, max(b - a for a, b in zip(hb, hb[1:]))
    locals_ = [x[torch.from_numpy(grp.local_tokens(j))].contiguous().cuda() for j in range(degree)]
    recv = [torch.full((grp.padded_tokens, 3, hm, D), 7, dtype=torch.int16, device="cuda")
            for _ in range(degree)]
    for j in range(degree):
        idx = torch.from_numpy(grp.pack_index(j)).cuda()
        src = locals_[j].view(locals_[j].shape[0], -1) if locals_[j].shape[0] else \
            locals_[j].reshape(0, 3 * H * D)
        ops.a2a("seq2head", src, [r.data_ptr() for r in recv], degree=degree, rank=j,
                rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D, dst_stride=3 * hm * D, index=idx,
                head_begin=hb)
    torch.cuda.synchronize()
    perm = grp.perm
    xp = np.zeros((grp.padded_tokens, 3, H, D), dtype=np.int16)
    xp[perm >= 0] = x.numpy()[perm[perm >= 0]]
    shards = [xp[j * R:(j + 1) * R] for j in range(degree)]
    ref = layout_ref.ulysses_seq2head(shards, 3, H, D)
    for j in range(degree):
        got = recv[j].cpu().numpy()
        np.testing.assert_array_equal(got[:, :, :hb[j + 1] - hb[j]], ref[j])
        assert (got[:, :, hb[j + 1] - hb[j]:] == 7).all()  # padding head slots untouched
    # head2seq back into loader-order local buffers: exact round trip
    outs = [torch.zeros_like(l) for l in locals_]
    table = torch.from_numpy(np.ascontiguousarray(grp.unpack_table().reshape(-1))).cuda()
    for j in range(degree):
        ops.a2a("head2seq", recv[j].view(grp.padded_tokens, -1), [o.data_ptr() for o in outs],
                degree=degree, rank=j, rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D,
                dst_stride=3 * H * D, index=table, head_begin=hb)
    torch.cuda.synchronize()
    for j in range(degree):
        assert torch.equal(outs[j].cpu(), locals_[j].cpu())


@pytest.mark.parametrize("degree,H,D", [(2, 4, 128), (4, 10, 128), (8, 13, 128), (2, 4, 64)])
def test_fused_head2seq_matches_separate_exchange(degree, H, D):
    """Eq. (4) fused into the attention epilogues (FspHeadScatter, ABI 4) stores exactly
    what the attention launch followed by fsp_a2a_head2seq stores: O (forward) and dK / dV
    (backward) bit for bit, dQ to the fp32 reduction order of its atomics; every member
    of an emulated group on one GPU, uneven head splits included."""
    ops = _ops()
    from paper_2412_01523_b200.layout import build_microbatch_layout, head_split
    lengths = [333, 1, 128, 77, 1000, 260]
    mb = {"selected_groups": [{"slot_id": 0, "degree": degree,
                               "sequence_indices": [2, 0, 4, 1, 3, 5]}]}
    lay = build_microbatch_layout(mb, lengths, degree, n_heads=H)
    grp = lay.groups[0]
    hb = head_split(H, degree)
    R, T = grp.rows_per_rank, grp.padded_tokens
    n_loc = [int((grp.shard(j) >= 0).sum()) for j in range(degree)]
    table = torch.from_numpy(np.ascontiguousarray(grp.unpack_table().reshape(-1))).cuda()
    g = torch.Generator().manual_seed(7 + degree)
    ref_o = [torch.zeros(n, H, D, dtype=torch.bfloat16, device="cuda") for n in n_loc]
    got_o = [torch.zeros_like(t) for t in ref_o]
    ref_d = [torch.zeros(n, 3, H, D, dtype=torch.bfloat16, device="cuda") for n in n_loc]
    got_d = [torch.zeros_like(t) for t in ref_d]
    for j in range(degree):
        hn = hb[j + 1] - hb[j]
        sched = ops.AttnSchedule.build(grp.cu_seqlens, "cuda", hn, total_rows=T, head_dim=D)
        qkv = torch.randn(T, 3, hn, D, generator=g).bfloat16().cuda()
        dout = torch.randn(T, hn, D, generator=g).bfloat16().cuda()
        q, k, v = qkv[:, 0], qkv[:, 1], qkv[:, 2]
        o, lse = ops.attn_fwd(q, k, v, sched)
        hm = max(b - a for a, b in zip(hb, hb[1:]))  # head slots of the head-sharded side
        o_pad = torch.zeros(T, hm, D, dtype=torch.bfloat16, device="cuda")
        o_pad[:, :hn] = o
        ops.a2a("head2seq", o_pad.view(T, hm * D), [t.data_ptr() for t in ref_o], degree=degree,
                rank=j, rows_per_rank=R, n_mats=1, n_heads=H, head_dim=D, dst_stride=H * D,
                index=table, head_begin=hb)
        sc = ops.HeadScatter(degree, R, hb[j], H * D, 0, table, [t.data_ptr() for t in got_o])
        o2, _ = ops.attn_fwd(q, k, v, sched, scatter=sc)
        n_real = int(grp.cu_seqlens[-1])  # rows past it are pad rows nobody writes
        assert torch.equal(o2[:n_real], o[:n_real])  # the local copy is still written
        dq, dk, dv = ops.attn_bwd(q, k, v, o, dout, lse, sched)
        dqkv = torch.zeros(T, 3, hm, D, dtype=torch.bfloat16, device="cuda")
        dqkv[:, :, :hn] = torch.stack([dq, dk, dv], dim=1)
        ops.a2a("head2seq", dqkv.view(T, 3 * hm * D), [t.data_ptr() for t in ref_d],
                degree=degree, rank=j, rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D,
                dst_stride=3 * H * D, index=table, head_begin=hb)
        sc = ops.HeadScatter(degree, R, hb[j], 3 * H * D, H * D, table,
                             [t.data_ptr() for t in got_d])
        assert ops.attn_bwd(q, k, v, o, dout, lse, sched, scatter=sc) == (None, None, None)
    torch.cuda.synchronize()
    for j in range(degree):
        assert torch.equal(got_o[j], ref_o[j])
        assert torch.equal(got_d[j][:, 1:], ref_d[j][:, 1:])
        torch.testing.assert_close(got_d[j][:, 0].float(), ref_d[j][:, 0].float(),
                                   atol=2e-2, rtol=2e-2)


def test_fused_head2seq_rejects_bad_tables():
    ops = _ops()
    sched = ops.AttnSchedule.build([0, 256], "cuda", 2, total_rows=256, head_dim=128)
    q = torch.zeros(256, 2, 128, dtype=torch.bfloat16, device="cuda")
    table = torch.zeros(256, dtype=torch.int32, device="cuda")
    dst = torch.zeros(256, 4, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):  # degree * rows_per_rank != total rows
        ops.attn_fwd(q, q, q, sched, scatter=ops.HeadScatter(2, 100, 0, 512, 0, table[:200],
                                                             [dst.data_ptr()] * 2))
    with pytest.raises(ValueError):  # destination row too short for head_offset + heads
        ops.attn_fwd(q, q, q, sched, scatter=ops.HeadScatter(2, 128, 3, 512, 0, table,
                                                             [dst.data_ptr()] * 2))


def _plan_n1(lengths, split):
    mbs = []
    for idx in split:
        mbs.append({"selected_groups": [{"slot_id": 0, "degree": 1, "sequence_indices": idx}]})
    return {"schema": 1, "strategy": "flexsp", "micro_batches": mbs}


def test_executor_world1_matches_oracle():
    """Full step through the executor (pack -> attn -> unpack, fwd+bwd) at N=1."""
    from paper_2412_01523_b200.executor import FlexSPExecutor
    H, D = 4, 128
    lengths = [700, 1, 130, 2048, 64, 300]
    plan = _plan_n1(lengths, [[3, 1, 5], [0, 2, 4]])
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    T = sum(lengths)
    g = torch.Generator().manual_seed(1)
    qkv = torch.randn(T, 3, H, D, generator=g).bfloat16()
    dout = torch.randn(T, H, D, generator=g).bfloat16()
    got_o = torch.zeros(T, H, D)
    got_d = torch.zeros(T, 3, H, D)
    ins, douts = [], []
    for mb in sp.micro_batches:
        tok = torch.from_numpy(mb.local_tokens)
        ins.append(qkv[tok].cuda())
        douts.append(dout[tok].cuda())

    def sink(m, out, dqkv):
        tok = torch.from_numpy(sp.micro_batches[m].local_tokens)
        got_o[tok] = out.float().cpu()
        got_d[tok] = dqkv.float().cpu()

    ex.step(sp, ins, douts, sink=sink)
    torch.cuda.synchronize()
    offs = np.concatenate([[0], np.cumsum(lengths)])
    cu = offs.astype(np.int32)  # loader order == per-sequence order for the oracle
    o_ref, _ = attention_fwd_ref(qkv[:, 0], qkv[:, 1], qkv[:, 2], cu)
    dq, dk, dv = attention_bwd_ref(qkv[:, 0], qkv[:, 1], qkv[:, 2], dout, cu)
    diff = (got_o - o_ref).abs()
    assert diff.max() <= 2e-2 and diff.mean() <= 2e-3
    for i, ref in enumerate((dq, dk, dv)):
        torch.testing.assert_close(got_d[:, i], ref, atol=5e-2, rtol=5e-2)


def test_attention_golden_vectors():
    """Kernel vs the committed oracle vectors (tests/golden/attn_small.npz, D=64)."""
    ops = _ops()
    z = np.load(GOLDEN / "attn_small.npz")
    bf = lambda a: torch.from_numpy(a).view(torch.bfloat16).cuda()  # noqa: E731
    q, k, v, do = bf(z["q"]), bf(z["k"]), bf(z["v"]), bf(z["do"])
    sched = ops.AttnSchedule.build(z["cu_seqlens"], "cuda", 1, head_dim=64)
    o, lse = ops.attn_fwd(q, k, v, sched)
    dq, dk, dv = ops.attn_bwd(q, k, v, o, do, lse, sched)
    torch.cuda.synchronize()
    assert (o.float().cpu() - torch.from_numpy(z["o"])).abs().max() <= 2e-2
    ref_lse = torch.from_numpy(z["lse"])
    # LSE: relative 1e-3 as stated in DESIGN.md §6 (absolute 1e-3 where |lse| < 1)
    assert ((lse.cpu() - ref_lse).abs() / ref_lse.abs().clamp(min=1.0)).max() <= 1e-3
    for got, key in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        torch.testing.assert_close(got.float().cpu(), torch.from_numpy(z[key]), atol=5e-2, rtol=5e-2)


def test_step_from_host_matches_device_step():
    """The pinned-host, copy-overlapped entry point computes the same step."""
    from paper_2412_01523_b200.executor import FlexSPExecutor
    H, D = 4, 128
    lengths = [700, 1, 130, 2048, 64, 300]
    plan = _plan_n1(lengths, [[3, 1, 5], [0, 2, 4]])
    ex = FlexSPExecutor(1, 0, H, D, "cuda", output_slots=2)
    sp = ex.prepare(plan, lengths)
    T = sum(lengths)
    g = torch.Generator().manual_seed(3)
    qkv = torch.randn(T, 3, H, D, generator=g).bfloat16()
    dout = torch.randn(T, H, D, generator=g).bfloat16()
    toks = [torch.from_numpy(mb.local_tokens) for mb in sp.micro_batches]
    res = {}

    def sink_for(tag):
        def sink(m, out, dqkv):
            res[(tag, m)] = (out.float().cpu(), dqkv.float().cpu())
        return sink

    ex.step(sp, [qkv[t].cuda() for t in toks], [dout[t].cuda() for t in toks], sink=sink_for("dev"))
    hq = [qkv[t].contiguous().pin_memory() for t in toks]
    hd = [dout[t].contiguous().pin_memory() for t in toks]
    ho = [torch.zeros((t.numel(), H, D), dtype=torch.bfloat16).pin_memory() for t in toks]
    hg = [torch.zeros((t.numel(), 3, H, D), dtype=torch.bfloat16).pin_memory() for t in toks]
    for _ in range(3):  # three times: buffers and output slots are reused across calls
        ex.step_from_host(sp, hq, hd, host_out=ho, host_dqkv=hg, sink=sink_for("host"))
    torch.cuda.synchronize()
    for m in range(len(toks)):
        torch.testing.assert_close(res[("host", m)][0], res[("dev", m)][0])
        torch.testing.assert_close(res[("host", m)][1], res[("dev", m)][1], atol=2e-2, rtol=2e-2)
        # the results copied back to pinned host memory are the device results
        assert torch.equal(ho[m].float(), res[("host", m)][0])
        assert torch.equal(hg[m].float(), res[("host", m)][1])


def test_step_from_host_prefetch_across_steps():
    """prefetch_next: the next step's first micro-batch is copied during this step's last
    one; consecutive steps with different inputs (and an odd micro-batch count, so the
    double-buffer slots alternate across steps) still compute exactly the device step,
    and a prefetch for other host tensors than the next call's is ignored."""
    from paper_2412_01523_b200.executor import FlexSPExecutor
    H, D = 4, 128
    lengths = [700, 1, 130, 2048, 64, 300]
    plan = _plan_n1(lengths, [[3], [1, 5, 0], [2, 4]])
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    T = sum(lengths)
    toks = [torch.from_numpy(mb.local_tokens) for mb in sp.micro_batches]
    inputs, ref = [], []
    for seed in range(3):
        g = torch.Generator().manual_seed(20 + seed)
        qkv = torch.randn(T, 3, H, D, generator=g).bfloat16()
        dout = torch.randn(T, H, D, generator=g).bfloat16()
        outs = {}
        ex.step(sp, [qkv[t].cuda() for t in toks], [dout[t].cuda() for t in toks],
                sink=lambda m, o, dq, outs=outs: outs.__setitem__(m, (o.float().cpu(), dq.float().cpu())))
        ref.append(outs)
        inputs.append(([qkv[t].contiguous().pin_memory() for t in toks],
                       [dout[t].contiguous().pin_memory() for t in toks]))
    # steps 0 -> 1 -> 2 prefetching the right next inputs, then step 0 after a prefetch of
    # step 1's tensors (mismatch: must copy its own)
    order = [(0, 1), (1, 2), (2, 1), (0, None)]
    for i, nxt in order:
        got = {}
        pre = None if nxt is None else (sp, inputs[nxt][0], inputs[nxt][1])
        ex.step_from_host(sp, inputs[i][0], inputs[i][1], prefetch_next=pre,
                          sink=lambda m, o, dq, got=got: got.__setitem__(m, (o.float().cpu(), dq.float().cpu())))
        torch.cuda.synchronize()
        for m in range(len(toks)):
            torch.testing.assert_close(got[m][0], ref[i][m][0])
            torch.testing.assert_close(got[m][1], ref[i][m][1], atol=2e-2, rtol=2e-2)


def test_flexsp_attention_autograd_two_layers():
    """FlexSPAttention.apply through torch autograd: two layers' forwards of every
    micro-batch run before any backward (so the heap regions are reused in between), and
    outputs and dK/dV equal the executor's own step bit for bit (dQ to fp32 reduction order)."""
    from paper_2412_01523_b200.attention import FlexSPAttention
    from paper_2412_01523_b200.executor import FlexSPExecutor
    H, D = 4, 128
    lengths = [700, 1, 130, 2048, 64, 300]
    plan = _plan_n1(lengths, [[3, 1, 5], [0, 2, 4]])
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    g = torch.Generator().manual_seed(11)
    toks = [torch.from_numpy(mb.local_tokens) for mb in sp.micro_batches]
    T = sum(lengths)
    layers = [(torch.randn(T, 3, H, D, generator=g).bfloat16(), torch.randn(T, H, D, generator=g).bfloat16())
              for _ in range(2)]
    ref = {}
    for li, (qkv, dout) in enumerate(layers):
        def sink(m, out, dqkv, li=li):
            ref[(li, m)] = (out.clone(), dqkv.clone())
        ex.step(sp, [qkv[t].cuda() for t in toks], [dout[t].cuda() for t in toks], sink=sink)
    leaves, outs = {}, {}
    for m, t in enumerate(toks):
        for li, (qkv, _) in enumerate(layers):
            x = qkv[t].cuda().requires_grad_(True)
            leaves[(li, m)] = x
            outs[(li, m)] = FlexSPAttention.apply(x, ex, sp, m)
    for m in reversed(range(len(toks))):
        for li in reversed(range(2)):
            outs[(li, m)].backward(layers[li][1][toks[m]].cuda())
    torch.cuda.synchronize()
    for key, (o_ref, d_ref) in ref.items():
        assert torch.equal(outs[key].detach(), o_ref), key
        grad = leaves[key].grad
        assert torch.equal(grad[:, 1:], d_ref[:, 1:]), key  # dK, dV: one writer per row
        # dQ sums fp32 reductions from several CTAs in whatever order they land
        torch.testing.assert_close(grad[:, 0].float(), d_ref[:, 0].float(), atol=1e-2, rtol=1e-2)


def test_step_from_host_shards_single_rank():
    """The data-loader path at one rank: the whole batch is the shard, the per-plan scatter
    is a local copy through the route table, results come back to pinned host memory —
    equal to the device step (O, dK, dV bit for bit; dQ to its atomics' order)."""
    from paper_2412_01523_b200.executor import FlexSPExecutor
    H, D = 4, 128
    lengths = [700, 1, 130, 2048, 64, 300]
    plan = _plan_n1(lengths, [[3], [1, 5, 0], [2, 4]])
    ex = FlexSPExecutor(1, 0, H, D, "cuda", output_slots=2)
    sp = ex.prepare(plan, lengths, sharded_loader=True)
    T = sum(lengths)
    assert sp.shard_tokens.tolist() == list(range(T))
    g = torch.Generator().manual_seed(9)
    qkv = torch.randn(T, 3, H, D, generator=g).bfloat16()
    dout = torch.randn(T, H, D, generator=g).bfloat16()
    toks = [torch.from_numpy(mb.local_tokens) for mb in sp.micro_batches]
    ref = {}
    ex.step(sp, [qkv[t].cuda() for t in toks], [dout[t].cuda() for t in toks],
            sink=lambda m, o, d: ref.__setitem__(m, (o.cpu(), d.cpu())))
    ho = [torch.zeros((t.numel(), H, D), dtype=torch.bfloat16).pin_memory() for t in toks]
    hg = [torch.zeros((t.numel(), 3, H, D), dtype=torch.bfloat16).pin_memory() for t in toks]
    hq, hd = qkv.pin_memory(), dout.pin_memory()
    for it in range(3):
        ex.step_from_host_shards(sp, hq, hd, host_out=ho, host_dqkv=hg,
                                 prefetch_next=(hq, hd) if it < 2 else None)
    torch.cuda.current_stream().wait_stream(ex.d2h_stream)
    torch.cuda.synchronize()
    for m in range(len(toks)):
        assert torch.equal(ho[m], ref[m][0])
        assert torch.equal(hg[m][:, 1:], ref[m][1][:, 1:])
        torch.testing.assert_close(hg[m][:, 0].float(), ref[m][1][:, 0].float(), atol=1e-2, rtol=1e-2)


@pytest.mark.parametrize("degree,H", [(2, 4), (4, 10)])
def test_fused_head2seq_persistent_matches_classic(degree, H, monkeypatch):
    """The fused head->seq epilogues on the persistent launches (the forward producer waits
    on epi_free before refilling the Q buffer the epilogue staged O in; the backward stages
    dK / dV through the dS^T region) write exactly what the classic one-CTA-per-entry launch
    writes — with far more schedule entries than SMs, so CTAs run several entries each."""
    ops = _ops()
    from paper_2412_01523_b200.layout import build_microbatch_layout, head_split
    D = 128
    lengths = [300] * 240 + [1, 129, 2048, 777]
    mb = {"selected_groups": [{"slot_id": 0, "degree": degree,
                               "sequence_indices": list(range(len(lengths)))}]}
    grp = build_microbatch_layout(mb, lengths, degree, n_heads=H).groups[0]
    hb = head_split(H, degree)
    R, T = grp.rows_per_rank, grp.padded_tokens
    n_loc = [int((grp.shard(j) >= 0).sum()) for j in range(degree)]
    table = torch.from_numpy(np.ascontiguousarray(grp.unpack_table().reshape(-1))).cuda()
    g = torch.Generator(device="cuda").manual_seed(5)
    ins = []
    for j in range(degree):
        hn = hb[j + 1] - hb[j]
        ins.append((torch.randn((T, 3, hn, D), generator=g, device="cuda", dtype=torch.bfloat16),
                    torch.randn((T, hn, D), generator=g, device="cuda", dtype=torch.bfloat16)))
    res = {}
    for mode in ("0", "1"):
        monkeypatch.setenv("FSP_FWD_PERSISTENT", mode)
        monkeypatch.setenv("FSP_BWD_PERSISTENT", mode)
        outs = [torch.zeros(n, H, D, dtype=torch.bfloat16, device="cuda") for n in n_loc]
        grads = [torch.zeros(n, 3, H, D, dtype=torch.bfloat16, device="cuda") for n in n_loc]
        for j in range(degree):
            hn = hb[j + 1] - hb[j]
            sched = ops.AttnSchedule.build(grp.cu_seqlens, "cuda", hn, total_rows=T, head_dim=D)
            if mode == "1":
                assert sched.n_fwd > 148 and sched.n_bwd > 148
            qkv, dout = ins[j]
            sc = ops.HeadScatter(degree, R, hb[j], H * D, 0, table, [t.data_ptr() for t in outs])
            o, lse = ops.attn_fwd(qkv[:, 0], qkv[:, 1], qkv[:, 2], sched, scatter=sc)
            sc2 = ops.HeadScatter(degree, R, hb[j], 3 * H * D, H * D, table,
                                  [t.data_ptr() for t in grads])
            ops.attn_bwd(qkv[:, 0], qkv[:, 1], qkv[:, 2], o, dout, lse, sched, scatter=sc2)
        torch.cuda.synchronize()
        res[mode] = (outs, grads)
    for j in range(degree):
        assert torch.equal(res["0"][0][j], res["1"][0][j])                  # O
        assert torch.equal(res["0"][1][j][:, 1:], res["1"][1][j][:, 1:])    # dK, dV
        torch.testing.assert_close(res["0"][1][j][:, 0].float(), res["1"][1][j][:, 0].float(),
                                   atol=2e-2, rtol=2e-2)                    # dQ (atomics)
