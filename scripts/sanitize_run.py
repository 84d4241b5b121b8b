"""Small launches of every FlexSP kernel, for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck).  Run under the sanitizer by scripts/sanitize.sh:

    compute-sanitizer --tool racecheck python scripts/sanitize_run.py [case ...]

Cases (all on cuda:0, sizes a sanitizer finishes in minutes):
  pack      fsp_pack_rows / fsp_unpack_rows
  a2a       seq2head + head2seq of an emulated d=4 group with an uneven head split (10 heads)
  barrier   fsp_group_barrier of member 0 of a d=2 group whose peer has already published
            (a serialised sanitizer run cannot host a second spinning member)
  fwd128 / bwd128   D=128 kernels, classic launch (FSP_*_PERSISTENT=0)
  fwd128p / bwd128p D=128 kernels, persistent launch (> 148 schedule entries)
  fused     D=128 fwd + bwd with the head->seq exchange fused into the epilogues (d=2 group
            emulated on one GPU: both members' destinations are local buffers)
  fwd64 / bwd64     D=64 kernels (the C1 shape: 4 heads of 64)
Each case checks its result loosely against a torch reference so a silent corruption
under the sanitizer is also caught.
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2412_01523_b200 import ops  # noqa: E402
from paper_2412_01523_b200.layout import build_microbatch_layout, head_split  # noqa: E402


def _ref_attn(q, k, v, cu):
    out = torch.empty_like(q, dtype=torch.float32)
    for a, b in zip(cu[:-1], cu[1:]):
        if b > a:
            x = torch.nn.functional.scaled_dot_product_attention(
                q[a:b].transpose(0, 1).float(), k[a:b].transpose(0, 1).float(),
                v[a:b].transpose(0, 1).float(), is_causal=True)
            out[a:b] = x.transpose(0, 1)
    return out


def case_pack():
    src = torch.randint(-100, 100, (1000, 384), dtype=torch.int16, device="cuda")
    idx = torch.randperm(1000, device="cuda")[:900].to(torch.int32)
    out = torch.empty((900, 384), dtype=torch.int16, device="cuda")
    ops.pack_rows(src, idx, out)
    back = torch.zeros_like(src)
    ops.unpack_rows(out, idx, back)
    torch.cuda.synchronize()
    assert torch.equal(out, src[idx.long()])


def case_a2a():
    H, D, degree = 10, 64, 4
    lengths = [333, 1, 128, 77, 1000]
    mb = {"selected_groups": [{"slot_id": 0, "degree": degree, "sequence_indices": [2, 0, 4, 1, 3]}]}
    grp = build_microbatch_layout(mb, lengths, degree, n_heads=H).groups[0]
    hb = head_split(H, degree)
    R, hm, T = grp.rows_per_rank, max(b - a for a, b in zip(hb, hb[1:])), grp.padded_tokens
    x = torch.randint(-100, 100, (sum(lengths), 3, H, D), dtype=torch.int16)
    locs = [x[torch.from_numpy(grp.local_tokens(j))].contiguous().cuda() for j in range(degree)]
    recv = [torch.zeros((T, 3, hm, D), dtype=torch.int16, device="cuda") for _ in range(degree)]
    for j in range(degree):
        ops.a2a("seq2head", locs[j].view(locs[j].shape[0], -1), [r.data_ptr() for r in recv],
                degree=degree, rank=j, rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D,
                dst_stride=3 * hm * D, index=torch.from_numpy(grp.pack_index(j)).cuda(),
                head_begin=hb)
    outs = [torch.zeros_like(l) for l in locs]
    table = torch.from_numpy(np.ascontiguousarray(grp.unpack_table().reshape(-1))).cuda()
    for j in range(degree):
        ops.a2a("head2seq", recv[j].view(T, -1), [o.data_ptr() for o in outs], degree=degree,
                rank=j, rows_per_rank=R, n_mats=3, n_heads=H, head_dim=D, dst_stride=3 * H * D,
                index=table, head_begin=hb)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(outs, locs))


def case_barrier():
    sig = [torch.zeros(1024, dtype=torch.int32, device="cuda") for _ in range(2)]
    sig[0][1] = 5  # member 1 already published epoch 5 into member 0's slot
    ops.group_barrier([s.data_ptr() for s in sig], 0, 0, 5)
    torch.cuda.synchronize()
    assert int(sig[1][0]) == 5 and int(sig[0][0]) == 0


def _attn(D, lengths, H, persistent, check=True):
    os.environ["FSP_FWD_PERSISTENT"] = os.environ["FSP_BWD_PERSISTENT"] = "1" if persistent else "0"
    cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
    T = int(cu[-1])
    g = torch.Generator(device="cuda").manual_seed(1)
    q, k, v, do = (torch.randn((T, H, D), generator=g, device="cuda", dtype=torch.bfloat16)
                   for _ in range(4))
    sched = ops.AttnSchedule.build(cu, "cuda", H, head_dim=D)
    o, lse = ops.attn_fwd(q, k, v, sched)
    dq, dk, dv = ops.attn_bwd(q, k, v, o, do, lse, sched)
    torch.cuda.synchronize()
    if check:
        ref = _ref_attn(q, k, v, cu)
        assert (o.float() - ref).abs().max().item() < 3e-2
        assert torch.isfinite(dq.float()).all() and torch.isfinite(dk.float()).all()
    return sched


def case_fwd128():
    _attn(128, [300, 1, 129, 700, 2048, 64], 2, False)


def case_fwd128p():
    s = _attn(128, [300] * 200 + [1, 1000], 1, True)
    assert s.n_fwd > 148 and s.n_bwd > 148


def case_fwd64():
    _attn(64, [300, 1, 129, 700, 2048, 64], 4, False)


def case_fwd64p():
    _attn(64, [300] * 100, 2, True)


def case_fused():
    from paper_2412_01523_b200 import ops as o_
    H, D, degree = 4, 128, 2
    lengths = [333, 1, 128, 77, 1000, 260]
    mb = {"selected_groups": [{"slot_id": 0, "degree": degree, "sequence_indices": [2, 0, 4, 1, 3, 5]}]}
    grp = build_microbatch_layout(mb, lengths, degree, n_heads=H).groups[0]
    hb = head_split(H, degree)
    R, T = grp.rows_per_rank, grp.padded_tokens
    n_loc = [int((grp.shard(j) >= 0).sum()) for j in range(degree)]
    table = torch.from_numpy(np.ascontiguousarray(grp.unpack_table().reshape(-1))).cuda()
    outs = [torch.zeros(n, H, D, dtype=torch.bfloat16, device="cuda") for n in n_loc]
    douts = [torch.zeros(n, 3, H, D, dtype=torch.bfloat16, device="cuda") for n in n_loc]
    g = torch.Generator(device="cuda").manual_seed(3)
    for j in range(degree):
        hn = hb[j + 1] - hb[j]
        sched = o_.AttnSchedule.build(grp.cu_seqlens, "cuda", hn, total_rows=T, head_dim=D)
        qkv = torch.randn((T, 3, hn, D), generator=g, device="cuda", dtype=torch.bfloat16)
        dout = torch.randn((T, hn, D), generator=g, device="cuda", dtype=torch.bfloat16)
        sc = o_.HeadScatter(degree, R, hb[j], H * D, 0, table, [t.data_ptr() for t in outs])
        o, lse = o_.attn_fwd(qkv[:, 0], qkv[:, 1], qkv[:, 2], sched, scatter=sc)
        sc2 = o_.HeadScatter(degree, R, hb[j], 3 * H * D, H * D, table, [t.data_ptr() for t in douts])
        o_.attn_bwd(qkv[:, 0], qkv[:, 1], qkv[:, 2], o, dout, lse, sched, scatter=sc2)
    torch.cuda.synchronize()
    assert all(torch.isfinite(t.float()).all() for t in outs + douts)


CASES = {"pack": case_pack, "a2a": case_a2a, "barrier": case_barrier, "fwd128": case_fwd128,
         "fwd128p": case_fwd128p, "fwd64": case_fwd64, "fwd64p": case_fwd64p, "fused": case_fused}


def main():
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        print(f"case {n}: ok", flush=True)


if __name__ == "__main__":
    main()
