"""Context-parallel (ring) attention over real NVSwitch peer memory, one process per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/ring_parity.py TOKENS [HEADS] [--no-check]

One causal sequence of TOKENS tokens in 2N zig-zag chunks (ring.RingAttention); rank 0
reassembles O / LSE / dQ / dK / dV and checks them against the dense fp32 CPU oracle, and
times the forward + backward of the whole ring (CUDA events, max over ranks)."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.attention_ref import attention_bwd_ref, attention_fwd_ref  # noqa: E402
from paper_2412_01523_b200.executor import PeerHeap  # noqa: E402
from paper_2412_01523_b200.ring import RingAttention, RingLayout, zigzag_rows  # noqa: E402


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    check = "--no-check" not in sys.argv
    sampled = "--sampled" in sys.argv  # long sequences: sampled rows against float64
    sys.argv = [a for a in sys.argv if a not in ("--no-check", "--sampled")]
    if sampled:
        check = False
    S = int(sys.argv[1])
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    D = 128
    rows = S // world
    heap = PeerHeap(RingLayout(rows, H, D).offsets(world)["end"], dev, world)
    ring = RingAttention(world, rank, H, D, heap)
    ring.prepare(rows)
    idx = torch.from_numpy(zigzag_rows(S, world, rank))
    if check:
        g = torch.Generator().manual_seed(11)
        qkv = torch.randn(S, 3, H, D, generator=g).bfloat16()
        dout = torch.randn(S, H, D, generator=g).bfloat16()
        loc = qkv[idx].to(dev)
        do = dout[idx].to(dev)
    elif sampled:  # every rank draws the whole sequence from one seed and keeps its rows
        g = torch.Generator(device=dev).manual_seed(11)
        full = torch.randn((S, 4, H, D), generator=g, device=dev, dtype=torch.bfloat16)
        loc = full[idx.to(dev), :3].contiguous()
        do = full[idx.to(dev), 3].contiguous()
    else:  # timing only (sequences too long for the dense CPU oracle)
        g = torch.Generator(device=dev).manual_seed(11 + rank)
        loc = torch.randn((rows, 3, H, D), generator=g, device=dev, dtype=torch.bfloat16)
        do = torch.randn((rows, H, D), generator=g, device=dev, dtype=torch.bfloat16)
    q, k, v = (loc[:, i].contiguous() for i in range(3))
    for _ in range(2):  # warm-up (and heap / barrier reuse)
        o, lse = ring.forward(q, k, v)
        grads = ring.backward(q, k, v, o, lse, do)
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(3):
        o, lse = ring.forward(q, k, v)
        grads = ring.backward(q, k, v, o, lse, do)
    e.record()
    torch.cuda.synchronize()
    ms = torch.tensor([s.elapsed_time(e) / 3], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ok = True
    flops = 7.0 * D * H * S * S  # causal fwd + bwd, flash-attn convention (2 + 5) * D * H * S^2
    if sampled:
        # sampled query rows (O, dQ) and key rows (dK, dV) of the first and last head against
        # oracle/sampled_ref.py in float64; per-row LSE from the ring itself, checked first
        sys.path.insert(0, str(ROOT / "tests"))
        from sampled_check import check_sequence, sample_rows  # noqa: E402
        rng = np.random.default_rng(0)
        qrows, krows = sample_rows(S, rng, 8), sample_rows(S, rng, 8)
        pos = {int(t): i for i, t in enumerate(idx.tolist())}
        mine = {t: pos[t] for t in set(qrows) | set(krows) if t in pos}
        sel = torch.tensor(sorted(mine.values()), device=dev, dtype=torch.long)
        toks = [t for t, _ in sorted(mine.items(), key=lambda kv: kv[1])]
        part = (toks, o[sel].float().cpu(), lse[:, sel].cpu(), [g_[sel].float().cpu() for g_ in grads])
        parts = [None] * world
        dist.all_gather_object(parts, part)
        report = []
        if rank == 0:
            at = {}
            for tk, oo, ll, gg in parts:
                for n, t in enumerate(tk):
                    at[t] = (oo[n], ll[:, n], [x[n] for x in gg])
            for h in (0, H - 1):
                qh, kh, vh, dh = (full[:, i, h].float().cpu() for i in range(4))
                o_rows = torch.stack([at[t][0][h] for t in qrows])
                dq_rows = torch.stack([at[t][2][0][h] for t in qrows])
                dk_rows = torch.stack([at[t][2][1][h] for t in krows])
                dv_rows = torch.stack([at[t][2][2][h] for t in krows])
                # per-row LSE / O of the whole sequence for the key-row check: one
                # single-GPU causal pass of this head with the repo's own kernel
                from paper_2412_01523_b200 import ops as ops_
                sched1 = ops_.AttnSchedule.build(np.array([0, S], np.int32), dev, 1, head_dim=D)
                o1, lse1 = ops_.attn_fwd(*(full[:, i, h].contiguous().view(S, 1, D) for i in range(3)),
                                         sched1)
                res = check_sequence(qh, kh, vh, dh, o_rows, dq_rows, dk_rows, dv_rows,
                                     o1[:, 0].cpu(), lse1[0].cpu(), qrows, krows,
                                     f"ring S={S} head {h}")
                ring_lse = torch.stack([at[t][1][h] for t in qrows])
                res["ring_lse_vs_single_gpu_max"] = float((ring_lse - lse1[0, qrows].cpu()).abs().max())
                res["ok"] = res["ok"] and res["ring_lse_vs_single_gpu_max"] <= 1e-2
                report.append(res)
            ok = all(r["ok"] for r in report)
            print(json.dumps({"tokens": S, "world": world, "heads": H, "mode": "sampled",
                              "ms_fwd_bwd": float(ms.item()),
                              "tflops_per_gpu": flops / (ms.item() / 1e3) / 1e12 / world,
                              "checked": report, "ok": ok}), flush=True)
        flag = torch.tensor([1 if ok else 0], device=dev)
        dist.broadcast(flag, 0)
        dist.destroy_process_group()
        sys.exit(0 if flag.item() else 1)
    if not check:
        if rank == 0:
            print(json.dumps({"tokens": S, "world": world, "heads": H,
                              "ms_fwd_bwd": float(ms.item()),
                              "tflops_whole_ring": flops / (ms.item() / 1e3) / 1e12,
                              "tflops_per_gpu": flops / (ms.item() / 1e3) / 1e12 / world,
                              "ok": True}), flush=True)
        dist.destroy_process_group()
        return
    parts = [None] * world
    dist.all_gather_object(parts, (idx, o.float().cpu(), lse.cpu(), [t.float().cpu() for t in grads]))
    if rank == 0:
        o_all, lse_all, g_all = torch.empty(S, H, D), torch.empty(H, S), torch.empty(S, 3, H, D)
        for ix, oo, ll, gg in parts:
            o_all[ix], lse_all[:, ix] = oo, ll
            for i in range(3):
                g_all[ix, i] = gg[i]
        cu = np.array([0, S], np.int32)
        o_ref, lse_ref = attention_fwd_ref(qkv[:, 0], qkv[:, 1], qkv[:, 2], cu)
        refs = attention_bwd_ref(qkv[:, 0], qkv[:, 1], qkv[:, 2], dout, cu)
        e_o = (o_all - o_ref).abs()
        ok = bool(e_o.max() <= 2e-2 and e_o.mean() <= 2e-3)
        errs = []
        for i, rf in enumerate(refs):
            errs.append(float((g_all[:, i] - rf).abs().max()))
            ok = ok and bool(torch.allclose(g_all[:, i], rf, atol=5e-2, rtol=5e-2))
        print(json.dumps({"tokens": S, "world": world, "heads": H, "o_max": float(e_o.max()),
                          "grad_max": errs, "ms_fwd_bwd": float(ms.item()),
                          "tflops_whole_ring": flops / (ms.item() / 1e3) / 1e12, "ok": ok}),
              flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
