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
    sys.argv = [a for a in sys.argv if a != "--no-check"]
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
