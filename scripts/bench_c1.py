"""BASELINE configs[0]: tiny GPT attention (hidden 256, 4 heads of 64,
2 layers), the reference planner's two-tier plan for 16 long-tail sequences <= 4K tokens
(tests/golden/c1_flexsp_2tier.json: micro-batches [1,1] [2] [1,1] [1,1]), the varlen SP
step fwd+bwd on 2 ranks — timed on the CPU oracle path (gloo, torch fp32, SURVEY §8d
"CPU path timed beside it" (2)) and on 2 B200s (this repo's executor).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/bench_c1.py --device cpu
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/bench_c1.py --device cuda

CPU path (TEST-INFRASTRUCTURE oracle code, timed as the baseline): per layer and
micro-batch, each rank packs its group's shard (layout_ref tables), runs Eq. (2) with gloo
all_to_all_single for d = 2 groups, causal attention fwd+bwd per sequence with torch's CPU
SDPA in fp32 (cores / 2 threads per rank), Eq. (4) back, and unpacks.  GPU path:
FlexSPExecutor.step per layer.  One JSON line per run (rank 0): tokens/s = the batch's
37,202 tokens / max-over-ranks time of one step (both layers).
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

H, D, LAYERS = 4, 64, 2


def cpu_layer(plan, lengths, rank, world, qkv, dout):
    """One layer's SP step on this rank (fwd + bwd); returns (out, dqkv) in loader order."""
    from oracle import layout_ref
    from oracle.ulysses_ref import head2seq, seq2head
    T = qkv.shape[0]
    out = torch.zeros(T, H, D)
    dqkv = torch.zeros(T, 3, H, D)
    for mb in plan["micro_batches"]:
        for g in layout_ref.microbatch_tables(mb, lengths, world):
            if not g["rank_begin"] <= rank < g["rank_begin"] + g["degree"]:
                continue
            d, j = g["degree"], rank - g["rank_begin"]
            R = g["padded"] // d
            tok = torch.as_tensor(g["perm"][j * R:(j + 1) * R], dtype=torch.long)
            live = tok >= 0
            shard = torch.zeros(R, 3, H, D)
            shard[live] = qkv[tok[live]]
            dshard = torch.zeros(R, 1, H, D)
            dshard[live, 0] = dout[tok[live]]
            if d > 1:  # Eq. (2): the d = 2 group is the whole gloo world here
                heads, dheads = seq2head(shard), seq2head(dshard)
            else:
                heads, dheads = shard, dshard
            cu = g["cu_seqlens"]
            o_h = torch.zeros(heads.shape[0], heads.shape[2], D)
            dqkv_h = torch.zeros_like(heads)
            for b in range(len(cu) - 1):
                s0, s1 = int(cu[b]), int(cu[b + 1])
                q, k, v = (heads[s0:s1, i].transpose(0, 1).clone().requires_grad_(True)
                           for i in range(3))
                o = torch.nn.functional.scaled_dot_product_attention(q[None], k[None], v[None],
                                                                     is_causal=True)
                o.backward(dheads[s0:s1, 0].transpose(0, 1)[None])
                o_h[s0:s1] = o[0].detach().transpose(0, 1)
                for i, t in enumerate((q, k, v)):
                    dqkv_h[s0:s1, i] = t.grad.transpose(0, 1)
            if d > 1:  # Eq. (4)
                o_sh = head2seq(o_h[:, None], n_heads=H)[:, 0]
                dqkv_sh = head2seq(dqkv_h, n_heads=H)
            else:
                o_sh, dqkv_sh = o_h, dqkv_h
            out[tok[live]] = o_sh[live]
            dqkv[tok[live]] = dqkv_sh[live]
    return out, dqkv


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--device", default="cpu", choices=["cpu", "cuda"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    plan = json.loads((ROOT / "tests" / "golden" / "c1_flexsp_2tier.json").read_text())
    lengths = plan["lengths"]
    T = sum(lengths)
    g = torch.Generator().manual_seed(1)
    qkv_all = [torch.randn(T, 3, H, D, generator=g).bfloat16() for _ in range(LAYERS)]
    dout_all = [torch.randn(T, H, D, generator=g).bfloat16() for _ in range(LAYERS)]
    if args.device == "cpu":
        dist.init_process_group("gloo")
        cores = max(1, len(os.sched_getaffinity(0)) // world)
        torch.set_num_threads(cores)
        qkv_f = [x.float() for x in qkv_all]
        dout_f = [x.float() for x in dout_all]

        def step():
            for layer in range(LAYERS):
                cpu_layer(plan, lengths, rank, world, qkv_f[layer], dout_f[layer])

        for _ in range(args.warmup):
            step()
        dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        secs = torch.tensor([(time.perf_counter() - t0) / args.steps], dtype=torch.float64)
        dist.all_reduce(secs, op=dist.ReduceOp.MAX)
        ms = float(secs.item()) * 1e3
        extra = {"impl": "cpu oracle (oracle/ulysses_ref.py + torch CPU SDPA fp32, gloo)",
                 "threads_per_rank": cores}
    else:
        from paper_2412_01523_b200.executor import FlexSPExecutor
        torch.cuda.set_device(local)
        dev = torch.device("cuda", local)
        dist.init_process_group("nccl", device_id=dev)
        ex = FlexSPExecutor(world, rank, H, D, dev)
        sp = ex.prepare(plan, lengths)
        ins = [[q[torch.from_numpy(mb.local_tokens)].to(dev) for mb in sp.micro_batches]
               for q in qkv_all]
        dos = [[o[torch.from_numpy(mb.local_tokens)].to(dev) for mb in sp.micro_batches]
               for o in dout_all]

        def step():
            for layer in range(LAYERS):
                ex.step(sp, ins[layer], dos[layer])

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        extra = {"impl": "FlexSPExecutor on B200 (sm_100a kernels)"}
    if rank == 0:
        print(json.dumps({
            "config": "C1 (BASELINE configs[0]): tiny GPT attention, hidden 256 = 4 heads x 64, "
                      "2 layers, 16 long-tail sequences <= 4K (37,202 tokens), reference "
                      "planner two-tier plan [1,1] [2] [1,1] [1,1], fwd+bwd",
            "device": args.device, "n_ranks": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "tokens_per_s": T / (ms / 1e3),
            "note": "tokens_per_s counts each of the 37,202 tokens once per step (2 layers)",
            **extra}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
