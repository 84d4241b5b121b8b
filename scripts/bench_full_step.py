"""C3 full training step (BASELINE.json configs[2]): GPT-13B-shape, 40 layers, fwd + bwd +
optimizer, adaptive (FlexSP) vs static Ulysses SP, one process per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_full_step.py \
        [--layers 40] [--steps 3] [--warmup 2] [--strategy both] [--replicated]

Model: 40 x FlexSPTransformerLayer(hidden 5120, 40 heads, 4x MLP), per-layer activation
checkpointing (the layer inputs of the 252,160-token batch would not fit otherwise).
Model state (default, "ZeRO with PyTorch FSDP" PAPER.md:917): ZeRO-3
sharding over all ranks (paper_2412_01523_b200/zero.py) — per-layer flat bf16 parameter
shards all-gathered before each layer (next layer prefetched on a communication stream),
per-layer gradient buckets reduce-scattered as soon as the layer's backward completes,
fp32 master shards with SGD-momentum (or --optimizer adamw).  --replicated: round 1's
baseline — bf16 replicas, a NCCL all-reduce per parameter after the backward, plain SGD.
One step = for every micro-batch of the plan: 40 layers forward on the rank's loader-order
rows, synthetic loss <out, dy>, backward (recomputing each layer, attention through
FlexSPAttention = the SP path of this repo); then the optimizer update.  Plans: tests/golden/c3_n{N}_{flexsp,static}.json (the
reference planner on the C3 batch).  Timing: CUDA events around the steps, max over ranks.
Prints one JSON line per strategy on rank 0.  Needs >= 2 GPUs (weights + gradients +
checkpoints exceed one GPU's 180 GB at 40 layers).
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist
from torch.utils.checkpoint import checkpoint

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2412_01523_b200.executor import FlexSPExecutor  # noqa: E402
from paper_2412_01523_b200.layer import FlexSPTransformerLayer  # noqa: E402
from bench import ClockSampler  # noqa: E402

HIDDEN, HEADS = 5120, 40


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--strategy", default="both", choices=["flexsp", "static", "both"])
    ap.add_argument("--config", default="c3full")
    ap.add_argument("--per-mb", action="store_true", help="split the SP-path spans per micro-batch")
    ap.add_argument("--replicated", action="store_true",
                    help="round-1 baseline: bf16 replicas + per-parameter all-reduce + SGD")
    ap.add_argument("--optimizer", default="sgd", choices=["sgd", "adamw"])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/fsp_nccl.{os.getpid()}.log")
    dist.init_process_group("nccl", device_id=dev)
    layers = [FlexSPTransformerLayer(HIDDEN, HEADS, device=dev, seed=1000 + i)
              for i in range(args.layers)]
    params = [p for l in layers for p in l.parameters()]
    zs = None
    if not args.replicated:
        from paper_2412_01523_b200.zero import ZeroStack
        zs = ZeroStack(layers, world, rank, optimizer=args.optimizer)
        torch.cuda.empty_cache()
    ex = FlexSPExecutor(world, rank, HEADS, HIDDEN // HEADS, dev)
    # the peak below is the training steps' (model construction materialises full layers
    # before ZeRO-3 shards them)
    torch.cuda.reset_peak_memory_stats(dev)
    strategies = ["flexsp", "static"] if args.strategy == "both" else [args.strategy]
    out = {}
    for strategy in strategies:
        plan = json.loads((ROOT / "tests" / "golden" / f"{args.config}_n{world}_{strategy}.json").read_text())  # noqa: E501
        sp = ex.prepare(plan, plan["lengths"])
        g = torch.Generator(device=dev).manual_seed(1234 + rank)
        xs = [torch.randn((mb.n_local, HIDDEN), generator=g, device=dev, dtype=torch.bfloat16)
              for mb in sp.micro_batches]
        dys = [torch.randn((mb.n_local, HIDDEN), generator=g, device=dev, dtype=torch.bfloat16)
               for mb in sp.micro_batches]

        def step():
            for m in range(len(sp.micro_batches)):
                ex.timer.tag = f"@mb{m}" if args.per_mb else ""
                if zs is not None:
                    zs.begin_micro_batch()
                h = xs[m]
                for layer in layers:
                    h = checkpoint(layer, h, ex, sp, m, use_reentrant=False)
                loss = (h.float() * dys[m].float()).sum()
                if zs is not None:
                    zs.begin_backward()
                if h.requires_grad:
                    loss.backward()
            if zs is not None:  # reduce-scatters already ran during the backward
                zs.step(1e-6)
                return
            for p in params:  # data/sequence-parallel gradient sum (library collective)
                if p.grad is None:
                    p.grad = torch.zeros_like(p)
                dist.all_reduce(p.grad)
            with torch.no_grad():
                torch._foreach_add_(params, [p.grad for p in params], alpha=-1e-6)
            for p in params:
                p.grad = None

        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ex.timer.start()
        clk = ClockSampler(local)
        s.record()
        for _ in range(args.steps):
            step()
        e.record()
        torch.cuda.synchronize()
        ex.timer.stop()
        clocks = clk.stop()
        kern = {k: {"ms": v["ms"] / args.steps, "launches": v["n"] // args.steps,
                    "tflops": v["work"] / v["ms"] / 1e9 if v["work"] and v["ms"] else None}
                for k, v in ex.timer.summary().items()}
        allk = [None] * world
        dist.all_gather_object(allk, kern)
        wall = time.perf_counter() - t0
        ms = torch.tensor([s.elapsed_time(e) / args.steps], dtype=torch.float64, device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        tokens = sum(plan["lengths"])
        out[strategy] = {"ms_per_step": float(ms.item()), "tokens_per_s": tokens / (ms.item() / 1e3),
                         "wall_s_per_step": wall / args.steps, "clocks_rank0": clocks,
                         "sp_path_ms_per_step_per_rank": allk,
                         "groups_per_micro_batch": [sorted((gg["degree"] for gg in mb["selected_groups"]),
                                                           reverse=True) for mb in plan["micro_batches"]]}
        del xs, dys
        torch.cuda.empty_cache()
    if rank == 0:
        line = {"metric": "tokens/sec/step, full fwd+bwd step (C3, GPT-13B shape)", "n_gpus": world,
                "layers": args.layers, "tokens": sum(plan["lengths"]), "steps": args.steps,
                "warmup": args.warmup, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": "C3: 40 x GPT-13B layer (h=5120, H=40, D=128, MLP 4h), "
                                       "gen_longtail(32, pareto(1.1, 1024), max 131072, seed 0) = "
                                       "252,160 tokens; per-layer activation checkpointing",
                           "model_state": ("bf16 replicas, per-parameter NCCL all-reduce, SGD"
                                           if zs is None else
                                           f"ZeRO-3 over {world} ranks: per-layer all-gather "
                                           "(prefetched) / reduce-scatter buckets, fp32 master "
                                           f"shards, {args.optimizer}"),
                           "model_state_bytes_per_rank": (None if zs is None else
                                                          zs.sharded_bytes()["bytes_per_rank"]),
                           "peak_mem_gb_rank0": torch.cuda.max_memory_allocated(dev) / 1e9},
                "strategies": out}
        if "flexsp" in out and "static" in out:
            line["speedup_flexsp_over_static"] = out["static"]["ms_per_step"] / out["flexsp"]["ms_per_step"]
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
