"""C3 full training step (BASELINE.json configs[2]): GPT-13B-shape, 40 layers, fwd + bwd +
gradient all-reduce + SGD, adaptive (FlexSP) vs static Ulysses SP, one process per GPU.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/bench_full_step.py \
        [--layers 40] [--steps 3] [--warmup 2] [--strategy both]

Model: 40 x FlexSPTransformerLayer(hidden 5120, 40 heads, 4x MLP), bf16 weights replicated
on every rank (FSDP/ZeRO is SURVEY §8f rank 4, out of scope), per-layer activation
checkpointing (the layer inputs of the 252,160-token batch would not fit otherwise).
One step = for every micro-batch of the plan: 40 layers forward on the rank's loader-order
rows, synthetic loss <out, dy>, backward (recomputing each layer, attention through
FlexSPAttention = the SP path of this repo); then a NCCL all-reduce of every gradient over
all ranks and an SGD update.  Plans: tests/golden/c3_n{N}_{flexsp,static}.json (the
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
    ex = FlexSPExecutor(world, rank, HEADS, HIDDEN // HEADS, dev)
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
                h = xs[m]
                for layer in layers:
                    h = checkpoint(layer, h, ex, sp, m, use_reentrant=False)
                loss = (h.float() * dys[m].float()).sum()
                if h.requires_grad:
                    loss.backward()
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
                                       "252,160 tokens; per-layer activation checkpointing; NCCL "
                                       "gradient all-reduce + SGD (bf16 replicas; FSDP out of scope)"},
                "strategies": out}
        if "flexsp" in out and "static" in out:
            line["speedup_flexsp_over_static"] = out["static"]["ms_per_step"] / out["flexsp"]["ms_per_step"]
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
