"""Planner/executor overlap in a training loop.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/train_demo.py \
        [--steps 6] [--layers 8] [--workers 2] [--lookahead 2]

Rank 0 runs a PlanPipeline: the reference planner (seqplan.solve_batch with the full-step
coefficients of tests/golden/c3full_*.json, 10 s MILP time limit) plans the next
`lookahead` long-tail batches in worker processes while the current step trains; each
plan is broadcast to every rank, turned into device tables (FlexSPExecutor.prepare) and
trained: `layers` x GPT-13B-shape layers (FlexSPTransformerLayer, activation
checkpointing), NCCL gradient all-reduce, SGD.  Prints one JSON line per step on rank 0
with the step time, the planner's solve time for that batch and how long training
waited for it (0 when planning is hidden), then a summary line.
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
from paper_2412_01523_b200.planning import PlanPipeline, broadcast_plan, import_seqplan  # noqa: E402

HIDDEN, HEADS = 5120, 40


def batches(n_steps: int):
    seqplan = import_seqplan()
    from seqplan.simulator import gen_longtail
    for i in range(n_steps):  # C3-like long-tail batches, a fresh draw per step
        yield gen_longtail(32, ("pareto", 1.1, 1024), 131072, seed=100 + i)[0]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--lookahead", type=int, default=2)
    ap.add_argument("--time-limit", type=float, default=10.0)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/fsp_nccl.{os.getpid()}.log")
    dist.init_process_group("nccl", device_id=dev)
    ref_plan = json.loads((ROOT / "tests" / "golden" / f"c3full_n{world}_flexsp.json").read_text())
    # the coefficients are per 40 layers; this demo trains `layers` of them
    coeffs = dict(ref_plan["coefficients"])
    for key in ("alpha1", "alpha2", "alpha3"):
        coeffs[key] *= args.layers / 40.0
    pipe = None
    if rank == 0:
        pipe = iter(PlanPipeline(batches(args.steps), ref_plan["cluster"], coeffs,
                                 {"jobs": 4, "time_limit": args.time_limit},
                                 lookahead=args.lookahead, workers=args.workers))
    layers = [FlexSPTransformerLayer(HIDDEN, HEADS, device=dev, seed=1000 + i)
              for i in range(args.layers)]
    params = [p for l in layers for p in l.parameters()]
    ex = FlexSPExecutor(world, rank, HEADS, HIDDEN // HEADS, dev)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    log = []
    t_loop = time.perf_counter()
    for step in range(args.steps):
        t0 = time.perf_counter()
        st = next(pipe) if rank == 0 else None
        info = broadcast_plan(None if st is None else {"plan": st.plan, "solve_s": st.solve_s,
                                                        "wait_s": st.wait_s})
        plan = info["plan"]
        sp = ex.prepare(plan, plan["lengths"])
        for m, mb in enumerate(sp.micro_batches):
            h = torch.randn((mb.n_local, HIDDEN), generator=g, device=dev, dtype=torch.bfloat16)
            dy = torch.randn((mb.n_local, HIDDEN), generator=g, device=dev, dtype=torch.bfloat16)
            for layer in layers:
                h = checkpoint(layer, h, ex, sp, m, use_reentrant=False)
            (h.float() * dy.float()).sum().backward()
        for p in params:
            if p.grad is None:
                p.grad = torch.zeros_like(p)
            dist.all_reduce(p.grad)
        with torch.no_grad():
            torch._foreach_add_(params, [p.grad for p in params], alpha=-1e-6)
        for p in params:
            p.grad = None
        torch.cuda.synchronize()
        step_s = time.perf_counter() - t0
        if rank == 0:
            rec = {"step": step, "tokens": sum(plan["lengths"]), "step_s": step_s,
                   "planner_solve_s": info["solve_s"], "trainer_waited_s": info["wait_s"],
                   "groups": [sorted((gg["degree"] for gg in mb["selected_groups"]), reverse=True)
                              for mb in plan["micro_batches"]]}
            log.append(rec)
            print(json.dumps(rec), flush=True)
    total = time.perf_counter() - t_loop
    if rank == 0:
        later = log[1:]
        print(json.dumps({
            "summary": True, "n_gpus": world, "layers": args.layers, "steps": args.steps,
            "workers": args.workers, "lookahead": args.lookahead, "loop_s": total,
            "mean_solve_s": sum(r["planner_solve_s"] for r in log) / len(log),
            "waited_after_first_step_s": sum(r["trainer_waited_s"] for r in later),
            "train_s_after_first_step": sum(r["step_s"] for r in later)}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
