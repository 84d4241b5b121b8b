"""Profile the SP step on B200 and fit the reference planner's cost model to it.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/calibrate.py [--out profiles/r01_calibration]

Writes <out>.csv (the reference's ProfileRecord CSV) and, when the reference package is
importable (baseline/_ref on the GPU box), <out>.json with the fitted CostCoefficients and
the fit's relative errors (seqplan.cost_model.fit_coefficients).  One process per GPU;
groups of every degree d <= N run on ranks [0, d).
"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
for cand in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
    if cand.is_dir():
        sys.path.insert(0, str(cand))

from paper_2412_01523_b200 import calibrate  # noqa: E402
from paper_2412_01523_b200.executor import FlexSPExecutor  # noqa: E402

H, D = 32, 128
BW = {1: 1e15}  # d = 1 exchanges nothing (the devices_per_node=1 tier of the B200 plans)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r01_calibration"))
    ap.add_argument("--per-degree", type=int, default=5)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--batches", default="c2,c3", help="golden batches the loads are drawn from")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG_FILE", f"/tmp/fsp_nccl.{os.getpid()}.log")
        dist.init_process_group("nccl", device_id=dev)
    # loads drawn from the C2 and C3 long-tail batches (1K .. 131K-token sequences), so the
    # fit covers the lengths the planner actually deals out
    lengths_all = []
    for name in args.batches.split(","):
        lengths_all += json.loads((ROOT / "tests" / "golden" / f"{name}_n1_flexsp.json").read_text())["lengths"]
    degrees = [d for d in (1, 2, 4, 8) if d <= world]
    loads = calibrate.group_loads(lengths_all, degrees, args.per_degree)
    ex = FlexSPExecutor(world, rank, H, D, dev)
    rows = []
    for d, lengths in loads:
        plan = {"schema": 1, "strategy": "profile", "micro_batches": [{"selected_groups": [
            {"slot_id": 0, "degree": d, "sequence_indices": list(range(len(lengths)))}]}]}
        sp = ex.prepare(plan, lengths)
        g = torch.Generator(device=dev).manual_seed(rank)
        qkv = [torch.randn((mb.n_local, 3, H, D), generator=g, device=dev, dtype=torch.bfloat16)
               for mb in sp.micro_batches]
        dout = [torch.randn((mb.n_local, H, D), generator=g, device=dev, dtype=torch.bfloat16)
                for mb in sp.micro_batches]
        for _ in range(2):
            ex.step(sp, qkv, dout)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ex.timer.start()
        for _ in range(args.reps):
            ex.step(sp, qkv, dout)
        torch.cuda.synchronize()
        ex.timer.stop()
        summ = ex.timer.summary()
        mine = {"comp": (summ.get("attn_fwd", {}).get("ms", 0.0) + summ.get("attn_bwd", {}).get("ms", 0.0))
                / args.reps / 1e3,
                # kernel-only exchange time: the a2a span minus the group barrier that
                # closes it (the barrier holds the other members' compute skew, which the
                # cost model's comm term does not describe)
                "comm": max(0.0, summ.get("a2a", {}).get("ms", 0.0) -
                            summ.get("group_barrier", {}).get("ms", 0.0)) / args.reps / 1e3}
        allr = [mine]
        if world > 1:
            allr = [None] * world
            dist.all_gather_object(allr, mine)
        members = allr[:d]
        rows.append(calibrate.GroupMeasurement(
            tuple(lengths), d, BW.get(d, 7.7e11), max(m["comp"] for m in members),
            max(m["comm"] for m in members),
            calibrate.step_bytes_per_device(lengths, d, H, D)))
    if rank == 0:
        calibrate.write_profile_csv(args.out + ".csv", rows)
        result = {"records": len(rows), "degrees": degrees, "world": world}
        try:
            fr, merged = calibrate.fit(rows, allow_underdetermined=len(degrees) < 2)
            pred = calibrate.predict(merged, rows)
            result["per_degree"] = calibrate.per_degree_errors(merged, rows)
            result.update({"coefficients": merged.to_json_dict(),
                           "comp_rel_error": fr.comp_rel_error, "mem_rel_error": fr.mem_rel_error,
                           "comm_rel_error_d_ge_2": pred["comm_rel_error_d_ge_2"],
                           "clamped": list(fr.clamped), "warnings": list(fr.warnings)})
        except ImportError as exc:  # reference package not shipped to this box
            result["fit"] = f"skipped: {exc}"
        Path(args.out + ".json").write_text(json.dumps(result, indent=2) + "\n")
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
