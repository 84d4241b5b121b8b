"""C5: Ulysses all-to-all sweep — fsp peer-memory a2a vs NCCL all_to_all_single.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/a2a_sweep.py [--max-mb 4096]

One group of degree d = N.  Per size S (bytes of the rank's shard, [R, 1, H=32, D=128]
bf16): time (CUDA events, max over ranks, median of iters)
  * fsp:       fsp_a2a_seq2head (pack fused, identity index) + fsp_group_barrier
  * nccl:      torch.distributed.all_to_all_single on a contiguous [d, S/d] buffer
               (best case: no Ulysses transposes)
  * nccl+perm: the Ulysses exchange done with NCCL: head-slice gather into [d, R, H/d, D],
               all_to_all_single, no further copy (receive layout already [d*R, H/d, D])
GB/s = bytes this rank sends to peers ((d-1)/d * S) / time  (= NCCL "busbw" for a2a).
Prints one JSON line per size on rank 0.
"""
import argparse
import json
import os
import statistics
import sys
from pathlib import Path

import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2412_01523_b200 import ops  # noqa: E402
from paper_2412_01523_b200.executor import PeerHeap  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mb", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    d = world
    H, D = 32, 128
    hs = H // d
    row = H * D * 2
    max_bytes = args.max_mb << 20
    R_max = max_bytes // row
    heap = PeerHeap(4096 + max_bytes + 4096, dev, world)
    recv_off = 4096
    src = torch.randn(R_max, H, D, device=dev, dtype=torch.bfloat16)
    epoch = [0]

    def barrier_kernel():
        epoch[0] += 1
        ops.group_barrier([heap.peer(r, 0) for r in range(d)], rank, 0, epoch[0])

    def fsp(R):
        ops.a2a("seq2head", src[:R].view(R, H * D), [heap.peer(r, recv_off) for r in range(d)],
                degree=d, rank=rank, rows_per_rank=R, n_mats=1, n_heads=H, head_dim=D,
                dst_stride=hs * D)
        barrier_kernel()

    nc_in = torch.empty(max_bytes // 2, device=dev, dtype=torch.bfloat16)
    nc_out = torch.empty_like(nc_in)

    def nccl(R):
        n = R * H * D
        dist.all_to_all_single(nc_out[:n], nc_in[:n])

    def nccl_perm(R):
        n = R * H * D
        send = nc_in[:n].view(d, R, hs, D)
        send.copy_(src[:R].view(R, d, hs, D).transpose(0, 1))
        dist.all_to_all_single(nc_out[:n], nc_in[:n])

    def timeit(fn, R):
        for _ in range(3):
            fn(R)
        torch.cuda.synchronize()
        dist.barrier()
        ts = []
        for _ in range(args.iters):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            fn(R)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        t = torch.tensor([statistics.median(ts)], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    size = 1 << 20
    while size <= max_bytes:
        R = max(1, size // row)
        S = R * row
        sent = S * (d - 1) / d
        res = {"degree": d, "bytes_per_rank": S}
        for name, fn in (("fsp", fsp), ("nccl", nccl), ("nccl_perm", nccl_perm)):
            ms = timeit(fn, R)
            res[name] = {"ms": ms, "gbs": sent / (ms / 1e3) / 1e9}
        res["fsp_over_nccl"] = res["nccl"]["ms"] / res["fsp"]["ms"]
        if rank == 0:
            print(json.dumps(res), flush=True)
        size *= 4
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
