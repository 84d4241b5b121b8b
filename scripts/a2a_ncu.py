"""Single-process multi-GPU harness for the Ulysses exchange kernels, for ncu NVLink counters.

    python scripts/a2a_ncu.py --degree 2 [--mb 1024] [--iters 5]
    ncu --metrics nvltx__bytes.sum,nvlrx__bytes.sum,gpu__time_duration.sum,... \
        -k regex:a2a python scripts/a2a_ncu.py --degree 2 --iters 1

One process drives d GPUs (CUDA peer access enabled between all of them), so ncu can
replay the exchange kernels without a multi-rank job (no barrier kernel is launched here:
the launches are ordered by host synchronisation instead).  Each member j runs
fsp_a2a_seq2head (Eq. 2, identity pack) and then fsp_a2a_head2seq (Eq. 4) on a
[R, H=32, D=128] bf16 shard; the bytes a member sends to peers are (d-1)/d of its shard.
Without ncu it prints the per-kernel CUDA-event times with all d members running
concurrently (the step's situation); under ncu the kernels are serialised, so each
launch shows one sender's NVLink TX bytes and duration.
"""
import argparse
import json
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2412_01523_b200 import ops  # noqa: E402


def enable_peer_access(d: int) -> None:
    from cuda.bindings import runtime as rt
    for i in range(d):
        rt.cudaSetDevice(i)
        for j in range(d):
            if i != j:
                err, = rt.cudaDeviceEnablePeerAccess(j, 0)
                if err not in (rt.cudaError_t.cudaSuccess,
                               rt.cudaError_t.cudaErrorPeerAccessAlreadyEnabled):
                    raise RuntimeError(f"peer access {i}->{j}: {err}")
    rt.cudaGetLastError()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--degree", type=int, default=2)
    ap.add_argument("--mb", type=int, default=1024, help="shard bytes per member (MiB)")
    ap.add_argument("--iters", type=int, default=5)
    args = ap.parse_args()
    d = args.degree
    if torch.cuda.device_count() < d:
        raise SystemExit(f"needs {d} GPUs")
    H, D = 32, 128
    hs = H // d
    row = H * D * 2
    R = (args.mb << 20) // row
    devs = [torch.device("cuda", i) for i in range(d)]
    for dev in devs:  # create the primary contexts before enabling peer access
        torch.empty(1, device=dev)
    enable_peer_access(d)
    src = [torch.randn(R, H, D, device=dev, dtype=torch.bfloat16) for dev in devs]
    recv = [torch.empty(d * R, hs, D, device=dev, dtype=torch.bfloat16) for dev in devs]
    back = [torch.empty(R, H, D, device=dev, dtype=torch.bfloat16) for dev in devs]

    def run(direction):
        ev = []
        for j, dev in enumerate(devs):
            with torch.cuda.device(dev):
                s, e = torch.cuda.Event(True), torch.cuda.Event(True)
                s.record()
                if direction == "seq2head":
                    ops.a2a("seq2head", src[j].view(R, H * D), [r.data_ptr() for r in recv],
                            degree=d, rank=j, rows_per_rank=R, n_mats=1, n_heads=H, head_dim=D,
                            dst_stride=hs * D)
                else:
                    ops.a2a("head2seq", recv[j].view(d * R, hs * D), [b.data_ptr() for b in back],
                            degree=d, rank=j, rows_per_rank=R, n_mats=1, n_heads=H, head_dim=D,
                            dst_stride=H * D)
                e.record()
                ev.append((s, e))
        for dev in devs:
            torch.cuda.synchronize(dev)
        return [s.elapsed_time(e) for s, e in ev]

    sent = R * row * (d - 1) / d
    out = {"degree": d, "bytes_per_member": R * row, "sent_per_member": sent}
    for direction in ("seq2head", "head2seq"):
        ts = [run(direction) for _ in range(args.iters)]
        worst = sorted(max(t) for t in ts)[len(ts) // 2]
        out[direction] = {"ms_max_over_members": worst, "gbs_per_member": sent / worst / 1e6}
    # round trip must restore the shards bit-exactly (identity pack / unpack)
    out["round_trip_exact"] = all(torch.equal(a, b) for a, b in zip(src, back))
    print(json.dumps(out), flush=True)
    if not out["round_trip_exact"]:
        raise SystemExit(1)


if __name__ == "__main__":
    main()
