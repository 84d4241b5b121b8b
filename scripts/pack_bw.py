"""HBM bandwidth of the standalone pack / unpack kernels (fsp_pack_rows / fsp_unpack_rows)
at the C2 row shape: 259,355 rows of q/k/v (3·h·2 B = 24 KB) permuted by the packing
permutation of the C2 static SP=8 plan (tests/golden/c2_n8_static.json, group-packed
order) — bytes per launch = read + write of every row.

    python scripts/pack_bw.py [--iters 10]
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:permute --clock-control none python scripts/pack_bw.py --iters 1

Prints one JSON line (CUDA-event ms, GB/s, fraction of MEASURED_PEAKS hbm_gbs) and checks
both directions bit-exact against torch indexing.
"""
import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_2412_01523_b200 import ops  # noqa: E402
from paper_2412_01523_b200.layout import build_plan_layouts  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    plan = json.loads((ROOT / "tests/golden/c2_n8_static.json").read_text())
    lengths = plan["lengths"]
    H, D = 32, 128
    lay = build_plan_layouts(plan, lengths, 8, H)[0]
    perm = np.concatenate([g.perm[g.perm >= 0] for g in lay.groups]).astype(np.int32)
    T = len(perm)
    dev = torch.device("cuda")
    src = torch.randn(T, 3 * H * D, device=dev, dtype=torch.bfloat16)
    packed = torch.empty_like(src)
    back = torch.empty_like(src)
    idx = torch.from_numpy(perm).to(dev)
    row = 3 * H * D * 2
    nbytes = 2 * T * row

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(args.iters):
            s, e = torch.cuda.Event(True), torch.cuda.Event(True)
            s.record()
            fn()
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        return sorted(ts)[len(ts) // 2]

    out = {"rows": T, "row_bytes": row, "bytes_per_launch": nbytes}
    peak = None
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peak = json.loads(pk.read_text()).get("hbm_gbs")
    for name, fn in (("pack", lambda: ops.pack_rows(src, idx, packed)),
                     ("unpack", lambda: ops.unpack_rows(packed, idx, back))):
        ms = timed(fn)
        gbs = nbytes / ms / 1e6
        out[name] = {"ms": ms, "gbs": gbs, "frac_of_hbm_peak": gbs / peak if peak else None}
    out["hbm_peak_gbs"] = peak
    out["pack_exact"] = bool(torch.equal(packed, src[idx.long()]))
    out["round_trip_exact"] = bool(torch.equal(back, src))
    print(json.dumps(out), flush=True)
    if not (out["pack_exact"] and out["round_trip_exact"]):
        raise SystemExit(1)


if __name__ == "__main__":
    main()
