"""A/B of an attention-kernel environment switch on one B200 (dev tool): forward and
backward TF/s with the switch off / on, interleaved 3 times, on the C2 batch and fixed
lengths, plus a bit-identity check of O / LSE / dQ / dK / dV between the two settings.

    python scripts/ab_env.py FSP_FWD_EARLY [--off 0 --on 1]
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2412_01523_b200 import ops  # noqa: E402

H, D = 32, 128


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("var")
    ap.add_argument("--off", default="0")
    ap.add_argument("--on", default="1")
    args = ap.parse_args()
    plan = json.loads((ROOT / "tests" / "golden" / "c2_n1_flexsp.json").read_text())
    loads = [("C2", np.asarray(plan["lengths"]))]
    loads += [(f"{s}x{262144 // s}", np.full(262144 // s, s)) for s in (1024, 2048, 4096, 16384)]
    loads += [("mixed 100..3000", np.random.default_rng(0).integers(100, 3000, 150))]
    dev = torch.device("cuda")
    for name, L in loads:
        cu = np.concatenate([[0], np.cumsum(L)]).astype(np.int32)
        T = int(cu[-1])
        ss = float((L.astype(np.float64) ** 2).sum())
        g = torch.Generator(device=dev).manual_seed(0)
        q, k, v, do = (torch.randn((T, H, D), generator=g, device=dev, dtype=torch.bfloat16)
                       for _ in range(4))
        sched = ops.AttnSchedule.build(cu, dev, H, head_dim=D)
        res, outs = {}, {}
        for rep in range(3):
            for val in (args.off, args.on):
                os.environ[args.var] = val
                ms_f = timeit(lambda: ops.attn_fwd(q, k, v, sched))
                o, lse = ops.attn_fwd(q, k, v, sched)
                ms_b = timeit(lambda: ops.attn_bwd(q, k, v, o, do, lse, sched))
                res.setdefault(val, []).append((2 * D * H * ss / ms_f / 1e9, 5 * D * H * ss / ms_b / 1e9))
                if rep == 0:
                    outs[val] = (o, lse) + tuple(ops.attn_bwd(q, k, v, o, do, lse, sched))
        same = all(torch.equal(a, b) for a, b in zip(outs[args.off][:2], outs[args.on][:2]))
        same_kv = all(torch.equal(a, b) for a, b in zip(outs[args.off][3:], outs[args.on][3:]))
        line = {"workload": name, "fwd_bit_identical": same, "dkdv_bit_identical": same_kv}
        for val in (args.off, args.on):
            f = [r[0] for r in res[val]]
            b = [r[1] for r in res[val]]
            line[f"{args.var}={val}"] = {"fwd_tflops": round(max(f), 1), "bwd_tflops": round(max(b), 1),
                                         "fwd_all": [round(x) for x in f], "bwd_all": [round(x) for x in b]}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
