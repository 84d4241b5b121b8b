"""Attention kernels against the strongest stock Blackwell kernels in the image, on the
same packed varlen batches (one B200; dev tool, not the bench).

    python scripts/perf_compare.py [--out profiles/r02_attention_compare.json]

Workloads (~262K tokens per launch, H=32, D=128, causal, bf16):
  C2 — the 259,355-token long-tail batch of BASELINE configs[1] (lengths from the
       committed reference plan), packed varlen;
  S x B fixed lengths 1K..32K, also passed as packed varlen batches.
Kernels:
  fsp       — this repo (fsp_attn_fwd / fsp_attn_bwd);
  cudnn     — cuDNN sm100 fused attention with ragged (cu_seqlens) offsets through
              aten._cudnn_attention_forward / _backward (the varlen path torch exposes);
  cudnn_dense — cuDNN fused SDPA on the fixed-length batches as a dense [B, H, S, D]
              batch (its fastest path; no varlen equivalent for C2);
  flashinfer— flashinfer 0.6 CUTLASS sm100a FMHA, fmha_varlen (forward only: it has no
              backward);
  fa2       — flash_attn_varlen_func 2.8.3 (the FA2 algorithm built for sm_100; the
              paper's own dependency).
TF/s in the flash-attn convention (fwd 2*D*H*sum s^2, bwd 2.5x).  Each timing: 3 warm-up +
10 timed launches, CUDA events; SM clocks sampled with nvidia-smi during the run.
"""
import argparse
import json
import os
import subprocess
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


def workloads():
    plan = json.loads((ROOT / "tests" / "golden" / "c2_n1_flexsp.json").read_text())
    out = [("C2 long-tail", np.asarray(plan["lengths"]))]
    for s in (1024, 2048, 4096, 8192, 16384, 32768):
        out.append((f"{s} x {262144 // s}", np.full(262144 // s, s)))
    return out


def run(name, L, fixed):
    cu = np.concatenate([[0], np.cumsum(L)]).astype(np.int32)
    T, smax = int(cu[-1]), int(L.max())
    ss = float((L.astype(np.float64) ** 2).sum())
    ffwd, fbwd = 2 * D * H * ss, 5 * D * H * ss
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, do = (torch.randn((T, H, D), generator=g, device=dev, dtype=torch.bfloat16)
                   for _ in range(4))
    cu_t = torch.from_numpy(cu).to(dev)
    res = {"workload": name, "tokens": T, "sum_s2": ss}
    sched = ops.AttnSchedule.build(cu, dev, H, head_dim=D)
    ms = timeit(lambda: ops.attn_fwd(q, k, v, sched))
    res["fsp_fwd"] = ffwd / ms / 1e9
    o, lse = ops.attn_fwd(q, k, v, sched)
    ms = timeit(lambda: ops.attn_bwd(q, k, v, o, do, lse, sched))
    res["fsp_bwd"] = fbwd / ms / 1e9
    scale = D ** -0.5
    try:
        f = lambda: torch.ops.aten._cudnn_attention_forward(  # noqa: E731
            q, k, v, None, cu_t, cu_t, smax, smax, True, 0.0, True, False, scale=scale)
        ms = timeit(f)
        res["cudnn_fwd"] = ffwd / ms / 1e9
        r = f()
        oc, lc, seed, off = r[0], r[1], r[6], r[7]
        b = lambda: torch.ops.aten._cudnn_attention_backward(  # noqa: E731
            do, q, k, v, oc, lc, seed, off, torch.empty(0, device=dev), cu_t, cu_t, smax, smax,
            0.0, True, scale=scale)
        res["cudnn_o_maxdiff_vs_fsp"] = float((oc.float() - o.float()).abs().max())
        res["cudnn_bwd"] = fbwd / ms / 1e9 if (ms := timeit(b)) else None
    except Exception as exc:  # noqa: BLE001
        res["cudnn_error"] = str(exc).splitlines()[0][:200]
    if fixed:
        # cuDNN's dense fused SDPA on the same fixed-length batch ([B, H, S, D]), fwd + bwd
        try:
            from torch.nn.attention import SDPBackend, sdpa_kernel
            B, S = len(L), int(L[0])
            qb, kb, vb, dob = (t.reshape(B, S, H, D).transpose(1, 2).contiguous()
                               for t in (q, k, v, do))
            with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
                f = lambda: torch.nn.functional.scaled_dot_product_attention(  # noqa: E731
                    qb, kb, vb, is_causal=True)
                ms = timeit(f)
                res["cudnn_dense_fwd"] = ffwd / ms / 1e9
                qr, kr, vr = (t.clone().requires_grad_(True) for t in (qb, kb, vb))
                ob = torch.nn.functional.scaled_dot_product_attention(qr, kr, vr, is_causal=True)
                ms = timeit(lambda: torch.autograd.grad(ob, (qr, kr, vr), dob, retain_graph=True))
                res["cudnn_dense_bwd"] = fbwd / ms / 1e9
        except Exception as exc:  # noqa: BLE001
            res["cudnn_dense_error"] = str(exc).splitlines()[0][:200]
    try:
        import flashinfer.prefill as fp
        from flashinfer.utils import PosEncodingMode
        mod = fp.get_fmha_module(q.dtype, k.dtype, v.dtype, torch.int32, D, D,
                                 PosEncodingMode.NONE.value, False, False, q.device)
        plan_info = fp.fmha_varlen_plan(mod, cu_t, cu_t, H, True)  # planned once, off the clock
        f = lambda: fp.fmha_varlen(q, k, v, cu_t, cu_t, plan_info=plan_info,  # noqa: E731
                                   max_qo_len=smax, causal=True, sm_scale=scale)
        ms = timeit(f)
        res["flashinfer_fwd"] = ffwd / ms / 1e9
        r = f()
        ofi = r[0] if isinstance(r, (tuple, list)) else r
        res["flashinfer_o_maxdiff_vs_fsp"] = float((ofi.float() - o.float()).abs().max())
    except Exception as exc:  # noqa: BLE001
        res["flashinfer_error"] = str(exc).splitlines()[0][:200]
    try:
        from flash_attn import flash_attn_varlen_func
        f = lambda: flash_attn_varlen_func(q, k, v, cu_t, cu_t, smax, smax, causal=True,  # noqa: E731
                                           softmax_scale=scale)
        ms = timeit(f)
        res["fa2_fwd"] = ffwd / ms / 1e9
        qf, kf, vf = (t.clone().requires_grad_(True) for t in (q, k, v))
        of = flash_attn_varlen_func(qf, kf, vf, cu_t, cu_t, smax, smax, causal=True,
                                    softmax_scale=scale)
        ms = timeit(lambda: torch.autograd.grad(of, (qf, kf, vf), do, retain_graph=True))
        res["fa2_bwd"] = fbwd / ms / 1e9
    except Exception as exc:  # noqa: BLE001
        res["fa2_error"] = str(exc).splitlines()[0][:200]
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/attention_compare.json")
    args = ap.parse_args()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks_event_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits", "-lms", "500"],
                           stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    rows = []
    for name, L in workloads():
        r = run(name, L, fixed=not name.startswith("C2"))
        print(json.dumps(r), flush=True)
        rows.append(r)
    smi.terminate()
    out, _ = smi.communicate()
    mhz = [float(x.split(",")[0]) for x in out.strip().splitlines() if x.strip()]
    clocks = {"sm_mhz_median": float(np.median(mhz)) if mhz else None,
              "sm_mhz_min": min(mhz) if mhz else None, "samples": len(mhz),
              "sw_power_cap_samples": sum(x.split(",")[1].strip() == "Active"
                                          for x in out.strip().splitlines() if "," in x)}
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps({"rows": rows, "clocks": clocks}, indent=1))
    print(json.dumps({"clocks": clocks}))


if __name__ == "__main__":
    main()
