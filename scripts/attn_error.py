"""Attention error vs the fp32 oracle (dev tool for numerics-affecting kernel variants).

    FSP_LIB=<variant.so> python scripts/attn_error.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.attention_ref import attention_bwd_ref, attention_fwd_ref  # noqa: E402
from paper_2412_01523_b200 import ops  # noqa: E402

H, D = 4, 128
lengths = [4096, 1000, 17, 2300]
cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
T = int(cu[-1])
g = torch.Generator().manual_seed(7)
res = {}
for scale_in in (1.0, 4.0):  # 4x inputs: peakier softmax
    q, k, v, do = (torch.randn(T, H, D, generator=g) * s for s in (scale_in, scale_in, 1.0, 1.0))
    q, k, v, do = (t.bfloat16() for t in (q, k, v, do))
    sched = ops.AttnSchedule.build(cu, "cuda", H, head_dim=D)
    o, lse = ops.attn_fwd(q.cuda(), k.cuda(), v.cuda(), sched)
    dq, dk, dv = ops.attn_bwd(q.cuda(), k.cuda(), v.cuda(), o, do.cuda(), lse, sched)
    torch.cuda.synchronize()
    o_ref, lse_ref = attention_fwd_ref(q, k, v, cu)
    grads = attention_bwd_ref(q, k, v, do, cu)
    eo = (o.float().cpu() - o_ref).abs()
    el = (lse.cpu() - lse_ref).abs()
    line = f"scale {scale_in}: O max {eo.max():.3e} mean {eo.mean():.3e} | lse max {el.max():.3e}"
    for name, got, ref in zip(("dq", "dk", "dv"), (dq, dk, dv), grads):
        e = (got.float().cpu() - ref).abs()
        line += f" | {name} max {e.max():.3e} mean {e.mean():.3e}"
    print(line, flush=True)
