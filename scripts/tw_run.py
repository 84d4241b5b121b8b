"""Run one fwd + two bwd launches (dev tool for the FSP_*_TIMING profiling builds)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2412_01523_b200 import ops  # noqa: E402

H, D = 32, 128
n, k = os.environ.get("WL", "32768x8").split("x")
L = np.full(int(k), int(n))
cu = np.concatenate([[0], np.cumsum(L)]).astype(np.int32)
T = int(cu[-1])
dev = torch.device("cuda")
qkv = torch.randn(T, 3, H, D, device=dev, dtype=torch.bfloat16)
do = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)
sched = ops.AttnSchedule.build(cu, dev, H, head_dim=D)
q, k_, v = qkv[:, 0], qkv[:, 1], qkv[:, 2]
for _ in range(2):
    o, lse = ops.attn_fwd(q, k_, v, sched)
if os.environ.get("BWD", "1") == "1":
    for _ in range(2):
        ops.attn_bwd(q, k_, v, o, do, lse, sched)
torch.cuda.synchronize()
