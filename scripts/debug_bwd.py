import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2412_01523_b200 import ops
lens = [int(x) for x in sys.argv[1].split(",")]
H = int(sys.argv[2]); D = 128
cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
T = int(cu[-1])
dev = torch.device("cuda")
qkv = torch.randn(T, 3, H, D, device=dev, dtype=torch.bfloat16)
do = torch.randn(T, H, D, device=dev, dtype=torch.bfloat16)
sched = ops.AttnSchedule.build(cu, dev, H, head_dim=D)
o, lse = ops.attn_fwd(qkv[:, 0], qkv[:, 1], qkv[:, 2], sched)
torch.cuda.synchronize(); print("fwd ok", flush=True)
dq, dk, dv = ops.attn_bwd(qkv[:, 0], qkv[:, 1], qkv[:, 2], o, do, lse, sched)
torch.cuda.synchronize(); print("bwd ok", lens, H, flush=True)
