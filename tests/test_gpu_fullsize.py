"""Parity at BASELINE's full sizes, through sampled rows (the dense CPU
oracle cannot hold a 32K–384K-token sequence).

* C2 (259,355 tokens, H=32): the whole step through FlexSPExecutor at N=1 with the
  reference planner's plan; O and dQ of sampled query rows and dK/dV of sampled key rows of
  a long, a medium and a short sequence are checked against oracle/sampled_ref.py.
* C4-scale sequence: one 393,216-token sequence (the C4 maximum) with the C4 head count
  H=52, so the fp32 dQ accumulator [H, T, D] spans 2.6e9 elements and the last head's rows
  sit beyond 2^31 (64-bit index math); the last query rows (attending to 384K keys) and
  the first key rows (receiving gradient from 384K queries) of the first and last head.
Key-row gradients use the kernel's own per-row LSE / delta after those are checked on the
sampled query rows (a consistency property of the backward given the forward statistics).
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from sampled_check import check_sequence, sample_rows

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def _check_sequence(q, k, v, do, o, dq, dk, dv, lse, rows, kv_rows, tag):
    """All arguments [s, D] for one (sequence, head) (lse [s]); o/dq/dk/dv from the GPU."""
    res = check_sequence(q, k, v, do, o[rows], dq[rows], dk[kv_rows], dv[kv_rows], o, lse, rows,
                         kv_rows, tag)
    assert res["ok"], res


def _rows(s, rng, n=12):
    return sample_rows(s, rng, n)


def test_c2_full_step_sampled_rows():
    from paper_2412_01523_b200 import ops
    from paper_2412_01523_b200.executor import FlexSPExecutor
    plan = json.loads((GOLDEN / "c2_n1_flexsp.json").read_text())
    lengths = plan["lengths"]
    H, D = 32, 128
    T = sum(lengths)
    offs = np.concatenate([[0], np.cumsum(lengths)])
    g = torch.Generator(device="cuda").manual_seed(4321)
    qkv = torch.randn((T, 3, H, D), generator=g, device="cuda", dtype=torch.bfloat16)
    dout = torch.randn((T, H, D), generator=g, device="cuda", dtype=torch.bfloat16)
    ex = FlexSPExecutor(1, 0, H, D, "cuda")
    sp = ex.prepare(plan, lengths)
    order = np.argsort(lengths)
    seqs = [int(order[-1]), int(order[len(order) // 2]), int(order[3])]  # long, medium, short
    o_full = torch.empty((T, H, D), dtype=torch.bfloat16, device="cuda")
    d_full = torch.empty((T, 3, H, D), dtype=torch.bfloat16, device="cuda")
    toks = [torch.from_numpy(mb.local_tokens).cuda() for mb in sp.micro_batches]

    def sink(m, out, dqkv):
        o_full[toks[m]] = out
        d_full[toks[m]] = dqkv

    ex.step(sp, [qkv[t] for t in toks], [dout[t] for t in toks], sink=sink)
    torch.cuda.synchronize()
    rng = np.random.default_rng(0)
    for kseq in seqs:
        s0, s1 = int(offs[kseq]), int(offs[kseq + 1])
        s = s1 - s0
        # per-row LSE of this sequence from the same kernel (checked below on sampled rows)
        sched = ops.AttnSchedule.build(np.array([0, s], np.int32), "cuda", H, head_dim=D)
        _, lse = ops.attn_fwd(qkv[s0:s1, 0], qkv[s0:s1, 1], qkv[s0:s1, 2], sched)
        for h in (0, 17, 31):
            _check_sequence(qkv[s0:s1, 0, h], qkv[s0:s1, 1, h], qkv[s0:s1, 2, h], dout[s0:s1, h],
                            o_full[s0:s1, h], d_full[s0:s1, 0, h], d_full[s0:s1, 1, h],
                            d_full[s0:s1, 2, h], lse[h], _rows(s, rng), _rows(s, rng),
                            f"C2 seq {kseq} (len {s}) head {h}")


def test_c4_max_length_sequence_sampled_rows():
    from paper_2412_01523_b200 import ops
    S, H, D = 393216, 52, 128
    assert H * S * D > 2 ** 31
    g = torch.Generator(device="cuda").manual_seed(99)
    q, k, v, do = (torch.randn((S, H, D), generator=g, device="cuda", dtype=torch.bfloat16)
                   for _ in range(4))
    sched = ops.AttnSchedule.build(np.array([0, S], np.int32), "cuda", H, head_dim=D)
    o, lse = ops.attn_fwd(q, k, v, sched)
    dq, dk, dv = ops.attn_bwd(q, k, v, o, do, lse, sched)
    torch.cuda.synchronize()
    rows = [S - 1, S - 2, S - 129, S // 2, 131071, 3]
    kv_rows = [0, 1, 127, 128, 4095, S // 3]
    for h in (0, H - 1):
        _check_sequence(q[:, h], k[:, h], v[:, h], do[:, h], o[:, h], dq[:, h], dk[:, h], dv[:, h],
                        lse[h], rows, kv_rows, f"C4-max seq head {h}")
