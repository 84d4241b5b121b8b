"""CPU checks of the oracle itself (no GPU): attention restatement vs golden vectors and
torch SDPA; Ulysses SP on gloo world_size=2 equals single-process attention; the
numpy data-movement restatement agrees with the gloo exchange."""
import os
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import layout_ref
from oracle.attention_ref import attention_bwd_ref, attention_fwd_ref, attention_sdpa_ref

GOLDEN = Path(__file__).resolve().parent / "golden"


def _golden():
    z = np.load(GOLDEN / "attn_small.npz")
    bf = lambda a: torch.from_numpy(a).view(torch.bfloat16)  # noqa: E731
    return z, bf(z["q"]), bf(z["k"]), bf(z["v"]), bf(z["do"])


def test_attention_oracle_matches_golden():
    z, q, k, v, do = _golden()
    cu = z["cu_seqlens"]
    o, lse = attention_fwd_ref(q, k, v, cu)
    np.testing.assert_allclose(o.numpy(), z["o"], atol=1e-6)
    np.testing.assert_allclose(lse.numpy(), z["lse"], atol=1e-6)
    dq, dk, dv = attention_bwd_ref(q, k, v, do, cu)
    for got, key in ((dq, "dq"), (dk, "dk"), (dv, "dv")):
        np.testing.assert_allclose(got.numpy(), z[key], atol=1e-5)


def test_attention_oracle_matches_sdpa():
    g = torch.Generator().manual_seed(5)
    cu = np.array([0, 1, 70, 70, 200], dtype=np.int32)
    q, k, v = (torch.randn(200, 3, 32, generator=g) for _ in range(3))
    o, _ = attention_fwd_ref(q, k, v, cu)
    torch.testing.assert_close(o, attention_sdpa_ref(q, k, v, cu), atol=1e-5, rtol=1e-5)


def test_attention_oracle_no_cross_sequence_leak():
    """Packing masks: changing sequence 1 must not change sequence 0."""
    g = torch.Generator().manual_seed(6)
    cu = np.array([0, 50, 120], dtype=np.int32)
    q, k, v = (torch.randn(120, 2, 16, generator=g) for _ in range(3))
    o1, _ = attention_fwd_ref(q, k, v, cu)
    k2 = k.clone()
    k2[60:] += 5.0
    o2, _ = attention_fwd_ref(q, k2, v, cu)
    torch.testing.assert_close(o1[:50], o2[:50])


def _ulysses_worker(rank, world, port, q, cu, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.ulysses_ref import ulysses_attention
    R = q.shape[0] // world
    out = ulysses_attention(q[rank * R:(rank + 1) * R], cu)
    torch.save(out, f"{out_path}.{rank}")
    dist.destroy_process_group()


@pytest.mark.parametrize("heads", [4, 5])
def test_ulysses_gloo_world2_equals_single_process(tmp_path, heads):
    """Eq. (2)-(4) on two gloo ranks == attention without SP (SP is an identity); 5 heads
    exercise the uneven head split (3 + 2)."""
    g = torch.Generator().manual_seed(11)
    lens = [97, 1, 200, 33]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T = int(cu[-1])
    Tp = -(-T // 2) * 2
    qkv = torch.zeros(Tp, 3, heads, 16)
    qkv[:T] = torch.randn(T, 3, heads, 16, generator=g)
    port = 29500 + os.getpid() % 1000
    mp.spawn(_ulysses_worker, args=(2, port, qkv, cu, str(tmp_path / "o")), nprocs=2)
    got = torch.cat([torch.load(tmp_path / f"o.{r}") for r in range(2)])[:T]
    ref, _ = attention_fwd_ref(qkv[:T, 0], qkv[:T, 1], qkv[:T, 2], cu)
    torch.testing.assert_close(got, ref, atol=1e-5, rtol=1e-5)


def test_numpy_exchange_restatement_roundtrip():
    rng = np.random.default_rng(0)
    d, R, M, H, D = 4, 3, 3, 8, 2
    shards = [rng.standard_normal((R, M, H, D)) for _ in range(d)]
    heads = layout_ref.ulysses_seq2head(shards, M, H, D)
    assert heads[1].shape == (d * R, M, H // d, D)
    np.testing.assert_array_equal(heads[2][R:2 * R, :, :, :], shards[1][:, :, 4:6, :])
    back = layout_ref.ulysses_head2seq(heads, M, H, D)
    for a, b in zip(back, shards):
        np.testing.assert_array_equal(a, b)


def test_head_split_uneven():
    assert layout_ref.head_split(52, 8) == [0, 7, 14, 21, 28, 34, 40, 46, 52]
    assert layout_ref.head_split(32, 4) == [0, 8, 16, 24, 32]
    assert layout_ref.head_split(3, 1) == [0, 3]


def test_numpy_exchange_restatement_roundtrip_uneven_heads():
    rng = np.random.default_rng(1)
    d, R, M, H, D = 8, 2, 3, 13, 2
    shards = [rng.standard_normal((R, M, H, D)) for _ in range(d)]
    heads = layout_ref.ulysses_seq2head(shards, M, H, D)
    b = layout_ref.head_split(H, d)
    for j in range(d):
        assert heads[j].shape == (d * R, M, b[j + 1] - b[j], D)
    np.testing.assert_array_equal(heads[5][3 * R:4 * R], shards[3][:, :, b[5]:b[6], :])
    back = layout_ref.ulysses_head2seq(heads, M, H, D)
    for a, c in zip(back, shards):
        np.testing.assert_array_equal(a, c)


def test_sampled_row_restatement_matches_dense_oracle():
    """oracle/sampled_ref.py (the full-size checker) == the dense restatement."""
    from oracle.sampled_ref import key_rows, query_rows
    g = torch.Generator().manual_seed(21)
    lens = [257, 40]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    T, H, D = int(cu[-1]), 2, 32
    q, k, v, do = (torch.randn(T, H, D, generator=g).bfloat16() for _ in range(4))
    o_ref, lse_ref = attention_fwd_ref(q, k, v, cu)
    dq_ref, dk_ref, dv_ref = attention_bwd_ref(q, k, v, do, cu)
    s0, s1, h = int(cu[0]), int(cu[1]), 1
    rows = [0, 1, 100, 256]
    qr = query_rows(q[s0:s1, h], k[s0:s1, h], v[s0:s1, h], do[s0:s1, h], rows)
    np.testing.assert_allclose(qr["o"], o_ref[s0:s1, h][rows].numpy(), atol=1e-5)
    np.testing.assert_allclose(qr["lse"], lse_ref[h, s0:s1][rows].numpy(), atol=1e-5)
    np.testing.assert_allclose(qr["dq"], dq_ref[s0:s1, h][rows].numpy(), atol=1e-4)
    all_rows = list(range(s1 - s0))
    full = query_rows(q[s0:s1, h], k[s0:s1, h], v[s0:s1, h], do[s0:s1, h], all_rows)
    kr = key_rows(q[s0:s1, h], k[s0:s1, h], v[s0:s1, h], do[s0:s1, h], [0, 7, 256],
                  full["lse"], full["delta"])
    np.testing.assert_allclose(kr["dk"], dk_ref[s0:s1, h][[0, 7, 256]].numpy(), atol=1e-4)
    np.testing.assert_allclose(kr["dv"], dv_ref[s0:s1, h][[0, 7, 256]].numpy(), atol=1e-4)


def _c1_worker(rank, world, port, plan, layers_qkv, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(max(1, (os.cpu_count() or 2) // world))
    from oracle.ulysses_ref import ulysses_attention
    lengths = plan["lengths"]
    outs = []
    for qkv in layers_qkv:
        T, _, H, D = qkv.shape
        out = torch.zeros(T, H, D)
        for mb in plan["micro_batches"]:
            for g in layout_ref.microbatch_tables(mb, lengths, world):
                if not g["rank_begin"] <= rank < g["rank_begin"] + g["degree"]:
                    continue
                d, j = g["degree"], rank - g["rank_begin"]
                R = g["padded"] // d
                shard_tok = torch.tensor(g["perm"][j * R:(j + 1) * R])
                live = shard_tok >= 0
                shard = torch.zeros(R, 3, H, D)
                shard[live] = qkv[shard_tok[live]]
                if d == 1:
                    o_sh, _ = attention_fwd_ref(shard[:, 0], shard[:, 1], shard[:, 2], g["cu_seqlens"])
                else:  # the d=2 group is the whole gloo world here
                    o_sh = ulysses_attention(shard, g["cu_seqlens"])
                out[shard_tok[live]] = o_sh[live]
        outs.append(out)
    torch.save(outs, f"{out_path}.{rank}")
    dist.destroy_process_group()


def test_c1_flexsp_plan_world2_equals_single_process(tmp_path):
    """BASELINE configs[0]: the reference planner's two-tier C1 plan
    (tests/golden/c1_flexsp_2tier.json: micro-batches [1,1] [2] [1,1] [1,1]) executed as
    the varlen SP step on 2 gloo ranks — tiny GPT attention, h=256, 4 heads, 2 layers —
    equals single-process attention of every sequence."""
    import json
    plan = json.loads((Path(__file__).resolve().parent / "golden" / "c1_flexsp_2tier.json").read_text())
    lengths = plan["lengths"]
    T, H, D = sum(lengths), 4, 64
    g = torch.Generator().manual_seed(1)
    layers_qkv = [torch.randn(T, 3, H, D, generator=g).bfloat16().float() for _ in range(2)]
    port = 29700 + os.getpid() % 1000
    mp.spawn(_c1_worker, args=(2, port, plan, layers_qkv, str(tmp_path / "c1")), nprocs=2)
    parts = [torch.load(tmp_path / f"c1.{r}") for r in range(2)]
    cu = np.concatenate([[0], np.cumsum(lengths)]).astype(np.int32)
    for li, qkv in enumerate(layers_qkv):
        got = parts[0][li] + parts[1][li]  # every token is produced on exactly one rank
        ref, _ = attention_fwd_ref(qkv[:, 0], qkv[:, 1], qkv[:, 2], cu)
        torch.testing.assert_close(got, ref, atol=1e-4, rtol=1e-4)
