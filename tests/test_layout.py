"""Bit-exact layout parity: host layout builder vs oracle restatement, on plans produced
by the reference planner itself (tests/golden/, made by tests/golden/make_golden.py)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import layout_ref
from paper_2412_01523_b200.layout import (LayoutError, build_microbatch_layout,
                                          build_plan_layouts, load_plan)

GOLDEN = Path(__file__).resolve().parent / "golden"
PLANS = sorted(p.name for p in GOLDEN.glob("*.json"))


def _world(plan: dict) -> int:
    if "cluster" in plan:
        return plan["cluster"]["total_devices"]
    return len(plan["micro_batches"][0]["group_selection"]) // 2 + 1  # catalog size 2N-1


@pytest.mark.parametrize("name", PLANS)
def test_layout_matches_oracle(name):
    plan = load_plan(GOLDEN / name)
    lengths = plan["lengths"]
    world = _world(plan)
    layouts = build_plan_layouts(plan, lengths, world)
    for mb, lay in zip(plan["micro_batches"], layouts):
        ref = layout_ref.microbatch_tables(mb, lengths, world)
        assert len(ref) == len(lay.groups)
        for r, g in zip(ref, lay.groups):
            assert g.rank_begin == r["rank_begin"]
            assert g.degree == r["degree"] and g.slot_id == r["slot_id"]
            assert g.padded_tokens == r["padded"]
            np.testing.assert_array_equal(g.cu_seqlens, np.asarray(r["cu_seqlens"], np.int32))
            np.testing.assert_array_equal(g.perm, np.asarray(r["perm"], np.int64))
            for j, (local, pack) in enumerate(r["shards"]):
                np.testing.assert_array_equal(g.local_tokens(j), np.asarray(local, np.int64))
                np.testing.assert_array_equal(g.pack_index(j), np.asarray(pack, np.int32))
            tab = g.unpack_table()
            assert tab.shape == (g.degree, g.rows_per_rank)


@pytest.mark.parametrize("name", [n for n in PLANS if "flexsp" in n])
def test_dispatch_rederived_from_assignment(name):
    """The plan's per-group sequence lists equal the oracle's re-derivation of the
    reference's dealing rule (planner.py:499-509) from the bucket assignment."""
    plan = load_plan(GOLDEN / name)
    lengths = plan["lengths"]
    for mb in plan["micro_batches"]:
        dealt = layout_ref.deal_sequences(mb["buckets"]["member_indices"], mb["assignment"],
                                          mb["group_selection"], lengths)
        got = {g["slot_id"]: g["sequence_indices"] for g in mb["selected_groups"]}
        assert got == dealt


def test_every_token_exactly_once():
    plan = load_plan(GOLDEN / "c2_n8_flexsp.json")
    lengths = plan["lengths"]
    layouts = build_plan_layouts(plan, lengths, 8)
    seen = np.concatenate([g.perm[g.perm >= 0] for lay in layouts for g in lay.groups])
    np.testing.assert_array_equal(np.sort(seen), np.arange(sum(lengths)))


def test_placement_is_buddy_aligned():
    for name in PLANS:
        plan = load_plan(GOLDEN / name)
        world = _world(plan)
        for lay in build_plan_layouts(plan, plan["lengths"], world):
            for g in lay.groups:
                assert g.rank_begin % g.degree == 0


def test_golden_plans_pinned():
    """the reference planner's C1 plans, byte-identical."""
    # Appendix B hashes are over Plan.to_json(); our fixture adds "lengths", so re-serialise.
    for name, prefix, t_star in (("c1_flexsp_2tier.json", "754b7317cdb3fa93", 0.390414),
                                 ("c1_flexsp_1tier.json", "0f73b86f27a09b11", 0.392397)):
        d = json.loads((GOLDEN / name).read_text())
        d.pop("lengths")
        text = json.dumps(d, indent=2) + "\n"
        assert hashlib.sha256(text.encode()).hexdigest()[:16] == prefix
        assert round(d["predicted_total_time"], 6) == t_star
    fig1 = json.loads((GOLDEN / "fig1_flexsp.json").read_text())
    assert fig1["predicted_total_time"] == pytest.approx(3.0)
    degs = sorted((g["degree"] for mb in fig1["micro_batches"] for g in mb["selected_groups"]),
                  reverse=True)
    assert degs == [32, 8, 8, 8, 8]
    st = json.loads((GOLDEN / "fig1_static32.json").read_text())
    assert st["predicted_total_time"] == 3.8977083333333336


def test_layout_errors():
    mb = {"selected_groups": [{"slot_id": 0, "degree": 2, "sequence_indices": [0, 0]}]}
    with pytest.raises(LayoutError):
        build_microbatch_layout(mb, [5], 2)
    mb = {"selected_groups": [{"slot_id": 0, "degree": 4, "sequence_indices": [0]}]}
    with pytest.raises(LayoutError):
        build_microbatch_layout(mb, [5], 2)
    mb = {"selected_groups": [{"slot_id": 0, "degree": 2, "sequence_indices": [3]}]}
    with pytest.raises(LayoutError):
        build_microbatch_layout(mb, [5], 2)
    mb = {"selected_groups": [{"slot_id": 0, "degree": 2, "sequence_indices": [0]}]}
    with pytest.raises(LayoutError):  # 1 head cannot be split over 2 members
        build_microbatch_layout(mb, [5], 2, n_heads=1)
    build_microbatch_layout(mb, [5], 2, n_heads=3)  # uneven split 2 + 1 is allowed (H5)
    with pytest.raises(LayoutError):
        load_plan({"schema": 2})


def test_padding_and_tiny_groups():
    # 5 tokens on a degree-4 group: R = 2, last two shard rows are pads
    mb = {"selected_groups": [{"slot_id": 0, "degree": 4, "sequence_indices": [1, 0]}]}
    lay = build_microbatch_layout(mb, [2, 3], 4)
    g = lay.groups[0]
    assert g.padded_tokens == 8 and g.rows_per_rank == 2
    np.testing.assert_array_equal(g.perm, [2, 3, 4, 0, 1, -1, -1, -1])
    np.testing.assert_array_equal(g.cu_seqlens, [0, 3, 5])
    assert g.local_tokens(3).size == 0
    np.testing.assert_array_equal(g.pack_index(2), [0, -1])


def test_head_split_matches_oracle():
    from oracle import layout_ref
    from paper_2412_01523_b200.layout import head_split
    for h in (1, 4, 5, 13, 32, 40, 52):
        for d in (1, 2, 4, 8):
            if h >= d:
                assert head_split(h, d) == layout_ref.head_split(h, d), (h, d)
    with pytest.raises(LayoutError):
        head_split(4, 8)


def test_scatter_routes_match_oracle_on_golden_plans():
    """layout.scatter_routes (the per-plan data scatter tables) equals the
    plain-loop restatement in oracle/layout_ref.py for every rank and micro-batch of the
    reference planner's plans, and together the routes deliver every token exactly once."""
    import json
    from oracle.layout_ref import place_groups, scatter_routes_ref
    from paper_2412_01523_b200.layout import build_plan_layouts, loader_shards, scatter_routes
    for name, world in (("rand1_n8_flexsp.json", 8), ("rand0_n4_flexsp.json", 4),
                        ("c1_flexsp_2tier.json", 2), ("idle_n4.json", 4), ("c2_n4_flexsp.json", 4)):
        plan = json.loads((GOLDEN / name).read_text())
        lengths = plan["lengths"]
        shards = loader_shards(lengths, world)
        assert sorted(np.concatenate(shards).tolist()) == list(range(sum(lengths)))
        delivered = 0
        for lay, mb in zip(build_plan_layouts(plan, lengths, world), plan["micro_batches"]):
            gs = mb["selected_groups"]
            starts = place_groups([g["degree"] for g in gs], world)
            ref = scatter_routes_ref(lengths, world, [(s, g["degree"], g["sequence_indices"])
                                                      for s, g in zip(starts, gs)])
            for r in range(world):
                got = scatter_routes(lay, shards[r])
                assert [tuple(x) for x in got.tolist()] == ref[r], (name, r)
                delivered += got.shape[0]
        assert delivered == sum(lengths)


def test_ring_zigzag_chunks_cover_the_sequence():
    """Context parallelism (ring.py): rank r's local rows are chunks r and 2R-1-r; every
    position of the sequence belongs to exactly one rank, each rank holds the same number of
    rows, and the causal work (positions below each row) is balanced within 1/R."""
    from paper_2412_01523_b200.ring import RingLayout, zigzag_rows
    for R in (1, 2, 4, 8):
        S = 2 * R * 96
        rows = [zigzag_rows(S, R, r) for r in range(R)]
        assert sorted(np.concatenate(rows).tolist()) == list(range(S))
        assert len({len(x) for x in rows}) == 1
        work = [int((x + 1).sum()) for x in rows]
        assert max(work) - min(work) <= S * S // (2 * R) // R
        off = RingLayout(S // R, 4, 128).offsets(R)
        assert off["kv"] % 4096 == 0 and off["dkv"] % 4096 == 0 and off["end"] > off["dkv"]
    with pytest.raises(ValueError):
        zigzag_rows(1000, 3, 0)
