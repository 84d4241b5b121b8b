"""C-ABI library checks that need no GPU: it builds, loads, exports every symbol the
header declares, host-side argument validation maps to ValueError, and the LPT tile
schedule (pure host code) matches a Python restatement."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent


@pytest.fixture(scope="module")
def lib():
    from paper_2412_01523_b200 import _build, capi
    if not capi.LIB_PATH.exists():
        _build.build()
    return capi.load()


def test_exports_every_declared_symbol(lib):
    header = (ROOT / "include" / "flexsp_b200.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int32_t|int64_t|const char\*)\s+(fsp_\w+)\(", header,
                              re.M))
    assert declared, "no declarations parsed"
    from paper_2412_01523_b200 import capi
    assert declared == set(capi.EXPORTED)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.fsp_abi_version() == capi.ABI_VERSION == 6


def _schedule(lib, lens, rev, heads=1, head_dim=64):
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    p = cu.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    n = lib.fsp_attn_schedule(p, len(lens), heads, head_dim, rev, None, 0)
    buf = np.zeros(max(2 * n, 2), dtype=np.int32)
    ptr = buf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
    assert lib.fsp_attn_schedule(p, len(lens), heads, head_dim, rev, ptr, n) == n
    w = buf[0::2].view(np.uint32)  # tile words are {seq << 16 | tile}, decoded unsigned
    return [(int(w[i]) >> 16, int(w[i]) & 0xFFFF, int(buf[2 * i + 1])) for i in range(n)]


@pytest.mark.parametrize("rev", [0, 1])
def test_schedule_complete_and_ordered(lib, rev):
    lens = [1, 128, 129, 0, 1000, 300, 4096]
    heads = 3
    tiles = _schedule(lib, lens, rev, heads)
    ntiles = [-(-s // 128) for s in lens]
    expect = sorted((s, t, h) for s, n in enumerate(ntiles) for t in range(n) for h in range(heads))
    assert sorted(tiles) == expect
    # sequences longest first; inside a sequence head-major, heaviest tile first
    seq_order = [s for s, _, _ in tiles]
    firsts = list(dict.fromkeys(seq_order))
    assert [ntiles[s] for s in firsts] == sorted((ntiles[s] for s in firsts), reverse=True)
    for s in firsts:
        block = [(t, h) for ss, t, h in tiles if ss == s]
        assert [h for _, h in block] == sorted(h for _, h in block)
        for h in range(heads):
            costs = [(ntiles[s] - t) if rev else (t + 1) for t, hh in block if hh == h]
            assert costs == sorted(costs, reverse=True)


def test_schedule_beyond_32768_sequences(lib):
    """A group with more than 2^15 sequences (40,000 one-token sequences): the tile word's
    sequence field is decoded unsigned, so every sequence index appears exactly once and
    none comes back negative; 65,536 sequences are rejected."""
    from paper_2412_01523_b200 import capi
    for kind in (0, 1):
        tiles = _schedule(lib, [1] * 40000, kind, heads=1, head_dim=128)
        assert sorted(s for s, _, _ in tiles) == list(range(40000))
        assert all(t == 0 for _, t, _ in tiles)
    cu = np.arange(65537, dtype=np.int32)
    assert lib.fsp_attn_schedule(cu.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 65536, 1,
                                 128, 0, None, 0) == capi.FSP_ERR_INVALID


def test_empty_group_calls_are_noops(lib):
    """An empty group (no rows: a selected group without sequences) or a member holding
    only pad rows is a valid no-op at the C-ABI even with null buffers, so such a rank
    does not raise while its peers wait in the group barrier."""
    from paper_2412_01523_b200 import capi
    a = capi.FspAttnFwd()
    a.head_dim, a.n_heads = 128, 4
    assert lib.fsp_attn_fwd(ctypes.byref(a), None) == capi.FSP_OK
    b = capi.FspAttnBwd()
    b.head_dim, b.n_heads = 128, 4
    b.scatter.degree, b.scatter.rows_per_rank = 2, 0
    assert lib.fsp_attn_bwd(ctypes.byref(b), None) == capi.FSP_OK
    x = capi.FspA2A(2, 1, 0, 3, 4, 64, 768, 384)  # R = 0: nothing to move, null src ok
    ptrs = (ctypes.c_void_p * 2)(16, 16)
    assert lib.fsp_a2a_seq2head(ctypes.byref(x), None, ptrs, None, None) == capi.FSP_OK
    x.rows_per_rank = 2  # rows to send but no src and no index: rejected
    assert lib.fsp_a2a_seq2head(ctypes.byref(x), None, ptrs, None, None) == capi.FSP_ERR_INVALID
    assert lib.fsp_a2a_head2seq(ctypes.byref(x), None, ptrs, None, None) == capi.FSP_ERR_INVALID


def test_integration_stub_matches_binding(lib):
    """The reference-side ctypes stub printed in INTEGRATION.md §2 is executed against
    the built library: its structures have capi.py's layouts, its argument lists equal
    capi.py's, and the host-only entry points give the same answers through it."""
    from paper_2412_01523_b200 import capi
    text = (ROOT / "INTEGRATION.md").read_text()
    sec = text[text.index("## 2. The ctypes stub"):]
    code = sec[sec.index("```python\n") + 10:]
    code = code[:code.index("```")]
    code = code.replace('"paper_2412_01523_b200/_lib/libflexsp_b200.so"', repr(str(capi.LIB_PATH)))
    ns: dict = {}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    stub = ns["lib"]
    for st in ("FspA2A", "FspHeadScatter", "FspAttnFwd", "FspAttnBwd"):
        mine, theirs = getattr(capi, st), ns[st]
        assert ctypes.sizeof(mine) == ctypes.sizeof(theirs), st
        assert [(f, getattr(mine, f).offset) for f, _ in mine._fields_] == \
            [(f, getattr(theirs, f).offset) for f, _ in theirs._fields_], st

    def sig(fn):
        return [getattr(t, "__name__", str(t)) for t in (fn.argtypes or [])], \
            getattr(fn.restype, "__name__", str(fn.restype))
    for name in capi.EXPORTED:
        if name == "fsp_selftest_umma":  # diagnostic, not part of the reference binding
            continue
        assert sig(getattr(stub, name)) == sig(getattr(lib, name)), name
    lens = [5, 300, 1, 4096, 77]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    for kind in (0, 1):
        p = cu.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        n = stub.fsp_attn_schedule(p, len(lens), 3, 128, kind, None, 0)
        a = np.zeros(2 * n, dtype=np.int32)
        b = np.zeros(2 * n, dtype=np.int32)
        stub.fsp_attn_schedule(p, len(lens), 3, 128, kind,
                               a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n)
        lib.fsp_attn_schedule(p, len(lens), 3, 128, kind,
                              b.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), n)
        assert n > 0 and np.array_equal(a, b)
    idx = np.array([2, 0, -1, 1], dtype=np.int32)
    ns["check"](stub.fsp_layout_check(idx.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 4, 3))
    bad = np.array([0, 0], dtype=np.int32)
    with pytest.raises(ValueError):
        ns["check"](stub.fsp_layout_check(bad.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)), 2, 2))
    assert stub.fsp_attn_bwd_workspace_bytes(1000, 8, 128) == lib.fsp_attn_bwd_workspace_bytes(1000, 8, 128)


def test_forward_schedule_pairs_for_head_dim_128(lib):
    lens = [1, 128, 129, 300, 1000]
    tiles = _schedule(lib, lens, 0, heads=2, head_dim=128)
    npairs = [-(-s // 256) for s in lens]
    assert sorted(tiles) == sorted((s, t, h) for s, n in enumerate(npairs) for t in range(n)
                                   for h in range(2))


def test_invalid_arguments_raise_valueerror(lib):
    from paper_2412_01523_b200 import capi
    # row_bytes not a multiple of 16 -> rejected on the host before any CUDA call
    rc = lib.fsp_pack_rows(16, 16, 16, 16, 16, 1, 10, None)
    assert rc == capi.FSP_ERR_INVALID
    with pytest.raises(ValueError):
        capi.check(rc)
    a = capi.FspAttnFwd()
    a.head_dim = 96
    a.n_heads = 1
    rc = lib.fsp_attn_fwd(ctypes.byref(a), None)
    assert rc == capi.FSP_ERR_INVALID
    assert b"head_dim" in lib.fsp_last_error()
    x = capi.FspA2A(3, 0, 1, 1, 4, 64, 256, 256)  # degree 3 is not a power of two
    ptrs = (ctypes.c_void_p * 3)(16, 16, 16)
    assert lib.fsp_a2a_seq2head(ctypes.byref(x), 16, ptrs, None, None) == capi.FSP_ERR_INVALID
    cu = (ctypes.c_int32 * 3)(0, 5, 3)  # decreasing cu_seqlens
    assert lib.fsp_attn_schedule(cu, 2, 1, 64, 0, None, 0) == capi.FSP_ERR_INVALID


def test_device_ops_reject_cpu_tensors(lib):
    from paper_2412_01523_b200 import ops
    x = torch.zeros(4, 8, dtype=torch.bfloat16)
    idx = torch.zeros(4, dtype=torch.int32)
    with pytest.raises(ValueError, match="CUDA"):
        ops.pack_rows(x, idx, x.clone())


def test_bwd_workspace_bytes(lib):
    assert lib.fsp_attn_bwd_workspace_bytes(1000, 8, 128) == (8 * 1000 * 128 + 8 * 1000) * 4
    assert lib.fsp_attn_bwd_workspace_bytes(0, 8, 128) == 0
    assert lib.fsp_attn_bwd_workspace_bytes(-1, 8, 128) < 0


def test_layout_check_accepts_permutations_and_rejects_the_rest(lib):
    from paper_2412_01523_b200 import ops
    ops.layout_check([2, 0, -1, 1], 3)
    ops.layout_check([], 0)
    ops.layout_check([-1, -1], 0)
    for bad, n in (([0, 0, 1], 3), ([0, 3], 2), ([0, 1], 3), ([0, -2, 1], 2)):
        with pytest.raises(ValueError):
            ops.layout_check(bad, n)


def test_layout_check_on_every_golden_plan(lib):
    """Every rank's pack index and unpack table of every committed plan passes the
    library's check (the executor runs the same check before uploading them)."""
    import json
    from paper_2412_01523_b200 import ops
    from paper_2412_01523_b200.layout import build_plan_layouts
    for path in sorted((ROOT / "tests" / "golden").glob("*.json")):
        plan = json.loads(path.read_text())
        if "micro_batches" not in plan or "lengths" not in plan:
            continue
        world = plan.get("cluster", {}).get("total_devices") or \
            len(plan["micro_batches"][0].get("group_selection", [0, 0, 0])) // 2 + 1
        for lay in build_plan_layouts(plan, plan["lengths"], world):
            for g in lay.groups:
                for j in range(g.degree):
                    ops.layout_check(g.pack_index(j), int((g.shard(j) >= 0).sum()))


def test_ctypes_structs_match_the_c_header(tmp_path):
    """The ctypes mirrors in capi.py have the C header's sizes and field offsets (a C
    program compiled against include/flexsp_b200.h prints them) — ABI 4 appended an
    FspHeadScatter to both attention argument structs."""
    import shutil
    import subprocess
    from paper_2412_01523_b200 import capi
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        pytest.skip("no C compiler")
    checks = {
        "FspA2A": ["degree", "rows_per_rank", "src_stride", "dst_stride", "head_begin"],
        "FspHeadScatter": ["degree", "head_offset", "dst_stride", "mat_stride", "d_unpack",
                           "peer_dst"],
        "FspAttnFwd": ["q", "lse", "o_stride", "d_seq_starts", "n_tiles", "softmax_scale",
                       "scatter", "flags"],
        "FspAttnBwd": ["dout", "dv", "dv_stride", "dq_accum", "d_tiles", "softmax_scale",
                       "scatter", "flags"],
    }
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "flexsp_b200.h"',
             "int main(void) {"]
    for st, fields in checks.items():
        lines.append(f'  printf("{st} size %zu\\n", sizeof({st}));')
        for f in fields:
            lines.append(f'  printf("{st} {f} %zu\\n", offsetof({st}, {f}));')
    lines.append("  return 0;\n}")
    src = tmp_path / "abi.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "abi"
    subprocess.run([cc, "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout
    got = {}
    for line in out.splitlines():
        st, field, val = line.split()
        got[(st, field)] = int(val)
    for st, fields in checks.items():
        cls = getattr(capi, st)
        assert ctypes.sizeof(cls) == got[(st, "size")], st
        for f in fields:
            assert getattr(cls, f).offset == got[(st, f)], (st, f)
