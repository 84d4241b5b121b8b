"""Sampled-row parity helpers shared by the full-size tests (tests/test_gpu_fullsize.py,
tests/vrank_parity.py): GPU rows of one (sequence, head) against oracle/sampled_ref.py.

Tolerances: O max|Δ| <= 2e-2; LSE |Δ| <= 1e-3 * max(1, |lse|) (relative
1e-3; absolute near zero, e.g. row 0 whose LSE is a single scaled dot product);
dQ / dK / dV allclose(atol=5e-2, rtol=5e-2)."""
import numpy as np

from oracle.sampled_ref import key_rows, query_rows


def sample_rows(s, rng, n=12):
    pick = {0, 1, s // 2, s - 2, s - 1} | set(rng.integers(0, s, size=n).tolist())
    return sorted(r for r in pick if 0 <= r < s)


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def check_sequence(q, k, v, do, o_rows, dq_rows, dk_rows, dv_rows, o_full, lse_full, rows,
                   kv_rows, tag):
    """q, k, v, do, o_full: [s, D] of one (sequence, head), lse_full [s] (the kernel's own
    per-row forward of the whole sequence, used for the key-row gradients after its
    sampled rows are checked); o_rows / dq_rows [len(rows), D] and dk_rows / dv_rows
    [len(kv_rows), D] are the step's outputs at the sampled rows.  Returns a dict of the
    max errors and `ok`."""
    ref = query_rows(q, k, v, do, rows)
    lse = _np(lse_full)
    e_o = np.abs(_np(o_rows) - ref["o"]).max()
    e_o1 = np.abs(_np(o_full)[rows] - ref["o"]).max()
    e_lse = (np.abs(lse[rows] - ref["lse"]) / np.maximum(1.0, np.abs(ref["lse"]))).max()
    dq_ok = np.allclose(_np(dq_rows), ref["dq"], atol=5e-2, rtol=5e-2)
    e_dq = np.abs(_np(dq_rows) - ref["dq"]).max()
    delta = (o_full.float() * do.float()).sum(-1).cpu().numpy()
    kr = key_rows(q, k, v, do, kv_rows, lse, delta)
    dk_ok = np.allclose(_np(dk_rows), kr["dk"], atol=5e-2, rtol=5e-2)
    dv_ok = np.allclose(_np(dv_rows), kr["dv"], atol=5e-2, rtol=5e-2)
    out = {"o_max": float(e_o), "o1_max": float(e_o1), "lse_rel": float(e_lse),
           "dq_max": float(e_dq), "dk_max": float(np.abs(_np(dk_rows) - kr["dk"]).max()),
           "dv_max": float(np.abs(_np(dv_rows) - kr["dv"]).max())}
    out["ok"] = bool(e_o <= 2e-2 and e_o1 <= 2e-2 and e_lse <= 1e-3 and dq_ok and dk_ok and
                     dv_ok and all(np.isfinite(x) for x in out.values()))
    out["tag"] = tag
    return out
