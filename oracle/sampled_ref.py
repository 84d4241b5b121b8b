"""Sampled-row restatement of causal attention fwd/bwd — TEST INFRASTRUCTURE ONLY.

Full-size parity (BASELINE configs at 259K–733K tokens, sequences up to 384K) cannot run
the dense CPU oracle (oracle/attention_ref.py is O(s^2) memory per sequence).  These
functions restate Eq. (3) and its gradient (flash-attn varlen semantics,
PAPER.md:916) for a handful of rows of ONE (sequence, head), in float64, at O(s·D) cost per
row:

  query row i:   s_ij = scale q_i·k_j (j <= i),  lse_i = log Σ_j e^{s_ij},
                 o_i = Σ_j e^{s_ij - lse_i} v_j,  delta_i = o_i·do_i,
                 dq_i = scale Σ_j P_ij (do_i·v_j - delta_i) k_j
  key row j:     dv_j = Σ_{i>=j} P_ij do_i,  dk_j = scale Σ_{i>=j} P_ij (do_i·v_j - delta_i) q_i

The key-row gradients need lse_i and delta_i of every later query row; the tests pass the
kernel's own per-row statistics (after checking them on sampled rows against
`query_rows`), which makes the key-row check a consistency property of the backward given
the forward statistics.  Only tests/ import this module.
"""
from __future__ import annotations

import math

import numpy as np


def _f64(x) -> np.ndarray:
    if hasattr(x, "detach"):
        x = x.detach().float().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def query_rows(q, k, v, do, rows, scale=None):
    """q, k, v, do: [s, D] of one (sequence, head).  Returns dict of o [r, D], lse [r],
    delta [r], dq [r, D] for the local query rows `rows`."""
    q, k, v, do = (_f64(t) for t in (q, k, v, do))
    D = q.shape[1]
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    out = {"o": [], "lse": [], "delta": [], "dq": []}
    for i in rows:
        s = (k[: i + 1] @ q[i]) * scale
        m = s.max()
        e = np.exp(s - m)
        lse = m + math.log(e.sum())
        p = np.exp(s - lse)
        o = p @ v[: i + 1]
        delta = float(o @ do[i])
        dp = v[: i + 1] @ do[i]
        dq = scale * ((p * (dp - delta)) @ k[: i + 1])
        for key, val in (("o", o), ("lse", lse), ("delta", delta), ("dq", dq)):
            out[key].append(val)
    return {key: np.asarray(val) for key, val in out.items()}


def key_rows(q, k, v, do, kv_rows, lse, delta, scale=None):
    """dk, dv [r, D] for local key rows `kv_rows`, given lse[s] and delta[s] of every query
    row of the sequence (natural-log units)."""
    q, k, v, do = (_f64(t) for t in (q, k, v, do))
    lse, delta = _f64(lse), _f64(delta)
    D = q.shape[1]
    scale = scale if scale is not None else 1.0 / math.sqrt(D)
    dk, dv = [], []
    for j in kv_rows:
        s = (q[j:] @ k[j]) * scale               # query rows i >= j
        p = np.exp(s - lse[j:])
        dp = do[j:] @ v[j]
        dv.append(p @ do[j:])
        dk.append(scale * ((p * (dp - delta[j:])) @ q[j:]))
    return {"dk": np.asarray(dk), "dv": np.asarray(dv)}
