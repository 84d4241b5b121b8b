"""Generate the committed golden fixtures from the REFERENCE planner (run in the build
container, where /root/reference is mounted; the GPU box only reads the outputs).

    python tests/golden/make_golden.py

Outputs (all small JSON/NPZ, committed):
  c1_*.json       SURVEY.md Appendix B config-1 plans (two-tier flexsp, one-tier flexsp,
                  static SP=2) — their sha256 prefixes are pinned in tests/test_golden.py
  fig1_*.json     PAPER Fig. 1 scenario (pkg/tests/conftest.py:14-45): flexsp T*=3.0,
                  degrees [32,8,8,8,8]; static SP=32
  c2_n{N}_{flexsp,static}.json   C2 long-tail batch (gen_longtail(64, pareto 1.1, 32K),
                  SURVEY.md §8d) planned for N = 1, 2, 4, 8 B200 with the B200
                  attention-layer coefficients below — these are the bench's plans
  c3_n{N}_*.json, c4_n{N}_*.json   C3 (13B-shape, H=40) / C4 (30B-shape, H=52) batches
                  planned with the fitted B200 coefficients (`--scale-configs` regenerates
                  only these)
  c3full_n{N}_*.json  C3 batch planned with full-step (40-layer) coefficients for
                  scripts/bench_full_step.py (`--full-step` regenerates only these)
  rand_*.json     random small instances (N = 4, 8) for layout parity
  attn_small.npz  attention golden vectors from oracle/attention_ref.py (fp32), checked
                  against torch SDPA when generated
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
for cand in ("/root/reference/pkg/src", str(ROOT / "baseline" / "_ref")):
    if os.path.isdir(cand) and cand not in sys.path:
        sys.path.insert(0, cand)
sys.path.insert(0, str(ROOT))

from seqplan.baselines import plan_static  # noqa: E402
from seqplan.domain import ClusterSpec, CostCoefficients, SequenceBatch  # noqa: E402
from seqplan.simulator import gen_longtail  # noqa: E402
from seqplan.workflow import SolveConfig, solve_batch  # noqa: E402

# ---- C1
C1_COEFFS = CostCoefficients(alpha1=3.584e-09, alpha2=9.437184e-06, beta1=1e-4, alpha3=8192,
                             beta2=5e-05, m_token=17408, m_ms=1e6)
C1_E = 143_606_336

# ---- B200 attention-layer coefficients for the C2 GPT-7B shape (h=4096, H=32, D=128).
# alpha1: measured round-1 kernel rates, fwd 2*D*H*s^2 FLOP at 718 TF/s + bwd 5*D*H*s^2 at
#         428 TF/s (profiles/r01_*); alpha2: ~160 KB/token of HBM traffic at 6.5 TB/s;
# alpha3: bytes crossing NVLink per token, fwd+bwd 2 x (3h + h) x 2 B;  bandwidth: d >= 2
#         groups ride NVLink 5 at the measured 770 GB/s peer rate, d = 1 groups exchange
#         nothing (the devices_per_node=1 tier trick).
B200_ATTN_COEFFS = CostCoefficients(alpha1=5.93e-11, alpha2=2.5e-8, beta1=1e-4, alpha3=65536,
                                    beta2=3e-5, m_token=2.0e5, m_ms=2e9)
B200_E = 180e9


def c2_fitted_coeffs() -> CostCoefficients:
    """The C2 plans' coefficients: fitted by the reference's fit_coefficients to the B200
    step itself (scripts/calibrate.py on 4xB200 with the round-1 final kernels and the fused
    head->seq exchange, profiles/r01_calibration_v2.json).  The hand-set
    B200_ATTN_COEFFS above predated the final kernels: their alpha1/alpha2 ratio made
    degree-1 groups of ~1K-token sequences look cheaper than they run."""
    cal = json.loads((ROOT / "profiles" / "r01_calibration_v2.json").read_text())["coefficients"]
    return CostCoefficients(alpha1=cal["alpha1"], alpha2=cal["alpha2"], beta1=cal["beta1"],
                            alpha3=cal["alpha3"], beta2=cal["beta2"],
                            m_token=cal["m_token"], m_ms=cal["m_ms"])


def b200_cluster(n: int) -> ClusterSpec:
    return ClusterSpec(n, 1, 1e15, 7.7e11, B200_E)


def c2_batch() -> SequenceBatch:
    return gen_longtail(64, ("pareto", 1.1, 1024), 32768, seed=0)[0]


def c1_batch() -> SequenceBatch:
    return gen_longtail(16, ("lognormal", 8.0, 1.4), 4096, seed=0)[0]


def dump(name: str, obj) -> str:
    text = json.dumps(obj, indent=2) + "\n"
    (HERE / name).write_text(text)
    return hashlib.sha256(text.encode()).hexdigest()[:16]


def plan_doc(plan, batch, extra=None) -> dict:
    d = plan.to_json_dict()
    d["lengths"] = list(batch.lengths)
    if extra:
        d.update(extra)
    return d


def main():
    meta = {}
    # C1
    b = c1_batch()
    two = ClusterSpec(2, 1, 1e15, 5e10, C1_E)
    one = ClusterSpec(2, 2, 5e10, 5e10, C1_E)
    p = solve_batch(b, two, C1_COEFFS, SolveConfig(jobs=1))
    meta["c1_flexsp_2tier"] = (p.to_json(), p.predicted_total_time)
    dump("c1_flexsp_2tier.json", plan_doc(p, b))
    p = solve_batch(b, one, C1_COEFFS, SolveConfig(jobs=1))
    meta["c1_flexsp_1tier"] = (p.to_json(), p.predicted_total_time)
    dump("c1_flexsp_1tier.json", plan_doc(p, b))
    p = plan_static(b, two, C1_COEFFS, 2)
    dump("c1_static2.json", plan_doc(p, b))
    # Fig. 1
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import FIG1_CLUSTER, FIG1_COEFFS, FIG1_LENGTHS  # noqa: E402
    fb = SequenceBatch(FIG1_LENGTHS, batch_id="fig1")
    p = solve_batch(fb, FIG1_CLUSTER, FIG1_COEFFS, SolveConfig(jobs=1))
    dump("fig1_flexsp.json", plan_doc(p, fb))
    p = plan_static(fb, FIG1_CLUSTER, FIG1_COEFFS, 32)
    dump("fig1_static32.json", plan_doc(p, fb))
    make_c2_plans()
    # random small instances for layout parity
    rng = np.random.default_rng(7)
    for i, n in enumerate((4, 8, 4)):
        lens = [int(x) for x in np.clip(rng.lognormal(6.0, 1.2, size=12), 1, 3000)]
        rb = SequenceBatch(lens, batch_id=f"rand{i}")
        coeffs = CostCoefficients(alpha1=1e-9, alpha2=1e-6, beta1=1e-4, alpha3=4096, beta2=1e-5,
                                  m_token=2e4, m_ms=1e6)
        cl = ClusterSpec(n, 1, 1e15, 2e10, 1e6 + 2e4 * 2500)
        p = solve_batch(rb, cl, coeffs, SolveConfig(jobs=1))
        dump(f"rand{i}_n{n}_flexsp.json", plan_doc(p, rb))
    # attention golden vectors (oracle, cross-checked with SDPA)
    import torch
    from oracle.attention_ref import attention_bwd_ref, attention_fwd_ref, attention_sdpa_ref
    lens = [37, 1, 130, 20]
    cu = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
    g = torch.Generator().manual_seed(2412)
    q, k, v, do = (torch.randn(int(cu[-1]), 1, 64, generator=g).bfloat16() for _ in range(4))
    o, lse = attention_fwd_ref(q, k, v, cu)
    o2 = attention_sdpa_ref(q, k, v, cu)
    assert torch.allclose(o, o2, atol=1e-5), (o - o2).abs().max()
    dq, dk, dv = attention_bwd_ref(q, k, v, do, cu)
    np.savez_compressed(HERE / "attn_small.npz", cu_seqlens=cu,
                        q=q.view(torch.int16).numpy(), k=k.view(torch.int16).numpy(),
                        v=v.view(torch.int16).numpy(), do=do.view(torch.int16).numpy(),
                        o=o.numpy(), lse=lse.numpy(), dq=dq.numpy(), dk=dk.numpy(), dv=dv.numpy())
    for key, (text, t) in meta.items():
        print(key, hashlib.sha256(text.encode()).hexdigest()[:16], round(t, 6))


def make_c2_plans(prefix: str = "c2"):
    """C2 at N = 1, 2, 4, 8 with the B200-fitted coefficients (the bench's plans)."""
    cb = c2_batch()
    co = c2_fitted_coeffs()
    for n in (1, 2, 4, 8):
        cl = b200_cluster(n)
        extra = {"coefficients": co.to_json_dict(), "cluster": cl.to_json_dict()}
        p = solve_batch(cb, cl, co, SolveConfig(jobs=8, time_limit=60))
        dump(f"{prefix}_n{n}_flexsp.json", plan_doc(p, cb, extra))
        s = plan_static(cb, cl, co, n)
        dump(f"{prefix}_n{n}_static.json", plan_doc(s, cb, extra))
        print(f"C2 N={n}: flexsp {p.predicted_total_time:.5f}s "
              f"{[sorted((g.degree for g in mb.selected_groups), reverse=True) for mb in p.micro_batches]}"
              f" static {s.predicted_total_time:.5f}s", flush=True)


# ---- C3 / C4: 13B-shape (H=40) and 30B-shape (H=52) attention layers.
# Coefficients: the B200-fitted C2 coefficients (profiles/r01_calibration.json, H=32,
# scripts/calibrate.py) with the per-head terms scaled by H/32 — attention FLOPs, HBM bytes,
# NVLink bytes and activation memory per token are all linear in H at fixed D=128.
SCALE_CONFIGS = {
    "c3": {"heads": 40, "gen": (32, ("pareto", 1.1, 1024), 131072)},
    "c4": {"heads": 52, "gen": (64, ("pareto", 0.9, 1024), 393216)},
}


def scaled_coeffs(heads: int) -> CostCoefficients:
    cal = json.loads((ROOT / "profiles" / "r01_calibration.json").read_text())["coefficients"]
    f = heads / 32.0
    return CostCoefficients(alpha1=cal["alpha1"] * f, alpha2=cal["alpha2"] * f, beta1=cal["beta1"],
                            alpha3=cal["alpha3"] * f, beta2=cal["beta2"],
                            m_token=cal["m_token"] * f, m_ms=cal["m_ms"])


# C3 full training step (scripts/bench_full_step.py: 40 layers with activation checkpointing,
# GEMMs + SP attention): coefficients measured on 4xB200 with an 8-layer run of that script
# (attention 186 ms and GEMMs 107 ms per layer at d=4 for 63,040 tokens per rank):
# alpha1 = 0.186 s * 4 / sum s^2 per layer x 40 layers; alpha2 = 107 ms / 63,040 tokens x 40;
# alpha3 = three exchanges (fwd, recompute, bwd) of 4h bf16 per token per layer x 40;
# m_token = 40 checkpointed layer inputs + one layer's transient activations per token;
# m_ms = bf16 weights + gradients of 40 layers (12.6 B parameters) + workspaces.
C3FULL_COEFFS = CostCoefficients(alpha1=1.62e-9, alpha2=6.8e-5, beta1=5e-3, alpha3=4.9e6,
                                 beta2=2e-3, m_token=7.2e5, m_ms=5.5e10)


def make_full_step_plans():
    b = gen_longtail(32, ("pareto", 1.1, 1024), 131072, seed=0)[0]
    for n in (2, 4, 8):
        cl = b200_cluster(n)
        extra = {"coefficients": C3FULL_COEFFS.to_json_dict(), "cluster": cl.to_json_dict(),
                 "heads": 40, "layers": 40}
        p = solve_batch(b, cl, C3FULL_COEFFS, SolveConfig(jobs=8, time_limit=60))
        dump(f"c3full_n{n}_flexsp.json", plan_doc(p, b, extra))
        s = plan_static(b, cl, C3FULL_COEFFS, n)
        dump(f"c3full_n{n}_static.json", plan_doc(s, b, extra))
        print(f"c3full N={n}: flexsp {p.predicted_total_time:.3f}s "
              f"{[sorted((g.degree for g in mb.selected_groups), reverse=True) for mb in p.micro_batches]}"
              f" static {s.predicted_total_time:.3f}s", flush=True)


def make_scale_configs():
    for name, spec in SCALE_CONFIGS.items():
        k, dist_, mx = spec["gen"]
        b = gen_longtail(k, dist_, mx, seed=0)[0]
        co = scaled_coeffs(spec["heads"])
        for n in (1, 2, 4, 8):
            cl = b200_cluster(n)
            extra = {"coefficients": co.to_json_dict(), "cluster": cl.to_json_dict(),
                     "heads": spec["heads"]}
            p = solve_batch(b, cl, co, SolveConfig(jobs=8, time_limit=60))
            dump(f"{name}_n{n}_flexsp.json", plan_doc(p, b, extra))
            s = plan_static(b, cl, co, n)
            dump(f"{name}_n{n}_static.json", plan_doc(s, b, extra))
            print(f"{name} N={n}: {len(b.lengths)} seqs, {sum(b.lengths)} tokens, max {max(b.lengths)}; "
                  f"flexsp {p.predicted_total_time:.4f}s "
                  f"{[sorted((g.degree for g in mb.selected_groups), reverse=True) for mb in p.micro_batches]}"
                  f" static {s.predicted_total_time:.4f}s", flush=True)


if __name__ == "__main__":
    if "--c2" in sys.argv:  # C2 plans only
        make_c2_plans()
    elif "--scale-configs" in sys.argv:  # C3 / C4 plans only
        make_scale_configs()
    elif "--full-step" in sys.argv:  # C3 full-step plans only
        make_full_step_plans()
    else:
        main()
