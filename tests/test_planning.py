"""Planner/executor overlap on CPU: PlanPipeline hands out the
reference planner's own plans (== seqplan.solve_stream, pkg/src/seqplan/workflow.py:174-182)
in step order, and hides planning behind the consumer's step time."""
import time

import pytest

from paper_2412_01523_b200.planning import PlanPipeline, import_seqplan

try:
    seqplan = import_seqplan()
except ImportError:  # pragma: no cover
    pytest.skip("reference planner not importable", allow_module_level=True)

from seqplan.domain import ClusterSpec, CostCoefficients, SequenceBatch  # noqa: E402

COEFFS = CostCoefficients(alpha1=1e-9, alpha2=1e-6, beta1=1e-4, alpha3=4096, beta2=1e-5,
                          m_token=2e4, m_ms=1e6)
CLUSTER = ClusterSpec(4, 1, 1e15, 2e10, 1e6 + 2e4 * 2500)


def _batches(n):
    import numpy as np
    rng = np.random.default_rng(5)
    return [SequenceBatch(tuple(int(x) for x in np.clip(rng.lognormal(6.0, 1.2, size=10), 1, 2500)),
                          batch_id=f"b{i}") for i in range(n)]


@pytest.mark.parametrize("workers,lookahead", [(0, 0), (2, 2)])
def test_pipeline_plans_equal_solve_stream(workers, lookahead):
    batches = _batches(4)
    ref = seqplan.solve_stream(batches, CLUSTER, COEFFS, seqplan.SolveConfig(), parallelism=1)
    pipe = PlanPipeline(batches, CLUSTER, COEFFS, seqplan.SolveConfig(), lookahead=lookahead,
                        workers=workers)
    got = list(pipe)
    assert [s.index for s in got] == list(range(4))
    for st, plan, b in zip(got, ref, batches):
        want = plan.to_json_dict()
        want["lengths"] = list(b.lengths)
        assert st.plan == want
        assert st.batch_id == b.batch_id and st.solve_s > 0


def test_pipeline_static_strategy_matches_plan_static():
    from seqplan.baselines import plan_static
    b = _batches(1)[0]
    (st,) = list(PlanPipeline([b], CLUSTER, COEFFS, strategy="static", static_degree=2, workers=0))
    want = plan_static(b, CLUSTER, COEFFS, 2).to_json_dict()
    want["lengths"] = list(b.lengths)
    assert st.plan == want


def test_pipeline_hides_planning_behind_steps():
    """The consumer 'trains' for longer than a solve; after the first step the trainer
    should not wait on the planner."""
    batches = _batches(5)
    pipe = PlanPipeline(batches, CLUSTER, COEFFS, lookahead=2, workers=2)
    steps = []
    for st in pipe:
        steps.append(st)
        time.sleep(max(0.5, 2.0 * st.solve_s))
    later_wait = sum(s.wait_s for s in steps[1:])
    later_solve = sum(s.solve_s for s in steps[1:])
    assert later_wait < 0.25 * later_solve + 0.2, (later_wait, later_solve)


def test_pipeline_plans_drive_the_layout():
    """A pipeline plan is directly consumable by the executor's layout builder."""
    from paper_2412_01523_b200.layout import build_plan_layouts
    (st,) = list(PlanPipeline(_batches(1), CLUSTER, COEFFS, workers=0))
    lays = build_plan_layouts(st.plan, st.lengths, 4, n_heads=8)
    covered = sorted(k for lay in lays for g in lay.groups for k in g.sequence_indices)
    assert covered == list(range(len(st.lengths)))


def test_pipeline_rejects_bad_arguments():
    with pytest.raises(ValueError):
        PlanPipeline([], CLUSTER, COEFFS, lookahead=-1)
    with pytest.raises(ValueError):
        PlanPipeline([], CLUSTER, COEFFS, strategy="ulysses")
