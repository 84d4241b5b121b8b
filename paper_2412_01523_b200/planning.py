"""Planner/executor overlap: plan steps t+1 .. t+k while step t trains.

FlexSP disaggregates solving (CPU) from training (GPU): a per-node solver service plans
upcoming batches concurrently, the plans go to a store, and "the executor sequentially
reads one plan per iteration to train", so solving overlaps training.
The reference ships the planning half only: `solve_stream` plans a list of batches on a
thread pool and returns every plan at once (pkg/src/seqplan/workflow.py:174-182).

`PlanPipeline` is the executor-facing form of that: an iterator over training steps that
keeps `lookahead` future batches in flight on a pool of worker *processes* (the planner is
Python + HiGHS; threads would contend with the training loop for the GIL), and hands
step t its plan the moment step t is reached.  Plans are the reference's own
`solve_batch` output (pkg/src/seqplan/workflow.py:81-171) — identical to `solve_stream`
on the same inputs — serialised as plan-JSON schema 1 dicts (domain.py:390-397) plus the
batch's `lengths`, which is what `FlexSPExecutor.prepare` consumes.  `wait_s` records how
long the trainer blocked on the planner at each step (0 when planning is fully hidden).

With one process per GPU, rank 0 runs the pipeline and `broadcast_plan` ships each plan
to the other ranks (a time-limited MILP is not guaranteed to be reproducible across
processes, so the ranks must not re-solve independently).
"""
from __future__ import annotations

import multiprocessing as mp
import sys
import time
from concurrent.futures import Future, ProcessPoolExecutor
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any, Iterable, Iterator, Sequence

_ROOT = Path(__file__).resolve().parent.parent


def import_seqplan():
    """The kept reference planner: `seqplan` from the environment, else the offline install
    under baseline/_ref (travels with the repo), else the read-only reference checkout."""
    try:
        import seqplan  # noqa: F401
    except ImportError:
        for cand in (_ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
            if cand.is_dir() and str(cand) not in sys.path:
                sys.path.append(str(cand))
        import seqplan  # noqa: F401
    return sys.modules["seqplan"]


def _solve_task(lengths: Sequence[int], batch_id: str, cluster: dict, coeffs: dict,
                config: dict, strategy: str, static_degree: int | None) -> tuple[dict, float]:
    """One batch through the reference planner (runs in a worker process)."""
    seqplan = import_seqplan()
    from seqplan.domain import ClusterSpec, CostCoefficients, SequenceBatch
    t0 = time.perf_counter()
    batch = SequenceBatch(tuple(int(s) for s in lengths), batch_id=batch_id)
    cl = ClusterSpec.from_json_dict(cluster)
    co = CostCoefficients.from_json_dict(coeffs)
    if strategy == "static":
        from seqplan.baselines import plan_static
        plan = plan_static(batch, cl, co, static_degree or cl.total_devices)
    else:
        plan = seqplan.solve_batch(batch, cl, co, seqplan.SolveConfig(**config))
    doc = plan.to_json_dict()
    doc["lengths"] = [int(s) for s in lengths]
    return doc, time.perf_counter() - t0


@dataclass
class PlannedStep:
    index: int
    batch_id: str
    lengths: list[int]
    plan: dict
    solve_s: float      # planner wall time of this batch (in its worker)
    wait_s: float       # time the trainer blocked waiting for it


@dataclass
class PlanPipeline:
    """Iterator of PlannedStep over `batches` with `lookahead` batches planned ahead.

    batches: iterable of SequenceBatch-like objects (`.lengths`, optional `.batch_id`) or
    plain length lists.  cluster / coeffs: seqplan ClusterSpec / CostCoefficients (or their
    JSON dicts).  config: seqplan.SolveConfig (or its kwargs).  strategy "flexsp" runs
    solve_batch, "static" runs plan_static(static_degree).  workers: planner processes
    (0 = plan synchronously in this process, the no-overlap baseline).
    """
    batches: Iterable[Any]
    cluster: Any
    coeffs: Any
    config: Any = None
    lookahead: int = 2
    workers: int = 2
    strategy: str = "flexsp"
    static_degree: int | None = None
    steps: list[PlannedStep] = field(default_factory=list, init=False)

    def __post_init__(self):
        if self.lookahead < 0 or self.workers < 0:
            raise ValueError("lookahead and workers must be >= 0")
        if self.strategy not in ("flexsp", "static"):
            raise ValueError(f"unknown strategy {self.strategy!r}")
        self._cluster = self.cluster if isinstance(self.cluster, dict) else self.cluster.to_json_dict()
        self._coeffs = self.coeffs if isinstance(self.coeffs, dict) else self.coeffs.to_json_dict()
        cfg = self.config
        if cfg is None:
            cfg = {}
        elif not isinstance(cfg, dict):
            cfg = {k: getattr(cfg, k) for k in cfg.__dataclass_fields__}
        self._config = cfg
        self._pool: ProcessPoolExecutor | None = None

    def _args(self, i: int, b: Any):
        lengths = [int(s) for s in (b.lengths if hasattr(b, "lengths") else b)]
        bid = str(getattr(b, "batch_id", None) or f"step{i}")
        return lengths, bid, (lengths, bid, self._cluster, self._coeffs, self._config,
                              self.strategy, self.static_degree)

    def __iter__(self) -> Iterator[PlannedStep]:
        src = enumerate(self.batches)
        inflight: list[tuple[int, list[int], str, Future | tuple]] = []
        if self.workers > 0:
            self._pool = ProcessPoolExecutor(max_workers=self.workers,
                                             mp_context=mp.get_context("spawn"))
        try:
            exhausted = False

            def refill():  # step t + the `lookahead` batches after it
                nonlocal exhausted
                while not exhausted and len(inflight) < self.lookahead + 1:
                    try:
                        i, b = next(src)
                    except StopIteration:
                        exhausted = True
                        return
                    lengths, bid, args = self._args(i, b)
                    fut = self._pool.submit(_solve_task, *args) if self._pool else args
                    inflight.append((i, lengths, bid, fut))

            while True:
                refill()
                if not inflight:
                    break
                i, lengths, bid, fut = inflight.pop(0)
                t0 = time.perf_counter()
                doc, solve_s = fut.result() if self._pool else _solve_task(*fut)
                wait = time.perf_counter() - t0
                # while the caller trains step t, steps t+1 .. t+lookahead keep planning
                st = PlannedStep(i, bid, lengths, doc, solve_s, wait)
                self.steps.append(st)
                yield st
        finally:
            self.close()

    def close(self) -> None:
        if self._pool is not None:
            self._pool.shutdown(wait=True, cancel_futures=True)
            self._pool = None


def broadcast_plan(plan: dict | None, src: int = 0, group=None) -> dict:
    """Ship rank `src`'s plan document to every rank of `group` (torch.distributed)."""
    import torch.distributed as dist
    box = [plan]
    dist.broadcast_object_list(box, src=src, group=group)
    return box[0]
