"""CUDA-event timing of individual device ops inside a timed region.

Events are recorded on the stream the op is launched on (torch's current stream, which
is the stream every C-ABI call in ops.py receives), so per-op durations are the device
time of that op's launches; `launches` counts the kernels each op issued.
"""
from __future__ import annotations

from collections import defaultdict

import torch


class EventTimer:
    def __init__(self):
        self.enabled = False
        self._pending: list[tuple[str, torch.cuda.Event, torch.cuda.Event, float]] = []
        self.work: dict[str, float] = defaultdict(float)
        self.tag = ""  # appended to every span name (e.g. "@mb1" for a per-micro-batch split)

    def start(self):
        self.enabled = True
        self._pending.clear()
        self.work.clear()

    def stop(self):
        self.enabled = False

    def span(self, name: str, work: float = 0.0):
        timer = self

        class _Span:
            def __enter__(self_inner):
                if timer.enabled:
                    self_inner.s = torch.cuda.Event(enable_timing=True)
                    self_inner.s.record()
                return self_inner

            def __exit__(self_inner, *exc):
                if timer.enabled:
                    e = torch.cuda.Event(enable_timing=True)
                    e.record()
                    timer._pending.append((name + timer.tag, self_inner.s, e, work))
                return False
        return _Span()

    def summary(self) -> dict[str, dict]:
        """{name: {"ms": total device ms, "n": launches, "work": summed work units}}."""
        torch.cuda.synchronize()
        out: dict[str, dict] = {}
        for name, s, e, work in self._pending:
            d = out.setdefault(name, {"ms": 0.0, "n": 0, "work": 0.0})
            d["ms"] += s.elapsed_time(e)
            d["n"] += 1
            d["work"] += work
        for name, w in self.work.items():  # counters without a device span (count())
            out.setdefault(name, {"ms": 0.0, "n": 0, "work": 0.0})["work"] += w
        return out

    def count(self, name: str, work: float) -> None:
        """Accumulate work that has no span of its own (e.g. bytes moved inside a kernel
        timed under another name)."""
        if self.enabled:
            self.work[name] += work


# Kernel launches issued by the C-ABI calls made through ops.py (the bench's
# `gpu_launches` claim): incremented by each wrapper with the kernels it launches.
LAUNCHES = [0]
