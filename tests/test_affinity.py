"""NUMA binding helper: a no-op (reported, not raised) where NVML has no GPU."""
import os

import torch

from paper_2412_01523_b200.affinity import bind_to_gpu_numa


def test_bind_reports_and_never_raises():
    before = os.sched_getaffinity(0)
    info = bind_to_gpu_numa(0)
    assert isinstance(info, dict) and "bound" in info and info["cpus"] >= 1
    if not torch.cuda.is_available():
        assert info["bound"] is False
        assert os.sched_getaffinity(0) == before
    os.sched_setaffinity(0, before)
