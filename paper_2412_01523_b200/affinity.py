"""Bind a rank's host thread (and so its pinned staging buffers) to its GPU's NUMA node.

The host-fed step (`FlexSPExecutor.step_from_host`) streams every micro-batch's q/k/v/dO
from pinned host memory; with one process per GPU, a rank whose pinned pages sit on the
other socket pays the inter-socket link on every H2D copy.  Binding the process to the
CPUs NVML reports as local to its GPU before the buffers are allocated (first touch) keeps
the copies on the GPU's own PCIe root.
"""
from __future__ import annotations

import os


def bind_to_gpu_numa(device_index: int) -> dict:
    """Set this process's CPU affinity to the CPUs local to CUDA device `device_index`.
    Returns {"bound": bool, "cpus": n} (bound False when NVML is unavailable)."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        nvml_index = device_index
        if hasattr(torch.cuda, "_get_nvml_device_index"):
            nvml_index = torch.cuda._get_nvml_device_index(device_index)
        handle = pynvml.nvmlDeviceGetHandleByIndex(nvml_index)
        pynvml.nvmlDeviceSetCpuAffinity(handle)
        cpus = sorted(os.sched_getaffinity(0))
        return {"bound": True, "cpus": len(cpus), "first_cpu": cpus[0] if cpus else None}
    except Exception as exc:  # no NVML / not permitted: leave the affinity alone
        return {"bound": False, "reason": str(exc)[:120], "cpus": len(os.sched_getaffinity(0))}
