"""Virtual ranks: the multi-rank SP step of one plan on ONE GPU.

`VirtualCluster(world, H, D)` runs `world` FlexSPExecutor instances in one process on one
device, each on its own CUDA stream with its own heap carved from device memory; every
executor's peer table points at the other virtual ranks' heaps, so the exact device code
of an N-GPU step runs: the fused-pack seq->head exchange kernels, the attention kernels
with the head->seq exchange fused into their epilogues (FspHeadScatter), the group entry
and exchange barriers (`fsp_group_barrier` spinning on the other streams' signal words),
idle ranks, uneven head splits and heap reuse across micro-batches.  Only the transport
differs: peer stores land in local HBM instead of crossing NVSwitch.

This is how a one-GPU box checks the degree >= 2 path of plans for 2/4/8 GPUs
(tests/test_gpu_multi.py, tests/vrank_parity.py).  Issue rules that keep it deadlock-free:
* the host must never wait on the device between the first and the last rank's issue of
  a step (a barrier of rank 0 spins until rank 1's stream reaches it, which needs rank 1's
  work to have been issued): `step()` issues every rank's whole step first and only then
  joins the streams; sinks must stay on the device (no .cpu(), no .item());
* enough hardware queues for one stream per rank: set CUDA_DEVICE_MAX_CONNECTIONS >= 16
  before CUDA initialises (tests run the harness in a subprocess for that reason), so a
  spinning barrier never sits in front of another rank's work in a shared queue;
* eager module loading (CUDA_MODULE_LOADING=EAGER before CUDA initialises): with lazy
  loading, the first launch of a kernel loads its module and that load waits for the
  kernels already running in the context — a spinning barrier of rank 0 then blocks the
  host before it has issued rank 1's arrival (observed: rank 0 timed out waiting for
  member 1 at its first barrier);
* FSP_BARRIER_TIMEOUT_S bounds every barrier spin: an issue bug becomes a device fault
  with a message, not a hang.
"""
from __future__ import annotations

import os
from typing import Callable, Sequence

import torch

from .executor import _SIGNAL_BYTES, FlexSPExecutor, LayoutError, PeerHeap, StepPlan


class VirtualHeap(PeerHeap):
    """One virtual rank's heap: a device buffer plus the shared table of every virtual
    rank's base address (filled in as the other ranks allocate)."""

    def __init__(self, nbytes: int, device: torch.device, ptrs: list[int], rank: int):
        self.device = device
        self.world_size = len(ptrs)
        self.nbytes = nbytes
        self.buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        self.ptrs = ptrs  # shared list: ptrs[r] = virtual rank r's base
        ptrs[rank] = self.buf.data_ptr()

    def peer(self, rank: int, offset: int) -> int:
        if not self.ptrs[rank]:
            raise LayoutError(f"virtual rank {rank} has no heap yet (prepare every rank first)")
        return self.ptrs[rank] + offset


class VirtualCluster:
    """`world` executors of one plan on one GPU (see the module docstring)."""

    def __init__(self, world: int, n_heads: int, head_dim: int, device="cuda", **kw):
        if os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8").isdigit() and \
                int(os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS", "8")) < world + 1:
            raise RuntimeError(
                f"VirtualCluster({world}) needs CUDA_DEVICE_MAX_CONNECTIONS >= {world + 1} "
                "set before CUDA initialises (one hardware queue per virtual rank)")
        if os.environ.get("CUDA_MODULE_LOADING", "LAZY").upper() != "EAGER":
            raise RuntimeError("VirtualCluster needs CUDA_MODULE_LOADING=EAGER set before CUDA "
                               "initialises (a lazy module load waits for the spinning barriers)")
        self.world = world
        self.device = torch.device(device)
        self.ptrs = [0] * world
        self.heaps: list[VirtualHeap | None] = [None] * world
        self.streams = [torch.cuda.Stream(self.device) for _ in range(world)]
        self.executors = [FlexSPExecutor(world, r, n_heads, head_dim, self.device,
                                         heap_factory=self._factory(r), **kw)
                          for r in range(world)]

    def _factory(self, rank: int) -> Callable[[int], VirtualHeap]:
        def make(nbytes: int) -> VirtualHeap:
            # a heap grows only between steps: nothing may still be queued on it
            torch.cuda.synchronize(self.device)
            self.heaps[rank] = None
            self.ptrs[rank] = 0
            h = VirtualHeap(nbytes, self.device, self.ptrs, rank)
            h.buf[:_SIGNAL_BYTES].zero_()
            self.heaps[rank] = h
            # every rank restarts its barrier epochs with a fresh heap; keep them in step
            for ex in self.executors:
                ex.epoch = 0
            for hh in self.heaps:
                if hh is not None:
                    hh.buf[:_SIGNAL_BYTES].zero_()
            torch.cuda.synchronize(self.device)
            return h
        return make

    def prepare(self, plan, lengths: Sequence[int], **kw) -> list[StepPlan]:
        sps = [ex.prepare(plan, lengths, **kw) for ex in self.executors]
        if len({sp.heap_bytes for sp in sps}) != 1:
            raise LayoutError("virtual ranks disagree on the heap layout")
        return sps

    def step(self, sps: Sequence[StepPlan], qkv_locals: Sequence[Sequence[torch.Tensor]],
             dout_locals: Sequence[Sequence[torch.Tensor]], sink=None) -> None:
        """Every rank's fwd+bwd of every micro-batch.  qkv_locals[r][m] / dout_locals[r][m]
        are rank r's loader-order rows; `sink(r, m, out, dqkv)` runs on rank r's stream
        and must not synchronise with the host."""
        cur = torch.cuda.current_stream(self.device)
        for r, ex in enumerate(self.executors):
            s = self.streams[r]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                ex.step(sps[r], qkv_locals[r], dout_locals[r],
                        sink=None if sink is None else (lambda m, o, d, r=r: sink(r, m, o, d)))
        for s in self.streams:
            cur.wait_stream(s)

    def run(self, fn: Callable[[int, FlexSPExecutor], None]) -> None:
        """Issue `fn(rank, executor)` for every rank on that rank's stream (same rules as
        step(): fn must not synchronise), then join the streams."""
        cur = torch.cuda.current_stream(self.device)
        for r, ex in enumerate(self.executors):
            s = self.streams[r]
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                fn(r, ex)
        for s in self.streams:
            cur.wait_stream(s)
