"""ZeRO-3 parameter / gradient / optimizer-state sharding for the layers around the SP step
("ZeRO with PyTorch FSDP").

In FlexSP every rank is a data-parallel replica of the model — SP groups split tokens and
heads, never parameters — so the whole world shards the model state ZeRO-3 style:

* each layer's parameters live as one flat bf16 buffer padded to a multiple of the world
  size; rank r keeps only shard r of it, with fp32 master weights and the optimizer state
  of that shard (1/W of the memory of a replica);
* before a layer runs (forward, and again when activation checkpointing recomputes it in
  the backward) its flat buffer is all-gathered (NCCL all_gather_into_tensor over NVLink)
  on a communication stream; the next layer's gather is issued while the current layer
  computes (prefetch), and a gathered buffer is released after the layer's use;
* gradients accumulate into a flat per-layer buffer (the parameters' .grad are views of
  it); when the layer's last gradient lands (post-accumulate-grad hooks) the buffer is
  reduce-scattered (sum) into the rank's fp32 gradient shard on the communication stream,
  overlapping the backward of the layers below — one bucket per layer;
* step() updates the fp32 master shard (SGD with momentum or AdamW) and refreshes the bf16
  shard the next gathers read.
Collectives are issued in the same order on every rank because every rank runs the same
layers for every micro-batch (idle ranks on zero rows), as the SP executor already requires.
"""
from __future__ import annotations

import contextlib
import math
from typing import Iterable, Sequence

import torch
import torch.distributed as dist


# CUDA: collectives on a side stream, ordered with events.  CPU (gloo, the CPU test suite):
# the same code path with every stream operation a no-op.
def _cur(dev: torch.device):
    return torch.cuda.current_stream(dev) if dev.type == "cuda" else None


def _on(stream):
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def _wait_stream(a, b) -> None:
    if a is not None and b is not None:
        a.wait_stream(b)


def _record(stream):
    if stream is None:
        return None
    ev = torch.cuda.Event()
    ev.record(stream)
    return ev


class ShardedLayer:
    """ZeRO-3 state of one module (all its parameters as one flat bucket)."""

    def __init__(self, module: torch.nn.Module, world: int, rank: int, group=None):
        self.module = module
        self.params = [p for p in module.parameters() if p.requires_grad]
        self.world, self.rank, self.group = world, rank, group
        self.shapes = [p.shape for p in self.params]
        self.numels = [p.numel() for p in self.params]
        n = sum(self.numels)
        self.padded = -(-n // world) * world
        self.shard_numel = self.padded // world
        dev = self.params[0].device
        self.dtype = self.params[0].dtype
        flat = torch.zeros(self.padded, dtype=self.dtype, device=dev)
        torch.cat([p.detach().reshape(-1) for p in self.params], out=flat[:n])
        lo = rank * self.shard_numel
        self.shard = flat[lo:lo + self.shard_numel].clone()              # bf16 shard
        self.master = self.shard.float()                                  # fp32 master shard
        self.grad_shard = torch.zeros(self.shard_numel, dtype=torch.float32, device=dev)
        self.full: torch.Tensor | None = None                             # gathered buffer
        self.flat_grad: torch.Tensor | None = None
        self.gather_done: torch.cuda.Event | None = None
        self.rs_done: torch.cuda.Event | None = None
        self.pending_grads = 0
        del flat
        for p in self.params:  # parameters hold no storage until gathered
            p.data = torch.empty(0, dtype=self.dtype, device=dev)
        for p in self.params:
            p.register_post_accumulate_grad_hook(self._grad_ready)

    # ---------------------------------------------------------------- all-gather
    def gather(self, stream: torch.cuda.Stream) -> None:
        """Issue the all-gather of this layer's parameters on `stream` (idempotent)."""
        if self.full is not None:
            return
        cur = _cur(self.shard.device)
        _wait_stream(stream, cur)  # the shard may just have been updated by step()
        with _on(stream):
            full = torch.empty(self.padded, dtype=self.dtype, device=self.shard.device)
            if self.world > 1:
                dist.all_gather_into_tensor(full, self.shard, group=self.group)
            else:
                full.copy_(self.shard)
            self.gather_done = _record(stream)
        if cur is not None:
            full.record_stream(cur)
        self.full = full

    def materialize(self) -> None:
        """Point the parameters at the gathered buffer (the compute stream waits for it)."""
        if self.gather_done is not None:
            _cur(self.shard.device).wait_event(self.gather_done)
        off = 0
        for p, shp, n in zip(self.params, self.shapes, self.numels):
            p.data = self.full[off:off + n].view(shp)
            off += n

    def release(self) -> None:
        """Drop the gathered parameters (storage returns to the caching allocator once the
        compute stream is past the layer)."""
        for p in self.params:
            p.data = torch.empty(0, dtype=self.dtype, device=self.shard.device)
        self.full = None

    # ---------------------------------------------------------------- reduce-scatter
    def prepare_grads(self) -> None:
        """Before the layer's backward (parameters materialized): their .grad become views of
        one zeroed flat buffer, so autograd accumulates straight into the reduce-scatter
        bucket."""
        self.flat_grad = torch.zeros(self.padded, dtype=self.dtype, device=self.shard.device)
        off = 0
        for p, shp, n in zip(self.params, self.shapes, self.numels):
            p.grad = self.flat_grad[off:off + n].view(shp)
            off += n
        self.pending_grads = len(self.params)

    def _grad_ready(self, p: torch.Tensor) -> None:
        self.pending_grads -= 1
        if self.pending_grads == 0:
            # the layer's backward is complete: nothing needs its weights any more
            self.reduce_scatter(self._comm)
            self.release()

    _comm: torch.cuda.Stream | None = None

    def reduce_scatter(self, stream: torch.cuda.Stream) -> None:
        cur = _cur(self.shard.device)
        _wait_stream(stream, cur)
        flat = self.flat_grad
        with _on(stream):
            part = torch.empty(self.shard_numel, dtype=self.dtype, device=flat.device)
            if self.world > 1:
                dist.reduce_scatter_tensor(part, flat, op=dist.ReduceOp.SUM, group=self.group)
            else:
                part.copy_(flat)
            self.grad_shard.add_(part.float())
            self.rs_done = _record(stream)
        if stream is not None:
            flat.record_stream(stream)
        for p in self.params:
            p.grad = None
        self.flat_grad = None


class ZeroStack:
    """ZeRO-3 over a sequence of layers run in order (the transformer stack).

    forward hooks gather layer i (and prefetch layer i+1) before it runs and release it
    after; backward hooks reduce-scatter each layer's gradients as soon as they are
    complete.  Use:
        zs = ZeroStack(layers, world, rank)
        zs.begin_micro_batch()           # before each micro-batch's forward
        ... forward through layers (per-layer activation checkpointing, required) ...
        zs.begin_backward(); loss.backward()
        zs.step(lr)                      # after the last micro-batch of the step
    """

    def __init__(self, layers: Sequence[torch.nn.Module], world: int, rank: int, group=None,
                 optimizer: str = "sgd", momentum: float = 0.9, betas=(0.9, 0.95),
                 eps: float = 1e-8, weight_decay: float = 0.0):
        self.layers = list(layers)
        self.shards = [ShardedLayer(l, world, rank, group) for l in self.layers]
        dev = self.shards[0].shard.device
        self.comm = torch.cuda.Stream(dev) if dev.type == "cuda" else None
        for s in self.shards:
            s._comm = self.comm
        self.optimizer = optimizer
        self.momentum, self.betas, self.eps, self.wd = momentum, betas, eps, weight_decay
        self.state = [torch.zeros_like(s.master) for s in self.shards]
        self.state2 = [torch.zeros_like(s.master) for s in self.shards] if optimizer == "adamw" else None
        self.t = 0
        self.backward_phase = False
        for i, l in enumerate(self.layers):
            l.register_forward_pre_hook(self._pre(i))
            l.register_forward_hook(self._post(i))

    def _pre(self, i: int):
        def hook(module, args):
            s = self.shards[i]
            s.gather(self.comm)
            # prefetch the layer that runs next: i+1 in the forward, i-1 when activation
            # checkpointing recomputes the layers in reverse during the backward
            nxt = i - 1 if self.backward_phase else i + 1
            if 0 <= nxt < len(self.shards):
                self.shards[nxt].gather(self.comm)
            s.materialize()
            if self.backward_phase and s.flat_grad is None:
                s.prepare_grads()  # the recomputed layer's backward accumulates into the bucket
        return hook

    def _post(self, i: int):
        def hook(module, args, out):
            # forward (checkpointed: nothing saved the weights) -> release now; in the
            # backward's recomputation the weights are still needed by the layer's own
            # backward, so they are released when its gradients are complete
            if not self.backward_phase:
                self.shards[i].release()
        return hook

    def begin_micro_batch(self) -> None:
        """Before a micro-batch's forward (forward phase: layers released after use)."""
        self.backward_phase = False

    def begin_backward(self) -> None:
        """Between the forward and loss.backward() of a micro-batch (the layers are then
        recomputed in reverse order by activation checkpointing)."""
        self.backward_phase = True

    def sharded_bytes(self) -> dict:
        """Per-rank bytes of model state (bf16 shard, fp32 master, fp32 grad, optimizer)."""
        n = sum(s.shard_numel for s in self.shards)
        opt = 4 * n * (2 if self.optimizer == "adamw" else 1)
        return {"params_total": sum(s.padded for s in self.shards), "shard_elems": n,
                "bytes_per_rank": 2 * n + 4 * n + 4 * n + opt}

    @torch.no_grad()
    def step(self, lr: float) -> None:
        """Optimizer step on the shards (waits for every reduce-scatter)."""
        _wait_stream(_cur(self.shards[0].shard.device), self.comm)
        self.t += 1
        masters = [s.master for s in self.shards]
        grads = [s.grad_shard for s in self.shards]
        if self.wd:
            torch._foreach_mul_(masters, 1.0 - lr * self.wd)
        if self.optimizer == "sgd":
            torch._foreach_mul_(self.state, self.momentum)
            torch._foreach_add_(self.state, grads)
            torch._foreach_add_(masters, self.state, alpha=-lr)
        else:  # adamw
            b1, b2 = self.betas
            torch._foreach_lerp_(self.state, grads, 1.0 - b1)
            torch._foreach_mul_(self.state2, b2)
            torch._foreach_addcmul_(self.state2, grads, grads, value=1.0 - b2)
            c1, c2 = 1.0 - b1 ** self.t, 1.0 - b2 ** self.t
            denom = torch._foreach_sqrt(self.state2)
            torch._foreach_div_(denom, math.sqrt(c2))
            torch._foreach_add_(denom, self.eps)
            torch._foreach_addcdiv_(masters, self.state, denom, value=-lr / c1)
        for s in self.shards:
            s.shard.copy_(s.master)
            s.grad_shard.zero_()

    def full_parameters(self) -> list[torch.Tensor]:
        """Gather every layer's full flat parameters (for checks); collective."""
        out = []
        for s in self.shards:
            s.gather(self.comm)
            if s.gather_done is not None:
                _cur(s.shard.device).wait_event(s.gather_done)
            out.append(s.full[:sum(s.numels)].clone())
            s.full = None
        return out


def params_iter(layers: Iterable[torch.nn.Module]):
    for l in layers:
        yield from l.parameters()
