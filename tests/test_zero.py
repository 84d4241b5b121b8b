"""ZeRO-3 sharding (paper_2412_01523_b200/zero.py) on CPU with gloo at
world size 2: sharded parameters gathered per layer, gradients reduce-scattered per layer,
SGD-momentum / AdamW on the fp32 master shards — after several steps with per-layer
activation checkpointing the gathered parameters equal a replicated fp32 reference that
all-reduces (sums) full gradients and applies the same optimizer."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class Block(torch.nn.Module):
    def __init__(self, h, seed):
        super().__init__()
        g = torch.Generator().manual_seed(seed)
        self.ln = torch.nn.LayerNorm(h)
        self.w1 = torch.nn.Parameter(torch.randn(2 * h, h, generator=g) * 0.1)
        self.w2 = torch.nn.Parameter(torch.randn(h, 2 * h, generator=g) * 0.1)

    def forward(self, x):
        return x + torch.nn.functional.linear(torch.tanh(torch.nn.functional.linear(self.ln(x), self.w1)), self.w2)


def _worker(rank, world, port, optimizer, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.manual_seed(0)
    from torch.utils.checkpoint import checkpoint
    from paper_2412_01523_b200.zero import ZeroStack
    h, L = 12, 3
    layers = [Block(h, 10 + i) for i in range(L)]
    ref = [Block(h, 10 + i) for i in range(L)]
    zs = ZeroStack(layers, world, rank, optimizer=optimizer, weight_decay=0.01)
    ref_params = [p for l in ref for p in l.parameters()]
    mom = [torch.zeros_like(p) for p in ref_params]
    v2 = [torch.zeros_like(p) for p in ref_params]
    lr = 0.05
    for step in range(3):
        for mb in range(2):  # two micro-batches of gradient accumulation, ranks see different data
            g = torch.Generator().manual_seed(100 * step + 10 * mb + rank)
            x = torch.randn(5 + rank, h, generator=g)
            zs.begin_micro_batch()
            y = x
            for l in layers:
                y = checkpoint(l, y, use_reentrant=False)
            zs.begin_backward()
            (y * y).mean().backward()
            yr = x
            for l in ref:
                yr = l(yr)
            (yr * yr).mean().backward()
        zs.step(lr)
        with torch.no_grad():
            for p in ref_params:
                dist.all_reduce(p.grad)
            for i, p in enumerate(ref_params):
                p.mul_(1 - lr * 0.01)
                if optimizer == "sgd":
                    mom[i].mul_(0.9).add_(p.grad)
                    p.add_(mom[i], alpha=-lr)
                else:
                    t = step + 1
                    mom[i].lerp_(p.grad, 0.1)
                    v2[i].mul_(0.95).addcmul_(p.grad, p.grad, value=0.05)
                    den = (v2[i].sqrt() / (1 - 0.95 ** t) ** 0.5).add_(1e-8)
                    p.addcdiv_(mom[i], den, value=-lr / (1 - 0.9 ** t))
                p.grad = None
    full = zs.full_parameters()
    flat_ref = [torch.cat([p.detach().reshape(-1) for p in l.parameters()]) for l in ref]
    # relative: the two sides sum the micro-batches' gradients in a different order
    err = max(float((a - b).abs().max() / b.abs().max()) for a, b in zip(full, flat_ref))
    out[rank] = err
    dist.destroy_process_group()


@pytest.mark.parametrize("optimizer", ["sgd", "adamw"])
def test_zero3_matches_replicated_allreduce(optimizer):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), optimizer, out), nprocs=world, join=True)
    assert max(out.values()) < 1e-5, dict(out)  # relative, fp32
