"""Model-config callers of the hot path (SURVEY §8 f, row 1; BASELINE configs 1-3).

Stock PyTorch forward/backward writes the gradient straight into the flat
buffer (``FlatParameters``: every ``p.grad`` is a view), then one
``SelSyncStep`` runs the hot path. Shapes and hyper-parameters follow the
paper:

  resnet101    torchvision resnet101(num_classes=10), CIFAR-10 32x32x3, batch 32/worker,
               SGD lr 0.1, momentum 0.9, weight decay 4e-4            P = 42,520,650
  vgg11        torchvision vgg11(num_classes=100), CIFAR-100 32x32x3, batch 32/worker,
               SGD lr 0.01, momentum 0.9, weight decay 5e-4           P = 129,176,036
  transformer  2-layer encoder LM, d = 200, 2 heads, nhid 200, dropout 0.2, bptt 35,
               WikiText-103 vocabulary (267,735), batch 20/worker, lr 2.0 decayed
               x0.8 every 2000 iterations, SelDP token-stream partitioning
                                                                      P = 107,845,735

Data are synthetic tensors of those shapes (no network for datasets); model
weights are random-init. BatchNorm running statistics are buffers, not
parameters: they stay per replica (the reference averages parameters only).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch
import torch.nn as nn

from .data import TokenStreamSampler
from .errors import ConfigError
from .model import LrSchedule, lr_at

WIKITEXT103_VOCAB = 267_735


class PositionalEncoding(nn.Module):
    def __init__(self, d_model: int, dropout: float, max_len: int = 5000):
        super().__init__()
        self.dropout = nn.Dropout(p=dropout)
        pe = torch.zeros(max_len, d_model)
        pos = torch.arange(0, max_len, dtype=torch.float).unsqueeze(1)
        div = torch.exp(torch.arange(0, d_model, 2).float() * (-math.log(10000.0) / d_model))
        pe[:, 0::2] = torch.sin(pos * div)
        pe[:, 1::2] = torch.cos(pos * div)
        self.register_buffer("pe", pe.unsqueeze(1))

    def forward(self, x):
        return self.dropout(x + self.pe[: x.size(0)])


class TransformerLM(nn.Module):
    """Encoder-only LM of the paper's WikiText-103 experiment."""

    def __init__(self, ntoken=WIKITEXT103_VOCAB, d_model=200, nhead=2, nhid=200, nlayers=2, dropout=0.2):
        super().__init__()
        self.encoder = nn.Embedding(ntoken, d_model)
        self.pos = PositionalEncoding(d_model, dropout)
        layer = nn.TransformerEncoderLayer(d_model, nhead, nhid, dropout)
        self.transformer = nn.TransformerEncoder(layer, nlayers, enable_nested_tensor=False)
        self.decoder = nn.Linear(d_model, ntoken)
        self.d_model = d_model
        self.register_buffer("mask", torch.empty(0), persistent=False)

    def forward(self, src):  # src: (bptt, batch) token ids
        n = src.size(0)
        if self.mask.size(0) != n:
            self.mask = torch.triu(torch.full((n, n), float("-inf"), device=src.device), diagonal=1)
        x = self.pos(self.encoder(src) * math.sqrt(self.d_model))
        # is_causal: skip the mask inspection (a host sync that would break graph capture)
        return self.decoder(self.transformer(x, self.mask, is_causal=True))


@dataclass
class Workload:
    name: str
    model: nn.Module
    lr: Callable[[int], float]
    momentum: float
    weight_decay: float
    make_batch: Callable[[int], tuple]  # step -> (inputs, targets) on the device
    loss: Callable[[nn.Module, tuple], torch.Tensor]
    host_batch_bytes: int  # bytes one host->device batch copy moves


def _cifar(name, ctor, num_classes, batch, lr0, wd, device, seed, channels_last=True):
    import torchvision

    model = getattr(torchvision.models, ctor)(num_classes=num_classes).to(device)
    if channels_last:
        model = model.to(memory_format=torch.channels_last)
    gen = torch.Generator(device=device).manual_seed(seed)
    x = torch.randn(batch, 3, 32, 32, generator=gen, device=device).contiguous(memory_format=torch.channels_last)
    y = torch.randint(0, num_classes, (batch,), generator=gen, device=device)
    ce = nn.CrossEntropyLoss()
    return Workload(name, model, lambda step: lr0, 0.9, wd, lambda step: (x, y),
                    lambda m, b: ce(m(b[0]), b[1]), host_batch_bytes=x.numel() * 4 + y.numel() * 8)


def build(name: str, device, *, rank: int = 0, world: int = 1, seed: int = 0) -> Workload:
    """BASELINE configs 1-3 by name."""
    device = torch.device(device)
    torch.manual_seed(seed)  # identical init on every rank (the bootstrap broadcast also enforces it)
    if name == "resnet101":
        return _cifar(name, "resnet101", 10, 32, 0.1, 4e-4, device, seed + rank)
    if name == "vgg11":
        return _cifar(name, "vgg11", 100, 32, 0.01, 5e-4, device, seed + rank)
    if name == "transformer":
        model = TransformerLM().to(device)
        bptt, batch = 35, 20
        n_tokens = 2_000_000  # synthetic WikiText-103-shaped stream (vocabulary 267,735)
        rng = np.random.default_rng(seed)
        stream = torch.from_numpy(rng.integers(0, WIKITEXT103_VOCAB, size=n_tokens, dtype=np.int64)).to(device)
        sampler = TokenStreamSampler(n_tokens, bptt, rank, world, batch, seed=seed + 1)
        offs = torch.arange(bptt + 1, device=device)
        ce = nn.CrossEntropyLoss()
        sched = LrSchedule(2.0, tuple((2000 * k, 0.8) for k in range(1, 64)), mode="per_step")

        def make_batch(step):
            starts, _src = sampler.next_windows()
            idx = torch.from_numpy(starts).to(device, non_blocking=True)[None, :] + offs[:, None]
            win = stream[idx]  # (bptt + 1, batch)
            return win[:-1], win[1:]

        def loss(m, b):
            out = m(b[0])
            return ce(out.reshape(-1, out.size(-1)), b[1].reshape(-1))

        return Workload(name, model, lambda step: lr_at(sched, step, 0), 0.0, 0.0, make_batch, loss,
                        host_batch_bytes=(bptt + 1) * batch * 8)
    raise ConfigError(f"unknown workload {name!r} (resnet101, vgg11, transformer)")


def parameter_count(model: nn.Module) -> int:
    return sum(p.numel() for p in model.parameters() if p.requires_grad)
