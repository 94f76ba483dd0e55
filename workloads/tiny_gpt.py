"""A small decoder-only transformer (GPT-style) and its seeded synthetic batches: the real eager
training workload of the runtime tests.  Plain PyTorch ops only
(attention written out as matmul + softmax so every kernel is deterministic), random init from a
seed.  No method arithmetic lives here."""
import math

import torch
import torch.nn as nn
import torch.nn.functional as F


class Block(nn.Module):
    def __init__(self, d: int, n_head: int):
        super().__init__()
        self.n_head = n_head
        self.ln1 = nn.LayerNorm(d)
        self.qkv = nn.Linear(d, 3 * d)
        self.proj = nn.Linear(d, d)
        self.ln2 = nn.LayerNorm(d)
        self.fc = nn.Linear(d, 4 * d)
        self.out = nn.Linear(4 * d, d)

    def forward(self, x, mask):
        B, S, D = x.shape
        h = self.ln1(x)
        q, k, v = self.qkv(h).split(D, dim=2)
        q = q.view(B, S, self.n_head, D // self.n_head).transpose(1, 2)
        k = k.view(B, S, self.n_head, D // self.n_head).transpose(1, 2)
        v = v.view(B, S, self.n_head, D // self.n_head).transpose(1, 2)
        att = (q @ k.transpose(-2, -1)) * (1.0 / math.sqrt(D // self.n_head))
        att = att.masked_fill(mask, float("-inf")).softmax(dim=-1)
        y = (att @ v).transpose(1, 2).reshape(B, S, D)
        x = x + self.proj(y)
        x = x + self.out(F.gelu(self.fc(self.ln2(x))))
        return x


class TinyGPT(nn.Module):
    def __init__(self, vocab: int = 64, d: int = 32, n_layer: int = 4, n_head: int = 4, seq: int = 16):
        super().__init__()
        self.wte = nn.Embedding(vocab, d)
        self.wpe = nn.Embedding(seq, d)
        self.blocks = nn.ModuleList([Block(d, n_head) for _ in range(n_layer)])
        self.ln_f = nn.LayerNorm(d)
        self.head = nn.Linear(d, vocab, bias=False)
        self.register_buffer("mask", torch.triu(torch.ones(seq, seq, dtype=torch.bool), diagonal=1))
        self.drift_layer = -1  # tests: insert one unrelated op before this block (sequence drift)

    def forward(self, idx, targets):
        B, S = idx.shape
        pos = torch.arange(S, device=idx.device)
        x = self.wte(idx) + self.wpe(pos)
        for li, blk in enumerate(self.blocks):
            if li == self.drift_layer:
                self._probe = self.wte.weight.norm()  # e.g. a logging read: one extra op
            x = blk(x, self.mask[:S, :S])
        logits = self.head(self.ln_f(x))
        return F.cross_entropy(logits.view(-1, logits.size(-1)), targets.view(-1))


def make(seed: int = 0, device="cpu", **kw) -> TinyGPT:
    g = torch.manual_seed(seed)  # noqa: F841
    return TinyGPT(**kw).to(device)


def batches(n: int, batch: int, seq: int, vocab: int, seed: int = 0, device="cpu"):
    g = torch.Generator().manual_seed(seed)
    out = []
    for _ in range(n):
        idx = torch.randint(0, vocab, (batch, seq), generator=g)
        tgt = torch.randint(0, vocab, (batch, seq), generator=g)
        out.append((idx.to(device), tgt.to(device)))
    return out
