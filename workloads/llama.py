"""Llama-2 architecture (RMSNorm, rotary embeddings, SwiGLU MLP, causal SDPA) in plain PyTorch
with seeded random init: the real model behind config C3 (Llama-2 7B: 32 layers, d 4096, 32
heads, MLP 11008, vocab 32000) for the runtime's end-to-end step.  No
method arithmetic lives here."""
import torch
import torch.nn as nn
import torch.nn.functional as F

LLAMA2_7B = dict(n_layer=32, d=4096, n_head=32, d_ff=11008, vocab=32000)


class RMSNorm(nn.Module):
    def __init__(self, d: int, eps: float = 1e-5):
        super().__init__()
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(d))

    def forward(self, x):
        xf = x.float()
        return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)).type_as(x) * self.weight


def _rope(x, cos, sin):
    x1, x2 = x[..., : x.shape[-1] // 2], x[..., x.shape[-1] // 2:]
    return x * cos + torch.cat((-x2, x1), dim=-1) * sin


class Layer(nn.Module):
    def __init__(self, d, n_head, d_ff):
        super().__init__()
        self.n_head = n_head
        self.attn_norm = RMSNorm(d)
        self.wq = nn.Linear(d, d, bias=False)
        self.wk = nn.Linear(d, d, bias=False)
        self.wv = nn.Linear(d, d, bias=False)
        self.wo = nn.Linear(d, d, bias=False)
        self.mlp_norm = RMSNorm(d)
        self.w1 = nn.Linear(d, d_ff, bias=False)
        self.w3 = nn.Linear(d, d_ff, bias=False)
        self.w2 = nn.Linear(d_ff, d, bias=False)

    def forward(self, x, cos, sin):
        B, S, D = x.shape
        hd = D // self.n_head
        h = self.attn_norm(x)
        q = self.wq(h).view(B, S, self.n_head, hd).transpose(1, 2)
        k = self.wk(h).view(B, S, self.n_head, hd).transpose(1, 2)
        v = self.wv(h).view(B, S, self.n_head, hd).transpose(1, 2)
        q, k = _rope(q, cos, sin), _rope(k, cos, sin)
        y = F.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + self.wo(y.transpose(1, 2).reshape(B, S, D))
        h = self.mlp_norm(x)
        return x + self.w2(F.silu(self.w1(h)) * self.w3(h))


class Llama(nn.Module):
    def __init__(self, n_layer, d, n_head, d_ff, vocab, max_seq=4096):
        super().__init__()
        self.tok = nn.Embedding(vocab, d)
        self.layers = nn.ModuleList([Layer(d, n_head, d_ff) for _ in range(n_layer)])
        self.norm = RMSNorm(d)
        self.head = nn.Linear(d, vocab, bias=False)
        hd = d // n_head
        inv = 1.0 / (10000 ** (torch.arange(0, hd, 2).float() / hd))
        ang = torch.outer(torch.arange(max_seq).float(), inv)
        ang = torch.cat((ang, ang), dim=-1)
        self.register_buffer("cos", ang.cos(), persistent=False)
        self.register_buffer("sin", ang.sin(), persistent=False)

    def forward(self, idx, targets):
        S = idx.shape[1]
        cos, sin = self.cos[:S].to(self.tok.weight.dtype), self.sin[:S].to(self.tok.weight.dtype)
        x = self.tok(idx)
        for layer in self.layers:
            x = layer(x, cos, sin)
        logits = self.head(self.norm(x))
        return F.cross_entropy(logits.view(-1, logits.size(-1)).float(), targets.view(-1))


def make(cfg=LLAMA2_7B, seed: int = 0, device="cuda", dtype=torch.bfloat16, max_seq=4096) -> Llama:
    torch.manual_seed(seed)
    with torch.device(device):
        m = Llama(max_seq=max_seq, **cfg)
    for p in m.parameters():
        if p.dim() > 1:
            nn.init.normal_(p, std=0.02)
    return m.to(dtype)


def batch(b: int, s: int, vocab: int, seed: int = 0, device="cuda"):
    g = torch.Generator().manual_seed(seed)
    idx = torch.randint(0, vocab, (b, s), generator=g)
    tgt = torch.randint(0, vocab, (b, s), generator=g)
    return idx.to(device), tgt.to(device)
