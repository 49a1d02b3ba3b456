"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no routing, no plan, no
FFN): it only draws random tensors with the shapes, scales and routing skew of
the paper's workloads (BASELINE.json configs C1-C5), so that both sides of a
parity test read exactly the same bits.

Recipe:
  * x ~ N(0, 1) with channel 0 set to 1.0 (a bias channel, exact in bf16).
  * Wr[e, j] ~ N(0, 1/d) for j >= 1 and Wr[e, 0] = b_e ~ N(0, sigma^2): the
    bias channel skews expert popularity while Eq. 8 stays bias-free.
    sigma = 0 "uniform", 0.5 "long-tail" (the paper's cold experts, P:48,
    P:122), 1.0 "heavy".
  * Wg, Wu ~ N(0, 1/d), Wd ~ N(0, 1/f)  (nn.Linear [out, in] layout:
    Wg, Wu [m, f, d], Wd [m, d, f]).
  * Everything is rounded once to the storage dtype (bf16 RNE; C1 stays fp32).
  * Seeds: weights 1000 + config id, tokens 2000 + batch index.

Draws use torch.Generator on the requested device ("cpu" draws are what the
oracle tests use; "cuda" draws are a fast path for full-size benches whose
parity samples copy the same generated tensors back to the host).
"""
from __future__ import annotations

from dataclasses import dataclass, replace

import torch


@dataclass(frozen=True)
class LayerConfig:
    name: str
    d: int            # hidden
    f: int            # ffn
    m: int            # experts
    K: int            # top-k
    way: int          # k of the paper (experts per united group)
    T: int            # tokens per batch
    ratio: float      # brownout ratio = 1 - threshold
    dtype: str        # "bf16" | "fp32"
    sigma: float = 0.5
    config_id: int = 0
    Ns: int = 0       # shared experts (Eq. 5 second term), each of width f

    @property
    def G(self) -> int:
        return -(-self.m // self.way)


# BASELINE.json configs (B:7-B:11)
C1 = LayerConfig("tiny", d=64, f=128, m=8, K=2, way=4, T=32, ratio=0.5, dtype="fp32",
                 sigma=0.0, config_id=1)
C2 = LayerConfig("mixtral_prefill", d=4096, f=14336, m=8, K=2, way=4, T=4096, ratio=0.5,
                 dtype="bf16", sigma=0.5, config_id=2)
C3 = LayerConfig("mixtral_decode", d=4096, f=14336, m=8, K=2, way=4, T=256, ratio=0.5,
                 dtype="bf16", sigma=0.5, config_id=3)
C4 = LayerConfig("qwen3_30b_a3b_prefill", d=2048, f=768, m=128, K=8, way=4, T=8192,
                 ratio=0.5, dtype="bf16", sigma=0.5, config_id=4)
C5 = LayerConfig("mixtral_ep", d=4096, f=14336, m=8, K=2, way=4, T=4096, ratio=0.5,
                 dtype="bf16", sigma=0.5, config_id=5)
# f2 (SURVEY.md §8 "next"): the paper's own model shape, Qwen1.5-MoE-A2.7B:
# 60 experts top-4, hidden 2048, expert ffn 1408, shared-expert width 5632 =
# 4 x 1408 (public model config) as N_s = 4 shared experts; the paper's
# (way, threshold) configs (2, 0), (4, 0.2), (8, 0.4) -> way 4, ratio
# 1 - 0.2 = 0.8 here (reading D2; way 8 gives the ragged 8th group of 4).
PAPER_WAY_THRESHOLD = ((2, 0.0), (4, 0.2), (8, 0.4))
F2 = LayerConfig("qwen15_moe_a27b_prefill", d=2048, f=1408, m=60, K=4, way=4, T=4096, ratio=0.8,
                 dtype="bf16", sigma=0.5, config_id=6, Ns=4)
CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5, F2)}
RATIO_SWEEP = (0.0, 0.25, 0.5, 1.0)


def torch_dtype(name: str):
    return {"bf16": torch.bfloat16, "fp32": torch.float32}[name]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def make_layer(cfg: LayerConfig, device="cpu", seed: int | None = None):
    """Router centroids and expert weights of one layer: dict of tensors."""
    seed = 1000 + cfg.config_id if seed is None else seed
    g = _gen(seed, device)
    dt = torch_dtype(cfg.dtype)
    d, f, m = cfg.d, cfg.f, cfg.m
    Wr = torch.randn(m, d, generator=g, device=device, dtype=torch.float32) * (1.0 / d) ** 0.5
    b = torch.randn(m, generator=g, device=device, dtype=torch.float32) * cfg.sigma
    Wr[:, 0] = b
    out = {"Wr": Wr.to(dt)}
    for name, shape, scale in (("Wg", (m, f, d), d), ("Wu", (m, f, d), d), ("Wd", (m, d, f), f)):
        w = torch.empty(shape, device=device, dtype=dt)
        for e in range(m):   # per-expert draws keep peak fp32 memory at one expert
            w[e] = (torch.randn(shape[1:], generator=g, device=device, dtype=torch.float32)
                    * (1.0 / scale) ** 0.5).to(dt)
        out[name] = w
    if cfg.Ns:   # shared experts: same scales, drawn after the routed ones
        for name, shape, scale in (("SWg", (cfg.Ns, f, d), d), ("SWu", (cfg.Ns, f, d), d),
                                   ("SWd", (cfg.Ns, d, f), f)):
            w = torch.empty(shape, device=device, dtype=dt)
            for e in range(cfg.Ns):
                w[e] = (torch.randn(shape[1:], generator=g, device=device, dtype=torch.float32)
                        * (1.0 / scale) ** 0.5).to(dt)
            out[name] = w
    return out


def make_united_random(cfg: LayerConfig, device="cpu", seed: int | None = None):
    """Independent random united weights (for tests that must not depend on
    any particular united-expert initialisation)."""
    seed = 3000 + cfg.config_id if seed is None else seed
    g = _gen(seed, device)
    dt = torch_dtype(cfg.dtype)
    d, f, G = cfg.d, cfg.f, cfg.G
    UWg = (torch.randn(G, f, d, generator=g, device=device) * (1.0 / d) ** 0.5).to(dt)
    UWu = (torch.randn(G, f, d, generator=g, device=device) * (1.0 / d) ** 0.5).to(dt)
    UWd = (torch.randn(G, d, f, generator=g, device=device) * (1.0 / f) ** 0.5).to(dt)
    return {"UWg": UWg, "UWu": UWu, "UWd": UWd}


def make_tokens(cfg: LayerConfig, batch_index: int = 0, T: int | None = None, device="cpu",
                seed: int | None = None):
    """Token batch x [T, d] with the bias channel x[:, 0] = 1."""
    T = cfg.T if T is None else T
    seed = 2000 + batch_index if seed is None else seed
    g = _gen(seed, device)
    x = torch.randn(T, cfg.d, generator=g, device=device, dtype=torch.float32)
    x[:, 0] = 1.0
    return x.to(torch_dtype(cfg.dtype))


def make_logits_with_counts(counts, K: int = 1, seed: int = 0):
    """fp32 logits [T, m] whose top-1 routing realises the given per-expert
    counts exactly (one-hot: the chosen expert gets logit 4, the rest 0), with
    tokens shuffled by a seeded permutation.  K must be 1."""
    assert K == 1
    m = len(counts)
    ids = []
    for e, c in enumerate(counts):
        ids += [e] * int(c)
    g = _gen(seed, "cpu")
    perm = torch.randperm(len(ids), generator=g)
    ids = torch.tensor(ids, dtype=torch.long)[perm]
    L = torch.zeros(len(ids), m, dtype=torch.float32)
    L[torch.arange(len(ids)), ids] = 4.0
    return L


def with_(cfg: LayerConfig, **kw) -> LayerConfig:
    return replace(cfg, **kw)


def make_logits(T: int, m: int, seed: int = 0, sigma: float = 0.5, device="cpu", ties: bool = False):
    """fp32 router logits [T, m] drawn directly (for routing parity with
    injected logits): N(0, 1) plus a per-expert N(0, sigma^2) popularity bias.
    ties=True draws small integers instead, so equal logits (and -0.0 / +0.0)
    are frequent."""
    g = _gen(seed, device)
    if ties:
        L = torch.randint(-2, 3, (T, m), generator=g, device=device).to(torch.float32)
        neg = torch.rand(T, m, generator=g, device=device) < 0.5
        L = torch.where((L == 0) & neg, torch.full_like(L, -0.0), L)
        return L
    bias = torch.randn(m, generator=g, device=device) * sigma
    return torch.randn(T, m, generator=g, device=device) + bias


def make_exact_router_inputs(cfg: LayerConfig, T: int | None = None, batch_index: int = 0, device="cpu",
                             ties: bool = False):
    """Tokens x [T, d] and router centroids Wr [m, d] whose Eq. 8 dot products
    are EXACT in fp32 (and tf32) accumulation in any order, so that the GPU
    router's logits equal the fp64 ones bit for bit and routing parity needs no
    clear-margin filter.

    ties=False ("dyadic"): x ~ N(0, 1) rounded to multiples of 1/8 in
    [-4, 4), x[:, 0] = 1; Wr ~ N(0, 1/d) rounded to multiples of 2^-10 in
    (-1/4, 1/4), bias channel Wr[:, 0] ~ N(0, sigma^2) on the same grid.  Every
    product is a multiple of 2^-13; the caller checks the partial-sum bound
    sum_j |x_tj||Wr_ej| < 2^11 (exactness_bound) so every partial sum has at
    most 24 significant bits.

    ties=True ("integer"): x in {-1, 0, 1} (x[:, 0] = 1), Wr in {-1, 0, 1} on
    16 channels plus an integer bias in [-2, 2]: logits are small integers and
    exact ties between experts are frequent (Eq. 7 tie rule, reading D8).
    """
    T = cfg.T if T is None else T
    g = _gen(5000 + 97 * cfg.config_id + batch_index, device)
    dt = torch_dtype(cfg.dtype)
    d, m = cfg.d, cfg.m
    if ties:
        x = torch.randint(-1, 2, (T, d), generator=g, device=device).to(torch.float32)
        x[:, 0] = 1.0
        Wr = torch.zeros(m, d, device=device)
        nz = min(16, d - 1)
        Wr[:, 1:1 + nz] = torch.randint(-1, 2, (m, nz), generator=g, device=device).to(torch.float32)
        Wr[:, 0] = torch.randint(-2, 3, (m,), generator=g, device=device).to(torch.float32)
    else:
        x = (torch.randn(T, d, generator=g, device=device) * 8.0).round().clamp(-32, 31) / 8.0
        x[:, 0] = 1.0
        Wr = (torch.randn(m, d, generator=g, device=device) * (1.0 / d) ** 0.5 * 1024.0).round().clamp(-255, 255)
        Wr[:, 0] = (torch.randn(m, generator=g, device=device) * cfg.sigma * 1024.0).round().clamp(-2047, 2047)
        Wr = Wr / 1024.0
    return x.to(dt), Wr.to(dt)


def exactness_bound(x: torch.Tensor, Wr: torch.Tensor) -> float:
    """max over (t, e) of sum_j |x_tj| |Wr_ej| (fp64) - with products on the
    2^-13 grid, partial sums below 2^11 carry at most 24 significant bits."""
    return float((x.double().abs() @ Wr.double().abs().T).max()) if x.numel() else 0.0
