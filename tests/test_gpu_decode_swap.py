"""Decode instantiation of the FFN GEMMs (GemmParams::swap_all, option decode_swap;
DESIGN.md §5): for decode-sized steps every executor whose rows fit (<= 288) is ONE
swapped CTA-pair tile — its weight rows on the MMA's M side, all of its rows on N
(a second MMA past 256 rows, a single-buffered accumulator then), GEMM1 with the
SwiGLU epilogue, GEMM2 with the Eq. 6 row weights and split-K partials.  Executors
past 288 rows fall back to the ordinary pair tiles in the same launch.

Executor sizes are set exactly with one-hot logits (K = 1, synthetic.make_logits_with_counts)
so the 256-row boundary (one MMA, double buffer) and the two-MMA / single-buffer path
(257..288 rows) and the fallback (> 288) are each hit; routing, plan and permutation
stay bit-exact vs the oracle (Alg. 1) and y is within the 2e-2 bar (Eq. 5)."""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu
OUT_TOL = 2e-2
C = S.LayerConfig


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _np(t):
    return t.detach().cpu().double().numpy()


def _rel(y, ref):
    den = np.abs(ref).max(1)
    den = np.where(den == 0, 1.0, den)
    return (np.abs(y - ref).max(1) / den).max()


def _run(cfg, L, ratio, env, monkeypatch, seed=7):
    from paper_2507_17133_b200 import BrownoutMoE
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    T = L.shape[0]
    lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=seed, T=T)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=T)
    moe.set_brownout(ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]), logits=L.cuda())
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    ref = O.moe_forward(_np(x), None, ex, un, cfg.K, cfg.way, ratio, logits=L.double().numpy())
    return y, dbg, ref


def _check(y, dbg, ref):
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    assert np.array_equal(dbg["exec_off"].cpu().numpy(), ref.perm.exec_off)
    assert np.array_equal(dbg["row_of"].cpu().numpy(), ref.perm.row_of)
    assert _rel(_np(y), ref.y) <= OUT_TOL


CFG = C("dec_swap", d=512, f=1024, m=8, K=1, way=4, T=512, ratio=1.0, dtype="bf16", sigma=0.5, config_id=91)
# per-expert counts (K = 1): at ratio 1 the two united executors hold sum(counts[0:4]) / sum(counts[4:8]) rows
COUNTS = {
    "united_271_241": [70, 70, 70, 61, 60, 60, 60, 61],    # C3-like: one tile past 256 rows (two MMAs)
    "united_256_256": [64] * 8,                              # exactly one MMA each, double buffer
    "united_288_224": [72, 72, 72, 72, 56, 56, 56, 56],    # the widest single pass (2 x 144 rows)
    "united_289_223": [73, 72, 72, 72, 56, 56, 56, 55],    # past 288: the launch falls back to pair tiles
    "united_17_495": [5, 4, 4, 4, 124, 124, 124, 123],     # tiny and fallback-sized executors together
}


@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("name", list(COUNTS), ids=list(COUNTS))
def test_decode_swap_tiles_match_oracle(name, ratio, monkeypatch):
    L = S.make_logits_with_counts(COUNTS[name], K=1, seed=3)
    y, dbg, ref = _run(CFG, L, ratio, {}, monkeypatch)
    _check(y, dbg, ref)


@pytest.mark.parametrize("cfg", [
    C("dec_k2_mixtral_like", d=512, f=2048, m=8, K=2, way=4, T=256, ratio=1.0, dtype="bf16", sigma=0.5, config_id=92),
    C("dec_k3_m16", d=384, f=768, m=16, K=3, way=4, T=200, ratio=0.5, dtype="bf16", sigma=0.7, config_id=93),
    C("dec_k2_ragged_way3", d=256, f=1536, m=11, K=2, way=3, T=333, ratio=0.7, dtype="bf16", sigma=0.5, config_id=94),
], ids=lambda c: c.name)
def test_decode_swap_random_routing(cfg, monkeypatch):
    L = S.make_logits(cfg.T, cfg.m, seed=11, sigma=cfg.sigma)
    y, dbg, ref = _run(cfg, L, cfg.ratio, {}, monkeypatch)
    _check(y, dbg, ref)


def test_decode_swap_off_agrees(monkeypatch):
    """BO_DECODE_SWAP=0 (ordinary pair / single-CTA tiles) gives the same routing and an
    output equal within fp32 summation-order noise."""
    L = S.make_logits_with_counts(COUNTS["united_271_241"], K=1, seed=3)
    y1, d1, ref = _run(CFG, L, 1.0, {}, monkeypatch)
    y0, d0, _ = _run(CFG, L, 1.0, {"BO_DECODE_SWAP": "0"}, monkeypatch)
    _check(y0, d0, ref)
    assert _rel(_np(y1), _np(y0)) <= 1e-2
