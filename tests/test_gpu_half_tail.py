"""GEMM2's half-width last wave (GemmParams::half_tail, option half_tail): on CTA pairs,
the X = tiles mod pairs tiles that would form a partial last wave run as two BN/2-column
halves each.  The halves compute disjoint columns with the same k order, so the output
is BITWISE the whole-tile result (Eq. 6 row weights, and the Eq. 5 combine fused into
the epilogue, whose arrival counters then count half-tile columns); and it matches the
fp64 oracle.  Shapes are chosen so that every tile is halved (32 tiles on 74 pairs) or a
partial wave of 22 tiles is (96 tiles)."""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu
C = S.LayerConfig
CFGS = [
    C("half_all", d=512, f=256, m=8, K=2, way=4, T=1500, ratio=0.5, dtype="bf16", sigma=0.5, config_id=95),
    C("half_partial_wave", d=512, f=256, m=8, K=2, way=4, T=6000, ratio=0.0, dtype="bf16", sigma=0.3, config_id=96),
    C("half_shared", d=512, f=256, m=8, K=2, way=4, T=2100, ratio=1.0, dtype="bf16", sigma=0.5,
      config_id=97, Ns=1),
]


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _np(t):
    return t.detach().cpu().double().numpy()


def _run(cfg, env, monkeypatch):
    from paper_2507_17133_b200 import BrownoutMoE
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=4)
    L = S.make_logits(cfg.T, cfg.m, seed=4, sigma=cfg.sigma)
    res = False
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T, num_shared=cfg.Ns,
                      add_residual=res)
    moe.set_brownout(cfg.ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    sh = (g["SWg"], g["SWu"], g["SWd"]) if cfg.Ns else None
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]), logits=L.cuda(),
                    shared=sh)
    torch.cuda.synchronize()
    return y.clone(), moe, lay, uni, x, L, res


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
def test_half_tail_bitwise_and_oracle(cfg, monkeypatch):
    y1, moe, lay, uni, x, L, res = _run(cfg, {}, monkeypatch)
    assert "gemm2_weighted_combine" in moe.last_kernels() or cfg.Ns, moe.last_kernels()
    y0, _, _, _, _, _, _ = _run(cfg, {"BO_HALF_TAIL": "0"}, monkeypatch)
    assert torch.equal(y1, y0), "half tiles must reproduce the whole-tile result bit for bit"
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    sh = tuple(_np(lay[k]) for k in ("SWg", "SWu", "SWd")) if cfg.Ns else None
    ref = O.moe_forward(_np(x), None, ex, un, cfg.K, cfg.way, cfg.ratio, logits=L.double().numpy(),
                        add_residual=res, shared=sh)
    yr, yg = ref.y, _np(y1)
    den = np.where(np.abs(yr).max(1) == 0, 1.0, np.abs(yr).max(1))
    assert (np.abs(yg - yr).max(1) / den).max() <= 2e-2
