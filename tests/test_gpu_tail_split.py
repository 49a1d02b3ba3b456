"""GEMM2's last-wave split (GemmParams::tail_split, option tail_split): on CTA pairs,
the tiles of a partial last wave are shared out by k-blocks over every pair; a tile's
finishing pair (the one owning its first k-block) adds the fp32 partials of the pairs
holding its other pieces, in unit order, before the Eq. 6 row weights and the Eq. 5
combine fused into the epilogue.  Only the fp32 summation order of Eq. 5's FFN
contraction changes, so outputs are compared with the fp64 oracle at the 2e-2
bar (on sampled tokens) and with the unsplit schedule at 1e-2; routing, plan and
permutation stay bit-exact.  Shapes: every tile split (48 tiles on 74 pairs, a tile
spread over 2-3 pairs) and a split partial wave after one whole tile per pair (96 tiles)."""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu
C = S.LayerConfig
CFGS = [
    C("ts_all_split", d=512, f=4096, m=8, K=2, way=4, T=3000, ratio=0.0, dtype="bf16", sigma=0.3, config_id=101),
    C("ts_partial_wave", d=1024, f=4096, m=8, K=2, way=4, T=3000, ratio=0.0, dtype="bf16", sigma=0.3,
      config_id=102),
    C("ts_united", d=512, f=4096, m=8, K=2, way=4, T=2600, ratio=0.5, dtype="bf16", sigma=0.6, config_id=103),
]
N_SAMPLE = 256


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
    x = S.make_tokens(cfg, batch_index=6)
    L = S.make_logits(cfg.T, cfg.m, seed=6, sigma=cfg.sigma)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T)
    moe.set_brownout(cfg.ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]), logits=L.cuda())
    torch.cuda.synchronize()
    return y.clone(), moe, lay, uni, x, L


def _rel(y, ref):
    den = np.where(np.abs(ref).max(1) == 0, 1.0, np.abs(ref).max(1))
    return (np.abs(y - ref).max(1) / den).max()


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
def test_tail_split_matches_oracle_and_unsplit(cfg, monkeypatch):
    y1, moe, lay, uni, x, L = _run(cfg, {}, monkeypatch)
    assert "gemm2_weighted_combine" in moe.last_kernels(), moe.last_kernels()
    dbg = moe.debug_arrays(cfg.T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    toks = np.sort(np.random.default_rng(cfg.config_id).choice(cfg.T, size=N_SAMPLE, replace=False))
    ref = O.moe_forward(_np(x), None, ex, un, cfg.K, cfg.way, cfg.ratio, logits=L.double().numpy(), tokens=toks)
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    assert np.array_equal(dbg["row_of"].cpu().numpy(), ref.perm.row_of)
    assert _rel(_np(y1)[toks], ref.y) <= 2e-2
    y0, _, _, _, _, _ = _run(cfg, {"BO_TAIL_SPLIT": "0"}, monkeypatch)
    assert _rel(_np(y1), _np(y0)) <= 1e-2
