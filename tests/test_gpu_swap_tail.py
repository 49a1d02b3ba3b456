"""Swapped-operand tail tiles of the CTA-pair GEMM1 (default; BO_SWAP_TAIL=0 turns them off).

An executor's last, ragged m-tile (rin < 256 rows) runs as D^T = [Wg; Wu] Xp^T with
the weight rows on the MMA's M side and its rows (rounded up to 32) on N; the
epilogue exchanges gate / up across half-warps.  The layer output must match the
fp64 oracle (Eq. 5-8, Alg. 1) within the same tolerance as the default path, for
every executor class (originals, united, shared) and for tail sizes below 32,
between 32 and 128, and above 128.
"""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu

OUT_TOL = 2e-2


def _np(t):
    return t.detach().cpu().double().numpy()


def _rel_err(y, ref):
    den = np.abs(ref).max(axis=1)
    den = np.where(den == 0, 1.0, den)
    return float((np.abs(y - ref).max(axis=1) / den).max())


def _run(cfg, ratio, mode="partial", seed=3, T=None, add_residual=False):
    from paper_2507_17133_b200 import BrownoutMoE
    T = cfg.T if T is None else T
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=seed, T=T)
    L = S.make_logits(T, cfg.m, seed=seed, sigma=cfg.sigma)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=T,
                      num_shared=cfg.Ns, add_residual=add_residual)
    moe.set_brownout(ratio, mode)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    shared = (g["SWg"], g["SWu"], g["SWd"]) if cfg.Ns else None
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]),
                    logits=L.cuda(), shared=shared)
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    sh = tuple(_np(lay[k]) for k in ("SWg", "SWu", "SWd")) if cfg.Ns else None
    ref = O.moe_forward(_np(x), None, ex, un, cfg.K, cfg.way, ratio, mode, logits=L.double().numpy(),
                        shared=sh, add_residual=add_residual)
    return y, dbg, ref


CFGS = [
    S.LayerConfig("sw_m8", d=256, f=512, m=8, K=2, way=4, T=1500, ratio=0.5, dtype="bf16", sigma=0.5,
                  config_id=51),
    S.LayerConfig("sw_m64_k4", d=384, f=256, m=64, K=4, way=4, T=700, ratio=0.5, dtype="bf16", sigma=0.8,
                  config_id=52),
    S.LayerConfig("sw_shared", d=256, f=384, m=8, K=2, way=4, T=611, ratio=0.5, dtype="bf16", sigma=0.5,
                  config_id=53, Ns=2),
]


@pytest.mark.parametrize("fc", ["auto", "1", "0"])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
def test_swap_tail_matches_oracle(cfg, ratio, fc, monkeypatch):
    """GEMM1 on CTA pairs with swapped tail tiles; GEMM2's fused combine on / off."""
    monkeypatch.setenv("BO_SWAP_TAIL", "1")
    monkeypatch.setenv("BO_PAIR_ROWS1", "1")
    monkeypatch.setenv("BO_PAIR_ROWS2", "1")
    if fc != "auto":
        monkeypatch.setenv("BO_FUSED_COMBINE", fc)
    y, dbg, ref = _run(cfg, ratio)
    rows = np.diff(dbg["exec_off"].cpu().numpy().astype(np.int64))
    tails = rows[rows > 0] % 256
    assert (tails > 0).any()          # the case exercises swapped tiles
    assert _rel_err(_np(y), ref.y) <= OUT_TOL


@pytest.mark.parametrize("T", [1, 5, 17, 40, 100, 129, 200, 255, 256, 257, 700])
def test_swap_tail_sizes(T, monkeypatch):
    """One expert (m = 1): the executor's rows are exactly T, so the tail is T % 256."""
    monkeypatch.setenv("BO_SWAP_TAIL", "1")
    monkeypatch.setenv("BO_PAIR_ROWS1", "1")
    monkeypatch.setenv("BO_PAIR_ROWS2", "1")
    monkeypatch.setenv("BO_FUSED_COMBINE", "1")
    cfg = S.LayerConfig("sw_one", d=256, f=256, m=1, K=1, way=1, T=T, ratio=0.0, dtype="bf16", sigma=0.0,
                        config_id=54)
    y, _, ref = _run(cfg, 0.0, add_residual=True)
    assert _rel_err(_np(y), ref.y) <= OUT_TOL


def test_swap_tail_same_as_default(monkeypatch):
    """Swapped and default tiles compute the same H up to fp32 summation order."""
    cfg = CFGS[0]
    monkeypatch.setenv("BO_PAIR_ROWS1", "1")
    monkeypatch.setenv("BO_PAIR_ROWS2", "1")
    monkeypatch.setenv("BO_SWAP_TAIL", "0")
    y0, _, _ = _run(cfg, 0.5)
    monkeypatch.setenv("BO_SWAP_TAIL", "1")
    y1, _, ref = _run(cfg, 0.5)
    a, b = _np(y0), _np(y1)
    assert _rel_err(b, a) <= 1e-2


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
def test_swap_tail_fused_combine_bitwise(cfg, monkeypatch):
    """After swapped GEMM1 tail tiles the fused combine still sums each token's Yp
    rows in slot order: bitwise the separate k_combine."""
    monkeypatch.setenv("BO_SWAP_TAIL", "1")
    monkeypatch.setenv("BO_PAIR_ROWS1", "1")
    monkeypatch.setenv("BO_PAIR_ROWS2", "1")
    monkeypatch.setenv("BO_FUSED_COMBINE", "1")
    y1, _, _ = _run(cfg, 0.5, add_residual=True)
    monkeypatch.setenv("BO_FUSED_COMBINE", "0")
    y0, _, _ = _run(cfg, 0.5, add_residual=True)
    assert torch.equal(y0.cpu(), y1.cpu())
