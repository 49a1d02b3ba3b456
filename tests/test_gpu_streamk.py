"""Stream-K decode GEMM1 (GemmParams::streamk): when the plan's CTA-pair
tiles outnumber the pairs, every pair takes an equal share of the (tile, k-block)
sequence and a tile cut in two is finished by the pair that owns its first k-block,
after adding the next pair's fp32 partial.  The split changes only the fp32 summation
order of Eq. 5's FFN contraction, so outputs are compared with the fp64 oracle
at the same 2e-2 bar; routing, plan and permutation stay bit-exact (injected logits)."""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu
OUT_TOL = 2e-2

C = S.LayerConfig
# decode-sized (T * K <= 1024 rows) with enough pair tiles to cut: f / 128 n-tiles per executor
CFGS = [
    C("sk_d512_f4096", d=512, f=4096, m=8, K=2, way=4, T=400, ratio=0.5, dtype="bf16", sigma=0.5, config_id=81),
    C("sk_d256_f8192_w2", d=256, f=8192, m=8, K=2, way=2, T=300, ratio=0.5, dtype="bf16", sigma=0.7, config_id=82),
    C("sk_m16_k3", d=384, f=3072, m=16, K=3, way=4, T=330, ratio=0.5, dtype="bf16", sigma=0.5, config_id=83),
]


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _np(t):
    return t.detach().cpu().double().numpy()


def _run(cfg, ratio, env, monkeypatch, seed=3):
    from paper_2507_17133_b200 import BrownoutMoE
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=seed)
    L = S.make_logits(cfg.T, cfg.m, seed=seed, sigma=cfg.sigma)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T)
    moe.set_brownout(ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]), logits=L.cuda())
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(cfg.T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    ref = O.moe_forward(_np(x), None, ex, un, cfg.K, cfg.way, ratio, logits=L.double().numpy())
    return y, dbg, ref


def _rel(y, ref):
    den = np.abs(ref).max(1)
    den = np.where(den == 0, 1.0, den)
    return (np.abs(y - ref).max(1) / den).max()


@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
def test_streamk_decode_gemm1_matches_oracle(cfg, ratio, monkeypatch):
    y, dbg, ref = _run(cfg, ratio, {}, monkeypatch)
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    assert np.array_equal(dbg["row_of"].cpu().numpy(), ref.perm.row_of)
    assert _rel(_np(y), ref.y) <= OUT_TOL
    # the tiles outnumber the pairs here, so the kernel really cut tiles: contributors counted 4 warps
    flags = dbg["sk_flag"].cpu().numpy()
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    assert set(np.unique(flags[:n_sm])) <= {0, 4}
    assert (flags[:n_sm] == 4).any(), "stream-K did not cut any tile"


@pytest.mark.parametrize("cfg", CFGS[:1], ids=lambda c: c.name)
def test_streamk_off_and_on_agree_to_fp32_order(cfg, monkeypatch):
    """BO_DECODE_STREAMK=0 (whole tiles) and the stream-K schedule differ only in fp32
    summation order: H and y agree far inside the oracle tolerance."""
    y1, d1, ref = _run(cfg, 1.0, {}, monkeypatch)
    h1 = d1["h"].clone()
    y0, d0, _ = _run(cfg, 1.0, {"BO_DECODE_STREAMK": "0"}, monkeypatch)
    assert _rel(_np(y0), ref.y) <= OUT_TOL
    R = int(ref.perm.exec_off[-1])
    hd = (h1[:R].float() - d0["h"][:R].float()).abs().max().item()
    assert hd <= 2e-2 * max(1.0, d0["h"][:R].float().abs().max().item())
    assert _rel(_np(y1), _np(y0)) <= 1e-2
