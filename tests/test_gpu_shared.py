"""GPU parity of the shared-expert term of Eq. 5:
h_t = sum_{i<=N_s} FFN_i^(s)(x_t) + sum p FFN^(r) + sum q FFN^(u).

The N_s shared experts run as a third executor class of the same grouped
GEMMs (rows appended after the m + G routed executors, every token, weight 1).
Checked against the fp64 oracle (oracle.moe_forward(shared=...)):
  * routed arrays bit-exact as in test_gpu_parity (injected fp32 logits);
  * the shared executors' offsets and row_of columns bit-exact against their
    definition (executor m + G + j holds tokens 0..T-1 in order);
  * outputs within 2e-2 relative error, in every engine variant.
"""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu

OUT_TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _np(t):
    return t.detach().cpu().double().numpy()


def _rel_err(y, ref):
    den = np.abs(ref).max(axis=1)
    den = np.where(den == 0, 1.0, den)
    return float((np.abs(y - ref).max(axis=1) / den).max())


CFGS = [
    S.LayerConfig("sh_small_bf16", d=256, f=512, m=8, K=2, way=4, T=300, ratio=0.5, dtype="bf16", sigma=0.7,
                  config_id=41, Ns=2),
    # the paper's 60 experts with the ragged 8th group (way 8), 4 shared experts of 1408
    S.LayerConfig("sh_qwen15_shape", d=256, f=1408, m=60, K=4, way=8, T=200, ratio=0.6, dtype="bf16", sigma=0.5,
                  config_id=42, Ns=4),
    S.LayerConfig("sh_tiny_fp32", d=64, f=128, m=8, K=2, way=4, T=32, ratio=0.5, dtype="fp32", sigma=0.0,
                  config_id=43, Ns=1),
    # R + N_s T >= 2048: 256-row CTA-pair tiles
    S.LayerConfig("sh_pairs_bf16", d=256, f=512, m=8, K=2, way=4, T=700, ratio=0.5, dtype="bf16", sigma=0.5,
                  config_id=44, Ns=2),
]


def _run(cfg, ratio, mode="partial", seed=0, T=None):
    from paper_2507_17133_b200 import BrownoutMoE
    T = cfg.T if T is None else T
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=seed, T=T)
    L = S.make_logits(T, cfg.m, seed=seed, sigma=cfg.sigma)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=max(T, 1),
                      num_shared=cfg.Ns)
    moe.set_brownout(ratio, mode)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    y = moe.forward(x.cuda(), g["Wr"], (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]),
                    logits=L.cuda(), shared=(g["SWg"], g["SWu"], g["SWd"]))
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    sh = tuple(_np(lay[k]) for k in ("SWg", "SWu", "SWd"))
    ref = O.moe_forward(_np(x), None, ex, un, cfg.K, cfg.way, ratio, mode, logits=L.double().numpy(), shared=sh)
    return y, dbg, ref


def _check_indices(cfg, dbg, ref, T):
    K, Ns, E = cfg.K, cfg.Ns, cfg.m + cfg.G
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    eo = dbg["exec_off"].cpu().numpy()
    assert len(eo) == E + Ns + 1
    assert np.array_equal(eo[:E + 1], ref.perm.exec_off)
    R = int(ref.perm.exec_off[-1])
    assert np.array_equal(eo[E:], R + T * np.arange(Ns + 1))
    ro = dbg["row_of"].cpu().numpy().reshape(T, K + Ns)
    assert np.array_equal(ro[:, :K].reshape(-1), ref.perm.row_of)
    for j in range(Ns):
        assert np.array_equal(ro[:, K + j], R + j * T + np.arange(T))
    Rt = R + Ns * T
    assert np.array_equal(dbg["row_tok"][:R].cpu().numpy(), ref.perm.row_tok)
    assert np.array_equal(dbg["row_tok"][R:Rt].cpu().numpy(), np.tile(np.arange(T), Ns))
    assert (dbg["row_w"][R:Rt].cpu().numpy() == 1.0).all()
    st = dbg["stats"].cpu().numpy()   # Alg. 1 statistics count routed rows only
    s = ref.plan.stats
    assert list(st[:7]) == [s["executors_accessed"], s["n_s1"], s["n_united"], s["n_singleton"],
                            s["rows_original"], s["rows_united"], s["rows_dropped"]]
    assert st[7] == T * K


@pytest.mark.parametrize("cfg", CFGS, ids=lambda c: c.name)
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_shared_experts_match_oracle(cfg, ratio):
    y, dbg, ref = _run(cfg, ratio, seed=3)
    _check_indices(cfg, dbg, ref, cfg.T)
    assert _rel_err(_np(y), ref.y) <= OUT_TOL


@pytest.mark.parametrize("cfg", CFGS[:2], ids=lambda c: c.name)
def test_shared_experts_full_brownout_keep_shared_term(cfg):
    """Full brownout at ratio 1 drops every routed slot: only Eq. 5's shared
    term remains, and it must still be there."""
    y, dbg, ref = _run(cfg, 1.0, mode="full", seed=4)
    _check_indices(cfg, dbg, ref, cfg.T)
    assert np.abs(ref.y).max() > 0
    assert _rel_err(_np(y), ref.y) <= OUT_TOL


@pytest.mark.parametrize("T", [1, 7, 129])
def test_shared_experts_ragged_T(T):
    cfg = CFGS[0]
    y, dbg, ref = _run(cfg, 0.5, seed=T, T=T)
    _check_indices(cfg, dbg, ref, T)
    assert _rel_err(_np(y), ref.y) <= OUT_TOL


@pytest.mark.parametrize("env", [{"BO_CTA_PAIRS": "0"}, {"BO_GEMM2_SPLITK": "1"}, {"BO_TILE_ALT": "0"}],
                         ids=["single_cta_gemm", "splitk_gemm2", "no_tile_alt"])
@pytest.mark.parametrize("cfg", [CFGS[0], CFGS[3]], ids=lambda c: c.name)
def test_shared_experts_engine_variants(cfg, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    y, dbg, ref = _run(cfg, 0.5, seed=8)
    _check_indices(cfg, dbg, ref, cfg.T)
    assert _rel_err(_np(y), ref.y) <= OUT_TOL


def test_shared_experts_required_and_ep_entries_refuse():
    """A handle created with N_s > 0 refuses to run without shared weights, and
    the expert-parallel dispatch entry reports BO_ERR_UNSUPPORTED."""
    from paper_2507_17133_b200 import BrownoutMoE
    from paper_2507_17133_b200.brownout import BrownoutError
    cfg = CFGS[0]
    lay = {k: v.cuda() for k, v in S.make_layer(cfg).items()}
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T, num_shared=cfg.Ns)
    x = S.make_tokens(cfg).cuda()
    with pytest.raises(BrownoutError):
        moe.forward(x, lay["Wr"], (lay["Wg"], lay["Wu"], lay["Wd"]), None)
