"""TILED weight layout (bo_pack_weights, BO_WEIGHTS_TILED): every 128-row x 128-byte
TMA box of the FFN GEMMs is one contiguous block.  Only the memory layout of the
weights changes, so the forward must equal the ROWMAJOR forward bit for bit (same
MMA operands, same order), at prefill and decode sizes, every ratio and mode, with
shared experts, and in fp32 (tf32) too."""
import numpy as np
import pytest
import torch

import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _moe(cfg, tiled, mode_T=None):
    from paper_2507_17133_b200 import BrownoutMoE
    return BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=mode_T or cfg.T,
                       num_shared=cfg.Ns, tiled=tiled)


@pytest.mark.parametrize("which", [0, 1])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_pack_is_the_documented_relayout(which, dtype):
    cfg = S.LayerConfig("pk", d=256, f=384, m=3, K=2, way=2, T=8, ratio=0.5, dtype=dtype, config_id=61)
    lay = {k: v.cuda() for k, v in S.make_layer(cfg).items()}
    moe = _moe(cfg, True)
    W = lay["Wg"] if which == 0 else lay["Wd"]
    P = moe.pack(W, which)
    torch.cuda.synchronize()
    n, rows, K = W.shape
    kc = 128 // W.element_size()
    want = W.reshape(n, rows // 128, 128, K // kc, kc).permute(0, 1, 3, 2, 4).contiguous().reshape(-1)
    assert torch.equal(P.reshape(-1), want)


CASES = [
    (S.LayerConfig("tiled_decode", d=256, f=512, m=8, K=2, way=4, T=300, ratio=0.5, dtype="bf16", sigma=0.7,
                   config_id=62), (0.0, 0.5, 1.0)),
    (S.LayerConfig("tiled_prefill_pairs", d=512, f=512, m=8, K=2, way=4, T=1500, ratio=0.5, dtype="bf16",
                   sigma=0.5, config_id=63), (0.0, 0.5, 1.0)),
    (S.LayerConfig("tiled_qwen_like", d=256, f=256, m=128, K=8, way=4, T=390, ratio=0.5, dtype="bf16",
                   sigma=0.5, config_id=64), (0.5,)),
    (S.LayerConfig("tiled_shared", d=256, f=384, m=8, K=2, way=4, T=333, ratio=0.5, dtype="bf16", sigma=0.5,
                   config_id=65, Ns=2), (0.5, 1.0)),
    (S.LayerConfig("tiled_fp32", d=128, f=256, m=8, K=2, way=4, T=64, ratio=0.5, dtype="fp32", sigma=0.0,
                   config_id=66), (0.5,)),
    (S.LayerConfig("tiled_decode_many_rows", d=256, f=512, m=8, K=2, way=4, T=500, ratio=1.0, dtype="bf16",
                   sigma=0.5, config_id=67), (1.0,)),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].name)
@pytest.mark.parametrize("mode", ["partial", "full"])
def test_tiled_forward_bitwise_equals_rowmajor(case, mode):
    cfg, ratios = case
    lay = {k: v.cuda() for k, v in S.make_layer(cfg).items()}
    x = S.make_tokens(cfg, batch_index=4).cuda()
    L = S.make_logits(cfg.T, cfg.m, seed=4, sigma=cfg.sigma).cuda()
    row = _moe(cfg, False)
    til = _moe(cfg, True)
    U = row.build_united(lay["Wg"], lay["Wu"], lay["Wd"])
    ex_t = til.pack_all(lay["Wg"], lay["Wu"], lay["Wd"])
    U_t = til.build_united(*ex_t)                 # element-wise mean: works on the packed stacks
    U_p = til.pack_all(*U)
    sh = (lay["SWg"], lay["SWu"], lay["SWd"]) if cfg.Ns else None
    sh_t = til.pack_all(*sh) if cfg.Ns else None
    torch.cuda.synchronize()
    for a, b in zip(U_t, U_p):
        assert torch.equal(a, b)                   # united init commutes with the packing
    for r in ratios:
        row.set_brownout(r, mode)
        til.set_brownout(r, mode)
        y0 = row.forward(x, lay["Wr"], (lay["Wg"], lay["Wu"], lay["Wd"]), U, logits=L, shared=sh)
        y1 = til.forward(x, lay["Wr"], ex_t, U_t, logits=L, shared=sh_t)
        torch.cuda.synchronize()
        assert torch.equal(y0, y1), (r, mode)


def test_tiled_layout_rejects_unaligned_shapes():
    from paper_2507_17133_b200 import BrownoutMoE
    from paper_2507_17133_b200.brownout import BrownoutError
    with pytest.raises(BrownoutError):
        BrownoutMoE(192, 256, 8, 2, 4, tiled=True)      # hidden not a multiple of 128
