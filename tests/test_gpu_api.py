"""GPU behaviour of the C ABI beyond numerics (include/brownout.h):
residual term of Eq. 5, CUDA-graph capture of the forward, argument / workspace
errors reported as status codes, and independence of handles and streams."""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu

CFG = S.LayerConfig("api_small", d=256, f=512, m=8, K=2, way=4, T=300, ratio=0.5, dtype="bf16", sigma=0.7,
                    config_id=61)


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _np(t):
    return t.detach().cpu().double().numpy()


def _layer(cfg=CFG):
    lay = {k: v.cuda() for k, v in S.make_layer(cfg).items()}
    uni = {k: v.cuda() for k, v in S.make_united_random(cfg).items()}
    return lay, (uni["UWg"], uni["UWu"], uni["UWd"])


def _rel(y, ref):
    den = np.abs(ref).max(axis=1)
    return float((np.abs(y - ref).max(axis=1) / np.where(den == 0, 1, den)).max())


def test_residual_term_of_eq5():
    """add_residual = 1 adds x_t (Eq. 5 first term, reading D12): y_res - y = x
    up to the bf16 rounding of each output."""
    from paper_2507_17133_b200 import BrownoutMoE
    lay, U = _layer()
    x = S.make_tokens(CFG).cuda()
    L = S.make_logits(CFG.T, CFG.m, seed=2, sigma=CFG.sigma).cuda()
    W = (lay["Wg"], lay["Wu"], lay["Wd"])
    outs = []
    for res in (False, True):
        moe = BrownoutMoE(CFG.d, CFG.f, CFG.m, CFG.K, CFG.way, add_residual=res, max_tokens=CFG.T)
        moe.set_brownout(0.5)
        outs.append(moe.forward(x, lay["Wr"], W, U, logits=L).double())
    xu = S.make_tokens(CFG)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(u) for u in U)
    ref = O.moe_forward(_np(xu), None, ex, un, CFG.K, CFG.way, 0.5, logits=_np(L), add_residual=True)
    assert _rel(_np(outs[1]), ref.y) <= 2e-2
    d = (outs[1] - outs[0]).cpu().numpy() - _np(x)
    assert np.abs(d).max() <= 2 ** -7 * (np.abs(_np(outs[1])).max() + 1)


def test_forward_is_cuda_graph_capturable_and_replays_new_inputs():
    """No host synchronisation inside the forward: a captured graph replays with
    fresh token contents in the captured buffer and matches the eager result."""
    from paper_2507_17133_b200 import BrownoutMoE
    lay, U = _layer()
    W = (lay["Wg"], lay["Wu"], lay["Wd"])
    moe = BrownoutMoE(CFG.d, CFG.f, CFG.m, CFG.K, CFG.way, max_tokens=CFG.T)
    moe.set_brownout(0.5)
    x = S.make_tokens(CFG, batch_index=1).cuda()
    y = torch.empty_like(x)
    ws = moe.workspace(CFG.T)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        moe.forward(x, lay["Wr"], W, U, y=y, workspace=ws)      # warm-up on the capture stream
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        moe.forward(x, lay["Wr"], W, U, y=y, workspace=ws)
    for b in (2, 3):
        x.copy_(S.make_tokens(CFG, batch_index=b).cuda())
        g.replay()
        torch.cuda.synchronize()
        got = y.clone()
        want = moe.forward(x.clone(), lay["Wr"], W, U)
        torch.cuda.synchronize()
        assert torch.equal(got, want)


def test_knob_changes_take_effect_per_call():
    """bo_set_brownout is snapshotted at enqueue: alternating ratios on one handle
    give each call its own plan (Alg. 1 on the same batch)."""
    from paper_2507_17133_b200 import BrownoutMoE
    lay, U = _layer()
    W = (lay["Wg"], lay["Wu"], lay["Wd"])
    moe = BrownoutMoE(CFG.d, CFG.f, CFG.m, CFG.K, CFG.way, max_tokens=CFG.T)
    x = S.make_tokens(CFG).cuda()
    L = S.make_logits(CFG.T, CFG.m, seed=5, sigma=CFG.sigma).cuda()
    res = {}
    for r in (0.0, 1.0, 0.0, 1.0):
        moe.set_brownout(r)
        y = moe.forward(x, lay["Wr"], W, U, logits=L)
        torch.cuda.synchronize()
        st = moe.debug_arrays(CFG.T)["stats"].cpu().tolist()
        if r in res:
            assert torch.equal(res[r][0], y) and res[r][1] == st
        else:
            res[r] = (y.clone(), st)
    assert res[0.0][1][5] == 0 and res[1.0][1][5] > 0      # united rows: none at ratio 0, some at ratio 1


def test_two_handles_on_two_streams_are_independent():
    from paper_2507_17133_b200 import BrownoutMoE
    cfg2 = S.LayerConfig("api_other", d=128, f=256, m=16, K=4, way=2, T=200, ratio=0.25, dtype="bf16", sigma=0.5,
                         config_id=62)
    lay1, U1 = _layer(CFG)
    lay2, U2 = _layer(cfg2)
    m1 = BrownoutMoE(CFG.d, CFG.f, CFG.m, CFG.K, CFG.way, max_tokens=CFG.T)
    m2 = BrownoutMoE(cfg2.d, cfg2.f, cfg2.m, cfg2.K, cfg2.way, max_tokens=cfg2.T)
    m1.set_brownout(0.5)
    m2.set_brownout(0.25)
    x1, x2 = S.make_tokens(CFG).cuda(), S.make_tokens(cfg2).cuda()
    ref1 = m1.forward(x1, lay1["Wr"], (lay1["Wg"], lay1["Wu"], lay1["Wd"]), U1).clone()
    ref2 = m2.forward(x2, lay2["Wr"], (lay2["Wg"], lay2["Wu"], lay2["Wd"]), U2).clone()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    w1 = torch.empty(m1.workspace_size(CFG.T), dtype=torch.uint8, device="cuda")
    w2 = torch.empty(m2.workspace_size(cfg2.T), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        with torch.cuda.stream(s1):
            y1 = m1.forward(x1, lay1["Wr"], (lay1["Wg"], lay1["Wu"], lay1["Wd"]), U1, workspace=w1, stream=s1)
        with torch.cuda.stream(s2):
            y2 = m2.forward(x2, lay2["Wr"], (lay2["Wg"], lay2["Wu"], lay2["Wd"]), U2, workspace=w2, stream=s2)
        torch.cuda.synchronize()
        assert torch.equal(y1, ref1) and torch.equal(y2, ref2)


def test_errors_are_status_codes():
    from paper_2507_17133_b200 import BrownoutMoE, BrownoutError
    from paper_2507_17133_b200.brownout import BO_ERR_INVALID_ARG, BO_ERR_SHAPE, BO_ERR_WORKSPACE
    lay, U = _layer()
    W = (lay["Wg"], lay["Wu"], lay["Wd"])
    moe = BrownoutMoE(CFG.d, CFG.f, CFG.m, CFG.K, CFG.way, max_tokens=CFG.T)
    moe.set_brownout(0.5)
    x = S.make_tokens(CFG).cuda()
    with pytest.raises(BrownoutError) as e:       # workspace too small
        moe.forward(x, lay["Wr"], W, U, workspace=torch.empty(1024, dtype=torch.uint8, device="cuda"))
    assert e.value.status == BO_ERR_WORKSPACE
    with pytest.raises(BrownoutError) as e:       # T > max_tokens
        moe.forward(torch.cat([x, x]), lay["Wr"], W, U)
    assert e.value.status == BO_ERR_INVALID_ARG
    with pytest.raises(BrownoutError) as e:       # misaligned token pointer
        xb = torch.empty(CFG.T * CFG.d + 1, dtype=torch.bfloat16, device="cuda")[1:].view(CFG.T, CFG.d)
        moe.forward(xb, lay["Wr"], W, U)
    assert e.value.status == BO_ERR_SHAPE
    with pytest.raises(BrownoutError) as e:       # ratio > 0 without united experts
        moe.forward(x, lay["Wr"], W, None)
    assert e.value.status == BO_ERR_INVALID_ARG
    with pytest.raises(BrownoutError):
        moe.set_brownout(1.5)
    # ratio 0 needs no united experts; full mode at ratio 1 drops every routed slot
    moe.set_brownout(0.0)
    moe.forward(x, lay["Wr"], W, None)
    moe.set_brownout(1.0, "full")
    y = moe.forward(x, lay["Wr"], W, U)
    torch.cuda.synchronize()
    assert float(y.float().abs().max()) == 0.0
