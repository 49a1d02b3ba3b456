"""Routing parity through EVERY router kernel with no clear-margin filter.

The inputs are drawn so that Eq. 8 is exact in fp32 / tf32 arithmetic
in any summation order (synthetic.make_exact_router_inputs): the GPU router's
logits must then equal the oracle's fp64 logits bit for bit, and everything
downstream is compared against the oracle's OWN fp64 path (Eq. 8 -> Eq. 7 ->
Alg. 1 -> Eq. 5-6, oracle.moe_forward with logits=None), with nothing taken
from the CUDA path:

  * logits                         exact (fp32 == fp64)
  * topk_id, in slot order         bit-exact (Eq. 7; ties -> lower id, D8)
  * topk_w                         |dg| <= 1e-6
  * counts, plan, permutation      bit-exact (Alg. 1)
  * y (residual off)               max row-relative error <= 2e-2

"integer" inputs make exact ties between experts frequent (the tie rule is
exercised on every path); "dyadic" inputs look like the seeded N(0, 1) recipe
on a 2^-3 / 2^-10 grid.  Router kernels: k_router_mma (bf16,
m <= 32, T >= 8 x #SM), k_router_split (m <= 32, T < 8 x #SM; 1 / 2 / 4 tokens
per CTA), k_router_small (BO_ROUTER_SPLIT=0 BO_ROUTER_MMA=0), and the tcgen05
router with the top-K fused into its epilogue (m > 32, or m <= 32 with Wr too
large for shared memory).
"""
import numpy as np
import pytest
import torch

import synthetic as S
from oracle import brownout_oracle as O

pytestmark = pytest.mark.gpu

OUT_TOL = 2e-2
W_TOL = 1e-6


@pytest.fixture(scope="module", autouse=True)
def _build():
    from paper_2507_17133_b200.build import build
    build()


def _np(t):
    return t.detach().cpu().double().numpy()


def _num_sms():
    return torch.cuda.get_device_properties(0).multi_processor_count


C = S.LayerConfig
# (config, router environment, the kernel that must run)
CASES = [
    (C("m8_mma", d=512, f=128, m=8, K=2, way=4, T=1300, ratio=0.5, dtype="bf16", config_id=61), {}, "mma"),
    (C("m20_k5_mma", d=256, f=128, m=20, K=5, way=4, T=1250, ratio=0.5, dtype="bf16", config_id=62), {}, "mma"),
    (C("m8_split_tpc1", d=512, f=128, m=8, K=2, way=4, T=100, ratio=0.5, dtype="bf16", config_id=63), {}, "split"),
    (C("m8_split_tpc2", d=512, f=128, m=8, K=2, way=4, T=400, ratio=0.5, dtype="bf16", config_id=64), {}, "split"),
    (C("m16_k3_split_tpc4", d=256, f=128, m=16, K=3, way=3, T=700, ratio=0.5, dtype="bf16", config_id=65), {},
     "split"),
    (C("m8_small", d=512, f=128, m=8, K=2, way=4, T=300, ratio=0.5, dtype="bf16", config_id=66),
     {"BO_ROUTER_SPLIT": "0", "BO_ROUTER_MMA": "0"}, "small"),
    (C("m32_k7_small", d=256, f=128, m=32, K=7, way=8, T=1300, ratio=0.5, dtype="bf16", config_id=67),
     {"BO_ROUTER_MMA": "0"}, "small"),
    (C("m8_fp32_small", d=64, f=128, m=8, K=2, way=4, T=32, ratio=0.5, dtype="fp32", config_id=68), {}, "split"),
    # the split-warp router as its own launch (BO_ROUTE_FUSED=0), not inside k_route_fused
    (C("m8_split_tpc1_unfused", d=512, f=128, m=8, K=2, way=4, T=100, ratio=0.5, dtype="bf16", config_id=75),
     {"BO_ROUTE_FUSED": "0"}, "split"),
    (C("m16_k3_split_tpc4_unfused", d=256, f=128, m=16, K=3, way=3, T=700, ratio=0.5, dtype="bf16",
       config_id=76), {"BO_ROUTE_FUSED": "0"}, "split"),
    # k_route_fused with shared experts' rows (Eq. 5 second term) and a ragged last group
    (C("m12_k3_fused_w5", d=256, f=128, m=12, K=3, way=5, T=150, ratio=0.5, dtype="bf16", config_id=77), {},
     "split"),
    (C("m32_tc_bn32", d=3072, f=128, m=32, K=4, way=8, T=200, ratio=0.5, dtype="bf16", config_id=69), {}, "tc"),
    (C("m64_k10_tc", d=256, f=128, m=64, K=10, way=5, T=390, ratio=0.5, dtype="bf16", config_id=70), {}, "tc"),
    (C("m128_k8_tc", d=512, f=128, m=128, K=8, way=4, T=390, ratio=0.5, dtype="bf16", config_id=71), {}, "tc"),
    (C("m128_k8_tc_t300", d=512, f=128, m=128, K=8, way=4, T=300, ratio=0.5, dtype="bf16", config_id=72), {},
     "tc"),
    (C("m256_k16_tc", d=256, f=128, m=256, K=16, way=8, T=260, ratio=0.5, dtype="bf16", config_id=73), {}, "tc"),
    (C("m64_k3_tc_tf32", d=128, f=64, m=64, K=3, way=4, T=150, ratio=0.5, dtype="fp32", config_id=74), {}, "tc"),
]


def _run(cfg, env, monkeypatch, ties, ratio):
    from paper_2507_17133_b200 import BrownoutMoE
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x, Wr = S.make_exact_router_inputs(cfg, ties=ties)
    assert S.exactness_bound(x, Wr) < 2.0 ** 11     # precondition of exact fp32 sums
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T)
    moe.set_brownout(ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    y = moe.forward(x.cuda(), Wr.cuda(), (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]))
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(cfg.T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    ref = O.moe_forward(_np(x), _np(Wr), ex, un, cfg.K, cfg.way, ratio)   # the oracle's own Eq. 8
    return moe, y, dbg, ref


def _expect_kernel(kind, cfg):
    if kind == "mma":
        assert cfg.T >= 8 * _num_sms()
    if kind == "split":
        assert cfg.T < 8 * _num_sms()


@pytest.mark.parametrize("ties", [True, False], ids=["integer", "dyadic"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0].name)
def test_every_router_exact_routing_and_output(case, ties, monkeypatch):
    cfg, env, kind = case
    _expect_kernel(kind, cfg)
    moe, y, dbg, ref = _run(cfg, env, monkeypatch, ties, cfg.ratio)
    # decode-sized split-router steps run a1-a5 in one cooperative launch by default
    fused = kind == "split" and env.get("BO_ROUTE_FUSED") != "0"
    assert moe.last_kernels()[0] == ("route_fused" if fused else "router_topk"), moe.last_kernels()
    st = dbg["stats"].cpu().numpy()
    s = ref.plan.stats
    assert list(st[:7]) == [s["executors_accessed"], s["n_s1"], s["n_united"], s["n_singleton"],
                            s["rows_original"], s["rows_united"], s["rows_dropped"]]
    mt = np.diff(ref.perm.exec_off)
    assert np.array_equal(np.diff(dbg["mtile_off"].cpu().numpy()[:len(mt) + 1]), (mt + 127) // 128)
    Lg = dbg["logits"].cpu().double().numpy()
    assert np.array_equal(Lg, ref.logits), "Eq. 8 not exact on exactly representable inputs"
    if ties:   # the tie rule is really exercised: some token has equal logits around its K-th choice
        Ls = np.sort(ref.logits, axis=1)[:, ::-1]
        k1 = min(cfg.K, cfg.m - 1)
        assert (Ls[:, k1 - 1] == Ls[:, k1]).any()
    ids = dbg["topk_id"].cpu().numpy()
    assert np.array_equal(ids, ref.ids), "ordered top-K ids differ from Eq. 7 (logit desc, id asc)"
    assert np.abs(dbg["topk_w"].cpu().double().numpy() - ref.g).max() <= W_TOL
    assert np.array_equal(dbg["counts"].cpu().numpy(), ref.plan.counts)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    assert np.array_equal(dbg["expert_row_off"].cpu().numpy(), ref.perm.expert_row_off)
    assert np.array_equal(dbg["exec_off"].cpu().numpy(), ref.perm.exec_off)
    assert np.array_equal(dbg["row_of"].cpu().numpy(), ref.perm.row_of)
    R = int(ref.perm.exec_off[-1])
    assert np.array_equal(dbg["row_tok"][:R].cpu().numpy(), ref.perm.row_tok)
    yg, yr = _np(y), ref.y
    den = np.abs(yr).max(1)
    den = np.where(den == 0, 1.0, den)
    assert (np.abs(yg - yr).max(1) / den).max() <= OUT_TOL


@pytest.mark.parametrize("ratio", [0.0, 1.0])
@pytest.mark.parametrize("case", [CASES[0], CASES[3], CASES[10], CASES[12]], ids=lambda c: c[0].name)
def test_router_paths_at_ratio_extremes(case, ratio, monkeypatch):
    """Ratio 0 is zero-brownout and ratio 1 delegates every S2 group
    (special case P:197) through the production router too."""
    cfg, env, kind = case
    _, y, dbg, ref = _run(cfg, env, monkeypatch, True, ratio)
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    assert np.array_equal(dbg["row_of"].cpu().numpy(), ref.perm.row_of)
    if ratio == 0.0:
        assert (ref.plan.exec_of_expert[ref.plan.counts > 0] < cfg.m).all()
    yg, yr = _np(y), ref.y
    den = np.where(np.abs(yr).max(1) == 0, 1.0, np.abs(yr).max(1))
    assert (np.abs(yg - yr).max(1) / den).max() <= OUT_TOL


def _rand_cfgs(n=10, seed=321):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        m = int(rng.choice([2, 5, 8, 16, 33, 60, 128, 256]))
        K = int(rng.integers(1, min(m, 16) + 1))
        way = int(rng.choice([1, 2, 3, 4, 8, m]))
        dt = "fp32" if rng.random() < 0.25 else "bf16"
        d = int(rng.choice([64, 128, 192, 320]))
        T = int(rng.choice([int(rng.integers(1, 300)), int(rng.integers(1184, 1500))]))
        out.append(C(f"xrand{i}_m{m}_K{K}_w{way}_{dt}_T{T}", d=d, f=128, m=m, K=K, way=way, T=T,
                     ratio=float(rng.choice([0.0, 0.3, 0.5, 1.0])), dtype=dt, config_id=200 + i))
    return out


@pytest.mark.parametrize("ties", [True, False], ids=["integer", "dyadic"])
@pytest.mark.parametrize("cfg", _rand_cfgs(), ids=lambda c: c.name)
def test_random_shapes_exact_router(cfg, ties, monkeypatch):
    """Random shapes over the envelope (whichever router kernel the shape picks)."""
    _, y, dbg, ref = _run(cfg, {}, monkeypatch, ties, cfg.ratio)
    assert np.array_equal(dbg["logits"].cpu().double().numpy(), ref.logits)
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.abs(dbg["topk_w"].cpu().double().numpy() - ref.g).max() <= W_TOL
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    assert np.array_equal(dbg["exec_off"].cpu().numpy(), ref.perm.exec_off)
    assert np.array_equal(dbg["row_of"].cpu().numpy(), ref.perm.row_of)
    yg, yr = _np(y), ref.y
    den = np.where(np.abs(yr).max(1) == 0, 1.0, np.abs(yr).max(1))
    assert (np.abs(yg - yr).max(1) / den).max() <= OUT_TOL


@pytest.mark.parametrize("fused", ["1", "0"], ids=["route_fused", "separate"])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_decode_routing_with_shared_experts(fused, ratio, monkeypatch):
    """k_route_fused (Alg. 1 run by every CTA from the same tile histograms, the
    permutation from each CTA's own copy of the plan) with the N_s shared experts of
    Eq. 5 appended after the routed executors, against the oracle's own
    Eq. 8 path; and the same step as separate launches."""
    from paper_2507_17133_b200 import BrownoutMoE
    monkeypatch.setenv("BO_ROUTE_FUSED", fused)
    cfg = C("sh_fused", d=256, f=256, m=8, K=2, way=4, T=120, ratio=ratio, dtype="bf16", Ns=2, config_id=78)
    x, Wr = S.make_exact_router_inputs(cfg, ties=True)
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T, num_shared=cfg.Ns)
    moe.set_brownout(ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    y = moe.forward(x.cuda(), Wr.cuda(), (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]),
                    shared=(g["SWg"], g["SWu"], g["SWd"]))
    torch.cuda.synchronize()
    assert moe.last_kernels()[0] == ("route_fused" if fused == "1" else "router_topk")
    dbg = moe.debug_arrays(cfg.T)
    ex = tuple(_np(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(_np(uni[k]) for k in ("UWg", "UWu", "UWd"))
    sh = tuple(_np(lay[k]) for k in ("SWg", "SWu", "SWd"))
    ref = O.moe_forward(_np(x), _np(Wr), ex, un, cfg.K, cfg.way, ratio, shared=sh)
    assert np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids)
    assert np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
    T, K, Ns, E = cfg.T, cfg.K, cfg.Ns, cfg.m + cfg.G
    eo = dbg["exec_off"].cpu().numpy()
    R = int(ref.perm.exec_off[-1])
    assert np.array_equal(eo[:E + 1], ref.perm.exec_off)
    assert np.array_equal(eo[E:], R + T * np.arange(Ns + 1))     # shared executors: every token, in order
    ro = dbg["row_of"].cpu().numpy().reshape(T, K + Ns)
    assert np.array_equal(ro[:, :K].reshape(-1), ref.perm.row_of)
    for j in range(Ns):
        assert np.array_equal(ro[:, K + j], R + j * T + np.arange(T))
    assert np.array_equal(dbg["row_tok"][:R].cpu().numpy(), ref.perm.row_tok)
    assert np.array_equal(dbg["row_tok"][R:R + Ns * T].cpu().numpy(), np.tile(np.arange(T), Ns))
    yg, yr = _np(y), ref.y
    den = np.where(np.abs(yr).max(1) == 0, 1.0, np.abs(yr).max(1))
    assert (np.abs(yg - yr).max(1) / den).max() <= OUT_TOL
