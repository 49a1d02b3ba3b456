"""Pins of the CPU oracle against what the paper and the mathematics fix.

None of these tests re-types an oracle formula: each checks the oracle against
(a) a value the paper prints (tests/golden/paper_examples.json, cited),
(b) a closed form, (c) brute force on tiny inputs, (d) an independent
reduction computed with torch fp64 dense masking, or (e) an invariant.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import brownout_oracle as O
import synthetic as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))
COUNTS = GOLD["counts_by_expert"]["value"]


# ---------------------------------------------------------------- Alg. 1 pins
def test_paper_partial_brownout_example():
    """5 executors: S1={E1,E3,E7}, UE0<-{E0,E2} (3), UE1<-{E4,E5,E6} (5)."""
    ex = GOLD["partial_brownout"]
    p = O.brownout_plan(COUNTS, ex["ratio"], ex["way"], O.PARTIAL)
    assert sorted(p.S1) == ex["S1"]
    assert p.stats["executors_accessed"] == ex["executors_accessed"]
    m = len(COUNTS)
    for j, u in ex["united"].items():
        members = [e for e in range(m) if p.exec_of_expert[e] == m + int(j)]
        assert members == u["members"]
        assert sum(COUNTS[e] for e in members) == u["rows"]
    assert p.stats["rows_original"] == 12 and p.stats["rows_united"] == 8


def test_paper_full_brownout_example():
    """12 tokens kept by E1,E3,E7; 8 ignored; 37.5% of experts accessed."""
    ex = GOLD["full_brownout"]
    p = O.brownout_plan(COUNTS, ex["ratio"], 4, O.FULL)
    assert sorted(p.S1) == ex["S1"]
    assert p.stats["rows_original"] == ex["rows_kept"]
    assert p.stats["rows_dropped"] == ex["rows_dropped"]
    assert p.stats["executors_accessed"] / len(COUNTS) == ex["access_fraction"]


def test_paper_special_case_example():
    """with k=3, E6 alone in its group keeps its original expert."""
    ex = GOLD["special_case"]
    p = O.brownout_plan(COUNTS, ex["ratio"], ex["way"], O.PARTIAL)
    m = len(COUNTS)
    assert sorted(p.S1) == ex["S1"]
    for e in ex["singleton_originals"]:
        assert p.exec_of_expert[e] == e and e in p.S2
    for j, u in ex["united"].items():
        members = [e for e in range(m) if p.exec_of_expert[e] == m + int(j)]
        assert members == u["members"]
        assert sum(COUNTS[e] for e in members) == u["rows"]
    assert p.stats["executors_accessed"] == ex["executors_accessed"]
    assert p.stats["n_singleton"] == 1


def test_literal_alg1_guard_contradicts_examples():
    """Reading D1: the printed guard of Alg. 1 line 10, evaluated before
    the increment, puts the largest expert (i = 0, sum_partial = 0) in S2 and
    so cannot reproduce P:173.  The oracle's prefix-until-coverage reading does."""
    cnt = np.array(COUNTS)
    A = sorted(range(8), key=lambda e: (-cnt[e], e))
    T = 20 * 0.6
    lit, sp = [], 0
    for i, e in enumerate(A):
        if sp >= T and (i == 0 or sp - cnt[e] < T):
            lit.append(e)
        sp += cnt[e]
    assert sorted(lit) != [1, 3, 7]
    assert sorted(O.brownout_plan(COUNTS, 0.4, 4).S1) == [1, 3, 7]


def _min_cover_bruteforce(counts, T):
    """Smallest number of experts whose counts sum to >= T (exhaustive)."""
    m = len(counts)
    if T <= 0:
        return 0
    for r in range(1, m + 1):
        for sub in itertools.combinations(range(m), r):
            if sum(counts[i] for i in sub) >= T:
                return r
    return None


def test_greedy_prefix_is_minimal_cover_bruteforce():
    """S:155-167 / P:173 'find fewer experts to handle more tokens': |S1| equals
    the exhaustive minimal cover size for random instances with m <= 12."""
    rng = np.random.default_rng(7)
    for _ in range(400):
        m = int(rng.integers(1, 13))
        counts = rng.integers(0, 30, size=m).tolist()
        ratio = float(rng.choice([0.0, 0.1, 0.25, 0.4, 0.5, 0.7, 0.9, 1.0, rng.random()]))
        p = O.brownout_plan(counts, ratio, int(rng.integers(1, 5)))
        need = _min_cover_bruteforce(counts, p.Tcov)
        if need is None:     # Tcov > S cannot happen (threshold <= 1)
            raise AssertionError
        assert len(p.S1) == need
        # coverage and prefix minimality
        assert sum(counts[e] for e in p.S1) >= p.Tcov
        if p.S1:
            smallest = min(p.S1, key=lambda e: (counts[e], -e))
            assert sum(counts[e] for e in p.S1) - counts[smallest] < p.Tcov or counts[smallest] == 0


def test_tcov_fp64_reading_d3():
    """Reading D3: T = S * (1 - ratio) in fp64.  ratio 0.7, S = 10 gives
    T = 3.0000000000000004 (not 3), so two experts (3 + 1 rows) are needed."""
    counts = [3, 1, 1, 1, 1, 1, 1, 1]
    p = O.brownout_plan(counts, 0.7, 4)
    assert p.Tcov == 10 * (1.0 - 0.7) and p.Tcov > 3.0
    assert sorted(p.S1) == [0, 1]


def test_zero_count_experts_join_neither_set():
    p = O.brownout_plan([0, 5, 0, 3], 1.0, 2)
    assert 0 not in p.S1 + p.S2 and 2 not in p.S1 + p.S2
    assert p.exec_of_expert[0] == O.INACTIVE


def test_ratio_extremes():
    """Ratio 0 (threshold 1, P:217 zero-brownout): every active expert in S1.
    Ratio 1 (threshold 0): S1 empty; all rows go to united experts except the
    special-case singletons (reading D7)."""
    rng = np.random.default_rng(3)
    for _ in range(100):
        m = int(rng.integers(2, 20))
        counts = rng.integers(0, 10, size=m)
        way = int(rng.integers(1, 6))
        p0 = O.brownout_plan(counts, 0.0, way)
        assert sorted(p0.S1) == [e for e in range(m) if counts[e] > 0]
        assert p0.stats["rows_united"] == 0
        p1 = O.brownout_plan(counts, 1.0, way)
        assert p1.S1 == []
        singles = sum(counts[e] for e in range(m) if 0 <= p1.exec_of_expert[e] < m)
        assert p1.stats["rows_united"] + singles == counts.sum()
        for j, mem in p1.groups.items():
            assert (len(mem) == 1) == (p1.exec_of_expert[mem[0]] == mem[0])


def test_monotone_in_ratio():
    """SPEC monotonicity: rows served by originals never increase with ratio."""
    rng = np.random.default_rng(5)
    for _ in range(100):
        counts = rng.integers(0, 50, size=int(rng.integers(2, 16)))
        prev = None
        for r in np.linspace(0, 1, 11):
            s1rows = sum(counts[e] for e in O.brownout_plan(counts, float(r), 4).S1)
            if prev is not None:
                assert s1rows <= prev
            prev = s1rows


# ------------------------------------------------------------- Eq. 7 / Eq. 8
def test_gate_closed_form():
    ex = GOLD["gate_closed_form"]
    ids, g = O.topk_gate(np.array([ex["scores"]]), ex["K"])
    assert ids.tolist() == [[0, 1]]
    assert g[0, 0] == pytest.approx(ex["g"][0], abs=1e-15)
    assert g[0, 1] == pytest.approx(ex["g"][1], abs=1e-15)
    assert g[0, 0] == pytest.approx(1.0 / (1.0 + math.exp(-1.0)), abs=1e-15)


def test_topk_matches_library_sort_and_sums_to_one():
    """Distinct logits: selection equals numpy argsort; ties: lexsort by
    (-logit, id); weights sum to 1 and are ordered like the logits."""
    rng = np.random.default_rng(11)
    L = rng.standard_normal((200, 16))
    ids, g = O.topk_gate(L, 4)
    assert (ids == np.argsort(-L, axis=1, kind="stable")[:, :4]).all()
    assert np.allclose(g.sum(1), 1.0, atol=1e-12)
    assert (np.diff(g, axis=1) <= 0).all()
    Lt = rng.integers(-2, 3, size=(300, 8)).astype(np.float64)
    Lt[Lt == 0] = np.where(rng.random((Lt == 0).sum()) < 0.5, -0.0, 0.0)
    assert np.signbit(Lt[Lt == 0]).any()
    ids, _ = O.topk_gate(Lt, 3)
    for t in range(Lt.shape[0]):
        ref = np.lexsort((np.arange(8), -Lt[t]))[:3]
        assert ids[t].tolist() == ref.tolist()


def test_router_logits_small_example():
    """S:50 example: x=[1,0], centroids [[2,0],[0,3],[1,1]] -> [2,0,1]."""
    s = O.router_logits(np.array([[1.0, 0.0]]), np.array([[2.0, 0.0], [0.0, 3.0], [1.0, 1.0]]))
    assert s.tolist() == [[2.0, 0.0, 1.0]]


def test_swiglu_scalar_closed_form():
    """d = f = 1, all weights 1, x = 1: FFN = silu(1) * 1 = 1 / (1 + e^-1)."""
    one = np.ones((1, 1))
    out = O.swiglu_ffn(one, one, one, one)
    assert out[0, 0] == pytest.approx(1.0 / (1.0 + math.exp(-1.0)), abs=1e-15)


# ---------------------------------------------------------- Eq. 5 reductions
def _tiny(seed, m=8, d=16, f=32, way=4, T=24, K=2, sigma=0.7):
    cfg = S.LayerConfig("t", d=d, f=f, m=m, K=K, way=way, T=T, ratio=0.5, dtype="fp32",
                        sigma=sigma, config_id=seed)
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=seed)
    ex = tuple(lay[k].double().numpy() for k in ("Wg", "Wu", "Wd"))
    un = tuple(uni[k].double().numpy() for k in ("UWg", "UWu", "UWd"))
    return cfg, x.double().numpy(), lay["Wr"].double().numpy(), ex, un


def _vanilla_moe_torch(x, Wr, Wg, Wu, Wd, K):
    """Independent top-K MoE in torch fp64 with dense masking (every expert runs
    on every token; the mask keeps the routed ones)."""
    x = torch.from_numpy(x)
    s = x @ torch.from_numpy(Wr).T
    top = torch.topk(s, K, dim=1)
    w = torch.softmax(top.values, dim=1)
    dense = torch.zeros_like(s).scatter(1, top.indices, w)
    y = torch.zeros_like(x)
    for e in range(s.shape[1]):
        a = x @ torch.from_numpy(Wg[e]).T
        b = x @ torch.from_numpy(Wu[e]).T
        h = torch.nn.functional.silu(a) * b
        y += dense[:, e:e + 1] * (h @ torch.from_numpy(Wd[e]).T)
    return y.numpy()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ratio0_equals_vanilla_topk_moe(seed):
    """P:217 'when threshold is equal to 1, Algorithm 1 describes the zero
    brownout process' = a plain top-K MoE."""
    cfg, x, Wr, ex, un = _tiny(seed)
    r = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, 0.0)
    ref = _vanilla_moe_torch(x, Wr, *ex, cfg.K)
    assert np.abs(r.y - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ratio1_without_singletons_equals_united_moe(seed):
    """Ratio 1 (threshold 0): every row goes to the united expert of its group
    (Eq. 5-6 with p = 0, q = g) whenever no group is a singleton (D7)."""
    cfg, x, Wr, ex, un = _tiny(seed, T=64)
    r = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, 1.0)
    assert r.plan.stats["n_singleton"] == 0
    m = cfg.m
    sub = tuple(np.stack([U[e // cfg.way] for e in range(m)]) for U in un)
    ref = _vanilla_moe_torch(x, Wr, *sub, cfg.K)
    assert np.abs(r.y - ref).max() <= 1e-12 * max(1.0, np.abs(ref).max())
    assert r.plan.stats["rows_united"] == cfg.T * cfg.K


def test_way1_is_ratio_independent():
    """Reading D7 corollary: k = 1 makes every delegated group a singleton, so
    the output equals zero-brownout for every ratio."""
    cfg, x, Wr, ex, un = _tiny(4, way=1)
    base = O.moe_forward(x, Wr, ex, un, cfg.K, 1, 0.0).y
    for ratio in (0.25, 0.5, 1.0):
        r = O.moe_forward(x, Wr, ex, un, cfg.K, 1, ratio)
        assert r.plan.stats["rows_united"] == 0
        assert np.array_equal(r.y, base)


def test_identical_group_experts_make_output_plan_independent():
    """S:85 substitution: if every expert of a group equals its united expert,
    Eq. 5 gives the same output for every plan."""
    cfg, x, Wr, ex, un = _tiny(5)
    G = cfg.G
    ex_same = tuple(np.stack([U[e // cfg.way] for e in range(cfg.m)]) for U in un)
    base = O.moe_forward(x, Wr, ex_same, un, cfg.K, cfg.way, 0.0).y
    for ratio in (0.25, 0.5, 0.75, 1.0):
        y = O.moe_forward(x, Wr, ex_same, un, cfg.K, cfg.way, ratio).y
        assert np.abs(y - base).max() <= 1e-12 * np.abs(base).max()


@pytest.mark.parametrize("ratio", [0.0, 0.3, 0.5, 0.8, 1.0])
@pytest.mark.parametrize("mode", [O.PARTIAL, O.FULL])
def test_permuted_forward_equals_per_token_definition(ratio, mode):
    """O10 vs O11: Alg. 1's concatenated processing equals Eq. 5-6 per token."""
    cfg, x, Wr, ex, un = _tiny(6, T=40, K=3, way=3)
    r = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, ratio, mode)
    y_def = O.moe_forward_definition(x, r.ids, r.g, r.plan, ex, un)
    assert np.abs(r.y - y_def).max() <= 1e-12 * max(1.0, np.abs(y_def).max())


def test_conservation_and_partition():
    """Every assignment lands in exactly one row (or is dropped in full mode);
    rows_original + rows_united + rows_dropped = S; p + q = g (Eq. 6)."""
    cfg, x, Wr, ex, un = _tiny(7, T=50, K=2)
    for mode in (O.PARTIAL, O.FULL):
        for ratio in (0.0, 0.4, 1.0):
            r = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, ratio, mode)
            st, perm = r.plan.stats, r.perm
            assert st["rows_original"] + st["rows_united"] + st["rows_dropped"] == cfg.T * cfg.K
            rows = perm.row_of[perm.row_of >= 0]
            assert len(set(rows.tolist())) == len(rows) == int(perm.exec_off[-1])
            for t in range(cfg.T):
                for s in range(cfg.K):
                    rr = perm.row_of[t * cfg.K + s]
                    if rr >= 0:
                        assert perm.row_tok[rr] == t and perm.row_w[rr] == r.g[t, s]
                        assert perm.exec_off[perm.row_exec[rr]] <= rr < perm.exec_off[perm.row_exec[rr] + 1]


def test_permutation_equivariance():
    """SPEC invariant: permuting tokens permutes y; counts and plan unchanged."""
    cfg, x, Wr, ex, un = _tiny(8, T=30)
    r = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, 0.5)
    pi = np.random.default_rng(0).permutation(cfg.T)
    r2 = O.moe_forward(x[pi], Wr, ex, un, cfg.K, cfg.way, 0.5)
    assert np.array_equal(r.plan.exec_of_expert, r2.plan.exec_of_expert)
    assert np.abs(r2.y - r.y[pi]).max() <= 1e-12 * np.abs(r.y).max()


def test_full_mode_ratio1_gives_residual_only():
    """SPEC moe_forward example: full brownout at threshold 0 with N_s = 0 ->
    h_t = x_t (every routed term is dropped, Eq. 6 p = q = 0)."""
    cfg, x, Wr, ex, un = _tiny(9)
    r = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, 1.0, O.FULL, add_residual=True)
    assert np.array_equal(r.y, x)


def test_sampled_forward_matches_full_forward():
    cfg, x, Wr, ex, un = _tiny(10, T=33)
    full = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, 0.5)
    toks = [0, 5, 17, 32]
    samp = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, 0.5, tokens=toks)
    assert np.array_equal(samp.y, full.y[toks])


# ---------------------------------------------------- bf16 rounding / united
def test_round_to_bf16_halfway_cases():
    one = 1.0
    cases = {
        one + 2.0 ** -8: 1.0,                         # tie -> even (down)
        one + 3 * 2.0 ** -8: one + 2.0 ** -6,         # tie -> even (up)
        one + 2.0 ** -8 + 2.0 ** -40: one + 2.0 ** -7,  # above half -> up
        -(one + 2.0 ** -8 + 2.0 ** -40): -(one + 2.0 ** -7),
        0.0: 0.0,
    }
    for v, want in cases.items():
        assert O.round_to_bf16(np.array([v]))[0] == want


def test_round_to_bf16_matches_torch_on_fp32_values():
    """For fp32-exact values torch's fp32 -> bf16 conversion is RNE, so it must
    agree with the fp64 -> bf16 rounding bit for bit."""
    v = torch.randn(100000, generator=torch.Generator().manual_seed(0)) * 3
    ref = v.to(torch.bfloat16).double().numpy()
    assert np.array_equal(O.round_to_bf16(v.double().numpy()), ref)


def test_build_united_mean_special_cases():
    rng = np.random.default_rng(0)
    W = torch.from_numpy(rng.standard_normal((6, 4, 8))).to(torch.bfloat16).double().numpy()
    # way 1: each group is one expert -> the mean is the expert itself
    U = O.build_united_mean(W, W, W, 1)[0]
    assert np.array_equal(U, W)
    # identical members -> the mean is the member; ragged last group (6 = 4 + 2)
    Wsame = np.repeat(W[:1], 6, axis=0)
    U = O.build_united_mean(Wsame, Wsame, Wsame, 4)[0]
    assert U.shape[0] == 2 and np.array_equal(U[0], W[0]) and np.array_equal(U[1], W[0])
    # hand example: mean of 1, 2, 4 = 7/3 -> bf16 2.328125 (7/3 = 10.0101010...b)
    Wh = np.array([1.0, 2.0, 4.0]).reshape(3, 1, 1)
    assert O.build_united_mean(Wh, Wh, Wh, 3)[0].item() == 2.328125


# --------------------------------------------- f3: united-row de-duplication
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_dedup_forward_equals_plain_forward(ratio):
    """Merging a token's slots delegated to the same united expert into one
    row with the summed weight is exact algebra on Eq. 5 (q1 F(x) + q2 F(x) =
    (q1 + q2) F(x)): the outputs agree to rounding."""
    cfg, x, Wr, ex, un = _tiny(12, T=60, K=3, way=4, m=8)
    a = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, ratio)
    b = O.moe_forward(x, Wr, ex, un, cfg.K, cfg.way, ratio, dedup=True)
    assert np.abs(a.y - b.y).max() <= 1e-12 * np.abs(a.y).max()
    # rows: originals unchanged, united rows = unique (token, united executor) pairs
    m = cfg.m
    uniq = {(t, int(a.plan.exec_of_expert[e])) for t in range(cfg.T) for e in a.ids[t]
            if a.plan.exec_of_expert[e] >= m}
    assert int(b.perm.exec_off[-1] - b.perm.exec_off[m]) == len(uniq)
    assert np.array_equal(a.perm.exec_off[:m + 1], b.perm.exec_off[:m + 1])
    # weights of a token's united rows sum to its delegated gate mass
    for t in range(cfg.T):
        rows = [r for r in b.perm.row_of[t * cfg.K:(t + 1) * cfg.K] if r >= 0]
        assert np.isclose(sum(b.perm.row_w[r] for r in rows), 1.0)


def test_dedup_hand_example():
    """Token 0 routed to experts 0 and 2 (same group of 4, both delegated at
    ratio 1) -> one united row carrying g0 + g2."""
    L = np.array([[3.0, 0.0, 2.0, -1.0, -5.0, -5.0, -5.0, -5.0],
                  [-5.0, 4.0, -5.0, -5.0, 3.0, -5.0, -5.0, -5.0]])
    ids, g = O.topk_gate(L, 2)
    plan = O.brownout_plan(O.expert_counts(ids, 8), 1.0, 4)
    # group 0 has experts {0, 1, 2} delegated (>= 2 members) -> UE0; group 1 has {4} -> singleton
    assert plan.exec_of_expert[0] == 8 and plan.exec_of_expert[2] == 8 and plan.exec_of_expert[4] == 4
    p = O.permutation_dedup(ids, g, plan)
    r0 = p.row_of[0]
    assert p.row_of[1] == -1 and p.row_w[r0] == pytest.approx(g[0, 0] + g[0, 1])
    assert p.exec_off[-1] == 3          # token 0 -> UE0 (merged), token 1 -> UE0 and E4


# ------------------------------------------------------- shared experts (f2)
def _shared_case(Ns=3, d=16, f=8, T=5, seed=4):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((T, d))
    SWg = rng.standard_normal((Ns, f, d)) / 4
    SWu = rng.standard_normal((Ns, f, d)) / 4
    SWd = rng.standard_normal((Ns, d, f)) / 3
    return x, (SWg, SWu, SWd)


def test_shared_experts_equal_one_wide_expert_with_gate_one():
    """Eq. 5 second term: N_s shared SwiGLU experts of width f summed with
    weight 1 equal ONE expert of width N_s f whose gate / up rows and down
    columns are the blocks concatenated (the SwiGLU is row-separable in f).
    The wide expert runs as the only routed expert of a top-1 layer, where Eq. 7's
    softmax over a single logit gives gate 1; the shared side runs next to a
    routed expert whose down-projection is zero."""
    x, (SWg, SWu, SWd) = _shared_case()
    T, d = x.shape
    Ns, f, _ = SWg.shape
    zero = (np.zeros((1, f, d)), np.zeros((1, f, d)), np.zeros((1, d, f)))
    L = np.zeros((T, 1))
    got = O.moe_forward(x, None, zero, zero, 1, 1, 0.0, logits=L, shared=(SWg, SWu, SWd)).y
    wide = (SWg.reshape(1, Ns * f, d), SWu.reshape(1, Ns * f, d),
            np.concatenate(list(SWd), axis=1)[None])
    want = O.moe_forward(x, None, wide, wide, 1, 1, 0.0, logits=L).y
    assert np.allclose(got, want, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("mode", [O.PARTIAL, O.FULL])
def test_shared_term_is_independent_of_brownout(mode):
    """Alg. 1 re-routes only original experts: the shared term of
    Eq. 5 is the same at every ratio / mode, also for tokens whose routed slots
    were all dropped (full brownout, ratio 1)."""
    cfg = S.with_(S.C1, T=24)
    lay = S.make_layer(cfg)
    ex = tuple(lay[k].double().numpy() for k in ("Wg", "Wu", "Wd"))
    un = O.build_united_mean(*ex, cfg.way)
    x = S.make_tokens(cfg).double().numpy()
    _, sh = _shared_case(Ns=2, d=cfg.d, f=cfg.f, T=cfg.T)
    L = S.make_logits(cfg.T, cfg.m, seed=3).double().numpy()
    deltas = []
    for ratio in (0.0, 0.5, 1.0):
        a = O.moe_forward(x, None, ex, un, cfg.K, cfg.way, ratio, mode, logits=L, shared=sh).y
        b = O.moe_forward(x, None, ex, un, cfg.K, cfg.way, ratio, mode, logits=L).y
        deltas.append(a - b)
    for dl in deltas[1:]:
        assert np.allclose(dl, deltas[0], rtol=1e-12, atol=1e-12)
    assert np.abs(deltas[0]).max() > 0.1
