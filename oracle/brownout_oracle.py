"""CPU fp64 oracle for the brownout MoE-layer forward (BrownoutServe, arXiv 2507.17133).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2507_17133_b200``) never imports it and
shares no code, headers, helpers or tables with it.

Citation format: ``P:n`` = line n of the paper text, with the
section / equation / algorithm it belongs to.  ``D<n>`` = a reading of the
paper recorded in DESIGN.md §"Readings" (where the paper is silent, garbled or
ambiguous).

Every step below follows the paper's own order and notation:

  Eq. 8      s_{i,t} = x_t^T e_i                       -> router_logits
  Eq. 7  g_{i,t} = softmax over TopK(s_{.,t}, K)   -> topk_gate
  Alg. 1  counts, sort, T = S*threshold, S1/S2,
                      group_experts, special case, concat       -> expert_counts,
                                                                   brownout_plan,
                                                                   permutation
  Eq. 5-6 h_t = x_t + sum p FFN^(r) + sum q FFN^(u)  -> moe_forward,
                                                                   moe_forward_definition

Arithmetic is IEEE binary64 throughout (inputs are widened exactly from their
bf16 / fp32 storage).  The only non-fp64 arithmetic is the Alg. 1 coverage
target, which is the fp64 product S * (1 - ratio) on both sides (reading D3).

Parity status: every function here is pinned by
at least one test in tests/test_oracle_pins.py against a value the paper prints,
a closed form, brute force, or an independent reduction.  The tie conventions
(D5 count-sort ties, D8 top-K ties, D11 row order inside a united executor) are
conventions: they are pinned by brute force on tiny inputs only ("parity
unpinned" beyond the stated convention).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PARTIAL = "partial"   # Alg. 1 with use_full_brownout = false
FULL = "full"         # Alg. 1 with use_full_brownout = true

# Executor codes for experts that do not execute (reading D6 / full mode).
INACTIVE = -1   # cnt_i == 0: joins neither S1 nor S2 (D6)
DROPPED = -2    # full-brownout: S2 experts' tokens are "ignored"


# --------------------------------------------------------------------------
# Eq. 8 and Eq. 7: gate
# --------------------------------------------------------------------------
def router_logits(x: np.ndarray, Wr: np.ndarray) -> np.ndarray:
    """Eq. 8: s_{i,t} = x_t^T e_i, where e_i = Wr[i] is the centroid.

    x [T, d], Wr [m, d]  ->  s [T, m] in fp64 (no bias, no scaling).
    """
    x = np.asarray(x, dtype=np.float64)
    Wr = np.asarray(Wr, dtype=np.float64)
    return x @ Wr.T


def topk_gate(logits: np.ndarray, K: int):
    """Eq. 7: pick the K highest affinities per token, softmax over them.

    Selection order: logit descending, ties -> lower expert id (reading D8).
    The comparison is on the logits themselves (not the probabilities), and
    -0.0 == +0.0 because IEEE comparison treats them as equal.
    Returns ids [T, K] int64 ordered by selection, and g [T, K] fp64 with
    g[t, s] = exp(s_sel - s_max) / sum_{s' in TopK} exp(s_sel' - s_max).
    """
    L = np.asarray(logits, dtype=np.float64)
    T, m = L.shape
    if not (1 <= K <= m):
        raise ValueError(f"K={K} out of range [1, {m}]")
    ids = np.empty((T, K), dtype=np.int64)
    g = np.empty((T, K), dtype=np.float64)
    for t in range(T):
        # Python's sort is stable; key (-logit, id) gives "logit desc, id asc".
        order = sorted(range(m), key=lambda i: (-L[t, i], i))
        sel = order[:K]
        ids[t] = sel
        vmax = L[t, sel[0]]
        num = np.array([math.exp(L[t, i] - vmax) for i in sel])
        g[t] = num / num.sum()
    return ids, g


# --------------------------------------------------------------------------
# Algorithm 1: the brownout plan
# --------------------------------------------------------------------------
def expert_counts(ids: np.ndarray, m: int) -> np.ndarray:
    """Alg. 1 input cnt_i: number of (token, slot) assignments routed to
    expert i.  With top-K routing S = sum cnt_i = T*K (reading D4)."""
    cnt = np.zeros(m, dtype=np.int64)
    for e in np.asarray(ids).reshape(-1):
        cnt[int(e)] += 1
    return cnt


@dataclass
class Plan:
    """Result of Alg. 1 lines 4-33 for one batch."""
    m: int
    way: int
    ratio: float
    mode: str
    counts: np.ndarray                 # cnt_i, [m]
    S: int                             # Alg. 1 line 6
    Tcov: float                        # Alg. 1 line 7, T = S * threshold
    sorted_experts: list               # Alg. 1 line 5 (cnt desc, id asc)
    S1: list                           # experts processed by their original FFN
    S2: list                           # experts delegated (partial) / ignored (full)
    groups: dict                       # group id j -> S2 members (ascending id)
    exec_of_expert: np.ndarray         # [m]: executor id, INACTIVE or DROPPED
    stats: dict = field(default_factory=dict)

    @property
    def G(self) -> int:
        return -(-self.m // self.way)

    @property
    def E(self) -> int:
        return self.m + self.G


def brownout_plan(counts, ratio: float, way: int, mode: str = PARTIAL) -> Plan:
    """Algorithm 1, BrownoutMoE, with the readings of DESIGN.md.

    Knob: ratio = 1 - threshold (D2; BASELINE's "brownout ratio").
    Line 5  sort A by cnt descending; ties -> lower id first (D5).
    Line 6  S = sum cnt.
    Line 7  T = S * threshold, threshold = 1.0 - ratio, both in fp64 (D3).
    Lines 9-15 (garbled guard, D1): the expert joins S1 iff it is active and
            the exclusive prefix sum_partial of the sorted list is < T
            ("prefix until coverage", reproduces P:173 and P:194).  Other
            active experts join S2 (partial) or are dropped (full).
            Zero-count experts join neither (D6).
    Lines 22-23 group_experts: group of expert e is floor(e / way) (P:149,
            P:154-155; ragged last group D15).
    Lines 24-26 special case: a group with exactly one S2 member keeps
            its original expert.
    Lines 27-30 otherwise the group's tokens go to united expert m + j.
    Executor ids: originals 0..m-1, united m..m+G-1.
    """
    cnt = np.asarray(counts, dtype=np.int64).copy()
    m = int(cnt.shape[0])
    if not (0.0 <= ratio <= 1.0):
        raise ValueError("ratio must be in [0, 1]")
    if way < 1:
        raise ValueError("way must be >= 1")
    if mode not in (PARTIAL, FULL):
        raise ValueError("mode must be 'partial' or 'full'")
    G = -(-m // way)

    # Alg. 1 lines 4-5
    A = sorted(range(m), key=lambda e: (-int(cnt[e]), e))
    # line 6
    S = int(cnt.sum())
    # line 7 (threshold = 1 - ratio, D2/D3)
    threshold = 1.0 - float(ratio)
    Tcov = float(S) * threshold
    # lines 8-15
    S1, S2 = [], []
    sum_partial = 0
    for e in A:
        if cnt[e] == 0:
            continue                       # D6
        if float(sum_partial) < Tcov:      # D1: exclusive prefix < T
            S1.append(e)
        else:
            S2.append(e)                   # partial: delegate; full: drop
        sum_partial += int(cnt[e])

    exec_of = np.full(m, INACTIVE, dtype=np.int64)
    for e in S1:
        exec_of[e] = e                     # lines 16-18: original expert
    # lines 22-23: group S2 by floor(e / way)
    groups: dict = {}
    for e in sorted(S2):
        groups.setdefault(e // way, []).append(e)
    n_singleton = 0
    n_united = 0
    for j, members in groups.items():
        if mode == FULL:
            for e in members:
                exec_of[e] = DROPPED       # P:173 "ignored"
        elif len(members) == 1:
            exec_of[members[0]] = members[0]   # lines 24-26, special case P:197
            n_singleton += 1
        else:
            for e in members:
                exec_of[e] = m + j         # lines 27-30, united expert of group j
            n_united += 1

    rows_orig = int(sum(cnt[e] for e in range(m) if 0 <= exec_of[e] < m))
    rows_united = int(sum(cnt[e] for e in range(m) if exec_of[e] >= m))
    rows_dropped = int(sum(cnt[e] for e in range(m) if exec_of[e] == DROPPED))
    accessed = len({int(x) for x in exec_of if x >= 0})
    stats = dict(executors_accessed=accessed, n_s1=len(S1), n_united=n_united,
                 n_singleton=n_singleton, rows_original=rows_orig,
                 rows_united=rows_united, rows_dropped=rows_dropped)
    return Plan(m=m, way=way, ratio=float(ratio), mode=mode, counts=cnt, S=S,
                Tcov=Tcov, sorted_experts=A, S1=S1, S2=S2, groups=groups,
                exec_of_expert=exec_of, stats=stats)


@dataclass
class Permutation:
    """concat_tokens (Alg. 1 line 27) laid out as one row array.

    Row order (reading D11): executor ascending, then original expert id
    ascending inside the executor, then token ascending.
    """
    exec_off: np.ndarray        # [E+1] first row of each executor
    expert_row_off: np.ndarray  # [m] first row of each expert's tokens (-1 if none)
    row_of: np.ndarray          # [T*K] row of assignment (t, s); -1 if dropped
    row_tok: np.ndarray         # [R] token of each row
    row_slot: np.ndarray        # [R] top-K slot of each row
    row_exec: np.ndarray        # [R] executor of each row
    row_w: np.ndarray           # [R] gate weight g of the row's original expert (Eq. 6)


def permutation(ids: np.ndarray, g: np.ndarray, plan: Plan) -> Permutation:
    """Build the rows each executor processes (Alg. 1 lines 16-30).

    The weight carried by a row is p_{i,t} = g_{i,t} for S1 experts and
    q_{i,t} = g_{i,t} for S2 experts (Eq. 6), i.e. always the gate
    weight of the ORIGINAL expert i (reading D10).
    """
    ids = np.asarray(ids)
    T, K = ids.shape
    m, E = plan.m, plan.E
    exec_of = plan.exec_of_expert
    cnt = plan.counts
    rows_of_exec = np.zeros(E, dtype=np.int64)
    for e in range(m):
        if exec_of[e] >= 0:
            rows_of_exec[exec_of[e]] += cnt[e]
    exec_off = np.zeros(E + 1, dtype=np.int64)
    exec_off[1:] = np.cumsum(rows_of_exec)
    expert_row_off = np.full(m, -1, dtype=np.int64)
    fill = exec_off[:-1].copy()
    for e in range(m):                    # experts ascending inside an executor
        x = exec_of[e]
        if x >= 0:
            expert_row_off[e] = fill[x]
            fill[x] += cnt[e]
    R = int(exec_off[-1])
    row_of = np.full(T * K, -1, dtype=np.int64)
    row_tok = np.empty(R, dtype=np.int64)
    row_slot = np.empty(R, dtype=np.int64)
    row_exec = np.empty(R, dtype=np.int64)
    row_w = np.empty(R, dtype=np.float64)
    nxt = expert_row_off.copy()
    for t in range(T):                    # tokens ascending inside an expert
        for s in range(K):
            e = int(ids[t, s])
            if exec_of[e] < 0:
                continue                  # dropped (full mode)
            r = int(nxt[e])
            nxt[e] += 1
            row_of[t * K + s] = r
            row_tok[r] = t
            row_slot[r] = s
            row_exec[r] = exec_of[e]
            row_w[r] = g[t, s]
    return Permutation(exec_off=exec_off, expert_row_off=expert_row_off,
                       row_of=row_of, row_tok=row_tok, row_slot=row_slot,
                       row_exec=row_exec, row_w=row_w)


def permutation_dedup(ids: np.ndarray, g: np.ndarray, plan: Plan) -> Permutation:
    """Row de-duplication variant (reading D10'):
    when several of a token's K slots are delegated to the SAME united expert
    (their experts share a group and are all in S2), Eq. 5 adds
    q_1 FFN_u(x_t) + q_2 FFN_u(x_t) + ... = (q_1 + q_2 + ...) FFN_u(x_t)
    (Eq. 6): one row with the summed weight (fp64, slot order)
    gives the same output.  Rows of original executors are unchanged.

    Row order: executor ascending; inside an original executor, token ascending;
    inside a united executor, token ascending (one row per token).  row_of of the
    first slot of a merged group points at the row; the other merged slots get -1
    (as dropped slots do: they have no row of their own).
    """
    ids = np.asarray(ids)
    T, K = ids.shape
    m, E = plan.m, plan.E
    exec_of = plan.exec_of_expert
    # unique (token, executor) pairs in token order, slots in slot order
    first = {}                        # (t, x) -> first slot
    wsum = {}
    for t in range(T):
        for s in range(K):
            x = int(exec_of[int(ids[t, s])])
            if x < 0:
                continue
            key = (t, x) if x >= m else (t, x, s)      # originals never merge (distinct experts)
            if key not in first:
                first[key] = s
                wsum[key] = 0.0
            wsum[key] += g[t, s]
    rows_of_exec = np.zeros(E, dtype=np.int64)
    for key in first:
        rows_of_exec[key[1]] += 1
    exec_off = np.zeros(E + 1, dtype=np.int64)
    exec_off[1:] = np.cumsum(rows_of_exec)
    R = int(exec_off[-1])
    expert_row_off = np.full(m, -1, dtype=np.int64)
    for e in range(m):
        if 0 <= exec_of[e] < m:
            expert_row_off[e] = exec_off[exec_of[e]]
    row_of = np.full(T * K, -1, dtype=np.int64)
    row_tok = np.empty(R, dtype=np.int64)
    row_slot = np.empty(R, dtype=np.int64)
    row_exec = np.empty(R, dtype=np.int64)
    row_w = np.empty(R, dtype=np.float64)
    nxt = exec_off[:-1].copy()
    for key in sorted(first, key=lambda k: (k[1], k[0])):   # executor, then token
        t, x = key[0], key[1]
        s = first[key]
        r = int(nxt[x])
        nxt[x] += 1
        row_of[t * K + s] = r
        row_tok[r] = t
        row_slot[r] = s
        row_exec[r] = x
        row_w[r] = wsum[key]
    return Permutation(exec_off=exec_off, expert_row_off=expert_row_off,
                       row_of=row_of, row_tok=row_tok, row_slot=row_slot,
                       row_exec=row_exec, row_w=row_w)


# --------------------------------------------------------------------------
# Expert FFN and Eq. 5
# --------------------------------------------------------------------------
def silu(z):
    """silu(z) = z / (1 + e^{-z}) (SwiGLU gate, reading D13)."""
    return z / (1.0 + np.exp(-z))


def swiglu_ffn(X: np.ndarray, Wg: np.ndarray, Wu: np.ndarray, Wd: np.ndarray) -> np.ndarray:
    """FFN(x) = Wd (silu(Wg x) * (Wu x)) for each row of X (reading D13).

    X [n, d]; Wg, Wu [f, d]; Wd [d, f] (nn.Linear [out, in] layout).
    """
    X = np.asarray(X, dtype=np.float64)
    a = X @ np.asarray(Wg, dtype=np.float64).T
    b = X @ np.asarray(Wu, dtype=np.float64).T
    h = silu(a) * b
    return h @ np.asarray(Wd, dtype=np.float64).T


def executor_weights(x_id: int, m: int, experts, united):
    """Weights of executor x_id: original expert x_id < m, else united x_id - m."""
    Wg, Wu, Wd = experts
    UWg, UWu, UWd = united
    if x_id < m:
        return Wg[x_id], Wu[x_id], Wd[x_id]
    j = x_id - m
    return UWg[j], UWu[j], UWd[j]


@dataclass
class ForwardResult:
    y: np.ndarray
    logits: np.ndarray
    ids: np.ndarray
    g: np.ndarray
    plan: Plan
    perm: Permutation
    rows_y: np.ndarray = None       # [R, d] weighted executor outputs (sampled forward: None)


def route(x, Wr, K, way, ratio, mode=PARTIAL, logits=None, dedup=False):
    """Eq. 8 -> Eq. 7 -> Alg. 1 -> concat order.  If ``logits`` is given it is
    used instead of Eq. 8 (parity entry: "given identical fp32 logits", B:5).
    dedup=True merges a token's slots delegated to the same united expert
    (permutation_dedup)."""
    L = router_logits(x, Wr) if logits is None else np.asarray(logits, dtype=np.float64)
    m = L.shape[1]
    ids, g = topk_gate(L, K)
    cnt = expert_counts(ids, m)
    plan = brownout_plan(cnt, ratio, way, mode)
    perm = permutation_dedup(ids, g, plan) if dedup else permutation(ids, g, plan)
    return L, ids, g, plan, perm


def moe_forward(x, Wr, experts, united, K, way, ratio, mode=PARTIAL,
                logits=None, add_residual=False, tokens=None, dedup=False, shared=None) -> ForwardResult:
    """Eq. 5 evaluated the way Alg. 1 processes it (lines 16-30).

    For each executor, its concatenated rows are run through that executor's
    FFN (process_tokens); each row's output is scaled by its gate
    weight (p or q of Eq. 6) and added to the row's token.

    ``shared``: optional (SWg [N_s, f, d], SWu [N_s, f, d], SWd [N_s, d, f]),
    the N_s shared experts of Eq. 5's second term, sum_{i=1}^{N_s}
    FFN_i^(s)(x_t): every token, weight 1, untouched by Alg. 1
    (which only re-routes original experts).  Added after the routed
    slots (reading D12).  None: N_s = 0.

    ``tokens``: optional list of token indices; when given, only those tokens'
    outputs are computed (routing and the plan still use the whole batch, since
    Alg. 1 counts over the whole batch, reading D18).  y then has one row per
    listed token.
    """
    x64 = np.asarray(x, dtype=np.float64)
    L, ids, g, plan, perm = route(x, Wr, K, way, ratio, mode, logits, dedup)
    T, d = x64.shape
    want = np.arange(T) if tokens is None else np.asarray(tokens, dtype=np.int64)
    R = int(perm.exec_off[-1])
    # rows whose outputs are needed: all rows, or the rows of the wanted tokens
    if tokens is None:
        needed = np.arange(R)
    else:
        rr = perm.row_of.reshape(T, K)[want].reshape(-1)
        needed = np.unique(rr[rr >= 0])
    rows_y = np.zeros((R, d), dtype=np.float64)
    # Alg. 1 lines 16-30: each executor processes its concatenated rows
    for xid in range(plan.E):
        r0, r1 = int(perm.exec_off[xid]), int(perm.exec_off[xid + 1])
        rows = needed[(needed >= r0) & (needed < r1)]
        if rows.size == 0:
            continue
        Wg, Wu, Wd = executor_weights(xid, plan.m, experts, united)
        out = swiglu_ffn(x64[perm.row_tok[rows]], Wg, Wu, Wd)
        rows_y[rows] = out * perm.row_w[rows][:, None]     # p / q of Eq. 6
    # Eq. 5: h_t = [x_t] + sum over the token's K slots, in slot order
    y = x64[want].copy() if add_residual else np.zeros((len(want), d), dtype=np.float64)
    for i, t in enumerate(want):
        for s in range(K):
            r = int(perm.row_of[int(t) * K + s])
            if r >= 0:
                y[i] += rows_y[r]
    if shared is not None:               # Eq. 5 second term: sum_i FFN_i^(s)(x_t)
        SWg, SWu, SWd = (np.asarray(a, dtype=np.float64) for a in shared)
        for j in range(SWg.shape[0]):
            y += swiglu_ffn(x64[want], SWg[j], SWu[j], SWd[j])
    return ForwardResult(y=y, logits=L, ids=ids, g=g, plan=plan, perm=perm,
                         rows_y=rows_y if tokens is None else None)


def moe_forward_definition(x, ids, g, plan: Plan, experts, united, add_residual=False):
    """Eq. 5-6 written per token, with no permutation (check O11):

        h_t = [x_t] + sum_{i in TopK(t)} p_{i,t} FFN_i^(r)(x_t) + q_{i,t} FFN_{f(i)}^(u)(x_t)

    p = g if i in S1 or i is a special-case singleton (executes as itself),
    q = g if i is delegated to united expert f(i) = floor(i / way), and both
    are 0 when i was dropped (full mode).  Equivalently: a vanilla top-K MoE
    whose expert table E' substitutes UE_{f(i)} for delegated experts.
    """
    x64 = np.asarray(x, dtype=np.float64)
    T, K = np.asarray(ids).shape
    y = x64.copy() if add_residual else np.zeros_like(x64)
    for t in range(T):
        for s in range(K):
            i = int(ids[t, s])
            xid = int(plan.exec_of_expert[i])
            if xid < 0:
                continue                   # p = q = 0 (dropped)
            Wg, Wu, Wd = executor_weights(xid, plan.m, experts, united)
            y[t] += g[t, s] * swiglu_ffn(x64[t][None, :], Wg, Wu, Wd)[0]
    return y


# --------------------------------------------------------------------------
# United experts (initialisation; distillation itself is out of scope)
# --------------------------------------------------------------------------
def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """Round fp64 values to the nearest bf16 (ties to even), returned as fp64.

    Done in two exact steps: fp64 -> the bf16 grid via integer manipulation of
    the fp64 bit pattern (no intermediate fp32 rounding, so no double rounding).
    """
    a = np.asarray(a, dtype=np.float64)
    bits = a.view(np.uint64)
    # bf16 keeps 8 significant bits (7 stored); fp64 has 53 -> drop 45 bits.
    drop = np.uint64(45)
    half = np.uint64(1) << (drop - np.uint64(1))
    mask = (np.uint64(1) << drop) - np.uint64(1)
    low = bits & mask
    base = bits & ~mask
    lsb = (bits >> drop) & np.uint64(1)
    up = (low > half) | ((low == half) & (lsb == np.uint64(1)))
    out = np.where(up, base + (np.uint64(1) << drop), base)
    r = out.view(np.float64)
    # Values outside the bf16 exponent range (|v| < 2^-133 or overflow) are not
    # produced by the generators; reject them loudly instead of mis-rounding.
    finite = np.isfinite(a)
    if np.any(finite & (a != 0) & ((np.abs(a) < 2.0 ** -126) | (np.abs(a) >= 2.0 ** 127))):
        raise ValueError("value outside the normal bf16 range")
    return r


def build_united_mean(Wg, Wu, Wd, way: int, out_dtype: str = "bf16"):
    """United-expert initialisation (reading D14): UE_j = element-wise mean of
    the weights of group j's members, group j = experts [j*way, min((j+1)*way, m))
    (P:149 grouping, ragged last group D15).  The mean is taken in fp64 and
    rounded once to the storage type (bf16 RNE, or fp32)."""
    outs = []
    for W in (Wg, Wu, Wd):
        W = np.asarray(W, dtype=np.float64)
        m = W.shape[0]
        G = -(-m // way)
        U = np.empty((G,) + W.shape[1:], dtype=np.float64)
        for j in range(G):
            members = W[j * way:min((j + 1) * way, m)]
            acc = np.zeros(W.shape[1:], dtype=np.float64)
            for w in members:            # member order ascending
                acc += w
            U[j] = acc / float(members.shape[0])
        if out_dtype == "bf16":
            U = round_to_bf16(U)
        elif out_dtype == "fp32":
            U = U.astype(np.float32).astype(np.float64)
        outs.append(U)
    return tuple(outs)
