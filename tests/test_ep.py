"""Expert parallelism (include/brownout.h "Expert parallelism").

CPU (no GPU): the library's host placement (bo_ep_placement) against the
reference of tests/ep_reference.py; the reference exchange tables' invariants;
and the staged orchestration (ep.ep_forward_staged) with gloo process groups of
world size 2 and 4 over a CPU stand-in of the stage calls, exact and padded,
against the single-process fp64 oracle on the rank-order concatenated batch
(reading D18: one global plan, rank 0's knob).

GPU (-m gpu): the device exchange tables (k_ep_tables) bit-exact against the
reference; the virtual EP forward (R logical ranks on one GPU, collectives
emulated by device copies) through the real kernels against the oracle, exact
and padded; the padded forward captured in a CUDA graph; two processes on one
GPU exchanging through gloo with the real kernels; and the library-owned NCCL
forward (world 1), graph-captured.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthetic as S
from oracle import brownout_oracle as O
from tests.ep_reference import EPPlanner, split_tables

CFG = S.LayerConfig("ep_tiny", d=64, f=512, m=8, K=2, way=4, T=24, ratio=0.5, dtype="fp32", sigma=0.7,
                    config_id=31)


# ------------------------------------------------------------ placement (host)
@pytest.mark.parametrize("m,way,f", [(8, 4, 14336), (8, 4, 512), (8, 2, 256), (60, 8, 1408), (128, 4, 768),
                                     (5, 3, 256), (16, 16, 1024), (256, 8, 512)])
@pytest.mark.parametrize("R", [1, 2, 3, 4, 8])
def test_library_placement_matches_reference(m, way, f, R):
    from paper_2507_17133_b200.ep import placement
    pl = EPPlanner(m, way, f, R)
    for q in range(R):
        p = placement(m, way, f, R, q)
        e0, e1 = pl.local_experts(q)
        assert (p["e0"], p["e1"]) == (e0, e1)
        assert p["slices"] == pl.local_slices(q)
        assert p["f_united"] == pl.f_u and p["nrep"] == pl.nrep and p["sliced"] == int(pl.sliced)
        assert p["n_exec"] == pl.V and p["n_local"] == len(pl.local_v[q])


def test_placement_mixtral_shape():
    for R in (1, 2, 4, 8):
        pl = EPPlanner(m=8, way=4, f=14336, world=R)
        assert pl.owner == [(e * R) // 8 for e in range(8)]
        assert pl.sliced and pl.f_u == 14336 // max(1, R // 2)
        for q in range(R):   # every rank executes at least one united slice at R >= 2 (balanced ratio 1)
            if R >= 2:
                assert pl.local_slices(q)
        assert pl.nrep == max(1, R // 2)


def test_placement_falls_back_to_whole_united_when_groups_differ():
    pl = EPPlanner(m=60, way=8, f=1408, world=8)   # the paper's 60 experts, ragged last group
    assert not pl.sliced and pl.nrep == 1
    assert all(len(o) == 1 for o in pl.group_owners)


def test_placement_rejects_bad_world():
    from paper_2507_17133_b200.brownout import BrownoutError
    from paper_2507_17133_b200.ep import placement
    with pytest.raises(BrownoutError):
        placement(8, 4, 512, 9, 0)
    with pytest.raises(BrownoutError):
        placement(8, 4, 512, 2, 2)


# ------------------------------------------------------- reference tables (host)
@pytest.mark.parametrize("padded", [False, True])
@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_tables_partition_every_row_exactly_once(R, ratio, padded):
    rng = np.random.default_rng(R)
    pl = EPPlanner(m=8, way=4, f=512, world=R)
    T, K = 20, 2
    C = rng.integers(0, 20, size=(R, 8))
    C = C * (T * K) // np.maximum(C.sum(1, keepdims=True), 1)     # each source <= T*K assignments
    cap = T * K
    plan = O.brownout_plan(C.sum(0), ratio, 4)
    tabs = [pl.tables(C, plan.exec_of_expert, q, padded, cap) for q in range(R)]
    for q in range(R):   # send / recv splits agree between the two ends
        assert list(tabs[q]["recv_rows"]) == [int(tabs[r]["send_rows"][q]) for r in range(R)]
        assert all(n <= cap for n in tabs[q]["send_rows"])
    reps = np.array([len(pl.group_owners[x - 8]) if x >= 8 else (1 if x >= 0 else 0) for x in plan.exec_of_expert])
    assert sum(int(t["totals"][0]) for t in tabs) == int((C.sum(0) * reps).sum())
    for r in range(R):   # row_base blocks of one source tile its send buffer without overlap
        rb = tabs[r]["row_base"].reshape(8, pl.nrep)
        cover = np.zeros(R * cap, dtype=int)
        for e in range(8):
            for rep in range(pl.nrep):
                if rb[e, rep] >= 0:
                    cover[rb[e, rep]:rb[e, rep] + C[r, e]] += 1
        assert cover.max() <= 1 and cover.sum() == int(tabs[r]["send_rows"].sum())
        if padded:   # destination q's rows lie inside [q cap, (q + 1) cap)
            for q in range(R):
                seg = cover[q * cap:(q + 1) * cap]
                assert seg.sum() == tabs[r]["send_rows"][q] and seg[:tabs[r]["send_rows"][q]].all()
    for q in range(R):
        t = tabs[q]
        assert t["exec_off"][-1] == t["totals"][0] and (np.diff(t["exec_off"]) >= 0).all()
        assert (np.diff(t["fwd_dst"]) == t["fwd_len"]).all()          # grouped blocks are contiguous
        assert (np.diff(t["inv_dst"]) >= t["inv_len"]).all()           # receive blocks ascending, disjoint
    fd = pl.feeds(plan.exec_of_expert)
    ex = plan.exec_of_expert
    for v, (q, kind, idx, _s) in enumerate(pl.vexec):
        used = (ex[idx] == idx) if kind == "o" else bool((ex == 8 + idx).any())
        assert (len(fd[v]) > 0) == used, (v, kind, idx)


# ------------------------------------------------------------------ gloo path
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_cpu_worker(rank, world, port, ratio, padded, q):
    import torch.distributed as dist
    from paper_2507_17133_b200.ep import TorchComm, ep_forward_staged
    from tests.ep_cpu_ops import CpuEPContext
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = CFG
        lay = S.make_layer(cfg)
        uni = S.make_united_random(cfg)
        Ts = [cfg.T - 5 * r for r in range(world)]            # uneven (bursty) local batches
        Tg = sum(Ts)
        x = S.make_tokens(cfg, T=Tg)
        L = S.make_logits(Tg, cfg.m, seed=9, sigma=cfg.sigma)
        t0 = sum(Ts[:rank])
        sl = slice(t0, t0 + Ts[rank])
        # rank 1 carries a different knob: the plan must use rank 0's (EP contract)
        ctx = CpuEPContext(cfg.m, cfg.f, cfg.d, cfg.K, cfg.way, world, rank, cfg.T,
                           ratio if rank == 0 else 0.0, padded=padded)
        ex, un = ctx.local_weights((lay["Wg"], lay["Wu"], lay["Wd"]), (uni["UWg"], uni["UWu"], uni["UWd"]))
        y = ep_forward_staged(ctx, x[sl], lay["Wr"], ex, un, TorchComm(), logits=L[sl].numpy())
        yp = torch.zeros(cfg.T, cfg.d, dtype=y.dtype)   # gloo gathers equal sizes: pad to the largest batch
        yp[:Ts[rank]] = y
        ys = [torch.empty_like(yp) for _ in range(world)]
        dist.all_gather(ys, yp)
        if rank == 0:
            q.put(torch.cat([ys[r][:Ts[r]] for r in range(world)]).numpy())
    finally:
        dist.destroy_process_group()


def _oracle_concat(cfg, Tg, ratio, lay, uni, L):
    x = S.make_tokens(cfg, T=Tg)
    ex = tuple(lay[k].double().numpy() for k in ("Wg", "Wu", "Wd"))
    un = tuple(uni[k].double().numpy() for k in ("UWg", "UWu", "UWd"))
    return O.moe_forward(x.double().numpy(), None, ex, un, cfg.K, cfg.way, ratio, logits=L.double().numpy())


@pytest.mark.parametrize("world,ratio,padded", [(2, 0.5, False), (2, 1.0, True), (4, 0.5, True), (4, 1.0, False)])
def test_ep_gloo_matches_single_process_oracle(world, ratio, padded):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_cpu_worker, args=(r, world, port, ratio, padded, q)) for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = CFG
    Tg = sum(cfg.T - 5 * r for r in range(world))
    lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
    ref = _oracle_concat(cfg, Tg, ratio, lay, uni, S.make_logits(Tg, cfg.m, seed=9, sigma=cfg.sigma))
    den = np.abs(ref.y).max(1, keepdims=True)
    assert (np.abs(y - ref.y) / den).max() < 1e-5     # fp32 storage of the exchanged rows


# ------------------------------------------------------------------ GPU paths
GCFG = S.LayerConfig("ep_gpu", d=256, f=512, m=8, K=2, way=4, T=96, ratio=0.5, dtype="bf16", sigma=0.7,
                     config_id=32)


def _gpu_layer(cfg, R, ratio, Ts=None):
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    Ts = Ts or [cfg.T] * R
    Tg = sum(Ts)
    x = S.make_tokens(cfg, T=Tg)
    L = S.make_logits(Tg, cfg.m, seed=11, sigma=cfg.sigma)
    ref = _oracle_concat(cfg, Tg, ratio, lay, uni, L)
    return lay, uni, x, L, Ts, ref


def _context(cfg, R, r, ratio, padded, g, u):
    from paper_2507_17133_b200 import BrownoutMoE
    from paper_2507_17133_b200.ep import EPContext
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T)
    moe.set_brownout(ratio)
    c = EPContext(moe, R, r, cfg.T, padded=int(padded))
    return c, c.local_weights((g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]))


def _contexts(cfg, R, ratio, padded, g, u):
    out = [_context(cfg, R, r, ratio, padded, g, u) for r in range(R)]
    return [c for c, _ in out], [w for _, w in out]


def _rel(y, ref):
    den = np.abs(ref).max(1, keepdims=True)
    den = np.where(den == 0, 1.0, den)
    return float((np.abs(y - ref) / den).max())


@pytest.mark.gpu
@pytest.mark.parametrize("padded", [False, True], ids=["exact", "padded"])
@pytest.mark.parametrize("R", [2, 4, 8])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_device_tables_match_reference(R, ratio, padded):
    """k_ep_tables (device) equals the reference tables on every rank, bit for bit."""
    from paper_2507_17133_b200.ep import virtual_ep_forward
    cfg = GCFG
    Ts = [cfg.T - 7 * r for r in range(R)]
    lay, uni, x, L, Ts, ref = _gpu_layer(cfg, R, ratio, Ts)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    ctxs, weights = _contexts(cfg, R, ratio, padded, g, u)
    offs = np.cumsum([0] + Ts)
    xs = [x[offs[r]:offs[r + 1]].cuda() for r in range(R)]
    Ls = [L[offs[r]:offs[r + 1]].cuda() for r in range(R)]
    virtual_ep_forward(ctxs, xs, g["Wr"], weights, logits=Ls)
    torch.cuda.synchronize()
    pl = EPPlanner(cfg.m, cfg.way, cfg.f, R)
    C = np.stack([np.bincount(ref.ids[offs[r]:offs[r + 1]].reshape(-1), minlength=cfg.m) for r in range(R)])
    for r, c in enumerate(ctxs):
        assert np.array_equal(c.plan()["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert)
        want = pl.tables(C, ref.plan.exec_of_expert, r, padded, c.cap)
        nl = len(pl.local_v[r])
        nb = nl * R
        n = cfg.m * pl.nrep + 2 * R + 6 * nb + 2 + 2 * (nl + 1) + 2
        got = split_tables(c._view(c.L.tables, n, torch.int32).cpu().numpy(), cfg.m, pl.nrep, R, nl)
        for k, v in got.items():
            assert np.array_equal(v, want[k]), (r, k, v, want[k])


@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"BO_PAIR_ROWS1": "1", "BO_PAIR_ROWS2": "1"}], ids=["default", "pairs"])
@pytest.mark.parametrize("padded", [False, True], ids=["exact", "padded"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_virtual_ep_on_gpu_matches_oracle(R, ratio, padded, env, monkeypatch):
    """EP through the real kernels on one GPU (R virtual ranks, uneven batches,
    f-sliced united experts) against the oracle on the concatenated batch."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_2507_17133_b200.ep import virtual_ep_forward
    cfg = GCFG
    Ts = [cfg.T - 9 * r for r in range(R)]
    lay, uni, x, L, Ts, ref = _gpu_layer(cfg, R, ratio, Ts)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    ctxs, weights = _contexts(cfg, R, ratio, padded, g, u)
    offs = np.cumsum([0] + Ts)
    xs = [x[offs[r]:offs[r + 1]].cuda() for r in range(R)]
    Ls = [L[offs[r]:offs[r + 1]].cuda() for r in range(R)]
    ys = virtual_ep_forward(ctxs, xs, g["Wr"], weights, logits=Ls)
    torch.cuda.synchronize()
    assert _rel(torch.cat(ys).double().cpu().numpy(), ref.y) <= 2e-2


@pytest.mark.gpu
@pytest.mark.parametrize("R", [2, 4])
def test_virtual_ep_padded_graph_capture(R):
    """Padded mode has no host synchronisation: the whole R-rank forward (route,
    count exchange, plan, tables, dispatch, exchanges, FFN, combine) is captured
    in one CUDA graph and replayed on a new batch."""
    from paper_2507_17133_b200.ep import virtual_ep_forward
    cfg = GCFG
    ratio = 0.5
    lay, uni, x, L, Ts, ref = _gpu_layer(cfg, R, ratio)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    ctxs, weights = _contexts(cfg, R, ratio, True, g, u)
    xs = [torch.zeros(cfg.T, cfg.d, dtype=torch.bfloat16, device="cuda") for _ in range(R)]
    Ls = [torch.zeros(cfg.T, cfg.m, dtype=torch.float32, device="cuda") for _ in range(R)]
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        virtual_ep_forward(ctxs, xs, g["Wr"], weights, logits=Ls)   # warm-up outside the capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        ys = virtual_ep_forward(ctxs, xs, g["Wr"], weights, logits=Ls)
    for r in range(R):
        xs[r].copy_(x[r * cfg.T:(r + 1) * cfg.T])
        Ls[r].copy_(L[r * cfg.T:(r + 1) * cfg.T])
    graph.replay()
    torch.cuda.synchronize()
    assert _rel(torch.cat(ys).double().cpu().numpy(), ref.y) <= 2e-2


def _gloo_gpu_worker(rank, world, port, ratio, padded, q):
    import torch.distributed as dist
    from paper_2507_17133_b200.ep import TorchComm, ep_forward_staged
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = GCFG
        Ts = [cfg.T - 9 * r for r in range(world)]
        lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
        Tg = sum(Ts)
        x = S.make_tokens(cfg, T=Tg)
        L = S.make_logits(Tg, cfg.m, seed=11, sigma=cfg.sigma)
        g = {k: v.cuda() for k, v in lay.items()}
        u = {k: v.cuda() for k, v in uni.items()}
        ctx, (ex, un) = _context(cfg, world, rank, ratio if rank == 0 else 0.0, padded, g, u)
        t0 = sum(Ts[:rank])
        y = ep_forward_staged(ctx, x[t0:t0 + Ts[rank]].cuda(), g["Wr"], ex, un, TorchComm(),
                              logits=L[t0:t0 + Ts[rank]].cuda())
        torch.cuda.synchronize()
        yp = torch.zeros(cfg.T, cfg.d, dtype=torch.float32)
        yp[:Ts[rank]] = y.float().cpu()
        ys = [torch.empty_like(yp) for _ in range(world)]
        dist.all_gather(ys, yp)
        if rank == 0:
            q.put(torch.cat([ys[r][:Ts[r]] for r in range(world)]).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("padded", [False, True], ids=["exact", "padded"])
def test_two_processes_one_gpu_gloo_real_kernels(padded):
    """Two processes (one CUDA context each on the same GPU) run the staged EP
    forward through the library's kernels and exchange over gloo; rank 1's knob
    differs and rank 0's must win.  y equals the oracle on the concatenated batch."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world, ratio = 2, 0.5
    procs = [ctx.Process(target=_gloo_gpu_worker, args=(r, world, port, ratio, padded, q)) for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = GCFG
    Ts = [cfg.T - 9 * r for r in range(world)]
    lay, uni, x, L, Ts, ref = _gpu_layer(cfg, world, ratio, Ts)
    assert _rel(y.astype(np.float64), ref.y) <= 2e-2


def _nccl_world1_worker(padded, q):
    """Child process of test_nccl_world1_library_forward: returns y's relative error."""
    from paper_2507_17133_b200.ep import EPContext
    cfg = GCFG
    ratio = 0.5
    lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    ctx, (ex, un) = _context(cfg, 1, 0, ratio, padded, g, u)
    ctx.init_nccl(EPContext.nccl_unique_id())
    xe, Wre = S.make_exact_router_inputs(cfg, T=cfg.T)
    ex64 = tuple(lay[k].double().numpy() for k in ("Wg", "Wu", "Wd"))
    un64 = tuple(uni[k].double().numpy() for k in ("UWg", "UWu", "UWd"))
    want = O.moe_forward(xe.double().numpy(), Wre.double().numpy(), ex64, un64, cfg.K, cfg.way, ratio).y
    xe, Wre = xe.cuda(), Wre.cuda()
    s = torch.cuda.Stream()
    xin = torch.zeros_like(xe)
    with torch.cuda.stream(s):
        y = ctx.forward(xin, Wre, ex, un)      # warm-up
    torch.cuda.synchronize()
    graph = None
    if padded:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            y = ctx.forward(xin, Wre, ex, un)
        xin.copy_(xe)
        graph.replay()
    else:
        xin.copy_(xe)
        with torch.cuda.stream(s):
            y = ctx.forward(xin, Wre, ex, un)
    torch.cuda.synchronize()
    err = _rel(y.double().cpu().numpy(), want)
    # A graph that captured NCCL work holds the communicator's persistent resources:
    # destroy it before the communicator (bo_ep_destroy; include/brownout.h).
    del graph
    torch.cuda.synchronize()
    ctx.close()
    q.put(float(err))


@pytest.mark.gpu
@pytest.mark.parametrize("padded", [True, False], ids=["padded_graph", "exact"])
def test_nccl_world1_library_forward(padded):
    """The library-owned NCCL path (bo_ep_init + bo_ep_forward: ncclAllGather of
    the count rows, grouped ncclSend / ncclRecv exchanges) on a world of one,
    captured in a CUDA graph in padded mode.  Router inputs are exactly
    representable, so the oracle's own Eq. 8 path is the reference.  Runs in a
    child process under a deadline, so a communicator that never finishes (or a
    teardown that blocks) fails the test instead of hanging the suite."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_world1_worker, args=(padded, q))
    p.start()
    try:
        err = q.get(timeout=300)
    except Exception:
        p.kill()
        pytest.fail("NCCL world-1 forward did not finish within 300 s")
    p.join(timeout=120)
    if p.is_alive():
        p.kill()
        pytest.fail("NCCL world-1 process did not exit (communicator teardown blocked)")
    assert p.exitcode == 0
    assert err <= 2e-2
