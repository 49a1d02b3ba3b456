"""Expert parallelism: placement / exchange logic on CPU with
gloo process groups (world size 2 and 4), and the virtual-EP forward on one
GPU through the C ABI, both against the single-process fp64 oracle on the
rank-order concatenated batch (reading D18: one global plan)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synthetic as S
from oracle import brownout_oracle as O
from paper_2507_17133_b200.ep import EPPlanner

CFG = S.LayerConfig("ep_tiny", d=64, f=512, m=8, K=2, way=4, T=24, ratio=0.5, dtype="fp32", sigma=0.7,
                    config_id=31)


# ------------------------------------------------------------ planner (host)
@pytest.mark.parametrize("R", [1, 2, 4, 8])
def test_placement_mixtral_shape(R):
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


@pytest.mark.parametrize("R", [2, 4])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_tables_partition_every_row_exactly_once(R, ratio):
    rng = np.random.default_rng(R)
    pl = EPPlanner(m=8, way=4, f=512, world=R)
    C = rng.integers(0, 20, size=(R, 8))
    plan = O.brownout_plan(C.sum(0), ratio, 4)
    tabs = pl.tables(C, plan.exec_of_expert)
    fd = pl.feeds(plan.exec_of_expert)
    # sends match receives
    for q in range(R):
        assert tabs[q]["recv_splits"] == [tabs[r]["send_splits"][q] for r in range(R)]
    # rows received by all ranks = sum over experts of count x replicas
    reps = np.array([len(pl.group_owners[x - 8]) if x >= 8 else (1 if x >= 0 else 0) for x in plan.exec_of_expert])
    assert sum(t["R_recv"] for t in tabs) == int((C.sum(0) * reps).sum())
    # row_base blocks of one source tile its send buffer exactly
    for r in range(R):
        rb = tabs[r]["row_base"].reshape(8, pl.nrep)
        cover = np.zeros(tabs[r]["R_send"], dtype=int)
        for e in range(8):
            for rep in range(pl.nrep):
                if rb[e, rep] >= 0:
                    cover[rb[e, rep]:rb[e, rep] + C[r, e]] += 1
        assert (cover == 1).all()
    for q in range(R):
        eo = tabs[q]["exec_off"]
        assert eo[-1] == tabs[q]["R_recv"] and (np.diff(eo) >= 0).all()
        assert len(eo) - 1 == tabs[q]["n_orig"] + tabs[q]["n_united"]
    # a virtual executor is fed exactly when the plan uses its executor: an original
    # expert that executes as itself, or a united expert some member is delegated to
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


def _gloo_worker(rank, world, port, ratio, q):
    import torch.distributed as dist
    from paper_2507_17133_b200.ep import EPMoE, EPPlanner, TorchComm
    from tests.ep_cpu_ops import CpuOps
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        cfg = CFG
        lay = S.make_layer(cfg)
        uni = S.make_united_random(cfg)
        Tg = cfg.T * world
        x = S.make_tokens(cfg, T=Tg)
        L = S.make_logits(Tg, cfg.m, seed=9, sigma=cfg.sigma)
        sl = slice(rank * cfg.T, (rank + 1) * cfg.T)
        pl = EPPlanner(cfg.m, cfg.way, cfg.f, world)
        ops = CpuOps(cfg.m, cfg.K, cfg.way, ratio)
        ep = EPMoE(ops, pl, rank, (lay["Wg"], lay["Wu"], lay["Wd"]), (uni["UWg"], uni["UWu"], uni["UWd"]),
                   cfg.d, cfg.K, torch.float32)
        y = ep.forward(x[sl], lay["Wr"], TorchComm(), logits=L[sl].numpy())
        ys = [torch.empty_like(y) for _ in range(world)]
        dist.all_gather(ys, y)
        if rank == 0:
            q.put(torch.cat(ys).numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("ratio", [0.5, 1.0])
def test_ep_gloo_matches_single_process_oracle(world, ratio):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, world, port, ratio, q)) for r in range(world)]
    for p in procs:
        p.start()
    y = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg = CFG
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    Tg = cfg.T * world
    x = S.make_tokens(cfg, T=Tg)
    L = S.make_logits(Tg, cfg.m, seed=9, sigma=cfg.sigma)
    ex = tuple(lay[k].double().numpy() for k in ("Wg", "Wu", "Wd"))
    un = tuple(uni[k].double().numpy() for k in ("UWg", "UWu", "UWd"))
    ref = O.moe_forward(x.double().numpy(), None, ex, un, cfg.K, cfg.way, ratio, logits=L.double().numpy())
    den = np.abs(ref.y).max(1, keepdims=True)
    assert (np.abs(y - ref.y) / den).max() < 1e-5     # fp32 storage of the exchanged rows


# ------------------------------------------------------------ one-GPU virtual EP
@pytest.mark.gpu
@pytest.mark.parametrize("env", [{}, {"BO_PAIR_ROWS1": "1", "BO_PAIR_ROWS2": "1", "BO_SWAP_TAIL": "1"}],
                         ids=["default", "pairs_swapped_tails"])
@pytest.mark.parametrize("R", [1, 2, 4, 8])
@pytest.mark.parametrize("ratio", [0.0, 0.5, 1.0])
def test_virtual_ep_on_gpu_matches_oracle(R, ratio, env, monkeypatch):
    """Expert parallelism on one GPU (R virtual ranks, f-sliced united experts);
    the second variant runs the FFN GEMMs on CTA pairs with swapped tail tiles,
    whose united class then has its own width f / R."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    from paper_2507_17133_b200 import BrownoutMoE
    from paper_2507_17133_b200.ep import EPMoE, virtual_ep_forward
    cfg = S.LayerConfig("ep_gpu", d=256, f=512, m=8, K=2, way=4, T=96, ratio=ratio, dtype="bf16", sigma=0.7,
                        config_id=32)
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    Tg = cfg.T * R
    x = S.make_tokens(cfg, T=Tg)
    L = S.make_logits(Tg, cfg.m, seed=11, sigma=cfg.sigma)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    pl = EPPlanner(cfg.m, cfg.way, cfg.f, R)
    ranks = []
    for r in range(R):
        moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype="bf16", max_tokens=cfg.T)
        moe.set_brownout(ratio)
        ranks.append(EPMoE(moe, pl, r, (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]), cfg.d, cfg.K,
                           torch.bfloat16))
    xs = [x[r * cfg.T:(r + 1) * cfg.T].cuda() for r in range(R)]
    Ls = [L[r * cfg.T:(r + 1) * cfg.T].cuda() for r in range(R)]
    ys = virtual_ep_forward(ranks, xs, g["Wr"], logits=Ls)
    torch.cuda.synchronize()
    y = torch.cat(ys).double().cpu().numpy()
    ex = tuple(lay[k].double().numpy() for k in ("Wg", "Wu", "Wd"))
    un = tuple(uni[k].double().numpy() for k in ("UWg", "UWu", "UWd"))
    ref = O.moe_forward(x.double().numpy(), None, ex, un, cfg.K, cfg.way, ratio, logits=L.double().numpy())
    den = np.abs(ref.y).max(1, keepdims=True)
    assert (np.abs(y - ref.y) / den).max() <= 2e-2
