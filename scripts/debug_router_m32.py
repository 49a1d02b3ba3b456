"""Debug: tcgen05 router (m = 32) top-K / plan vs the oracle on exact inputs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import synthetic as S
from oracle import brownout_oracle as O
from paper_2507_17133_b200 import BrownoutMoE
C = S.LayerConfig
cfg = C("m32_tc_bn32", d=3072, f=128, m=32, K=4, way=8, T=200, ratio=0.5, dtype="bf16", config_id=69)
for ties in (True, False):
    x, Wr = S.make_exact_router_inputs(cfg, ties=ties)
    lay, uni = S.make_layer(cfg), S.make_united_random(cfg)
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T)
    moe.set_brownout(0.5)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    moe.forward(x.cuda(), Wr.cuda(), (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]))
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(cfg.T)
    L, ids, gw, plan, perm = O.route(x.double().numpy(), Wr.double().numpy(), cfg.K, cfg.way, 0.5, O.PARTIAL, None, False)
    gi = dbg["topk_id"].cpu().numpy()
    print("kernels", moe.last_kernels())
    print("ties", ties, "logits equal", np.array_equal(dbg["logits"].cpu().double().numpy(), L),
          "ids equal", np.array_equal(gi, ids), "bad rows", np.where((gi != ids).any(1))[0][:10].tolist())
    bad = np.where((gi != ids).any(1))[0][:3]
    for t in bad:
        print("  t", t, "gpu", gi[t].tolist(), "ref", ids[t].tolist(), "logits", sorted(L[t].tolist(), reverse=True)[:6])
    print("  counts equal", np.array_equal(dbg["counts"].cpu().numpy(), plan.counts),
          "exec equal", np.array_equal(dbg["exec_of_expert"].cpu().numpy(), plan.exec_of_expert))
    print("  stats gpu", dbg["stats"].cpu().tolist(), "ref", plan.stats)
