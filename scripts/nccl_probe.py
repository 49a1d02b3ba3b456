"""Probe of the library-owned NCCL EP path on a world of one (step-by-step prints)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2507_17133_b200 import BrownoutMoE  # noqa: E402
from paper_2507_17133_b200.ep import EPContext  # noqa: E402

t0 = time.time()
log = lambda *a: print(f"[{time.time() - t0:7.2f}s]", *a, flush=True)
cfg = S.LayerConfig("ep_gpu", d=256, f=512, m=8, K=2, way=4, T=96, ratio=0.5, dtype="bf16", sigma=0.7, config_id=32)
lay = {k: v.cuda() for k, v in S.make_layer(cfg).items()}
uni = {k: v.cuda() for k, v in S.make_united_random(cfg).items()}
moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype="bf16", max_tokens=cfg.T)
moe.set_brownout(0.5)
padded = int(sys.argv[1]) if len(sys.argv) > 1 else 1
ctx = EPContext(moe, 1, 0, cfg.T, padded=padded)
ex, un = ctx.local_weights((lay["Wg"], lay["Wu"], lay["Wd"]), (uni["UWg"], uni["UWu"], uni["UWd"]))
log("ctx ok, padded", ctx.padded)
uid = EPContext.nccl_unique_id()
log("unique id ok")
ctx.init_nccl(uid)
log("comm init ok")
x = S.make_tokens(cfg).cuda()
y = ctx.forward(x, lay["Wr"], ex, un)
torch.cuda.synchronize()
log("eager forward ok", float(y.float().abs().sum()))
if ctx.padded:
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        y2 = ctx.forward(x, lay["Wr"], ex, un)
    log("captured")
    g.replay()
    torch.cuda.synchronize()
    log("replayed", bool(torch.equal(y, y2)))
