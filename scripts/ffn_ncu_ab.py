"""Kernel-time A/B under ncu's serialised launch list: one workload, one handle
per env setting (argv[3:] = NAME=VALUE, applied before bo_create), `reps`
forwards each.  Usage: ncu --metrics gpu__time_duration.sum -k regex:k_grouped_gemm --csv \
    python scripts/ffn_ncu_ab.py mixtral_prefill 0.5 BO_SWAP_TAIL=0
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
import torch
import synthetic as S
from paper_2507_17133_b200 import BrownoutMoE

cfg = S.CONFIGS[sys.argv[1]]
ratio = float(sys.argv[2])
lay = S.make_layer(cfg, device="cuda")
uni = S.make_united_random(cfg, device="cuda")
x = S.make_tokens(cfg, device="cuda")
moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T, num_shared=cfg.Ns)
moe.set_brownout(ratio)
shared = (lay["SWg"], lay["SWu"], lay["SWd"]) if cfg.Ns else None
for _ in range(int(os.environ.get("REPS", "6"))):
    moe.forward(x, lay["Wr"], (lay["Wg"], lay["Wu"], lay["Wd"]), (uni["UWg"], uni["UWu"], uni["UWd"]), shared=shared)
torch.cuda.synchronize()
