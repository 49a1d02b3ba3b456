"""Small forwards over the library's code paths, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): bf16 decode and CTA-pair prefill,
fp32 (tf32), shared experts, united-row de-duplication, full brownout, the fused
combine, the decode split-K GEMM2 and the swapped GEMM1 tail tiles.  Exits
non-zero if the fused combine disagrees bitwise with the separate kernel."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2507_17133_b200 import BrownoutMoE  # noqa: E402


def run(cfg, ratio=0.5, mode="partial", dedup=False, logits=True):
    lay = {k: v.cuda() for k, v in S.make_layer(cfg).items()}
    x = S.make_tokens(cfg, batch_index=2).cuda()
    moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T, dedup=dedup,
                      num_shared=cfg.Ns)
    ex = (lay["Wg"], lay["Wu"], lay["Wd"])
    sh = (lay["SWg"], lay["SWu"], lay["SWd"]) if cfg.Ns else None
    U = moe.build_united(*ex)
    moe.set_brownout(ratio, mode)
    L = S.make_logits(cfg.T, cfg.m, seed=2, sigma=cfg.sigma).cuda() if logits else None
    y = moe.forward(x, lay["Wr"], ex, U, logits=L, shared=sh)
    torch.cuda.synchronize()
    return y


def run_env(env, *a, **k):
    old = {n: os.environ.get(n) for n in env}
    os.environ.update(env)
    try:
        return run(*a, **k)
    finally:
        for n, v in old.items():
            if v is None:
                os.environ.pop(n, None)
            else:
                os.environ[n] = v


def main():
    small = S.LayerConfig("s", d=256, f=512, m=8, K=2, way=4, T=200, ratio=0.5, dtype="bf16", sigma=0.7,
                          config_id=71)
    pair = S.LayerConfig("p", d=256, f=256, m=8, K=2, way=4, T=1100, ratio=0.5, dtype="bf16", sigma=0.5,
                         config_id=72)
    fp32 = S.LayerConfig("f", d=64, f=128, m=8, K=2, way=4, T=32, ratio=0.5, dtype="fp32", sigma=0.0, config_id=1)
    qwen = S.LayerConfig("q", d=256, f=256, m=128, K=8, way=4, T=130, ratio=0.5, dtype="bf16", sigma=0.5,
                         config_id=73)
    shared = S.LayerConfig("sh", d=256, f=256, m=8, K=2, way=4, T=150, ratio=0.5, dtype="bf16", sigma=0.5,
                           config_id=74, Ns=2)
    # GEMM2's last-wave split: 48 pair tiles of 64 k-blocks shared out over the pairs
    tail = S.LayerConfig("ts", d=512, f=4096, m=8, K=2, way=4, T=3000, ratio=0.0, dtype="bf16", sigma=0.3,
                         config_id=101)
    bad = 0
    for name, f in [
        ("decode", lambda: run(small)),
        ("decode_ratio1", lambda: run(small, ratio=1.0)),
        ("router_gpu", lambda: run(small, logits=False)),   # k_route_fused (decode-sized, m <= 32)
        ("router_gpu_unfused", lambda: run_env({"BO_ROUTE_FUSED": "0"}, small, logits=False)),
        ("router_gpu_fused_shared", lambda: run(shared, logits=False)),
        ("prefill_pairs_fused_combine", lambda: run(pair)),   # GEMM1 swapped tail tiles (default)
        ("prefill_gemm2_tail_split", lambda: run(tail)),
        ("decode_gemm2_splitk", lambda: run_env({"BO_GEMM2_SPLITK": "1"}, small)),
        ("fp32", lambda: run(fp32)),
        ("qwen_like_tc_router", lambda: run(qwen, logits=False)),
        ("shared", lambda: run(shared)),
        ("dedup", lambda: run(small, ratio=1.0, dedup=True)),
        ("full_mode", lambda: run(small, ratio=0.6, mode="full")),
    ]:
        f()
        print("ok", name, flush=True)
    for name, a, b in [("fused_combine", lambda: run_env({"BO_FUSED_COMBINE": "0"}, pair),
                        lambda: run_env({"BO_FUSED_COMBINE": "1"}, pair))]:
        if not torch.equal(a(), b()):
            bad += 1
            print("MISMATCH", name)
        else:
            print("ok", name, flush=True)
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
