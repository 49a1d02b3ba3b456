"""Interleaved A/B timing of library knobs (env vars read at bo_create).

    python scripts/ab.py --env BO_FUSED_COMBINE=0 [--env "BO_X=1;BO_Y=2" ...] \
        --workloads mixtral_prefill:0.5,mixtral_decode:1.0 --reps 6

Arm A = default handle; arm B, C, ... = handles created with each --env's
variables set.  All arms share the layer's weights / tokens / output and
alternate graph replays of K steps (bench.time_steps, rotating order), so GPU
clock / power drift hits every arm alike.  Prints one JSON line: per workload
the median ms/step and per-kernel medians of each arm.
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--env", action="append", required=True, help="NAME=VALUE[;NAME=VALUE] for one extra arm")
    ap.add_argument("--workloads", default="mixtral_prefill:0.5,mixtral_decode:0.0,mixtral_decode:0.5,"
                                           "mixtral_decode:1.0,qwen3_30b_a3b_prefill:0.5")
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import bench
    import synthetic as S
    from paper_2507_17133_b200 import BrownoutMoE
    arms = {"A": {}}
    for i, e in enumerate(args.env):
        arms[chr(ord("B") + i)] = dict(kv.split("=", 1) for kv in e.split(";"))
    out = {"arms": arms}
    cache = {}
    for wl in args.workloads.split(","):
        wname, ratio = wl.split(":")
        cfg = S.CONFIGS[wname]
        if wname not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[wname] = bench.Layer(cfg, "cuda")
        layer = cache[wname]
        moes, weights, wss = {}, {}, {}
        base_w = (layer.lay, layer.united)
        base_ws = layer.ws
        for arm, env in arms.items():
            if arm == "A":
                moes[arm] = layer.moe
                weights[arm] = base_w
                wss[arm] = base_ws
                continue
            env = dict(env)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=layer.T,
                              num_shared=cfg.Ns)
            lay = layer.lay
            uni = layer.united
            weights[arm] = (lay, uni)
            if cfg.Ns:
                moe.set_shared_experts(lay["SWg"], lay["SWu"], lay["SWd"])
            for k, v in old.items():
                if v is None:
                    del os.environ[k]
                else:
                    os.environ[k] = v
            moes[arm] = moe
            wss[arm] = moe.workspace(layer.T, "cuda")   # an arm's options may change the layout
        moe_a = layer.moe
        res = {arm: {"ms": [], "k": []} for arm in arms}
        names = list(arms)
        for rep in range(args.reps):
            order = names[rep % len(names):] + names[:rep % len(names)]
            for arm in order:
                layer.moe = moes[arm]
                layer.lay, layer.united = weights[arm]
                layer.ws = wss[arm]
                layer.moe.set_brownout(float(ratio))
                ms, kern = bench.time_steps(layer, args.steps, 3, False)
                res[arm]["ms"].append(ms / args.steps)
                res[arm]["k"].append(kern)
        layer.moe = moe_a
        layer.lay, layer.united = base_w
        layer.ws = base_ws
        summ = {}
        for arm in names:
            ks = {}
            for k in res[arm]["k"][0]:
                if not k.startswith("_"):
                    ks[k] = round(statistics.median(x[k] for x in res[arm]["k"] if k in x), 4)
            summ[arm] = {"ms_median": round(statistics.median(res[arm]["ms"]), 4),
                         "ms_all": [round(v, 4) for v in res[arm]["ms"]], "kernel_ms": ks}
        out[wl] = summ
        print(wl, " ".join(f"{a}={summ[a]['ms_median']}" for a in names), file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
