"""Interleaved A/B timing of one library knob (env var read at bo_create).

    python scripts/ab.py --env BO_FUSED_COMBINE=0 \
        --workloads mixtral_prefill:0.5,mixtral_decode:1.0 --reps 6

A = default handle, B = handle created with the env var set; both share the
layer's weights / tokens / output and alternate graph replays of K steps
(bench.time_steps), so GPU clock / power drift hits both arms alike.  Prints
one JSON line: per workload the median ms/step and per-kernel medians of each arm.
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
    ap.add_argument("--env", required=True, help="NAME=VALUE for arm B")
    ap.add_argument("--workloads", default="mixtral_prefill:0.5,mixtral_decode:0.0,mixtral_decode:0.5,"
                                           "mixtral_decode:1.0,qwen3_30b_a3b_prefill:0.5")
    ap.add_argument("--reps", type=int, default=6)
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    import torch
    import bench
    import synthetic as S
    from paper_2507_17133_b200 import BrownoutMoE
    name, val = args.env.split("=", 1)
    out = {"env_b": args.env}
    cache = {}
    for wl in args.workloads.split(","):
        wname, ratio = wl.split(":")
        cfg = S.CONFIGS[wname]
        if wname not in cache:
            cache.clear()
            torch.cuda.empty_cache()
            cache[wname] = bench.Layer(cfg, "cuda")
        layer = cache[wname]
        moe_a = layer.moe
        old = os.environ.get(name)
        os.environ[name] = val
        moe_b = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=layer.T,
                            num_shared=cfg.Ns)
        if cfg.Ns:
            moe_b.set_shared_experts(layer.lay["SWg"], layer.lay["SWu"], layer.lay["SWd"])
        if old is None:
            del os.environ[name]
        else:
            os.environ[name] = old
        res = {"A": {"ms": [], "k": []}, "B": {"ms": [], "k": []}}
        for rep in range(args.reps):
            for arm, moe in (("A", moe_a), ("B", moe_b)) if rep % 2 == 0 else (("B", moe_b), ("A", moe_a)):
                layer.moe = moe
                moe.set_brownout(float(ratio))
                ms, kern = bench.time_steps(layer, args.steps, 3, False)
                res[arm]["ms"].append(ms / args.steps)
                res[arm]["k"].append(kern)
        layer.moe = moe_a
        summ = {}
        for arm in ("A", "B"):
            ks = {}
            for k in res[arm]["k"][0]:
                if not k.startswith("_"):
                    ks[k] = round(statistics.median(x[k] for x in res[arm]["k"] if k in x), 4)
            summ[arm] = {"ms_median": round(statistics.median(res[arm]["ms"]), 4),
                         "ms_all": [round(v, 4) for v in res[arm]["ms"]], "kernel_ms": ks}
        summ["B_over_A"] = round(summ["B"]["ms_median"] / summ["A"]["ms_median"], 4)
        out[wl] = summ
        print(wl, summ["A"]["ms_median"], summ["B"]["ms_median"], summ["B_over_A"], file=sys.stderr, flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
