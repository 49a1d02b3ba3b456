"""Parity soak: many random layer shapes / ratios / modes / library knobs against
the fp64 oracle (the contract of tests/test_gpu_parity.py at a larger scale).

    python scripts/soak.py --n 200 --seed 1        # prints one line per failure + a summary

Each case draws m, K, way, d, f, T, dtype, sigma, ratio, mode (partial / full),
de-duplication, shared experts, residual, T up to 2500 (decode and CTA-pair
prefill schedules) and one engine knob; routing, plan and permutation must be
bit-exact given injected fp32 logits, the output within 2e-2 (row-relative)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as S  # noqa: E402
from oracle import brownout_oracle as O  # noqa: E402

KNOBS = [{}, {"BO_FUSED_COMBINE": "1"}, {"BO_FUSED_COMBINE": "0"}, {"BO_CTA_PAIRS": "0"}, {"BO_GEMM2_SPLITK": "1"},
         {"BO_TILE_ALT": "0"}, {"BO_DECODE_PAIR2": "0"},
         {"BO_PAIR_ROWS1": "1", "BO_PAIR_ROWS2": "1"}, {"BO_B_POLICY": "1"},
         {"BO_PAIR_ROWS1": "1", "BO_SWAP_TAIL": "0"}, {"BO_TMA_STORE": "0", "BO_PDL": "0"},
         {"BO_ROUTE_FUSED": "0"}]


def case(rng, i):
    m = int(rng.choice([2, 5, 8, 16, 60, 128]))
    K = int(rng.integers(1, min(m, 8) + 1))
    way = int(rng.choice([1, 2, 3, 4, 8, m]))
    dt = "fp32" if rng.random() < 0.2 else "bf16"
    d = int(rng.choice([128, 256, 384, 512]))
    f = int(rng.choice([128, 256, 384, 512]))
    T = int(rng.choice([1, 7, 64, 200, 513, 1100, 2500]))
    Ns = int(rng.choice([0, 0, 0, 1, 2]))
    dedup = Ns == 0 and rng.random() < 0.2
    mode = "full" if (not dedup and rng.random() < 0.15) else "partial"
    ratio = float(rng.choice([0.0, 0.25, 0.5, 0.75, 0.9, 1.0]))
    cfg = S.LayerConfig(f"soak{i}", d=d, f=f, m=m, K=K, way=way, T=T, ratio=ratio, dtype=dt,
                        sigma=float(rng.choice([0.0, 0.5, 1.0])), config_id=500 + i, Ns=Ns)
    knob = KNOBS[int(rng.integers(0, len(KNOBS)))]
    # 30 %: the production router (Eq. 8 on the GPU, the fused decode routing launch for small
    # T) on exactly representable inputs, compared with the oracle's own Eq. 8 path
    prod = bool(rng.random() < 0.3)
    return cfg, mode, dedup, bool(rng.random() < 0.3), knob, prod


def run(cfg, mode, dedup, residual, knob, prod=False):
    from paper_2507_17133_b200 import BrownoutMoE
    old = {k: os.environ.get(k) for k in knob}
    os.environ.update(knob)
    try:
        moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, add_residual=residual,
                          max_tokens=cfg.T, dedup=dedup, num_shared=cfg.Ns)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    lay = S.make_layer(cfg)
    uni = S.make_united_random(cfg)
    x = S.make_tokens(cfg, batch_index=cfg.config_id)
    L = S.make_logits(cfg.T, cfg.m, seed=cfg.config_id, sigma=cfg.sigma)
    Wr = lay["Wr"]
    if prod:
        x, Wr = S.make_exact_router_inputs(cfg, ties=cfg.config_id % 2 == 0)
        prod = S.exactness_bound(x, Wr) < 2.0 ** 11   # else injected logits as usual
    moe.set_brownout(cfg.ratio, mode)
    g = {k: v.cuda() for k, v in lay.items()}
    u = {k: v.cuda() for k, v in uni.items()}
    sh = (g["SWg"], g["SWu"], g["SWd"]) if cfg.Ns else None
    y = moe.forward(x.cuda(), Wr.cuda(), (g["Wg"], g["Wu"], g["Wd"]), (u["UWg"], u["UWu"], u["UWd"]),
                    logits=None if prod else L.cuda(), shared=sh)
    torch.cuda.synchronize()
    dbg = moe.debug_arrays(cfg.T)
    npd = lambda t: t.detach().cpu().double().numpy()
    ex = tuple(npd(lay[k]) for k in ("Wg", "Wu", "Wd"))
    un = tuple(npd(uni[k]) for k in ("UWg", "UWu", "UWd"))
    shn = tuple(npd(lay[k]) for k in ("SWg", "SWu", "SWd")) if cfg.Ns else None
    ref = O.moe_forward(npd(x), npd(Wr) if prod else None, ex, un, cfg.K, cfg.way, cfg.ratio,
                        mode=O.FULL if mode == "full" else O.PARTIAL, logits=None if prod else L.double().numpy(),
                        add_residual=residual, dedup=dedup, shared=shn)
    errs = []
    if not np.array_equal(dbg["topk_id"].cpu().numpy(), ref.ids):
        errs.append("topk")
    if not np.array_equal(dbg["exec_of_expert"].cpu().numpy(), ref.plan.exec_of_expert):
        errs.append("plan")
    ro = dbg["row_of"].cpu().numpy().reshape(cfg.T, cfg.K + cfg.Ns)[:, :cfg.K].reshape(-1)   # routed slots
    if not np.array_equal(ro, ref.perm.row_of):
        errs.append("row_of")
    yr = ref.y
    den = np.abs(yr).max(axis=1)
    den = np.where(den == 0, 1.0, den)
    e = float((np.abs(npd(y) - yr).max(axis=1) / den).max())
    if e > 2e-2:
        errs.append(f"y rel err {e:.3e}")
    return errs


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=100)
    ap.add_argument("--seed", type=int, default=1)
    args = ap.parse_args()
    from paper_2507_17133_b200.build import build
    build()
    rng = np.random.default_rng(args.seed)
    fails = 0
    for i in range(args.n):
        cfg, mode, dedup, residual, knob, prod = case(rng, i)
        try:
            errs = run(cfg, mode, dedup, residual, knob, prod)
        except Exception as ex:   # noqa: BLE001
            errs = [f"exception {type(ex).__name__}: {ex}"]
        if errs:
            fails += 1
            print("FAIL", cfg, mode, "dedup" if dedup else "", "res" if residual else "", "router" if prod else "",
                  knob, errs, flush=True)
    print(f"soak: {args.n - fails}/{args.n} passed", flush=True)
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
