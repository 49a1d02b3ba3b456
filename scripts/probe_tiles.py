"""Per-tile timeline of the grouped GEMMs from the instrumentation build
(build.py --variant probe; loaded with BO_LIB=probe).

    BO_LIB=probe python scripts/probe_tiles.py mixtral_decode 1.0 [NAME=VALUE ...] > out.json

Runs a few forwards of the workload, then reads the globaltimer stamps of the last
one: per CTA and work item [producer starts the tile, MMA has its first stage, MMA
committed the last k-block, epilogue done] and the tile id.  Prints per launch class
(0 = GEMM1 SwiGLU, 1 = GEMM2 / router) the kernel span, per-CTA busy / idle time,
tile durations by executor and m-tile, and the first-data latency."""
import ctypes as C
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
for kv in sys.argv[3:]:
    k, v = kv.split("=", 1)
    os.environ[k] = v
os.environ["BO_LIB"] = "probe"
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synthetic as S  # noqa: E402
from paper_2507_17133_b200 import BrownoutMoE  # noqa: E402
from paper_2507_17133_b200 import brownout as B  # noqa: E402

cfg = S.CONFIGS[sys.argv[1]]
ratio = float(sys.argv[2])
lay = S.make_layer(cfg, device="cuda")
uni = S.make_united_random(cfg, device="cuda")
x = S.make_tokens(cfg, device="cuda")
moe = BrownoutMoE(cfg.d, cfg.f, cfg.m, cfg.K, cfg.way, dtype=cfg.dtype, max_tokens=cfg.T, num_shared=cfg.Ns)
moe.set_brownout(ratio)
shared = (lay["SWg"], lay["SWu"], lay["SWd"]) if cfg.Ns else None
for _ in range(4):
    moe.forward(x, lay["Wr"], (lay["Wg"], lay["Wu"], lay["Wd"]), (uni["UWg"], uni["UWu"], uni["UWd"]), shared=shared)
torch.cuda.synchronize()
NC, NI = 160, 48
stamps = np.zeros((2, NC, NI, 6), dtype=np.uint64)
ids = np.zeros((2, NC, NI), dtype=np.int32)
lib = B._lib
lib.bo_probe_copy.argtypes = [C.c_void_p, C.c_void_p]
assert lib.bo_probe_copy(stamps.ctypes.data, ids.ctypes.data) == 0
dbg = moe.debug_arrays(cfg.T)
out = {"workload": cfg.name, "ratio": ratio, "env": sys.argv[3:], "kernels": moe.last_kernels(),
       "exec_rows": np.diff(dbg["exec_off"].cpu().numpy()).tolist()}
for cls in range(2):
    st = stamps[cls].astype(np.int64)
    valid = st[:, :, 0] > 0
    if not valid.any():
        continue
    t0 = st[:, :, 0][valid].min()
    rel = np.where(st > 0, (st - t0) / 1e3, np.nan)   # us
    ncta = int(valid.any(axis=1).sum())
    items = []
    for c in range(NC):
        for j in range(NI):
            if valid[c, j]:
                tid = int(ids[cls, c, j])
                items.append({"cta": c, "item": j, "x": tid & 1023, "mi": (tid >> 10) & 63, "n": tid >> 16,
                              "start": rel[c, j, 0], "first": rel[c, j, 1], "mma_done": rel[c, j, 2],
                              "epi_done": rel[c, j, 3], "tempty": rel[c, j, 4], "issue0": rel[c, j, 5]})
    end = np.nanmax(rel[:, :, 3])
    cta_end = [np.nanmax(rel[c, :, 3]) for c in range(NC) if valid[c].any()]
    cta_first = [rel[c, 0, 1] for c in range(NC) if valid[c].any()]
    dur = {}
    for it in items:
        key = f"x{it['x']}_mi{it['mi']}"
        dur.setdefault(key, []).append(it["mma_done"] - it["first"])
    summ = {"ctas": ncta, "span_us": float(end), "first_data_us_median": float(np.median(cta_first)),
            "cta_end_us_min_med_max": [float(min(cta_end)), float(np.median(cta_end)), float(max(cta_end))],
            "busy_frac": float(np.mean(cta_end) / end),
            "items_per_cta": np.bincount([it["cta"] for it in items]).tolist()[:ncta],
            "mainloop_us_by_tile_class": {k: [round(min(v), 2), round(statistics.median(v), 2), round(max(v), 2),
                                              len(v)] for k, v in sorted(dur.items())},
            "epi_lag_us_median": float(np.nanmedian([it["epi_done"] - it["mma_done"] for it in items]))}
    out[f"class{cls}"] = summ
    out[f"class{cls}_items"] = [{k: (round(v, 2) if isinstance(v, float) else v) for k, v in it.items()}
                                for it in items]
print(json.dumps(out))
