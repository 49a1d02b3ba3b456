"""Phase timeline of the fused decode routing launch (k_route_fused) from the
instrumentation build (build.py --variant probe; loaded with BO_LIB=probe).

    BO_LIB=probe python scripts/probe_route.py mixtral_decode 1.0 [NAME=VALUE ...]

Runs a few forwards, then reads each CTA's globaltimer stamps of the last launch
[entry, router tile done, grid barrier passed, histograms staged, plan done, permute
done] and prints, per phase, the median / max over CTAs of the time since the
earliest entry (ns)."""
import ctypes as C
import json
import os
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
out = {"workload": sys.argv[1], "ratio": ratio, "runs": []}
for rep in range(5):
    for _ in range(3):
        moe.forward(x, lay["Wr"], (lay["Wg"], lay["Wu"], lay["Wd"]), (uni["UWg"], uni["UWu"], uni["UWd"]))
    torch.cuda.synchronize()
    st = np.zeros((1024, 6), dtype=np.uint64)
    assert B._lib.bo_probe_rf_copy(st.ctypes.data_as(C.c_void_p)) == 0
    used = st[:, 0] > 0
    st = st[used].astype(np.int64)
    t0 = st[:, 0].min()
    rel = st - t0
    out["runs"].append({"ctas": int(used.sum()), "kernels": moe.last_kernels(),
                        "phase_median_ns": [int(v) for v in np.median(rel, axis=0)],
                        "phase_max_ns": [int(v) for v in rel.max(axis=0)],
                        "entry_spread_ns": int(rel[:, 0].max())})
print(json.dumps(out))
