"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of bench.py:
per-step durations of the library's kernels (bo::*) and each kernel's share of the step.

    python scripts/launch_summary.py gpurun_out/launches.csv > profiles/<name>.json
"""
import csv
import json
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    seq = []
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[ki].lstrip("void ").startswith("bo::"):
            continue
        name = r[ki].replace("void ", "").split("(")[0]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "nsecond": 1e-3}[r[ui]]
        seq.append((name, float(r[vi].replace(",", "")) * scale))
    # steps start at the router (first kernel of a forward)
    steps, cur = [], []
    for name, us in seq:
        # a forward starts at its router: k_router_*, the fused decode routing kernel, or the
        # tcgen05 router (k_grouped_gemm with EPI_ROUTER = 2 as its third template argument)
        starts = "router" in name or "route_fused" in name or \
            (name.startswith("bo::k_grouped_gemm<") and name.split(",")[2].strip() == "2")
        if starts and cur:
            steps.append(cur)
            cur = []
        if "united_mean" in name:
            continue
        cur.append((name, us))
    if cur:
        steps.append(cur)
    # the bench's timed forwards: the most common launch pattern
    pats = {}
    for s in steps:
        pats.setdefault(tuple(n for n, _ in s), []).append(s)
    pat, group = max(pats.items(), key=lambda kv: len(kv[1]))
    n = len(group)
    per = [sum(s[i][1] for s in group) / n for i in range(len(pat))]
    tot = sum(per)
    out = {"source": path, "steps_averaged": n, "step_us": tot,
           "kernels": [{"kernel": k, "us": round(u, 2), "share": round(u / tot, 4)} for k, u in zip(pat, per)]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
