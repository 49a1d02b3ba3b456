# Interleaved rounds of kernel-time A/B under ncu launch lists:
#   bash scripts/ncu_ab_rounds.sh ROUNDS "<workload> <ratio>" ENV1 ENV2 ...  ("-" = defaults)
# prints per arm the GEMM1 / GEMM2 medians over all rounds (6 forwards per round).
rounds=$1; shift; wl=$1; shift
tmp=$(mktemp -d)
for r in $(seq 1 $rounds); do
  for e in "$@"; do
    f=$tmp/$(echo "$e" | tr '=;/ ' '____')
    ee=$e; if [ "$ee" = "-" ]; then ee=""; fi
    ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grouped_gemm --csv python scripts/ffn_ncu_ab.py $wl $ee 2>/dev/null | grep k_grouped | awk -F'"' '{print $(NF-1)}' >> $f
  done
done
for e in "$@"; do
  f=$tmp/$(echo "$e" | tr '=;/ ' '____')
  python3 - "$f" "$wl" "$e" <<'PY'
import sys, statistics
v = [float(x) for x in open(sys.argv[1]).read().split()]
g1, g2 = v[0::2], v[1::2]
print(f"{sys.argv[2]} {sys.argv[3]:>20s}  GEMM1 {statistics.median(g1)/1e3:8.1f} us  GEMM2 {statistics.median(g2)/1e3:7.1f} us  (n={len(g1)})")
PY
done
