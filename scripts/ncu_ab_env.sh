# usage: bash scripts/ncu_ab_env.sh "<workload> <ratio>" ENV1 ENV2 ...   (each ENV = NAME=VALUE or "-" for defaults)
wl=$1; shift
for e in "$@"; do
  echo "== $wl $e"
  if [ "$e" = "-" ]; then e=""; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grouped_gemm --csv python scripts/ffn_ncu_ab.py $wl $e 2>/dev/null | grep k_grouped | awk -F'"' '{print $(NF-1)}' | tr '\n' ' '; echo
done
