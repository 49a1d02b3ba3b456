for wl in "mixtral_prefill 0.5" "mixtral_prefill 0.0" "mixtral_prefill 0.25"; do
 for sw in 0 1; do
  echo "== $wl sw=$sw"
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_grouped_gemm --csv python scripts/ffn_ncu_ab.py $wl BO_SWAP_TAIL=$sw 2>/dev/null | grep k_grouped | awk -F'"' '{print $(NF-1)}' | tr '\n' ' '; echo
 done
done
