for cfg in "200 1 100" "110 1 50" "110 1 100" "110 2 100" "64 1 30" "64 2 60" "48 2 50"; do
  set -- $cfg
  echo "== smem $1 KB, ctas/SM $2, carveout $3"
  BILU_SMEM_KB=$1 BILU_CTAS_PER_SM=$2 BILU_CARVEOUT=$3 BILU_DEBUG_TIMEOUT=30 timeout 120 python tools/block_profile.py c2 2>&1 | grep -E "factor|heaviest|lightest"
done
