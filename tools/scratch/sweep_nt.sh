#!/bin/bash
# launch-geometry sweep of the factor kernel on c2
cd "$(dirname "$0")/.."
for smem in 96 110; do
  echo "NT512 1/SM smem $smem: $(BILU_SMEM_KB=$smem timeout 100 python tools/run_one.py c2 3 2>&1 | tail -1)"
  echo "NT256 1/SM smem $smem: $(BILU_LIB=$PWD/paper_1908_10169_b200/libbilu_nt256.so BILU_SMEM_KB=$smem timeout 100 python tools/run_one.py c2 3 2>&1 | tail -1)"
  echo "NT256 2/SM smem $smem: $(BILU_LIB=$PWD/paper_1908_10169_b200/libbilu_nt256.so BILU_CTAS_PER_SM=2 BILU_SMEM_KB=$smem timeout 100 python tools/run_one.py c2 3 2>&1 | tail -1)"
done
