#!/bin/bash
# split-parameter sweep of the factor kernel on c2 (t_factor_ms incl. merge post-pass)
cd "$(dirname "$0")/.."
for T in ${SWEEP_T:-256 512 1024}; do for PI in ${SWEEP_PI:-256 512}; do for I in ${SWEEP_I:-2 8}; do
  echo "heavy_T=$T part_items=$PI idle=$I: $(BILU_HEAVY_T=$T BILU_PART_ITEMS=$PI BILU_HEAVY_IDLE=$I timeout 60 python tools/run_one.py c2 3 2>&1 | tail -1)"
done; done; done
