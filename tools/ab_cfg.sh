#!/bin/bash
# A/B of library builds on one config (factor time of the last of 4 reps), interleaved:
#   bash tools/ab_cfg.sh c4 libA.so libB.so ...   (paths relative to paper_1908_10169_b200/)
cd "$(dirname "$0")/.."
L=$(pwd)/paper_1908_10169_b200
CFG=$1; shift
for rep in 1 2; do for lib in "$@"; do
  echo -n "$lib "; BILU_LIB=$L/$lib timeout 300 python tools/run_cfg.py $CFG 4 2>/dev/null | tail -1
done; done
