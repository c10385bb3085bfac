#!/bin/bash
cd "$(dirname "$0")/.."
for a in "c5 N=24" "c5 N=32" "c5 N=48" "c5 N=64" "c3 N=16" "c3 N=24" "c3 N=32"; do
  set -- $a
  echo "$a: $(timeout 300 python tools/run_full.py $1 1 $2 2>&1 | tail -1 | cut -c1-300)"
done
