#!/bin/bash
# A/B of library builds on the bench's own timing (c2, 20 steps, L2 flushed), interleaved:
#   bash tools/ab_bench.sh libA.so libB.so ...   (paths relative to paper_1908_10169_b200/)
cd "$(dirname "$0")/.."
L=$(pwd)/paper_1908_10169_b200
for rep in 1 2; do for lib in "$@"; do
  BILU_LIB=$L/$lib timeout 300 python bench.py --steps 20 --warmup 5 --no-extra --no-cpu-baseline --no-solve --no-e2e \
    2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['ms_per_step'], d['roofline']['kernel_ms'])"
done; done
