#!/bin/bash
# quick GPU iteration: parity subset (pytest -k expression in $K) + timings of $CFGS (3 reps each)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-q}
K=${K:-"random_small or c2_reduced or c1_full or flop_count or c5_reduced or c3_reduced or c4_reduced or c4_2000"}
CFGS=${CFGS:-"c2 c4 c5"}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in $CFGS; do timeout 300 python tools/run_cfg.py $c 3 >> gpurun_out/${TAG}_time.log 2>&1; done
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_time.log
