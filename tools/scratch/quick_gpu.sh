#!/bin/bash
# quick GPU iteration: selected parity tests + timings of c2/c3/c5 (args: pytest -k expression)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-q}
K=${1:-"random_small or c2_reduced or c1_full or flop_count or c5_reduced or c3_reduced or c4_reduced"}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "$K" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
for c in c2 c2 c3 c5; do timeout 300 python tools/run_cfg.py $c 3 >> gpurun_out/${TAG}_time.log 2>&1; done
tail -3 gpurun_out/${TAG}_pytest.log; cat gpurun_out/${TAG}_time.log
