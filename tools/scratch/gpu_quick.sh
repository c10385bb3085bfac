#!/bin/bash
# quick GPU iteration: parity tests, bench (no CPU baseline), block profile of c2
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
BILU_DEBUG_TIMEOUT=60 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dgemm.py -x -q > gpurun_out/tq.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/tq.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bq.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bq.log').read().strip().splitlines()[-1]); print('bench ms/step', d['ms_per_step'], 'factor kernel ms', d['roofline']['kernel_ms'])" 2>&1 | tail -1
if [ "$1" == "prof" ]; then timeout 300 python tools/block_profile.py c2 > gpurun_out/blkq.log 2>&1; tail -4 gpurun_out/blkq.log; fi
