#!/bin/bash
# per-block timeline of c4 (diagnostic build) + plain timing
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-p}
timeout 600 python tools/block_profile.py c4 > gpurun_out/blk_c4_$TAG.log 2>&1
timeout 300 python tools/run_cfg.py c4 3 > gpurun_out/time_c4_$TAG.log 2>&1
tail -30 gpurun_out/blk_c4_$TAG.log; cat gpurun_out/time_c4_$TAG.log
