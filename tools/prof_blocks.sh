#!/bin/bash
# per-block timelines (diagnostic build) + critical paths of c2 and c4 -> gpurun_out/blk_*.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-p}
for c in ${CFGS:-c2 c4}; do
  timeout 600 python tools/block_profile.py $c > gpurun_out/blk_${c}_$TAG.log 2>&1
  cp gpurun_out/blkprof_$c.npy gpurun_out/blkprof_${c}_$TAG.npy
  timeout 900 python tools/crit_path.py gpurun_out/blkprof_$c.npy $c >> gpurun_out/blk_${c}_$TAG.log 2>&1
done
tail -n 30 gpurun_out/blk_*_$TAG.log
