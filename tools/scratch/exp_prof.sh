#!/bin/bash
# per-block profile of c2 (diagnostic build) -> gpurun_out/${TAG}_blk.log + npy
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-p}
timeout 300 python tools/block_profile.py c2 > gpurun_out/${TAG}_blk.log 2>&1
cp gpurun_out/blkprof_c2.npy gpurun_out/${TAG}_blkprof_c2.npy
cat gpurun_out/${TAG}_blk.log | head -8
