#!/bin/bash
# quick GPU iteration: parity subset + timings + c4 block profile
cd "$(dirname "$0")/.."
TAG=${1:-q}
bash tools/gq.sh $TAG
timeout 600 python tools/block_profile.py c4 > gpurun_out/blk_c4_$TAG.log 2>&1
head -12 gpurun_out/blk_c4_$TAG.log
