#!/bin/bash
# quick GPU iteration + c4 block profile + pair-cap sweep
cd "$(dirname "$0")/.."
TAG=${1:-q}
bash tools/gq.sh $TAG
timeout 600 python tools/block_profile.py c4 > gpurun_out/blk_c4_$TAG.log 2>&1
for pc in 32 1024; do echo "pair_cap $pc" >> gpurun_out/${TAG}_time.log; for c in c2 c4; do BILU_PAIR_CAP=$pc timeout 300 python tools/run_cfg.py $c 3 >> gpurun_out/${TAG}_time.log 2>&1; done; done
head -12 gpurun_out/blk_c4_$TAG.log; cat gpurun_out/${TAG}_time.log
