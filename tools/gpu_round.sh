#!/bin/bash
# One GPU session: build, tests, smoke, bench (plain), then ncu launch list + full capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-v}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "$SKIP_TESTS" != "1" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
if [ "$1" == "ncu" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
     python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
  echo "ncu1 rc=$?" >> gpurun_out/ncu_launch.log
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:factor_kernel -s 1 -c 1 \
     -o gpurun_out/prof_factor_$TAG python tools/run_one.py c2 2 > gpurun_out/ncu_full.log 2>&1
  echo "ncu2 rc=$?" >> gpurun_out/ncu_full.log
fi
tail -3 gpurun_out/pytest_gpu.log 2>/dev/null; cat gpurun_out/smoke.log; tail -2 gpurun_out/bench_$TAG.log | cut -c1-300
