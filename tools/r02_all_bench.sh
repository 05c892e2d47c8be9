#!/usr/bin/env bash
# Every config's bench line (with its CPU baseline) + the GPU test suite: the round's evidence.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02}
for w in ${WL:-C4 C1 C2 C3 C5}; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 5 ${BENCH_ARGS} > $O/${T}_bench_$w.json 2> $O/${T}_bench_$w.err
  echo bench_${w}_rc=$?
done
if [ -z "$NOTESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -2 $O/${T}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.log 2>&1; echo smoke_rc=$?; tail -1 $O/${T}_smoke.log
fi
