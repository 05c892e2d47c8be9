#!/usr/bin/env bash
# C4 bench (timed + per-phase profile) and ncu --set full of one LU-update and one backward zgemm.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02b}
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo bench_rc=$?
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel --launch-skip 2 -c 1 -f -o $O/${T}_c4_zgemm_lu \
  python bench.py --steps 1 --warmup 0 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline > $O/${T}_ncu1.log 2>&1; echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel --launch-skip 420 -c 1 -f -o $O/${T}_c4_zgemm_bwd \
  python bench.py --steps 1 --warmup 0 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline > $O/${T}_ncu2.log 2>&1; echo ncu2_rc=$?
fi
