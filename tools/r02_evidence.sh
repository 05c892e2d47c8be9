#!/usr/bin/env bash
# Round-2 evidence in one box session: every config's bench line, the GPU test suite and smoke,
# the ncu per-config dominant-kernel counters + C4 launch list, one --set full capture of the
# C4 top kernel, and the reference arm on the headline config.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02z}
TAG=$T tools/r02_all_bench.sh
TAG=$T tools/r02_ncu_pass.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel --launch-skip 40 -c 1 -f \
  -o $O/${T}_c4_zgemm_full python bench.py --steps 1 --warmup 0 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline \
  > $O/${T}_c4_full.log 2>&1; echo ncu_full_rc=$?
timeout 1500 python bench.py --impl reference --steps 20 --warmup 5 > $O/${T}_ref_C4.json 2> $O/${T}_ref_C4.err; echo ref_rc=$?
