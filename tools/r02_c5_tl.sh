#!/usr/bin/env bash
# C5 per-launch timeline of one evaluation (profiled, direct launches) -> chain breakdown
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02c5tl}
rm -f $O/${T}_timeline.txt
PFX_PROF_TIMELINE=$O/${T}_timeline.txt timeout 600 python bench.py --workload ${WL:-C5} --steps 2 --warmup 1 --prof-steps 1 \
  --no-cpu-baseline --e2e-steps 0 > $O/${T}_tl_bench.json 2> $O/${T}_tl_bench.err; echo tl_rc=$?
python tools/timeline_chain.py $O/${T}_timeline.txt > $O/${T}_chain.txt 2>&1; cat $O/${T}_chain.txt
