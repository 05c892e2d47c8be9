#!/usr/bin/env bash
# C5 critical chain: a per-launch timeline of one evaluation (profiled, direct launches) and
# the graph-replayed step time with parts of the work skipped (PFX_BD_SKIP; results wrong,
# timing only): 4 = no far trailing update, 2 = no RHS chain, 1 = no back substitution.
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02c5}
rm -f $O/${T}_timeline.txt
PFX_PROF_TIMELINE=$O/${T}_timeline.txt timeout 600 python bench.py --workload C5 --steps 2 --warmup 1 --prof-steps 1 \
  --no-cpu-baseline --e2e-steps 0 > $O/${T}_tl_bench.json 2> $O/${T}_tl_bench.err; echo tl_rc=$?
python tools/timeline_chain.py $O/${T}_timeline.txt > $O/${T}_chain.txt 2>&1; head -30 $O/${T}_chain.txt
for sk in 0 4 6 7 16 8; do
  PFX_BD_SKIP=$sk timeout 600 python bench.py --workload C5 --steps 5 --warmup 2 --no-cpu-baseline --e2e-steps 0 \
    > $O/${T}_skip$sk.json 2> $O/${T}_skip$sk.err
  echo "skip=$sk rc=$? $(python -c "import json;d=json.load(open('$O/${T}_skip$sk.json'));print(round(d['ms_per_step'],2))" 2>/dev/null)"
done
