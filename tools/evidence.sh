#!/bin/bash
# One GPU call that regenerates the round's evidence into gpurun_out/ev/ (copied to profiles/ by hand).
# Order matters: every ncu capture runs only after the same command exited 0 without ncu.
out=gpurun_out/ev
mkdir -p $out
python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $out/smoke.log 2>&1; echo "smoke rc=$?" >> $out/smoke.log
for w in C2 C1 C3 C4 C5; do
  python bench.py --workload $w > $out/bench_$w.json 2> $out/bench_$w.err
done
python bench.py --impl reference > $out/bench_reference_C2.json 2> $out/bench_reference_C2.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $out/c2_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --prof-steps 0 --e2e-steps 0 > $out/ncu_c2_launches.log 2>&1
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --prof-steps 0 > /dev/null 2>&1 && \
  ncu --set full --import-source on -k 'regex:tri_ls|tri_fixz' -c 2 -o $out/c2_tri_ls \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --prof-steps 0 --e2e-steps 0 > $out/ncu_c2_full.log 2>&1
python tools/run_c5_once.py 512 1 > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $out/c5_launches.csv \
    python tools/run_c5_once.py 512 1 > $out/ncu_c5_launches.log 2>&1
python tools/run_c3_once.py 512 > /dev/null 2>&1 && \
  ncu --set full --import-source on -k regex:dense_batched -c 1 -o $out/c3_dense \
    python tools/run_c3_once.py 512 > $out/ncu_c3_full.log 2>&1
PFX_DENSE_PHASES=1 python tools/run_c3_once.py 512 > $out/c3_phases.log 2>&1
python tools/time_c2_rows.py 8 > $out/c2_rows_scaling.txt 2>&1
echo done > $out/DONE
