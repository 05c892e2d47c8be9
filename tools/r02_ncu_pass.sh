#!/usr/bin/env bash
# ncu evidence per config: the dominant kernel's per-launch DRAM bytes and pipe utilisation
# over one bench step (-> profiles/ncu_summary.json via tools/ncu_summary.py), and the full
# launch list of the headline command (C4).
cd "$(dirname "$0")/.."
O=gpurun_out
T=${TAG:-r02}
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
for spec in ${SPECS:-C4:zgemm_kernel C5:zgemm_kernel C3:dense_batched_kernel C1:dense_batched_kernel C2:tri_ls}; do
  w=${spec%%:*}; pat=${spec#*:}
  timeout 900 ncu --metrics $M --clock-control none -k regex:$pat --csv --log-file $O/${T}_ncu_$w.csv \
    python bench.py --workload $w --steps 1 --warmup 0 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline > $O/${T}_ncu_$w.log 2>&1
  echo ncu_${w}_rc=$?
  python tools/ncu_summary.py $w $pat $O/${T}_ncu_$w.csv profiles/${T}_ncu_$w.csv
  cp $O/${T}_ncu_$w.csv profiles/ 2>/dev/null
done
cp profiles/ncu_summary.json $O/${T}_ncu_summary.json
if [ -z "$NOLIST" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/${T}_c4_launches.csv \
    python bench.py --steps 1 --warmup 1 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline > $O/${T}_c4_list.log 2>&1; echo list_rc=$?
fi
