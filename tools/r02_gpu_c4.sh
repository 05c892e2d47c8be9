#!/usr/bin/env bash
# One GPU-box session: parity tests of the dense path, the C4 headline bench, the ncu launch
# list of the same command, one `ncu --set full` capture of a C4 trailing-update zgemm, and the
# CPU-baseline calibration (BASELINE.md §3 settings) for every config.
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_pivoting_gpu.py tests/test_configs_gpu.py tests/test_dense_large_gpu.py -m gpu -q -rA > $O/r02_dense_tests.log 2>&1; echo dense_tests_rc=$?
tail -2 $O/r02_dense_tests.log
timeout 900 python bench.py --steps 10 --warmup 3 > $O/r02_bench_c4.json 2> $O/r02_bench_c4.err; echo bench_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $O/r02_c4_launches.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline > $O/r02_c4_ncu_launch.log 2>&1; echo ncu_list_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zgemm_kernel --launch-skip 2 -c 1 -f -o $O/r02_c4_zgemm \
  python bench.py --steps 1 --warmup 0 --e2e-steps 0 --prof-steps 1 --no-cpu-baseline > $O/r02_c4_ncu_full.log 2>&1; echo ncu_full_rc=$?
for w in ${CALIB:-C4 C1 C3 C2 C5}; do
  timeout 1500 python bench.py --cpu-calibrate --workload $w >> $O/r02_cpu_calibrate.log 2>&1; echo calib_${w}_rc=$?
done
cp profiles/cpu_settings.json $O/r02_cpu_settings.json 2>/dev/null
