#!/bin/bash
# C2 sweep phase ablation (timing only; results are wrong for EXP != 0). Rebuilds the library on the box.
for e in 0 1 2; do
  PFX_NVCC_FLAGS="-DPFX_TRI_EXP=$e" python -m paper_2306_16778_b200.build --force > /dev/null 2>&1
  python bench.py --workload C2 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']
print('EXP=$e', 'ms/step %.3f' % d['ms_per_step'], {n: round(v['total_ms']/v['launches'],4) for n,v in k.items()})"
done
python -m paper_2306_16778_b200.build --force > /dev/null 2>&1
