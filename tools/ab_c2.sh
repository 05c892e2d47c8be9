#!/bin/bash
# A/B of compile-time variants on C2 (timing only). Usage: tools/ab_c2.sh "-DFOO=1" "-DFOO=2" ...
for v in "$@"; do
  PFX_NVCC_FLAGS="$v" python -m paper_2306_16778_b200.build --force > /dev/null 2>&1
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read())
print('variant [$v]', 'ms/step %.4f' % d['ms_per_step'], {n: round(v['total_ms']/v['launches'],4) for n,v in d['kernels'].items()})"
done
python -m paper_2306_16778_b200.build --force > /dev/null 2>&1
