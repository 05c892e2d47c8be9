#!/bin/bash
# A/B of compile-time variants on the C2 host-entry (e2e) call. Usage: tools/ab_c2_host.sh "-DFOO=1" ...
for v in "$@"; do
  PFX_NVCC_FLAGS="$v" python -m paper_2306_16778_b200.build --force > /dev/null 2>&1
  echo "variant [$v]"; python tools/time_c2_host.py | tail -2
done
python -m paper_2306_16778_b200.build --force > /dev/null 2>&1
