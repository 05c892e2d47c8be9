#!/usr/bin/env bash
# Install the UNMODIFIED reference package (and its own test suite) into baseline/_ref, the
# reference arm's location (git-ignored, travels to the GPU box with the gpurun snapshot).
#   * pfexpm itself: the offline pip install the task prescribes (from a /tmp copy, because
#     the build writes into the source tree and /root/reference is read-only);
#   * its tests (pkg/tests, unmodified) next to it, so tests/test_reference_dropin_gpu.py can
#     run the reference's own engine tests through the libpfx.so drop-in on the GPU box,
#     where /root/reference does not exist.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference}"
rm -rf /tmp/pfx_refpkg "$ROOT/baseline/_ref"
cp -r "$SRC/pkg" /tmp/pfx_refpkg
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" /tmp/pfx_refpkg
cp -r "$SRC/pkg/tests" "$ROOT/baseline/_ref/pfexpm_ref_tests"
echo "installed: $(ls "$ROOT/baseline/_ref")"
