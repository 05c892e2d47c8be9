// Banded path (config C5): placeholder until the banded LU lands.
#include "pfx_common.cuh"

namespace pfx {

int banded_run(const double*, int64_t, int64_t, const double*, int64_t, double, const double2*, const double2*, int,
               double*, cudaStream_t, float*) {
  return fail(PFX_BADARG, "banded path is not built yet");
}

}  // namespace pfx
