// Large dense path (config C4, d > 512): placeholder until the blocked multi-CTA LU lands.
#include "pfx_common.cuh"

namespace pfx {

int dense_large_run(const double*, int, int, const double*, int, int, int, int, double, const double2*,
                    const double2*, int, double*, cudaStream_t, float*) {
  return fail(PFX_BADARG, "dense path for d > 512 is not built yet");
}

}  // namespace pfx
