// Two-stage fast path (placeholder until the coarse kernel lands).
#include "gd_fast.cuh"

namespace gdk {

cudaError_t launch_fast(const DevPocket&, const DevParams&, const DevBatch&, int, cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace gdk
