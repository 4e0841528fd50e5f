// Two-stage fast path (FP32 coarse screen + FP64 refinement). Filled in by the fast kernel.
#pragma once

#include "gd_internal.h"

namespace gdk {

cudaError_t launch_fast(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                        cudaStream_t stream);

}  // namespace gdk
