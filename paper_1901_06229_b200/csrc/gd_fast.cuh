// Two-stage fast path (FP32 coarse screen + FP64 refinement). Filled in by the fast kernel.
#pragma once

#include "gd_internal.h"

namespace gdk {

// K1a then K1b; `mid` (nullable) is recorded between them.
cudaError_t launch_fast(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                        cudaStream_t stream, cudaEvent_t mid = nullptr);

}  // namespace gdk
