// Two-stage fast path (FP32 coarse screen + FP64 refinement). Filled in by the fast kernel.
#pragma once

#include "gd_internal.h"

namespace gdk {

// K1a then K1b; `mid` (nullable) is recorded between them. With stream_b (and mid), K1b runs on
// stream_b after mid, so the next batch's K1a can follow on `stream` while this K1b runs.
cudaError_t launch_fast(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                        cudaStream_t stream, cudaEvent_t mid = nullptr, cudaStream_t stream_b = nullptr);

// K1a alone for ligands of 129..256 atoms (NS = 8): their candidates feed the FP64 kernel, which
// then skips its own all-FP64 alignment (the FP32 sweep does not fit registers at that size).
cudaError_t launch_align_big(const DevPocket& pk, const DevParams& pr, const DevBatch& b, int n_sms,
                             cudaStream_t stream);

}  // namespace gdk
