// Blocking host<->device copy that is also complete on the DEVICE when it returns.
// A plain cudaMemcpy from pageable memory returns once the data is staged, and a
// device-to-device cudaMemcpy returns before the copy runs; both are ordered only on the
// legacy stream, while this library's kernels and copies run on non-blocking streams.
// Every setup upload that later work on those streams reads therefore goes through here.
#pragma once
#include <cuda_runtime.h>

namespace sparsla_b200 {
inline cudaError_t memcpy_sync(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    cudaError_t e = cudaMemcpy(dst, src, bytes, kind);
    if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
    return e;
}
}  // namespace sparsla_b200
