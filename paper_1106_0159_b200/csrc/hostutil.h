// Host-side helpers shared by the context (shtc.cu) and the multi-GPU group (group.cu):
// page-locked detection and the host copy pool that stages pageable buffers on all cores.
#pragma once

#include <cuda_runtime.h>

#include "hostcopy.h"

namespace shtc_host {

// host memory the copy engines can read / write directly (cudaHostAlloc, cudaHostRegister,
// pinned torch tensors); pageable memory (std::vector, numpy) goes through PinnedBuf staging
inline bool host_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace shtc_host
