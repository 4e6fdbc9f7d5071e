// Host <-> device copies of large PAGEABLE buffers (numpy arrays handed to
// the host entries) through a library-owned pinned staging ring: the host
// side of each chunk is copied by several threads (pageable memcpy is
// DRAM-bound, one thread reaches a fraction of it) while the previous
// chunk's DMA runs, instead of the driver's single-threaded pageable path.
#pragma once
#include <cstddef>
#include <cuda_runtime.h>

namespace bse {

// dst (device) <- src (host, pageable), `rows` rows of `row_bytes` with the
// given pitches.  Ordered on s; returns after the last host copy is issued
// (the staging buffers are reused only after their DMA completes).
cudaError_t h2d_staged(void* dst, size_t dpitch, const void* src, size_t spitch,
                       size_t row_bytes, size_t rows, cudaStream_t s);
// dst (host, pageable) <- src (device); returns when dst is complete.
cudaError_t d2h_staged(void* dst, size_t dpitch, const void* src, size_t spitch,
                       size_t row_bytes, size_t rows, cudaStream_t s);

}  // namespace bse
