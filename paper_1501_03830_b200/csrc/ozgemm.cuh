// FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme II), see ozgemm.cu.
#pragma once
#include <cuda_runtime.h>
#include "gemm.cuh"

namespace bse {

// Workspace for an M x N x K product processed in column chunks of `chunk`.
size_t ozgemm_bytes(int M, int N, int K, int chunk);

// C := alpha op(A) op(B) + beta C with the operand masks of GemmProblem
// (view-relative, as in gemm()), the output mask (relative to the unmapped
// column) and the optional output column map p.ccol (device array).  reuse_a: the workspace already holds the slices of this
// op(A) from the previous call (same A, M, K and workspace).
cudaError_t ozgemm(bool transA, bool transB, const GemmProblem& p, void* work, size_t work_bytes,
                   int chunk, cudaStream_t s, bool reuse_a = false);

// Contraction kernel behind the engine: 0 = hand-written tcgen05 kernel on CTA
// pairs (default), 1 = the same on single CTAs, 2 = CUTLASS kernel + INT32
// planes (A/B measurements).  Returns the previous setting.
int oz_set_engine(int engine);

// Products at least this large (M N K) go to the emulated engine.
// (2^34 by default -- retuned in round 2 for the byte-plane CRT and the
// tile-skipping contraction kernel: 2^36 -> 2^34 is worth 8-10 ms of the cfg2
// solve; BSE_OZ_MIN_WORK_LOG2 overrides it for tuning)
double oz_min_work();

}  // namespace bse
