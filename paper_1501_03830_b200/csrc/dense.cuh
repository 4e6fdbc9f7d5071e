// Dense triangular building blocks: recursive POTRF, TRSM, TRMM and the
// congruence W = L^T M L, all expressed as small in-CTA leaf kernels plus the
// masked DMMA GEMM engine.
#pragma once
#include <cuda_runtime.h>
#include "gemm.cuh"

namespace bse {

// Device-side status written by factorization kernels.
struct DevStatus {
  int info;       // -1: ok; >= 0: index of the first non-positive pivot
  int conv_fail;  // nonzero: an iterative kernel did not converge
  double value;   // failing pivot value
  double aux;     // min pivot L_jj^2 (initialise to +inf; atomicMin over the leaves)
};

// In-place lower Cholesky of the n x n matrix A (column-major, lda); the
// strict upper triangle is zeroed.  Failure is reported through `st`
// (first failing pivot, as kernels.py:56-61 in the reference).
// inv_cache (optional): ceil(n/64) blocks of 64 x 64 doubles receiving the
// inverses of the 64-wide diagonal blocks of L, reused by trsm_* (pass the
// same cache there) so each leaf inverse is computed once.
// Workspace for the emulated-FP64 (INT8 tensor core) engine: the large
// off-diagonal updates of the recursive POTRF / TRSM run there when given.
struct OzWork {
  void* p = nullptr;
  size_t bytes = 0;
  int chunk = 2048;
};
size_t trsm_llt_oz_bytes(int n, int ncols, int chunk);

size_t potrf_inv_cache_doubles(int n);
// hook (optional): lets a caller stream the matrix in by column pieces while
// the Cholesky runs.  Piece 0 = columns [0, s_depth) must be present at the
// call; piece L (1 <= L <= depth) = columns [s_{depth-L+1}, s_{depth-L}) with
// s_0 = n and s_{k+1} = potrf_top_split(s_k), i.e. the top-left recursion
// chain.  fn(ctx, L, s) is called on the stream before piece L is first read.
struct PotrfHook {
  cudaError_t (*fn)(void* ctx, int level, cudaStream_t s);
  void* ctx;
  int depth;
};
int potrf_top_split(int n);
cudaError_t potrf_lower(double* A, long long lda, int n, DevStatus* st, cudaStream_t s,
                        double* inv_cache = nullptr, const OzWork* oz = nullptr,
                        const PotrfHook* hook = nullptr);

// The same for a diagonal block whose first row/column is global index `off`
// (a failing pivot is reported as off + j): the tile factorizations of the
// distributed right-looking Cholesky.
cudaError_t potrf_lower_at(double* A, long long lda, int n, int off, DevStatus* st, cudaStream_t s);

// A (m x n) <- A * L^{-T}, L n x n lower (right, lower, transposed).
cudaError_t trsm_rlt(const double* L, long long ldl, int n, double* A, long long lda, int m,
                     cudaStream_t s, const double* inv = nullptr, const OzWork* oz = nullptr);


// Called on the stream as soon as rows [r0, r1) of a TRSM solution are final
// (bottom-up: L^T is upper triangular); `depth` levels of the recursion
// report separately (2^depth row pieces), `base` offsets the row indices.
struct RowHook {
  cudaError_t (*fn)(void* ctx, int r0, int r1, cudaStream_t s);
  void* ctx;
  int depth;
  int base;
};

// B (n x ncols) <- L^{-T} * B (left, lower, transposed: solves L^T X = B).
cudaError_t trsm_llt(const double* L, long long ldl, int n, double* B, long long ldb, int ncols,
                     cudaStream_t s, const double* inv = nullptr, const OzWork* oz = nullptr,
                     const RowHook* hook = nullptr);

// B (n x ncols) <- L^{-1} * B (left, lower, no transpose).
cudaError_t trsm_lln(const double* L, long long ldl, int n, double* B, long long ldb, int ncols,
                     cudaStream_t s);

// Zero the strict upper triangle of an n x n matrix.
cudaError_t zero_strict_upper(double* A, long long lda, int n, cudaStream_t s);

// Copy lower triangle to upper (make symmetric).
cudaError_t symmetrize_from_lower(double* A, long long lda, int n, cudaStream_t s);

}  // namespace bse
