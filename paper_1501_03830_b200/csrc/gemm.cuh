// Masked FP64 GEMM engine (DMMA + cp.async multistage), the contraction
// workhorse behind POTRF/TRSM/TRMM, the congruence W = L^T M L, SY2SB's
// SYMM/SYR2K, the D&C merge products and the WY back-transforms.
//
//   C := alpha * op(A) * op(B) + beta * C      (column-major, FP64)
//
// Masks select a diagonal band of a *stored* operand (view-relative (r, c)):
// an element is kept iff lo <= c - r <= hi; `unit` forces the diagonal to 1
// (implicit-unit Householder storage).  The output mask restricts which C
// elements are written (e.g. the lower triangle for SYRK/SYR2K).  Masked
// operands also shrink the k-range, so triangular products cost half.
#pragma once
#include <cuda_runtime.h>
#include "common.cuh"

namespace bse {

struct Mask {
  int lo = kNoMaskLo, hi = kNoMaskHi, unit = 0;
  BSE_HD static Mask none() { return Mask{}; }
  BSE_HD static Mask lower() { return Mask{kNoMaskLo, 0, 0}; }          // tril(X)
  BSE_HD static Mask strict_lower() { return Mask{kNoMaskLo, -1, 0}; }  // tril(X, -1)
  BSE_HD static Mask unit_lower() { return Mask{kNoMaskLo, -1, 1}; }    // tril(X,-1) + I
  BSE_HD static Mask upper() { return Mask{0, kNoMaskHi, 0}; }          // triu(X)
  BSE_HD static Mask strict_upper() { return Mask{1, kNoMaskHi, 0}; }
  BSE_HD bool active() const { return lo != kNoMaskLo || hi != kNoMaskHi || unit; }
};

struct GemmProblem {
  int M = 0, N = 0, K = 0;
  const double* A = nullptr;
  long long lda = 0;
  const double* B = nullptr;
  long long ldb = 0;
  double* C = nullptr;
  long long ldc = 0;
  double alpha = 1.0, beta = 0.0;
  Mask ma, mb, mc;
  const int* ccol = nullptr;  // optional column map: C column n is written at ccol[n]
  bool mirror = false;        // also store every strictly-lower C(m, n) at C(n, m) (symmetric result)
};

// Single problem.  transA/transB: op(X) = X^T.
cudaError_t gemm(bool transA, bool transB, const GemmProblem& p, cudaStream_t s);

// Grouped: `probs` is a DEVICE array of `count` problems sharing (transA,
// transB); maxM/maxN bound the grid.  Masks inside each problem are honoured.
cudaError_t gemm_grouped(bool transA, bool transB, const GemmProblem* probs_dev, int count,
                         int maxM, int maxN, cudaStream_t s, bool all_aligned16 = false,
                         int cfg = 1);

// Split-K for short-and-wide outputs (M*N small, K large): `splits` partial
// products go to `ws` (>= splits*M*N doubles), then a fixed-order reduction
// applies alpha/beta (deterministic).  Masks on A/B are honoured; the output
// mask must be inactive.
cudaError_t gemm_splitk(bool transA, bool transB, const GemmProblem& p, int splits, double* ws,
                        GemmProblem* probs_dev_scratch, cudaStream_t s);

// Convenience wrappers ------------------------------------------------------
inline GemmProblem make_gemm(int M, int N, int K, double alpha, const double* A, long long lda,
                             const double* B, long long ldb, double beta, double* C,
                             long long ldc) {
  GemmProblem p;
  p.M = M; p.N = N; p.K = K; p.alpha = alpha; p.beta = beta;
  p.A = A; p.lda = lda; p.B = B; p.ldb = ldb; p.C = C; p.ldc = ldc;
  return p;
}

}  // namespace bse
