// Complex Hermitian BSE on the device (complex.cu): real embedding, the real
// product-form solve with column selection, complex extraction.
#pragma once
#include <cuda_runtime.h>
#include "solver.cuh"
#include "workspace.cuh"

namespace bse {

// Doubled eigenvalues of the embedding are grouped when their lambda^2 differ
// by <= kComplexGroupTol * N * eps * lambda^2_max (the reference groups
// doubled Hermitian eigenvalues at 20 N eps scale, kernels.py:644-650).
constexpr double kComplexGroupTol = 20.0;

struct ComplexCarve {
  long long ld;
  double* M;      // M' (N x N), later X2r
  double* K;      // K' (N x N), later X1r
  double* lam2;   // N
  int* src;       // n
  char* cls;      // cluster descriptors
  char* ws;       // solve workspace (solve_bytes(N)); extraction scratch after the solve
  size_t ws_bytes;
  size_t scratch_bytes;  // extraction scratch at the start of ws
};
ComplexCarve carve_complex(Arena& a, int n, int flags);
size_t complex_bytes(int n, int flags);

// A, B: n x n complex128 row-major (lda, ldb complex elements), on the
// device; X1c, X2c likewise (ldx1, ldx2).  lam_dev / lam_host (either may be
// null): the n eigenvalues, descending.  Synchronises `s` before returning.
cudaError_t solve_complex(int n, const double2* A, long long lda, const double2* B, long long ldb,
                          double* lam_dev, double* lam_host, double2* X1c, long long ldx1,
                          double2* X2c, long long ldx2, const ComplexCarve& c, int flags,
                          cudaStream_t s, SolveStatus* out);

}  // namespace bse
