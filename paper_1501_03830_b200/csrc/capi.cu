// extern "C" boundary (include/bse_b200.h).  Never throws across the ABI:
// every entry point returns a bse_status and records a message retrievable
// with bse_last_error().
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include "../../include/bse_b200.h"
#include "comm.cuh"
#include "complex.cuh"
#include "dense.cuh"
#include "hostio.cuh"
#include "ozgemm.cuh"
#include "solver.cuh"
#include "dist.cuh"

namespace {
thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(BSE_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}
bse::Mask mask_from(const int32_t* m) {
  bse::Mask k;
  k.lo = m[0];
  k.hi = m[1];
  k.unit = m[2];
  return k;
}
}  // namespace

#define BSE_TRY_CUDA(expr, where)                 \
  do {                                            \
    cudaError_t _e = (expr);                      \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

extern "C" {

int bse_version(void) { return 100; }  // 0.1.0

const char* bse_last_error(void) { return g_last_error.c_str(); }

int bse_gemm_dev(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                 const double* dA, int64_t lda, const double* dB, int64_t ldb, double beta,
                 double* dC, int64_t ldc, const int32_t* masks, void* stream) {
  if (M < 0 || N < 0 || K < 0) return fail(BSE_BAD_ARGUMENT, "negative dimension");
  bse::GemmProblem p = bse::make_gemm((int)M, (int)N, (int)K, alpha, dA, lda, dB, ldb, beta, dC, ldc);
  if (masks) {
    p.ma = mask_from(masks);
    p.mb = mask_from(masks + 3);
    p.mc = mask_from(masks + 6);
  }
  BSE_TRY_CUDA(bse::gemm(transA != 0, transB != 0, p, (cudaStream_t)stream), "gemm");
  return BSE_OK;
}

int bse_ozgemm_dev(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                   const double* dA, int64_t lda, const double* dB, int64_t ldb, double beta,
                   double* dC, int64_t ldc, const int32_t* masks, int64_t chunk, void* stream) {
  if (M < 0 || N < 0 || K < 0) return fail(BSE_BAD_ARGUMENT, "negative dimension");
  if (M == 0 || N == 0) return BSE_OK;
  bse::GemmProblem p = bse::make_gemm((int)M, (int)N, (int)K, alpha, dA, lda, dB, ldb, beta, dC, ldc);
  if (masks) {
    p.ma = mask_from(masks);
    p.mb = mask_from(masks + 3);
    p.mc = mask_from(masks + 6);
  }
  const int ch = chunk > 0 ? (int)chunk : (int)N;
  cudaStream_t s = (cudaStream_t)stream;
  const size_t wb = bse::ozgemm_bytes((int)M, (int)N, (int)K, ch);
  void* ws = nullptr;
  BSE_TRY_CUDA(cudaMallocAsync(&ws, wb, s), "ozgemm workspace");
  cudaError_t e = bse::ozgemm(transA != 0, transB != 0, p, ws, wb, ch, s);
  cudaFreeAsync(ws, s);
  BSE_TRY_CUDA(e, "ozgemm");
  return BSE_OK;
}

int bse_oz_set_engine(int engine) { return bse::oz_set_engine(engine); }

int bse_trsm_dev(int kind, int64_t n, const double* dL, int64_t ldl, double* dB, int64_t ldb,
                 int64_t m, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e;
  if (kind == 0) e = bse::trsm_rlt(dL, ldl, (int)n, dB, ldb, (int)m, s);
  else if (kind == 1) e = bse::trsm_llt(dL, ldl, (int)n, dB, ldb, (int)m, s);
  else if (kind == 2) e = bse::trsm_lln(dL, ldl, (int)n, dB, ldb, (int)m, s);
  else return fail(BSE_BAD_ARGUMENT, "trsm kind must be 0, 1 or 2");
  BSE_TRY_CUDA(e, "trsm");
  return BSE_OK;
}

int bse_potrf_dev(int64_t n, double* dA, int64_t lda, void* stream, bse_info* info) {
  if (n < 0 || lda < (n > 0 ? n : 1)) return fail(BSE_BAD_ARGUMENT, "bad dimension");
  cudaStream_t s = (cudaStream_t)stream;
  bse::DevStatus* st = nullptr;
  BSE_TRY_CUDA(cudaMallocAsync((void**)&st, sizeof(bse::DevStatus), s), "alloc status");
  bse::DevStatus h0{-1, 0, 0.0, HUGE_VAL};
  BSE_TRY_CUDA(cudaMemcpyAsync(st, &h0, sizeof(h0), cudaMemcpyHostToDevice, s), "status init");
  double* inv = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&inv, sizeof(double) * bse::potrf_inv_cache_doubles((int)n), s);
  if (e == cudaSuccess) e = bse::potrf_lower(dA, lda, (int)n, st, s, inv);
  if (inv) cudaFreeAsync(inv, s);
  bse::DevStatus h;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(st, s);
  BSE_TRY_CUDA(e, "potrf");
  if (h.info >= 0) {
    if (info) { info->pivot_index = h.info; info->pivot_value = h.value; info->failed_factor = 0; }
    return fail(BSE_NOT_POSITIVE_DEFINITE, "matrix is not positive definite");
  }
  if (info) {
    info->pivot_index = -1;
    info->pivot_value = 0.0;
    info->failed_factor = -1;
    info->min_pivot = n > 0 ? h.aux : 0.0;
  }
  return BSE_OK;
}

size_t bse_solve_workspace_bytes(int64_t n, int flags) {
  return n > 0 ? bse::solve_bytes((int)n, flags) : 0;
}

static int map_solve_status(const bse::SolveStatus& st, bse_info* info) {
  if (info) {
    info->pivot_index = st.pivot_index;
    info->pivot_value = st.pivot_value;
    info->failed_factor = st.failed_factor;
    info->min_pivot = st.min_pivot;
    info->clusters = st.clusters;
  }
  switch (st.code) {
    case 0: return BSE_OK;
    case 2: return fail(BSE_NO_CONVERGENCE, "divide and conquer: a secular root did not converge");
    case 5: return fail(BSE_SPECTRUM_NOT_POSITIVE,
                        "all eigenvalues must be strictly positive (A+B and A-B factor, but "
                        "L^T (A+B) L has a non-positive eigenvalue in floating point)");
    default:
      return fail(BSE_NOT_POSITIVE_DEFINITE, st.failed_factor == 1 ? "A+B is not positive definite"
                                                                   : "A-B is not positive definite");
  }
}

// Flags accepted by the solve entries: BSE_FLAG_NATIVE_FP64 only.  Values-only
// is a bse_syevd_dev mode (the recovery of X needs the eigenvectors).
static int check_solve_flags(int flags) {
  if (flags & ~BSE_FLAG_NATIVE_FP64)
    return fail(BSE_BAD_ARGUMENT, "unsupported flag for a solve (only BSE_FLAG_NATIVE_FP64)");
  return BSE_OK;
}

// Library-owned stream-ordered pool for the host entries' device buffers
// (one per device).  Freed blocks stay reserved in THIS pool between calls
// (a 0 release threshold would unmap ~20 n^2 doubles every solve); the
// device's default pool, which torch or other libraries may use, is left
// untouched.  bse_release_cached_memory() trims it.
static cudaError_t host_pool(cudaMemPool_t* out) {
  static cudaMemPool_t pools[64] = {};
  static std::mutex mu;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[dev & 63]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p;
    if ((e = cudaMemPoolCreate(&p, &props)) != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;
    if ((e = cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr)) != cudaSuccess)
      return e;
    pools[dev & 63] = p;
  }
  *out = pools[dev & 63];
  return cudaSuccess;
}

int bse_solve_spd_pair_dev(int64_t n, const double* dM, int64_t ldm, const double* dK,
                           int64_t ldk, double* dLam, double* dX1, int64_t ldx1, double* dX2,
                           int64_t ldx2, void* dWork, size_t work_bytes, int flags, void* stream,
                           bse_info* info) {
  if (n < 0 || ldm < n || ldk < n || ldx1 < n || ldx2 < n)
    return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (check_solve_flags(flags) != BSE_OK) return BSE_BAD_ARGUMENT;
  if (n > 0 && work_bytes < bse::solve_bytes((int)n, flags))
    return fail(BSE_BAD_ARGUMENT, "workspace too small (see bse_solve_workspace_bytes)");
  bse::SolveStatus st{};
  BSE_TRY_CUDA(bse::solve_spd_pair((int)n, dM, ldm, dK, ldk, dLam, dX1, ldx1, dX2, ldx2, dWork,
                                   work_bytes, flags, (cudaStream_t)stream, &st),
               "solve");
  return map_solve_status(st, info);
}

int bse_solve_spd_pair_host(int64_t n, const double* M, int64_t ldm, const double* K,
                            int64_t ldk, double* lam, double* X1, int64_t ldx1, double* X2,
                            int64_t ldx2, int flags, bse_info* info) {
  if (n < 0 || ldm < n || ldk < n || ldx1 < n || ldx2 < n)
    return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (check_solve_flags(flags) != BSE_OK) return BSE_BAD_ARGUMENT;
  if (n == 0) return BSE_OK;
  {
    // graded-input guard decided on the host: K and M reach the device in
    // pieces overlapped with the Cholesky, so the solve cannot read their
    // diagonals up front
    double mlo = HUGE_VAL, mhi = -HUGE_VAL, klo = HUGE_VAL, khi = -HUGE_VAL;
    for (int64_t i = 0; i < n; ++i) {
      const double m = M[i + i * ldm], k = K[i + i * ldk];
      mlo = std::min(mlo, m); mhi = std::max(mhi, m);
      klo = std::min(klo, k); khi = std::max(khi, k);
    }
    flags |= (bse::diag_graded(mlo, mhi) || bse::diag_graded(klo, khi)) ? bse::kFlagGraded
                                                                       : bse::kFlagNotGraded;
  }
  cudaMemPool_t pool;
  BSE_TRY_CUDA(host_pool(&pool), "memory pool");
  cudaStream_t s, s2;
  BSE_TRY_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  BSE_TRY_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking), "stream");
  cudaEvent_t evM;
  cudaEventCreateWithFlags(&evM, cudaEventDisableTiming);
  const long long ld = bse::pad_ld(n);
  const size_t mat = sizeof(double) * (size_t)ld * n;
  const size_t wb = bse::solve_bytes((int)n, flags);
  const size_t lam_bytes = ((sizeof(double) * n + 255) / 256) * 256;
  char* buf = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void**)&buf, 4 * mat + lam_bytes + wb, pool, s);
  if (e != cudaSuccess) {
    cudaStreamDestroy(s);
    cudaStreamDestroy(s2);
    cudaEventDestroy(evM);
    return cuda_fail(e, "alloc");
  }
  double* dM = (double*)buf;
  double* dK = (double*)(buf + mat);
  double* dX1 = (double*)(buf + 2 * mat);
  double* dX2 = (double*)(buf + 3 * mat);
  double* dLam = (double*)(buf + 4 * mat);
  void* dW = buf + 4 * mat + lam_bytes;
  bse::SolveStatus st{};
  const size_t row = sizeof(double) * (size_t)n;
  // K by column pieces (the Cholesky starts on piece 0 as soon as it lands
  // and waits for each later piece just before first reading it), then M, on
  // a second stream after piece 0: the copies share the host link in that
  // order, overlapping the factorization; M is joined before the congruence.
  bse::KPieces kp{};
  bse::kpieces_plan((int)n, 2, &kp);
  e = cudaMemcpy2DAsync(dK, ld * 8, K, ldk * 8, row, kp.c1[0], cudaMemcpyHostToDevice, s);
  cudaEvent_t evAlloc;
  cudaEventCreateWithFlags(&evAlloc, cudaEventDisableTiming);
  cudaEventRecord(evAlloc, s);
  cudaStreamWaitEvent(s2, evAlloc, 0);
  for (int L = 1; L <= kp.depth; ++L) {
    cudaEventCreateWithFlags(&kp.ready[L], cudaEventDisableTiming);
    const int c0 = kp.c0[L], c1 = kp.c1[L];
    if (e == cudaSuccess && c1 > c0)
      e = cudaMemcpy2DAsync(dK + (long long)c0 * ld, ld * 8, K + (long long)c0 * ldk, ldk * 8, row,
                            c1 - c0, cudaMemcpyHostToDevice, s2);
    if (e == cudaSuccess) e = cudaEventRecord(kp.ready[L], s2);
  }
  if (e == cudaSuccess)
    e = cudaMemcpy2DAsync(dM, ld * 8, M, ldm * 8, row, n, cudaMemcpyHostToDevice, s2);
  if (e == cudaSuccess) e = cudaEventRecord(evM, s2);
  // X1/X2 column blocks stream back on s2 while later blocks are recovered
  bse::HostOut hout{X1, ldx1, X2, ldx2, lam, s2};
  if (e == cudaSuccess)
    e = bse::solve_spd_pair((int)n, dM, ld, dK, ld, dLam, dX1, ld, dX2, ld, dW, wb, flags, s, &st,
                            evM, &hout, nullptr, &kp);
  cudaEvent_t evDone;
  cudaEventCreateWithFlags(&evDone, cudaEventDisableTiming);
  cudaEventRecord(evDone, s2);
  cudaStreamWaitEvent(s, evDone, 0);  // device buffers stay alive until the copies finish
  cudaFreeAsync(buf, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  cudaEventDestroy(evDone);
  cudaStreamDestroy(s);
  cudaStreamDestroy(s2);
  cudaEventDestroy(evM);
  cudaEventDestroy(evAlloc);
  for (int L = 1; L <= kp.depth; ++L)
    if (kp.ready[L]) cudaEventDestroy(kp.ready[L]);
  BSE_TRY_CUDA(e, "solve_host");
  BSE_TRY_CUDA(e2, "solve_host sync");
  return map_solve_status(st, info);
}

/* ---- complex Hermitian BSE (solvers.solve_complex) ---------------------- */

size_t bse_solve_complex_workspace_bytes(int64_t n, int flags) {
  return n > 0 ? bse::complex_bytes((int)n, flags) : 0;
}

static int complex_args_ok(int64_t n, int64_t lda, int64_t ldb, int64_t ldx1, int64_t ldx2,
                           int flags) {
  if (n < 0 || lda < n || ldb < n || ldx1 < n || ldx2 < n)
    return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (n > (1 << 29)) return fail(BSE_BAD_ARGUMENT, "n too large");
  return check_solve_flags(flags);
}

int bse_solve_complex_dev(int64_t n, const double* dA, int64_t lda, const double* dB,
                          int64_t ldb, double* dLam, double* dX1, int64_t ldx1, double* dX2,
                          int64_t ldx2, void* dWork, size_t work_bytes, int flags, void* stream,
                          bse_info* info) {
  if (complex_args_ok(n, lda, ldb, ldx1, ldx2, flags) != BSE_OK) return BSE_BAD_ARGUMENT;
  if (n == 0) return BSE_OK;
  if (work_bytes < bse::complex_bytes((int)n, flags))
    return fail(BSE_BAD_ARGUMENT, "workspace too small (see bse_solve_complex_workspace_bytes)");
  bse::Arena a{static_cast<char*>(dWork), work_bytes, 0, false};
  const bse::ComplexCarve c = bse::carve_complex(a, (int)n, flags);
  bse::SolveStatus st{};
  BSE_TRY_CUDA(bse::solve_complex((int)n, (const double2*)dA, lda, (const double2*)dB, ldb, dLam,
                                  nullptr, (double2*)dX1, ldx1, (double2*)dX2, ldx2, c, flags,
                                  (cudaStream_t)stream, &st),
               "solve_complex");
  return map_solve_status(st, info);
}

int bse_solve_complex_host(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                           double* lam, double* X1, int64_t ldx1, double* X2, int64_t ldx2,
                           int flags, bse_info* info) {
  if (complex_args_ok(n, lda, ldb, ldx1, ldx2, flags) != BSE_OK) return BSE_BAD_ARGUMENT;
  if (n == 0) return BSE_OK;
  cudaMemPool_t pool;
  BSE_TRY_CUDA(host_pool(&pool), "memory pool");
  cudaStream_t s;
  BSE_TRY_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
  const size_t wb = bse::complex_bytes((int)n, flags);
  char* buf = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void**)&buf, wb, pool, s);
  if (e != cudaSuccess) {
    cudaStreamDestroy(s);
    return cuda_fail(e, "alloc");
  }
  bse::Arena a{buf, wb, 0, false};
  const bse::ComplexCarve c = bse::carve_complex(a, (int)n, flags);
  // inputs and outputs live in the solve workspace region: A, B are consumed
  // by the embedding before the solve starts; X1c, X2c are written after it,
  // behind the extraction scratch
  const size_t cb = ((16 * (size_t)n * n + 255) / 256) * 256;
  double2* dA = reinterpret_cast<double2*>(c.ws);
  double2* dB = reinterpret_cast<double2*>(c.ws + cb);
  char* outs = c.ws + ((c.scratch_bytes + 255) / 256) * 256;
  double2* dX1 = reinterpret_cast<double2*>(outs);
  double2* dX2 = reinterpret_cast<double2*>(outs + cb);
  const size_t row = 16 * (size_t)n;
  // pageable numpy buffers: pinned staging ring, multi-threaded host copies
  e = bse::h2d_staged(dA, row, A, 16 * lda, row, n, s);
  if (e == cudaSuccess) e = bse::h2d_staged(dB, row, B, 16 * ldb, row, n, s);
  bse::SolveStatus st{};
  if (e == cudaSuccess)
    e = bse::solve_complex((int)n, dA, n, dB, n, nullptr, lam, dX1, n, dX2, n, c, flags, s, &st);
  if (e == cudaSuccess && st.code == 0) {
    e = bse::d2h_staged(X1, 16 * ldx1, dX1, row, row, n, s);
    if (e == cudaSuccess) e = bse::d2h_staged(X2, 16 * ldx2, dX2, row, row, n, s);
  }
  cudaFreeAsync(buf, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  BSE_TRY_CUDA(e, "solve_complex_host");
  BSE_TRY_CUDA(e2, "solve_complex_host sync");
  return map_solve_status(st, info);
}

size_t bse_syevd_workspace_bytes(int64_t n, int flags) {
  return n > 0 ? bse::syevd_bytes((int)n, flags) : 0;
}

int bse_syevd_dev(int64_t n, double* dA, int64_t lda, double* dW, double* dZ, int64_t ldz,
                  void* dWork, size_t work_bytes, int flags, void* stream) {
  if (n < 0 || lda < n || ldz < n) return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (n > 0 && work_bytes < bse::syevd_bytes((int)n, flags))
    return fail(BSE_BAD_ARGUMENT, "workspace too small (see bse_syevd_workspace_bytes)");
  if (flags & ~(BSE_FLAG_VALUES_ONLY | BSE_FLAG_NATIVE_FP64))
    return fail(BSE_BAD_ARGUMENT, "unsupported flag for bse_syevd_dev");
  if (n == 0) return BSE_OK;
  cudaStream_t s = (cudaStream_t)stream;
  int* conv = nullptr;
  BSE_TRY_CUDA(cudaMallocAsync((void**)&conv, sizeof(int), s), "alloc flag");
  cudaError_t e = bse::syevd((int)n, dA, lda, dW, dZ, ldz, dWork, work_bytes, flags, s, 0, -1, conv);
  int h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, conv, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(conv, s);
  BSE_TRY_CUDA(e, "syevd");
  if (h) return fail(BSE_NO_CONVERGENCE, "syevd: the tridiagonal eigensolver did not converge");
  return BSE_OK;
}

size_t bse_stedc_workspace_bytes(int64_t n) {
  return n > 0 ? bse::stedc_bytes((int)n) + 4096 : 0;
}

int bse_stedc_dev(int64_t n, double* dD, double* dE, double* dQ, int64_t ldq, void* dWork,
                  size_t work_bytes, void* stream) {
  if (n < 0 || ldq < n) return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (n == 0) return BSE_OK;
  if (work_bytes < bse::stedc_bytes((int)n)) return fail(BSE_BAD_ARGUMENT, "workspace too small");
  bse::Arena a{static_cast<char*>(dWork), work_bytes, 0, false};
  bse::StedcWork w = bse::stedc_carve(a, (int)n);
  cudaStream_t s = (cudaStream_t)stream;
  BSE_TRY_CUDA(bse::stedc((int)n, dD, dE, dD, dQ, ldq, w, s), "stedc");
  int h = 0;
  BSE_TRY_CUDA(cudaMemcpyAsync(&h, w.fail, sizeof(int), cudaMemcpyDeviceToHost, s), "stedc flag");
  BSE_TRY_CUDA(cudaStreamSynchronize(s), "stedc sync");
  if (h) return fail(BSE_NO_CONVERGENCE, "stedc: a secular root did not converge");
  return BSE_OK;
}

int bse_absorption_dev(int64_t n, const double* dLam, const double* dX1c, int64_t ldx1,
                       const double* dX2c, int64_t ldx2, const double* dDr, const double* dDl,
                       int64_t ngrid, const double* dGrid, double sigma, double* dWeights,
                       double* dValues, double* dDefect, double* dMinPair, void* stream) {
  if (n < 0 || ngrid < 0 || !(sigma > 0.0)) return fail(BSE_BAD_ARGUMENT, "bad argument");
  BSE_TRY_CUDA(bse::absorption((int)n, dLam, dX1c, ldx1, dX2c, ldx2, dDr, dDl, (int)ngrid, dGrid,
                               sigma, dWeights, dValues, dDefect, dMinPair, (cudaStream_t)stream),
               "absorption");
  return BSE_OK;
}

size_t bse_residual_workspace_bytes(int64_t n) { return n > 0 ? bse::verify_bytes((int)n) : 0; }

int bse_pair_residuals_dev(int64_t n, const double* dM, int64_t ldm, const double* dK, int64_t ldk,
                           const double* dLam, const double* dX1, int64_t ldx1, const double* dX2,
                           int64_t ldx2, double* dRes, double* dXnorm, double* dBio, void* dWork,
                           size_t work_bytes, void* stream) {
  if (n < 0 || (n > 0 && (ldm < n || ldk < n || ldx1 < n || ldx2 < n)))
    return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (n == 0) return BSE_OK;
  if (work_bytes < bse::verify_bytes((int)n)) return fail(BSE_BAD_ARGUMENT, "workspace too small");
  BSE_TRY_CUDA(bse::pair_residuals((int)n, dM, ldm, dK, ldk, dLam, dX1, ldx1, dX2, ldx2, dRes,
                                   dXnorm, dBio, dWork, work_bytes, (cudaStream_t)stream),
               "pair_residuals");
  return BSE_OK;
}

int bse_profile_enable(int on) {
  bse::StageLog& L = bse::stage_log();
  L.on = on != 0;
  L.used = 0;
  return BSE_OK;
}

int bse_profile_read(int max_stages, double* ms, char* names) {
  bse::StageLog& L = bse::stage_log();
  if (L.used < 2) { L.used = 0; return 0; }
  cudaError_t e = cudaEventSynchronize(L.ev[L.used - 1]);
  if (e != cudaSuccess) return -cuda_fail(e, "profile");
  int k = 0;
  for (; k < L.used - 1 && k < max_stages; ++k) {
    float t = 0.f;
    cudaEventElapsedTime(&t, L.ev[k], L.ev[k + 1]);
    ms[k] = t;
    std::snprintf(names + 32 * k, 32, "%s", L.names[k].c_str());
  }
  L.used = 0;
  return k;
}

int bse_memcpy2d_staged(int to_device, void* dst, size_t dpitch, const void* src, size_t spitch,
                        size_t width_bytes, size_t rows, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = to_device ? bse::h2d_staged(dst, dpitch, src, spitch, width_bytes, rows, s)
                            : bse::d2h_staged(dst, dpitch, src, spitch, width_bytes, rows, s);
  BSE_TRY_CUDA(e, "memcpy2d_staged");
  return BSE_OK;
}

int bse_profile_count(void) {
  const bse::StageLog& L = bse::stage_log();
  return L.used > 1 ? L.used - 1 : 0;
}

long long bse_launch_count(void) { return bse::launch_counter().load(); }

int bse_release_cached_memory(void) {
  cudaMemPool_t pool;
  BSE_TRY_CUDA(host_pool(&pool), "memory pool");
  BSE_TRY_CUDA(cudaMemPoolTrimTo(pool, 0), "trim");
  return BSE_OK;
}

int bse_peak_fp64(int which, int blocks, int iters, int reps, double* flops, double* ms) {
  double* sink = nullptr;
  BSE_TRY_CUDA(cudaMalloc(&sink, 256 * sizeof(double)), "alloc");
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  bse::launch_peak(which, blocks, iters, sink, 0);  // warm-up
  cudaEventRecord(a, 0);
  double f = 0.0;
  for (int r = 0; r < reps; ++r) f = bse::launch_peak(which, blocks, iters, sink, 0);
  cudaEventRecord(b, 0);
  cudaError_t e = cudaEventSynchronize(b);
  float t = 0.f;
  cudaEventElapsedTime(&t, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  BSE_TRY_CUDA(e, "peak");
  *flops = f;
  *ms = t / reps;
  return BSE_OK;
}

/* ---- column-sharded multi-GPU solve ------------------------------------- */

struct bse_comm {
  bse::Comm* impl;
};

int bse_comm_nccl_unique_id(void* id128) {
  std::string err;
  if (!id128) return fail(BSE_BAD_ARGUMENT, "null id buffer");
  if (bse::nccl_unique_id(id128, &err) != 0) return fail(BSE_CUDA_ERROR, "nccl: " + err);
  return BSE_OK;
}

int bse_comm_create_nccl(int rank, int world, const void* id128, bse_comm** out) {
  if (!out || !id128 || world < 1 || rank < 0 || rank >= world)
    return fail(BSE_BAD_ARGUMENT, "bad communicator argument");
  std::string err;
  bse::Comm* c = bse::make_nccl_comm(rank, world, id128, &err);
  if (!c) return fail(BSE_CUDA_ERROR, "nccl: " + err);
  *out = new bse_comm{c};
  return BSE_OK;
}

int bse_comm_create_host(int rank, int world, bse_host_bcast_fn fn, void* ctx, bse_comm** out) {
  if (!out || !fn || world < 1 || rank < 0 || rank >= world)
    return fail(BSE_BAD_ARGUMENT, "bad communicator argument");
  *out = new bse_comm{bse::make_host_comm(rank, world, fn, ctx)};
  return BSE_OK;
}

int bse_comm_create_solo(int rank, int world, bse_comm** out) {
  if (!out || world < 1 || rank < 0 || rank >= world)
    return fail(BSE_BAD_ARGUMENT, "bad communicator argument");
  *out = new bse_comm{bse::make_solo_comm(rank, world)};
  return BSE_OK;
}

int bse_comm_destroy(bse_comm* comm) {
  if (comm) {
    delete comm->impl;
    delete comm;
  }
  return BSE_OK;
}

int bse_shard_range(int64_t n, int world, int rank, int64_t* c0, int64_t* c1) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !c0 || !c1)
    return fail(BSE_BAD_ARGUMENT, "bad shard argument");
  long long a, b;
  bse::shard_range(n, world, rank, &a, &b);
  *c0 = a;
  *c1 = b;
  return BSE_OK;
}

int bse_comm_allgather_cols_dev(bse_comm* comm, double* dA, int64_t ld, int64_t n, void* stream) {
  if (!comm || n < 0 || ld < 1) return fail(BSE_BAD_ARGUMENT, "bad argument");
  cudaError_t e = bse::allgather_cols(*comm->impl, dA, ld, n, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    const std::string why = comm->impl->error();
    return fail(BSE_CUDA_ERROR, "allgather_cols: " + (why.empty() ? std::string(cudaGetErrorString(e)) : why));
  }
  return BSE_OK;
}

int bse_solve_spd_pair_dist_dev(bse_comm* comm, int64_t n, const double* dM, int64_t ldm,
                                const double* dK, int64_t ldk, double* dLam, double* dX1,
                                int64_t ldx1, double* dX2, int64_t ldx2, void* dWork,
                                size_t work_bytes, int flags, void* stream, bse_info* info) {
  if (!comm) return fail(BSE_BAD_ARGUMENT, "null communicator");
  if (check_solve_flags(flags) != BSE_OK) return BSE_BAD_ARGUMENT;
  if (n < 0 || ldm < n || ldk < n || ldx1 < n || ldx2 < n)
    return fail(BSE_BAD_ARGUMENT, "bad dimension");
  if (n > 0 && work_bytes < bse::solve_bytes((int)n, flags))
    return fail(BSE_BAD_ARGUMENT, "workspace too small (see bse_solve_workspace_bytes)");
  bse::SolveStatus st{};
  cudaError_t e = bse::solve_spd_pair((int)n, dM, ldm, dK, ldk, dLam, dX1, ldx1, dX2, ldx2, dWork,
                                      work_bytes, flags, (cudaStream_t)stream, &st, nullptr,
                                      nullptr, comm->impl);
  if (e != cudaSuccess) {
    const std::string why = comm->impl->error();
    return fail(BSE_CUDA_ERROR, "solve_dist: " + (why.empty() ? std::string(cudaGetErrorString(e)) : why));
  }
  return map_solve_status(st, info);
}

/* ---- memory-distributed multi-GPU solve (block-cyclic column tiles) ------ */

static bool bc_args_ok(int64_t n, int nb, int world, int rank) {
  return n >= 0 && n < (1ll << 31) && nb >= 64 && nb % 64 == 0 && world >= 1 && rank >= 0 &&
         rank < world;
}

int64_t bse_bc_local_cols(int64_t n, int nb, int world, int rank) {
  if (!bc_args_ok(n, nb, world, rank)) return -1;
  bse::BcLayout lay;
  lay.n = (int)n; lay.nb = nb; lay.world = world; lay.rank = rank;
  return lay.ncols_of(rank);
}

int64_t bse_bc_global_col(int64_t local_col, int nb, int world, int rank) {
  if (local_col < 0 || !bc_args_ok(0, nb, world, rank)) return -1;
  return ((local_col / nb) * world + rank) * (int64_t)nb + local_col % nb;
}

size_t bse_solve_bc_workspace_bytes(int64_t n, int nb, int world, int rank, int flags,
                                    size_t* distributed, size_t* replicated) {
  if (!bc_args_ok(n, nb, world, rank)) return 0;
  const bse::DistBytes b = bse::dist_solve_bytes((int)n, nb, world, rank, flags);
  if (distributed) *distributed = b.distributed;
  if (replicated) *replicated = b.replicated;
  return b.total;
}

int bse_solve_spd_pair_bc_dev(bse_comm* comm, int64_t n, int nb, const double* dMloc, int64_t ldm,
                              const double* dKloc, int64_t ldk, double* dLam, double* dX1loc,
                              int64_t ldx1, double* dX2loc, int64_t ldx2, void* dWork,
                              size_t work_bytes, int flags, void* stream, bse_info* info) {
  if (!comm) return fail(BSE_BAD_ARGUMENT, "null communicator");
  if (check_solve_flags(flags) != BSE_OK) return BSE_BAD_ARGUMENT;
  if (!bc_args_ok(n, nb, comm->impl->world, comm->impl->rank))
    return fail(BSE_BAD_ARGUMENT, "bad dimension or tile (nb must be a multiple of 64)");
  if (ldm < n || ldk < n || ldx1 < n || ldx2 < n) return fail(BSE_BAD_ARGUMENT, "bad leading dimension");
  if (n > 0 && work_bytes < bse::dist_solve_bytes((int)n, nb, comm->impl->world, comm->impl->rank,
                                                  flags).total)
    return fail(BSE_BAD_ARGUMENT, "workspace too small (see bse_solve_bc_workspace_bytes)");
  bse::SolveStatus st{};
  cudaError_t e = bse::solve_spd_pair_bc(*comm->impl, (int)n, nb, dMloc, ldm, dKloc, ldk, dLam,
                                         dX1loc, ldx1, dX2loc, ldx2, dWork, work_bytes, flags,
                                         (cudaStream_t)stream, &st);
  if (e != cudaSuccess) {
    const std::string why = comm->impl->error();
    return fail(BSE_CUDA_ERROR, "solve_bc: " + (why.empty() ? std::string(cudaGetErrorString(e)) : why));
  }
  return map_solve_status(st, info);
}

int bse_comm_allreduce_sum_dev(bse_comm* comm, double* dptr, size_t count, void* stream) {
  if (!comm || (!dptr && count)) return fail(BSE_BAD_ARGUMENT, "bad argument");
  cudaError_t e = comm->impl->allreduce_sum(dptr, count, (cudaStream_t)stream);
  if (e != cudaSuccess) {
    const std::string why = comm->impl->error();
    return fail(BSE_CUDA_ERROR, "allreduce: " + (why.empty() ? std::string(cudaGetErrorString(e)) : why));
  }
  return BSE_OK;
}

}  // extern "C"
