// extern "C" boundary (include/bse_b200.h).  Never throws across the ABI:
// every entry point returns a bse_status and records a message retrievable
// with bse_last_error().
#include <cstdio>
#include <cstring>
#include <string>
#include "../../include/bse_b200.h"
#include "dense.cuh"
#include "solver.cuh"

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
  bse::DevStatus h0{-1, 0, 0.0, 0.0};
  BSE_TRY_CUDA(cudaMemcpyAsync(st, &h0, sizeof(h0), cudaMemcpyHostToDevice, s), "status init");
  cudaError_t e = bse::potrf_lower(dA, lda, (int)n, st, s);
  bse::DevStatus h;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFreeAsync(st, s);
  BSE_TRY_CUDA(e, "potrf");
  if (h.info >= 0) {
    if (info) { info->pivot_index = h.info; info->pivot_value = h.value; info->failed_factor = 0; }
    return fail(BSE_NOT_POSITIVE_DEFINITE, "matrix is not positive definite");
  }
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

}  // extern "C"
