// Stage 2: band -> tridiagonal by bulge chasing (Schwarz/Lang element
// annihilation, the task structure of LAPACK's SB2ST kernels), as one
// persistent cooperative kernel.  Sweep s is owned by CTA s mod G; step j of
// sweep s may start once sweep s-1 has finished step j+1 (a release/acquire
// progress counter per sweep), so ~N/(2b) sweeps are in flight at once.  The
// band (ldab = 2b doubles per column) stays L2-resident; every reflector is
// stored for the Q2 back-transform.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "eig.cuh"

namespace bse {
namespace {

constexpr int kSbThreads = 256;
constexpr int kDone = 0x7fffffff;
constexpr int kLd = kMaxPanel + 1;
constexpr int kSlots = kMaxPanel * kMaxPanel / kSbThreads;  // 16 block slots per thread

struct SbSmem {
  double D[kMaxPanel * kLd];  // symmetric block, full, [c*kLd + r]
  double O[kMaxPanel * kLd];  // off-diagonal block, [c*kLd + r]
  double v[kMaxPanel];        // current reflector
  double vn[kMaxPanel];       // new reflector
  double w[kMaxPanel];
  double part[4 * kMaxPanel];
  double sc[4];
};

BSE_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Householder of x[0..len) (one warp, LAPACK dlarfg conventions): v (v[0]=1),
// sc[0] = tau, sc[1] = beta.
BSE_DEV void warp_house(const double* x, int len, double* v, double* sc) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
  for (int i = 1 + lane; i < len; i += 32) s += x[i] * x[i];
  s = warp_sum(s);
  const double x0 = x[0];
  double tau = 0.0, beta = x0, scale = 0.0;
  if (s > 0.0) {
    beta = -copysign(sqrt(x0 * x0 + s), x0);
    tau = (beta - x0) / beta;
    scale = 1.0 / (x0 - beta);
  }
  for (int i = lane; i < kMaxPanel; i += 32)
    v[i] = (i == 0) ? 1.0 : ((i < len && tau != 0.0) ? x[i] * scale : 0.0);
  if (lane == 0) { sc[0] = tau; sc[1] = beta; }
}

__constant__ int c_sb_flags;  // tuning variants (BSE_SB2ST_VARIANT), default 0

BSE_DEV void wait_progress(const int* progress, int s, int need) {
  if (s > 0 && threadIdx.x == 0) {
    // relaxed polling (no L1 invalidation per probe), one acquire fence after
    if (ld_relaxed(progress + s - 1) < need) {
      const int ns = (c_sb_flags & 1) ? 256 : 0;
      while (ld_relaxed(progress + s - 1) < need) {
        if (ns) __nanosleep(ns);
      }
    }
    fence_acquire();
  }
  __syncthreads();
}

BSE_DEV void signal_progress(int* progress, int s, int val) {
  __syncthreads();
  if (threadIdx.x == 0) {
    if (c_sb_flags & 2) fence_acquire();  // acq_rel fence (cheaper than sc)
    else __threadfence();
    st_release(progress + s, val);
  }
}

// Stage the len x len symmetric block at (q0, q0) (lower triangle in the band)
// and, optionally, the lq x lp off-diagonal block at (q0, p0) into smem with
// cp.async: every load of the step is in flight at once (one L2 round trip).
BSE_DEV void stage_blocks(SbSmem& sm, const double* AB, int ldab, int q0, int len, bool with_o,
                          int p0, int lp) {
  const int tid = threadIdx.x;
#pragma unroll 4
  for (int k = 0; k < kSlots; ++k) {
    const int idx = tid + k * kSbThreads;
    const int r = idx & (kMaxPanel - 1), c = idx >> 6;
    const bool dv = r < len && c <= r;
    const double* ds = dv ? AB + (long long)(q0 + c) * ldab + (r - c) : AB;
    cp_async8(&sm.D[c * kLd + r], ds, dv);
    if (with_o) {
      const bool ov = r < len && c < lp;
      const double* os = ov ? AB + (long long)(p0 + c) * ldab + (q0 + r - p0 - c) : AB;
      cp_async8(&sm.O[c * kLd + r], os, ov);
    }
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  // mirror the lower triangle of D into the upper one
#pragma unroll 4
  for (int k = 0; k < kSlots; ++k) {
    const int idx = tid + k * kSbThreads;
    const int r = idx & (kMaxPanel - 1), c = idx >> 6;
    if (c > r) sm.D[c * kLd + r] = sm.D[r * kLd + c];
  }
  __syncthreads();
}

// Column-sum matvec out_c = scale * sum_r X[c][r] x[r] (X column-major in smem,
// 8 columns per warp, lanes over rows: conflict-free, shuffle-reduced).
BSE_DEV void colsum(const double* X, const double* x, int nrows, double scale, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int u = 0; u < kMaxPanel / 8; ++u) {
    const int c = warp + 8 * u;
    double a = 0.0;
    if (lane < nrows) a = X[c * kLd + lane] * x[lane];
    if (lane + 32 < nrows) a += X[c * kLd + lane + 32] * x[lane + 32];
    a = warp_sum(a);
    if (lane == 0) out[c] = scale * a;
  }
}

// Two-sided D <- H D H (H = I - tau v v^T) on the staged symmetric block; the
// lower triangle of the result is stored straight to the band.
BSE_DEV void two_sided_store(SbSmem& sm, int len, const double* v, double tau, double* AB,
                             int ldab, int q0) {
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  colsum(sm.D, v, len, tau, sm.w);  // D symmetric: column sums == row sums
  __syncthreads();
  if (tid < 32) {
    double a = 0.0;
    for (int i = lane; i < len; i += 32) a += sm.w[i] * v[i];
    a = warp_sum(a);
    if (lane == 0) sm.sc[2] = -0.5 * tau * a;
  }
  __syncthreads();
  const double alpha = sm.sc[2];
#pragma unroll
  for (int k = 0; k < kSlots; ++k) {
    const int idx = tid + k * kSbThreads;
    const int r = idx & (kMaxPanel - 1), c = idx >> 6;
    if (r < len && c <= r) {
      const double wr = sm.w[r] + alpha * v[r], wc = sm.w[c] + alpha * v[c];
      const double val = sm.D[c * kLd + r] - (v[r] * wc + wr * v[c]);
      AB[(long long)(q0 + c) * ldab + (r - c)] = val;
    }
  }
}

__global__ void __launch_bounds__(kSbThreads) sb2st_kernel(double* AB, int ldab, int n, int b,
                                                           double* V2, double* tau2,
                                                           int maxsteps, int* progress,
                                                           unsigned long long* trace) {
  extern __shared__ __align__(16) unsigned char raw[];
  SbSmem& sm = *reinterpret_cast<SbSmem*>(raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const bool tr = trace != nullptr && blockIdx.x == 1 && threadIdx.x == 0;
  int tcount = 0;
  auto bidx = [&](int i, int j) -> long long { return (long long)j * ldab + (i - j); };

  for (int s = blockIdx.x; s < n - 2; s += gridDim.x) {
    const bool trs = tr && s < 1 + 2 * (int)gridDim.x;
    // ---------------- step 0: annihilate column s ----------------
    if (trs) trace[8 * tcount] = gtimer();
    wait_progress(progress, s, 2);
    if (trs) trace[8 * tcount + 1] = gtimer();
    int p0 = s + 1, p1 = min(s + b, n - 1);
    int lp = p1 - p0 + 1;
    if (tid < kMaxPanel) sm.w[tid] = tid < lp ? __ldcg(AB + bidx(p0 + tid, s)) : 0.0;
    stage_blocks(sm, AB, ldab, p0, lp, false, 0, 0);
    if (tid < 32) warp_house(sm.w, lp, sm.v, sm.sc);
    __syncthreads();
    double tau = sm.sc[0];
    if (tid < lp) AB[bidx(p0 + tid, s)] = (tid == 0) ? sm.sc[1] : 0.0;
    if (tid < b) V2[((long long)s * maxsteps) * b + tid] = sm.v[tid];
    if (tid == 0) tau2[(long long)s * maxsteps] = tau;
    if (tau != 0.0) two_sided_store(sm, lp, sm.v, tau, AB, ldab, p0);
    signal_progress(progress, s, 1);
    if (trs) { for (int q = 2; q < 8; ++q) trace[8 * tcount + q] = gtimer(); ++tcount; }

    // ---------------- steps j >= 1: chase the bulge ----------------
    for (int j = 1;; ++j) {
      const int q0 = p1 + 1;
      if (q0 > n - 1) break;
      const int q1 = min(p1 + b, n - 1);
      const int lq = q1 - q0 + 1;
      if (trs) trace[8 * tcount] = gtimer();
      wait_progress(progress, s, j + 2);
      if (trs) trace[8 * tcount + 1] = gtimer();
      stage_blocks(sm, AB, ldab, q0, lq, true, p0, lp);
      if (trs) trace[8 * tcount + 2] = gtimer();
      if (tau != 0.0) {
        // right-apply: w = tau O v (row sums: 4 partial sums per row, lanes
        // over consecutive rows -> conflict-free), O -= w v^T
        {
          const int r = tid & (kMaxPanel - 1), q = tid >> 6;
          double a = 0.0;
          for (int c = q; c < lp; c += 4) a += sm.O[c * kLd + r] * sm.v[c];
          sm.part[q * kMaxPanel + r] = a;
        }
        __syncthreads();
        if (tid < kMaxPanel)
          sm.w[tid] = tau * ((sm.part[tid] + sm.part[kMaxPanel + tid]) +
                             (sm.part[2 * kMaxPanel + tid] + sm.part[3 * kMaxPanel + tid]));
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kSlots; ++k) {
          const int idx = tid + k * kSbThreads;
          const int rr = idx & (kMaxPanel - 1), c = idx >> 6;
          sm.O[c * kLd + rr] -= sm.w[rr] * sm.v[c];
        }
        __syncthreads();
      }
      if (trs) trace[8 * tcount + 3] = gtimer();
      if (tid < 32) warp_house(sm.O, lq, sm.vn, sm.sc);
      __syncthreads();
      if (trs) trace[8 * tcount + 4] = gtimer();
      const double taun = sm.sc[0], betan = sm.sc[1];
      // left-apply to columns >= 1: y_c = taun * vn^T O[:, c] (column sums)
      if (taun != 0.0) {
        colsum(sm.O, sm.vn, lq, taun, sm.w);
        __syncthreads();
      }
      // store O (column 0 = (beta, 0, ...)), reflector, then the two-sided D update
#pragma unroll
      for (int k = 0; k < kSlots; ++k) {
        const int idx = tid + k * kSbThreads;
        const int r = idx & (kMaxPanel - 1), c = idx >> 6;
        if (r < lq && c < lp) {
          double val;
          if (c == 0) val = (r == 0) ? betan : 0.0;
          else val = taun != 0.0 ? sm.O[c * kLd + r] - sm.vn[r] * sm.w[c] : sm.O[c * kLd + r];
          AB[bidx(q0 + r, p0 + c)] = val;
        }
      }
      if (tid < b) V2[((long long)s * maxsteps + j) * b + tid] = sm.vn[tid];
      if (tid == 0) tau2[(long long)s * maxsteps + j] = taun;
      __syncthreads();
      if (trs) trace[8 * tcount + 5] = gtimer();
      if (taun != 0.0) two_sided_store(sm, lq, sm.vn, taun, AB, ldab, q0);
      if (trs) trace[8 * tcount + 6] = gtimer();
      __syncthreads();
      if (tid < kMaxPanel) sm.v[tid] = sm.vn[tid];
      tau = taun;
      signal_progress(progress, s, j + 1);
      if (trs) { trace[8 * tcount + 7] = gtimer(); ++tcount; }
      p0 = q0;
      p1 = q1;
      lp = lq;
    }
    signal_progress(progress, s, kDone);
    __syncthreads();
  }
  (void)lane;
  (void)warp;
}

__global__ void band_to_tridiag_kernel(const double* AB, int ldab, int n, double* d, double* e) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    d[i] = AB[(long long)i * ldab];
    if (i < n - 1) e[i] = AB[(long long)i * ldab + 1];
  }
}

}  // namespace

int sb2st_maxsteps(int n, int b) { return (int)ceil_div(n, b) + 1; }

cudaError_t sb2st(double* AB, int ldab, int n, int b, double* d, double* e, double* V2,
                  double* tau2, int* progress, int num_sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err;
  if (n > 2) {
    if ((err = cudaMemsetAsync(progress, 0, sizeof(int) * n, s)) != cudaSuccess) return err;
    const size_t smem = sizeof(SbSmem);
    static bool attr = false;
    if (!attr) {
      err = cudaFuncSetAttribute(sb2st_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (err != cudaSuccess) return err;
      attr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sb2st_kernel, kSbThreads, smem);
    int flags = 0;
    if (const char* v = std::getenv("BSE_SB2ST_VARIANT")) flags = std::atoi(v);
    cudaMemcpyToSymbolAsync(c_sb_flags, &flags, sizeof(int), 0, cudaMemcpyHostToDevice, s);
    if (!(flags & 8)) per_sm = 1;  // default 1 CTA/SM (flag 8 restores full occupancy)
    int grid = std::max(1, std::min(n - 2, std::max(1, per_sm) * num_sms));
    int maxsteps = sb2st_maxsteps(n, b);
    unsigned long long* trace = nullptr;
    const bool want_trace = std::getenv("BSE_SB2ST_TRACE") != nullptr;
    const int tmax = 2 * (maxsteps + 1);
    if (want_trace) {
      cudaMalloc(&trace, sizeof(unsigned long long) * 8 * tmax);
      cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 8 * tmax, s);
    }
    void* args[] = {&AB, &ldab, &n, &b, &V2, &tau2, &maxsteps, &progress, &trace};
    count_launch();
    err = cudaLaunchCooperativeKernel((void*)sb2st_kernel, dim3(grid), dim3(kSbThreads), args, smem, s);
    if (err != cudaSuccess) return err;
    if (want_trace) {
      std::vector<unsigned long long> h(8 * tmax);
      cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      cudaFree(trace);
      double acc[8] = {0};
      int cnt = 0;
      for (int k = 0; k < tmax; ++k) {
        if (!h[8 * k + 7]) break;
        for (int q = 1; q < 8; ++q) acc[q] += (double)(h[8 * k + q] - h[8 * k + q - 1]);
        ++cnt;
      }
      const double d = std::max(cnt, 1) * 1e3;
      std::fprintf(stderr, "[sb2st trace] grid=%d steps=%d us: wait %.2f load %.2f right %.2f house %.2f "
                   "left+storeO %.2f twosided %.2f signal %.2f\n", grid, cnt, acc[1] / d, acc[2] / d,
                   acc[3] / d, acc[4] / d, acc[5] / d, acc[6] / d, acc[7] / d);
    }
  }
  band_to_tridiag_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(AB, ldab, n, d, e);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bse
