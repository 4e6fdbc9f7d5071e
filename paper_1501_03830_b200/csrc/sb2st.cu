// Stage 2: band -> tridiagonal by bulge chasing (Schwarz/Lang element
// annihilation, the task structure of LAPACK's SB2ST kernels), as one
// persistent cooperative kernel.  Sweep s is owned by CTA s mod G; step j of
// sweep s may start once sweep s-1 has finished step j+1 (a release/acquire
// progress counter per sweep), so ~N/(2b) sweeps are in flight at once.  The
// band (ldab = 2b doubles per column) stays L2-resident; every reflector is
// stored for the Q2 back-transform.
#include "eig.cuh"

namespace bse {
namespace {

constexpr int kSbThreads = 128;
constexpr int kDone = 0x7fffffff;

struct SbSmem {
  double D[kMaxPanel * (kMaxPanel + 1)];  // symmetric block, [c*(b+1) + r]
  double O[kMaxPanel * (kMaxPanel + 1)];  // off-diagonal block, [c*(b+1) + r]
  double v[kMaxPanel];
  double vn[kMaxPanel];
  double w[kMaxPanel];
  double red[32];
  double sc[4];
};

// Householder of x[0..len) held in smem (one warp); writes v (v[0]=1) and
// returns tau/beta through sc.  LAPACK dlarfg conventions.
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
  for (int i = lane; i < len; i += 32) v[i] = (i == 0) ? 1.0 : (tau != 0.0 ? x[i] * scale : 0.0);
  if (lane == 0) { sc[0] = tau; sc[1] = beta; }
}

BSE_DEV void wait_progress(const int* progress, int s, int need) {
  if (s <= 0) return;
  if (threadIdx.x == 0) {
    while (ld_acquire(progress + s - 1) < need) __nanosleep(64);
  }
  __syncthreads();
}

BSE_DEV void signal_progress(int* progress, int s, int val) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    st_release(progress + s, val);
  }
}

// D (len x len symmetric, full in smem) <- H D H, H = I - tau v v^T.
BSE_DEV void two_sided(double* D, int ldd, int len, const double* v, double tau, double* w,
                       double* red) {
  const int tid = threadIdx.x;
  if (tau == 0.0) return;
  // p = tau D v
  for (int i = tid; i < len; i += blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < len; ++k) s += D[k * ldd + i] * v[k];
    w[i] = tau * s;
  }
  __syncthreads();
  // alpha = -0.5 tau p^T v
  if (tid < 32) {
    double s = 0.0;
    for (int i = tid; i < len; i += 32) s += w[i] * v[i];
    s = warp_sum(s);
    if (tid == 0) red[0] = -0.5 * tau * s;
  }
  __syncthreads();
  const double alpha = red[0];
  for (int i = tid; i < len; i += blockDim.x) w[i] += alpha * v[i];
  __syncthreads();
  for (int idx = tid; idx < len * len; idx += blockDim.x) {
    const int r = idx % len, c = idx / len;
    D[c * ldd + r] -= v[r] * w[c] + w[r] * v[c];
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kSbThreads) sb2st_kernel(double* AB, int ldab, int n, int b,
                                                           double* V2, double* tau2,
                                                           int maxsteps, int* progress) {
  extern __shared__ __align__(16) unsigned char raw[];
  SbSmem& sm = *reinterpret_cast<SbSmem*>(raw);
  const int tid = threadIdx.x;
  const int ld = kMaxPanel + 1;
  auto band = [&](int i, int j) -> double* { return AB + (long long)j * ldab + (i - j); };

  for (int s = blockIdx.x; s < n - 2; s += gridDim.x) {
    // ---------------- step 0: annihilate column s ----------------
    wait_progress(progress, s, 2);
    int p0 = s + 1, p1 = min(s + b, n - 1);
    int lp = p1 - p0 + 1;
    for (int i = tid; i < lp; i += blockDim.x) sm.w[i] = __ldcg(band(p0 + i, s));
    __syncthreads();
    if (tid < 32) warp_house(sm.w, lp, sm.v, sm.sc);
    __syncthreads();
    double tau = sm.sc[0];
    const double beta0 = sm.sc[1];
    for (int i = tid; i < lp; i += blockDim.x) *band(p0 + i, s) = (i == 0) ? beta0 : 0.0;
    double* vslot = V2 + ((long long)s * maxsteps) * b;
    for (int i = tid; i < b; i += blockDim.x) vslot[i] = i < lp ? sm.v[i] : 0.0;
    if (tid == 0) tau2[(long long)s * maxsteps] = tau;
    // D block
    for (int idx = tid; idx < lp * lp; idx += blockDim.x) {
      const int r = idx % lp, c = idx / lp;
      if (r >= c) {
        const double x = __ldcg(band(p0 + r, p0 + c));
        sm.D[c * ld + r] = x;
        sm.D[r * ld + c] = x;
      }
    }
    __syncthreads();
    two_sided(sm.D, ld, lp, sm.v, tau, sm.w, sm.red);
    for (int idx = tid; idx < lp * lp; idx += blockDim.x) {
      const int r = idx % lp, c = idx / lp;
      if (r >= c) *band(p0 + r, p0 + c) = sm.D[c * ld + r];
    }
    signal_progress(progress, s, 1);

    // ---------------- steps j >= 1: chase the bulge ----------------
    int j = 1;
    while (true) {
      const int q0 = p1 + 1;
      if (q0 > n - 1) break;
      const int q1 = min(p1 + b, n - 1);
      const int lq = q1 - q0 + 1;
      wait_progress(progress, s, j + 2);
      // O block rows q0..q1, cols p0..p1
      for (int idx = tid; idx < lq * lp; idx += blockDim.x) {
        const int r = idx % lq, c = idx / lq;
        sm.O[c * ld + r] = __ldcg(band(q0 + r, p0 + c));
      }
      __syncthreads();
      if (tau != 0.0) {
        // right-apply: O <- O (I - tau v v^T)
        for (int r = tid; r < lq; r += blockDim.x) {
          double acc = 0.0;
          for (int c = 0; c < lp; ++c) acc += sm.O[c * ld + r] * sm.v[c];
          sm.w[r] = tau * acc;
        }
        __syncthreads();
        for (int idx = tid; idx < lq * lp; idx += blockDim.x) {
          const int r = idx % lq, c = idx / lq;
          sm.O[c * ld + r] -= sm.w[r] * sm.v[c];
        }
        __syncthreads();
      }
      // new reflector from the first column of O
      if (tid < 32) warp_house(sm.O, lq, sm.vn, sm.sc);
      __syncthreads();
      const double taun = sm.sc[0], betan = sm.sc[1];
      // left-apply to O[:, 1:]: y_c = vn^T O[:, c]
      if (taun != 0.0) {
        for (int c = 1 + tid; c < lp; c += blockDim.x) {
          double acc = 0.0;
          for (int r = 0; r < lq; ++r) acc += sm.vn[r] * sm.O[c * ld + r];
          sm.w[c] = taun * acc;
        }
        __syncthreads();
        for (int idx = tid; idx < lq * (lp - 1); idx += blockDim.x) {
          const int r = idx % lq, c = 1 + idx / lq;
          sm.O[c * ld + r] -= sm.vn[r] * sm.w[c];
        }
      }
      __syncthreads();
      if (tid == 0) sm.O[0] = betan;
      for (int r = 1 + tid; r < lq; r += blockDim.x) sm.O[r] = 0.0;
      __syncthreads();
      for (int idx = tid; idx < lq * lp; idx += blockDim.x) {
        const int r = idx % lq, c = idx / lq;
        *band(q0 + r, p0 + c) = sm.O[c * ld + r];
      }
      // store reflector (s, j)
      double* vs = V2 + ((long long)s * maxsteps + j) * b;
      for (int i = tid; i < b; i += blockDim.x) vs[i] = i < lq ? sm.vn[i] : 0.0;
      if (tid == 0) tau2[(long long)s * maxsteps + j] = taun;
      // two-sided on the next diagonal block
      for (int idx = tid; idx < lq * lq; idx += blockDim.x) {
        const int r = idx % lq, c = idx / lq;
        if (r >= c) {
          const double x = __ldcg(band(q0 + r, q0 + c));
          sm.D[c * ld + r] = x;
          sm.D[r * ld + c] = x;
        }
      }
      __syncthreads();
      two_sided(sm.D, ld, lq, sm.vn, taun, sm.w, sm.red);
      for (int idx = tid; idx < lq * lq; idx += blockDim.x) {
        const int r = idx % lq, c = idx / lq;
        if (r >= c) *band(q0 + r, q0 + c) = sm.D[c * ld + r];
      }
      for (int i = tid; i < lq; i += blockDim.x) sm.v[i] = sm.vn[i];
      tau = taun;
      signal_progress(progress, s, j + 1);
      p0 = q0;
      p1 = q1;
      lp = lq;
      ++j;
    }
    signal_progress(progress, s, kDone);
    __syncthreads();
  }
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
    int grid = std::max(1, std::min(n - 2, std::max(1, per_sm) * num_sms));
    int maxsteps = sb2st_maxsteps(n, b);
    void* args[] = {&AB, &ldab, &n, &b, &V2, &tau2, &maxsteps, &progress};
    count_launch();
    err = cudaLaunchCooperativeKernel((void*)sb2st_kernel, dim3(grid), dim3(kSbThreads), args, smem, s);
    if (err != cudaSuccess) return err;
  }
  band_to_tridiag_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(AB, ldab, n, d, e);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bse
