// Dipole-weighted absorption spectrum (spectra.py:120-151 restated on the
// GPU): one warp per eigenpair for the projections d_r^H x_j, y_j^H d_l and
// the pairing y_j^H x_j (HBM-bound: X1, X2 are read once), then one thread
// per grid point accumulating the truncated Gaussians in eigenvalue order,
// which is the reference's accumulation order (spectra.py:83-85) and keeps
// the curve deterministic.
#include "solver.cuh"

namespace bse {
namespace {

struct cplx { double re, im; };

__global__ void absorption_weights_kernel(int n, const cplx* __restrict__ X1, long long ldx1,
                                          const cplx* __restrict__ X2, long long ldx2,
                                          const cplx* __restrict__ dr, const cplx* __restrict__ dl,
                                          double* __restrict__ weights, double* __restrict__ pair_abs,
                                          double* __restrict__ pair_defect) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= n) return;
  const cplx* x1 = X1 + (long long)j * ldx1;
  const cplx* x2 = X2 + (long long)j * ldx2;
  // p = y^H x = sum conj(x1) x1 - conj(x2) x2 (complex, as the reference forms it)
  double pr = 0, pi = 0, rr = 0, ri = 0, lr = 0, li = 0;
  for (int i = lane; i < n; i += 32) {
    const cplx a = x1[i], b = x2[i];
    pr += a.re * a.re + a.im * a.im - (b.re * b.re + b.im * b.im);
    pi += (a.re * a.im - a.im * a.re) - (b.re * b.im - b.im * b.re);
    // right = d_r^H x: conj(dr_i) x_i over the stacked [x1; x2]
    const cplx d1 = dr[i], d2 = dr[n + i];
    rr += d1.re * a.re + d1.im * a.im + d2.re * b.re + d2.im * b.im;
    ri += d1.re * a.im - d1.im * a.re + d2.re * b.im - d2.im * b.re;
    // left = y^H d_l with y = [x1; -x2]: conj(x1) dl1 - conj(x2) dl2
    const cplx e1 = dl[i], e2 = dl[n + i];
    lr += a.re * e1.re + a.im * e1.im - (b.re * e2.re + b.im * e2.im);
    li += a.re * e1.im - a.im * e1.re - (b.re * e2.im - b.im * e2.re);
  }
  pr = warp_sum(pr); pi = warp_sum(pi);
  rr = warp_sum(rr); ri = warp_sum(ri);
  lr = warp_sum(lr); li = warp_sum(li);
  if (lane == 0) {
    // w = Re[(right * left) / p]
    const double nr = rr * lr - ri * li, ni = rr * li + ri * lr;
    const double den = pr * pr + pi * pi;
    weights[j] = den > 0.0 ? (nr * pr + ni * pi) / den : 0.0;
    pair_abs[j] = sqrt(den);
    pair_defect[j] = hypot(pr - 1.0, pi);
  }
}

__global__ void reduce_minmax_kernel(int n, const double* pair_abs, const double* pair_defect,
                                     double* minpair, double* defect) {
  __shared__ double smin[32], smax[32];
  double mn = 1e300, mx = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    mn = fmin(mn, pair_abs[i]);
    mx = fmax(mx, pair_defect[i]);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = mn; smax[threadIdx.x >> 5] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mn = fmin(mn, smin[w]); mx = fmax(mx, smax[w]); }
    mn = fmin(mn, smin[0]);
    mx = fmax(mx, smax[0]);
    *minpair = n ? mn : 1.0;
    *defect = n ? mx : 0.0;
  }
}

__global__ void gaussian_mix_kernel(int n, const double* __restrict__ lam,
                                    const double* __restrict__ w, int ngrid,
                                    const double* __restrict__ grid, double sigma,
                                    double* __restrict__ out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngrid) return;
  const double x = grid[g];
  const double peak = 1.0 / (sqrt(2.0 * 3.141592653589793) * sigma);
  const double reach = 8.0 * sigma;
  double acc = 0.0;
  for (int j = 0; j < n; ++j) {
    const double c = lam[j];
    if (x >= c - reach && x <= c + reach) {
      const double t = (x - c) / sigma;
      acc += (w[j] * peak) * exp(-0.5 * t * t);
    }
  }
  out[g] = acc;
}

}  // namespace

cudaError_t absorption(int n, const double* lam, const double* X1c, long long ldx1,
                       const double* X2c, long long ldx2, const double* dr, const double* dl,
                       int ngrid, const double* grid, double sigma, double* weights,
                       double* values, double* defect, double* minpair, cudaStream_t s) {
  double* tmp = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&tmp, sizeof(double) * 2 * (size_t)std::max(n, 1), s);
  if (e != cudaSuccess) return e;
  if (n > 0)
    absorption_weights_kernel<<<(unsigned)ceil_div(n, 8), 256, 0, s>>>(
        n, reinterpret_cast<const cplx*>(X1c), ldx1, reinterpret_cast<const cplx*>(X2c), ldx2,
        reinterpret_cast<const cplx*>(dr), reinterpret_cast<const cplx*>(dl), weights, tmp, tmp + n);
    count_launch();
  reduce_minmax_kernel<<<1, 1024, 0, s>>>(n, tmp, tmp + n, minpair, defect);
  count_launch();
  if (ngrid > 0)
    gaussian_mix_kernel<<<(unsigned)ceil_div(ngrid, 128), 128, 0, s>>>(n, lam, weights, ngrid, grid,
                                                                       sigma, values);
    count_launch();
  e = cudaGetLastError();
  cudaFreeAsync(tmp, s);
  return e;
}

}  // namespace bse
