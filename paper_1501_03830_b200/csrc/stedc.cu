// Symmetric tridiagonal divide and conquer (Cuppen splitting, LAPACK
// dlaed2-style deflation, Gu-Eisenstat Loewner z-hat for orthogonal
// vectors), level-synchronous on the GPU.  Replaces the reference's
// bisection + inverse iteration + Gram-Schmidt (kernels.py:262-535), whose
// two CGS passes against all previous vectors are O(m k^2) BLAS-2.
//
// Tree: leaves are 1x1; level l merges nodes [i*2^l, min((i+1)*2^l, n)) from
// children of size 2^(l-1).  Every node's eigenvectors live in the diagonal
// block Q[lo:hi, lo:hi] of a ping-pong pair of n x n buffers; per level:
//   prepare (z, merge-sort, deflation scan) -> secular roots (one thread per
//   root) -> z-hat -> output ordering -> eigenvector columns -> deflation
//   rotations -> grouped DMMA GEMM Q_out = diag(Q1, Q2) * U.
#include <cstdio>
#include <cstdlib>
#include "eig.cuh"
#include "ozgemm.cuh"

namespace bse {
namespace {

constexpr int kDcThreads = 256;

struct Level {
  int size;  // 2^l
  int half;  // 2^(l-1)
  int nnodes;
};

BSE_DEV void node_range(const Level& L, int n, int i, int& lo, int& mid, int& hi) {
  lo = i * L.size;
  hi = min(lo + L.size, n);
  mid = min(lo + L.half, hi);
}

__global__ void dc_init_kernel(int n, const double* d, const double* e, double* D, double* Q,
                               long long ld, const double* scal, int r0, int r1) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double inv = scal[0] > 0.0 ? 1.0 / scal[0] : 1.0;
  double v = d[i] * inv;
  // Cuppen splitting at every boundary: T = diag(T^1, T^2) + |b| w w^T
  if (i > 0) v -= fabs(e[i - 1] * inv);
  if (i < n - 1) v -= fabs(e[i] * inv);
  D[i] = v;
  if (i >= r0 && i < r1) Q[(i - r0) + (long long)i * ld] = 1.0;
}

// Non-finite input guard: the D&C's index logic (sorting, deflation) assumes
// finite data, so NaN / Inf in d or e are replaced by 0 in private copies and
// reported through *fail (BSE_NO_CONVERGENCE) instead of reaching it.
__global__ void sanitize_kernel(int n, const double* d, const double* e, double* ds, double* es,
                                int* fail) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool bad = false;
  double v = d[i];
  if (!isfinite(v)) { v = 0.0; bad = true; }
  ds[i] = v;
  if (i < n - 1) {
    double f = e[i];
    if (!isfinite(f)) { f = 0.0; bad = true; }
    es[i] = f;
  }
  if (bad && fail) atomicOr(fail, 1);
}

__global__ void absmax_kernel(int n, const double* d, const double* e, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    m = fmax(m, fabs(d[i]));
    if (i < n - 1) m = fmax(m, fabs(e[i]));
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    t = warp_max(t);
    if (threadIdx.x == 0) out[0] = t;
  }
}

// Row-distributed mode: zrow[c] = the entry of column c in its child's
// boundary row (last row of the first child, first row of the second), from
// the rank that owns that row; 0 elsewhere, so a sum over ranks is exact.
__global__ void dc_zrow_kernel(Level L, int n, const double* __restrict__ Qin, long long ld, int r0,
                               int r1, double* __restrict__ zrow) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  int lo, mid, hi;
  node_range(L, n, c / L.size, lo, mid, hi);
  double v = 0.0;
  if (mid < hi) {
    const int row = c < mid ? mid - 1 : mid;
    if (row >= r0 && row < r1) v = Qin[(row - r0) + (long long)c * ld];
  }
  zrow[c] = v;
}

// ---- 1. z vector, merge-sort of the children's eigenvalues, deflation ----
constexpr int kDcScanChunk = 2048;
__global__ void __launch_bounds__(kDcThreads) dc_prepare_kernel(
    Level L, int n, const double* __restrict__ e, const double* __restrict__ scal,
    const double* __restrict__ Din, double* __restrict__ Dout, const double* __restrict__ Qin,
    double* __restrict__ Qout, long long ld, StedcWork w, int r0, int r1,
    const double* __restrict__ zrow) {
  // Rows [r0, r1) of every eigenvector block live here (Q(r, c) at
  // Q[(r - r0) + c * ld]); zrow (row-distributed mode) holds the children's
  // boundary rows gathered from their owners, else they are read from Qin.
  __shared__ double red[32];
  int lo, mid, hi;
  node_range(L, n, blockIdx.x, lo, mid, hi);
  const int m = hi - lo, n1 = mid - lo;
  const int tid = threadIdx.x;
  int* cnt = w.counts + 3 * blockIdx.x;
  if (mid >= hi) {  // pass-through node: copy the block
    const int ra = max(lo, r0), rb = min(hi, r1), mr = rb - ra;
    for (long long idx = tid; mr > 0 && idx < (long long)mr * m; idx += blockDim.x) {
      const int r = (int)(idx % mr), c = (int)(idx / mr);
      Qout[(ra - r0 + r) + (long long)(lo + c) * ld] = Qin[(ra - r0 + r) + (long long)(lo + c) * ld];
    }
    for (int t = tid; t < m; t += blockDim.x) Dout[lo + t] = Din[lo + t];
    if (tid == 0) { cnt[0] = -1; cnt[1] = 0; cnt[2] = 0; }
    return;
  }
  const double inv = scal[0] > 0.0 ? 1.0 / scal[0] : 1.0;
  const double beta = e[mid - 1] * inv;
  const double rho = 2.0 * fabs(beta);
  const double sgn = beta >= 0.0 ? 1.0 : -1.0;
  const double rs2 = 0.70710678118654752440;
  const double* D1 = Din + lo;
  const double* D2 = Din + mid;
  const int n2 = hi - mid;
  double amax = 0.0;
  for (int t = tid; t < m; t += blockDim.x) {
    double val, zval;
    int r;
    if (t < n1) {
      val = D1[t];
      zval = (zrow ? zrow[lo + t] : Qin[(mid - 1 - r0) + (long long)(lo + t) * ld]) * rs2;
      int a = 0, b = n2;  // count of D2 < val
      while (a < b) { const int c = (a + b) >> 1; if (D2[c] < val) a = c + 1; else b = c; }
      r = t + a;
    } else {
      const int u = t - n1;
      val = D2[u];
      zval = sgn * (zrow ? zrow[mid + u] : Qin[(mid - r0) + (long long)(mid + u) * ld]) * rs2;
      int a = 0, b = n1;  // count of D1 <= val
      while (a < b) { const int c = (a + b) >> 1; if (D1[c] <= val) a = c + 1; else b = c; }
      r = u + a;
    }
    w.ds[lo + r] = val;
    w.zs[lo + r] = zval;
    w.perm[lo + r] = t;
    amax = fmax(amax, fmax(fabs(val), fabs(zval)));
  }
  amax = warp_max(amax);
  if ((tid & 31) == 0) red[tid >> 5] = amax;
  __syncthreads();
  double tol = 0.0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) tol = fmax(tol, red[i]);
  tol *= 8.0 * kEps;
  // sequential deflation scan (dlaed2 logic) in sorted order.  The scan only
  // ever rewrites the entries of the current candidate pj and of j, so pj's
  // (possibly rotated) d and z live in registers and every j is a fresh read
  // of the sorted arrays, staged chunk-wise into shared memory by the whole
  // block: the serial loop then runs at shared-memory instead of L2 latency.
  __shared__ double sd[kDcScanChunk], sz[kDcScanChunk];
  const double* ds = w.ds + lo;
  const double* zs = w.zs + lo;
  int K = 0, nd = 0, nr = 0, pj = -1;
  double dpj = 0.0, zpj = 0.0;
  for (int c0 = 0; c0 < m; c0 += kDcScanChunk) {
    const int cl = min(kDcScanChunk, m - c0);
    __syncthreads();
    for (int t = tid; t < cl; t += blockDim.x) { sd[t] = ds[c0 + t]; sz[t] = zs[c0 + t]; }
    __syncthreads();
    if (tid != 0) continue;
    for (int jj = 0; jj < cl; ++jj) {
      const int j = c0 + jj;
      const double zj = sz[jj], dj = sd[jj];
      if (rho * fabs(zj) <= tol) {
        w.defl[lo + nd] = j;
        w.val[lo + (m - 1 - nd)] = dj;  // deflated values fill from the back
        ++nd;
        continue;
      }
      if (pj < 0) { pj = j; dpj = dj; zpj = zj; continue; }
      double s = zpj, c = zj;
      const double tau = hypot(c, s);
      const double t = dj - dpj;
      c /= tau;
      s = -s / tau;
      if (fabs(t * c * s) <= tol) {
        w.rotp[lo + nr] = pj; w.rotq[lo + nr] = j; w.rotc[lo + nr] = c; w.rots[lo + nr] = s;
        ++nr;
        const double tt = dpj * c * c + dj * s * s;
        const double dnew = dpj * s * s + dj * c * c;
        w.defl[lo + nd] = pj;
        w.val[lo + (m - 1 - nd)] = tt;
        ++nd;
        pj = j; dpj = dnew; zpj = tau;
      } else {
        w.keep[lo + K] = pj; w.dk[lo + K] = dpj; w.zk[lo + K] = zpj;
        ++K;
        pj = j; dpj = dj; zpj = zj;
      }
    }
  }
  if (tid != 0) return;
  if (pj >= 0) { w.keep[lo + K] = pj; w.dk[lo + K] = dpj; w.zk[lo + K] = zpj; ++K; }
  cnt[0] = K; cnt[1] = nd; cnt[2] = nr;
  w.zh[lo] = rho;  // stash rho for the secular / z-hat kernels
}

// ---- 2. secular equation: one thread per root ----
// Root i of f(lam) = 1 + rho sum_j z_j^2 / (d_j - lam) lies in (d_i, d_{i+1})
// (last root: (d_{K-1}, d_{K-1} + rho |z|^2]).  It is computed as an offset
// tau from the closer pole (relative accuracy in tau is what the Loewner
// formula needs) by a safeguarded rational iteration: f is modelled by
// c + rho b1/(d_l - x) + rho b2/(d_r - x), fitted to f and f' at the current
// iterate (the "middle way" of Li / LAPACK dlaed4), with bisection whenever
// the model step leaves the bracket.  Converges in a handful of sweeps.
// kSecLanes lanes share one root: each sums a strided slice of the K poles
// and a butterfly (xor) reduction gives every lane of the group the same
// bitwise sum (a + b == b + a), so the group's control flow stays uniform.
// One thread per root left the top merges at ~3 warps per SM, latency-bound
// on the dependent FP64 reciprocals.
constexpr int kSecLanes = 8;
// iteration budget per root: the safeguarded rational step converges in a
// handful of sweeps (LAPACK's dlaed4 gives up after 30 and fails the whole
// dstedc); a root still unconverged after 200 is reported, not returned
constexpr int kSecMaxIter = 200;

__device__ __forceinline__ double group_sum(double v, unsigned mask) {
#pragma unroll
  for (int o = kSecLanes / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, kSecLanes);
  return v;
}

__global__ void dc_secular_kernel(Level L, int n, StedcWork w) {
  int lo, mid, hi;
  node_range(L, n, blockIdx.y, lo, mid, hi);
  const int* cnt = w.counts + 3 * blockIdx.y;
  const int K = cnt[0];
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = gt / kSecLanes;
  const int lane = gt % kSecLanes;
  const unsigned mask = ((1u << kSecLanes) - 1u) << ((threadIdx.x & 31) & ~(kSecLanes - 1));
  if (K <= 0 || i >= K) return;
  const double rho = w.zh[lo];
  const double* dk = w.dk + lo;
  const double* zk = w.zk + lo;
  if (K == 1) {
    if (lane != 0) return;
    const double t = rho * zk[0] * zk[0];
    w.org[lo] = 0;
    w.tau[lo] = t;
    w.val[lo] = dk[0] + t;
    return;
  }
  int org, pl, pr;
  double a, b;  // bracket for tau with f(a) < 0 <= f(b)
  if (i < K - 1) {
    const double half = 0.5 * (dk[i + 1] - dk[i]);
    double f = 0.0;
    for (int j = lane; j < K; j += kSecLanes) f += zk[j] * zk[j] / ((dk[j] - dk[i]) - half);
    f = 1.0 + rho * group_sum(f, mask);
    if (f >= 0.0) { org = i; a = 0.0; b = half; }
    else { org = i + 1; a = -half; b = 0.0; }
    pl = i; pr = i + 1;
  } else {
    double s = 0.0;
    for (int j = lane; j < K; j += kSecLanes) s += zk[j] * zk[j];
    org = K - 1; a = 0.0; b = rho * group_sum(s, mask);
    pl = K - 2; pr = K - 1;
  }
  const double d0 = dk[org];
  const double dl = dk[pl] - d0, dr = dk[pr] - d0;
  double t = 0.5 * (a + b);
  bool conv = false;
  for (int it = 0; it < kSecMaxIter; ++it) {
    double psi = 0.0, dpsi = 0.0, phi = 0.0, dphi = 0.0;
    for (int j = lane; j <= pl; j += kSecLanes) {
      const double inv = 1.0 / ((dk[j] - d0) - t);
      const double q = zk[j] * zk[j] * inv;
      psi += q;
      dpsi += q * inv;
    }
    for (int j = pr + lane; j < K; j += kSecLanes) {
      const double inv = 1.0 / ((dk[j] - d0) - t);
      const double q = zk[j] * zk[j] * inv;
      phi += q;
      dphi += q * inv;
    }
    psi = group_sum(psi, mask);
    dpsi = group_sum(dpsi, mask);
    phi = group_sum(phi, mask);
    dphi = group_sum(dphi, mask);
    const double f = 1.0 + rho * (psi + phi);
    // rounding-error bound of the computed f (cf. dlaed4's ERRETM): once |f|
    // is below it the iterate is a root to working accuracy
    const double erretm = 8.0 * rho * (fabs(psi) + fabs(phi)) + 2.0;
    if (fabs(f) <= kEps * erretm) { conv = true; break; }
    if (f > 0.0) b = t; else a = t;
    if (b - a <= 2.0 * kEps * fmax(fabs(a), fabs(b))) { t = 0.5 * (a + b); conv = true; break; }
    const double P0 = dl - t, Q0 = dr - t;
    const double b1 = dpsi * P0 * P0, a1 = psi - dpsi * P0;
    const double b2 = dphi * Q0 * Q0, a2 = phi - dphi * Q0;
    const double c = 1.0 + rho * (a1 + a2);
    const double B = c * (P0 + Q0) + rho * (b1 + b2);
    const double C0 = f * P0 * Q0;
    const double disc = B * B - 4.0 * c * C0;
    double tn;
    if (disc >= 0.0 && B != 0.0) {
      const double eta = 2.0 * C0 / (B + copysign(sqrt(disc), B));
      tn = t + eta;
    } else {
      tn = 0.5 * (a + b);
    }
    if (!(tn > a && tn < b)) tn = 0.5 * (a + b);
    const bool done = fabs(tn - t) <= 2.0 * kEps * fabs(tn);
    t = tn;
    if (done) { conv = true; break; }
  }
  if (lane != 0) return;
  // the bracket never reached working accuracy (or the data are not finite):
  // reported as BSE_NO_CONVERGENCE rather than returned silently
  if (w.fail && (!conv || !isfinite(t))) atomicOr(w.fail, 1);
  w.org[lo + i] = org;
  w.tau[lo + i] = t;
  w.val[lo + i] = d0 + t;
}

// ---- 3. Loewner z-hat ----
__global__ void dc_zhat_kernel(Level L, int n, StedcWork w, const double* rho_src) {
  int lo, mid, hi;
  node_range(L, n, blockIdx.y, lo, mid, hi);
  const int K = w.counts[3 * blockIdx.y];
  const int gt = blockIdx.x * blockDim.x + threadIdx.x;
  const int j = gt / kSecLanes;
  const int lane = gt % kSecLanes;
  const unsigned mask = ((1u << kSecLanes) - 1u) << ((threadIdx.x & 31) & ~(kSecLanes - 1));
  if (K <= 0 || j >= K) return;
  const double rho = rho_src[lo];
  const double* dk = w.dk + lo;
  const int* org = w.org + lo;
  const double* tau = w.tau + lo;
  const double dj = dk[j];
  // each factor is a ratio of neighbouring pole/root gaps (O(1)), so the
  // per-lane partial products stay in range
  double p = 1.0;
  for (int i = lane; i < K; i += kSecLanes) {
    const double li = (dk[org[i]] - dj) + tau[i];
    if (i < K - 1) p *= li / (i < j ? (dk[i] - dj) : (dk[i + 1] - dj));
    else p *= li;
  }
#pragma unroll
  for (int o = kSecLanes / 2; o > 0; o >>= 1) p *= __shfl_xor_sync(mask, p, o, kSecLanes);
  if (lane != 0) return;
  w.zh2[lo + j] = copysign(sqrt(fmax(p, 0.0) / rho), w.zk[lo + j]);
}

// ---- 4. output ordering (roots ascending merged with deflated values) ----
__global__ void dc_order_kernel(Level L, int n, StedcWork w, double* Dout) {
  int lo, mid, hi;
  node_range(L, n, blockIdx.y, lo, mid, hi);
  const int K = w.counts[3 * blockIdx.y];
  if (K < 0) return;
  const int m = hi - lo, nd = m - K;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= m) return;
  const double* val = w.val + lo;  // roots at [0,K), deflated at [m-1-c] for c < nd
  int pos;
  double v;
  if (t < K) {
    v = val[t];
    int c = 0;
    for (int q = 0; q < nd; ++q) c += val[m - 1 - q] < v;
    pos = t + c;
  } else {
    const int cidx = t - K;  // deflated #cidx
    v = val[m - 1 - cidx];
    int a = 0, b = K;  // roots <= v
    while (a < b) { const int c = (a + b) >> 1; if (val[c] <= v) a = c + 1; else b = c; }
    int c = 0;
    for (int q = 0; q < nd; ++q) {
      const double u = val[m - 1 - q];
      c += (u < v) || (u == v && q < cidx);
    }
    pos = a + c;
  }
  w.pos[lo + t] = pos;
  Dout[lo + pos] = v;
}

// ---- 5. eigenvector matrix U (rows in the node's original order) ----
// Column chunk [cc0, cc0 + cw) of every node (cw = L.size: all columns): node
// i's column t is stored at U column (i % slots) * cw + (t - cc0), rows by
// global index: nodes sharing a column slot own disjoint rows of U.
__global__ void __launch_bounds__(kDcThreads) dc_vectors_kernel(Level L, int n, StedcWork w,
                                                                long long ld, int cc0, int cw,
                                                                int slots) {
  int lo, mid, hi;
  node_range(L, n, blockIdx.y, lo, mid, hi);
  const int K = w.counts[3 * blockIdx.y];
  if (K < 0) return;
  const int m = hi - lo;
  const int lane = threadIdx.x & 31;
  const int t = cc0 + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);  // column source index
  if (t >= m || t >= cc0 + cw) return;
  // compact order: roots first (t < K), then deflated columns; the merge GEMM
  // scatters its output to the sorted positions w.pos through a column map
  double* U = w.U + lo + ((long long)(blockIdx.y % slots) * cw + (t - cc0)) * ld;
  for (int r = lane; r < m; r += 32) U[r] = 0.0;
  __syncwarp();
  const int* perm = w.perm + lo;
  if (t < K) {
    const double* dk = w.dk + lo;
    const double* zh = w.zh2 + lo;
    const int* keep = w.keep + lo;
    const double d0 = dk[w.org[lo + t]], tt = w.tau[lo + t];
    double s = 0.0;
    for (int j = lane; j < K; j += 32) {
      const double x = zh[j] / ((dk[j] - d0) - tt);
      s += x * x;
    }
    s = warp_sum(s);
    const double inv = 1.0 / sqrt(s);
    for (int j = lane; j < K; j += 32) U[perm[keep[j]]] = zh[j] / ((dk[j] - d0) - tt) * inv;
  } else if (lane == 0) {
    U[perm[w.defl[lo + (t - K)]]] = 1.0;
  }
}

// ---- 6. deflation rotations on the rows of U (reverse order) ----
__global__ void dc_rotate_kernel(Level L, int n, StedcWork w, long long ld, int cc0, int cw,
                                 int slots) {
  int lo, mid, hi;
  node_range(L, n, blockIdx.y, lo, mid, hi);
  const int K = w.counts[3 * blockIdx.y];
  const int nr = w.counts[3 * blockIdx.y + 2];
  if (K < 0 || nr == 0) return;
  const int m = hi - lo;
  const int col = cc0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (col >= m || col >= cc0 + cw) return;
  double* U = w.U + lo + ((long long)(blockIdx.y % slots) * cw + (col - cc0)) * ld;
  const int* perm = w.perm + lo;
  for (int r = nr - 1; r >= 0; --r) {
    const int p = perm[w.rotp[lo + r]], q = perm[w.rotq[lo + r]];
    const double c = w.rotc[lo + r], s = w.rots[lo + r];
    const double up = U[p], uq = U[q];
    U[p] = c * up - s * uq;
    U[q] = s * up + c * uq;
  }
}

// ---- 7. GEMM descriptors: Q_out = diag(Q1, Q2) * U per node ----
__global__ void dc_probs_kernel(Level L, int n, StedcWork w, const double* Qin, double* Qout,
                                long long ld, long long ldu, int r0, int r1, int cc0, int cw,
                                int slots) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.nnodes) return;
  int lo, mid, hi;
  node_range(L, n, i, lo, mid, hi);
  GemmProblem top, bot;
  if (mid < hi) {
    const int n1 = mid - lo, n2 = hi - mid, m = hi - lo;
    const int K = w.counts[3 * i], nr = w.counts[3 * i + 2];
    // deflated columns are unit vectors unless a Givens rotation touched the
    // node: then they join the GEMM, else dc_copy_deflated moves them
    const int ncols = (nr > 0) ? m : K;
    // this chunk's columns [cc0, cc0 + cw) of the node, this rank's rows
    const int nc = max(0, min(ncols, cc0 + cw) - cc0);
    const int ta = max(lo, r0), tb = min(mid, r1);
    const int ba = max(mid, r0), bb = min(hi, r1);
    const long long ucol = (long long)(i % slots) * cw;
    top.M = max(0, tb - ta); top.N = nc; top.K = n1;
    top.ccol = w.pos + lo + cc0; bot.ccol = w.pos + lo + cc0;
    bot.N = nc;
    top.A = Qin + (ta - r0) + (long long)lo * ld; top.lda = ld;
    top.B = w.U + lo + ucol * ldu; top.ldb = ldu;
    top.C = Qout + (ta - r0) + (long long)lo * ld; top.ldc = ld;
    bot.M = max(0, bb - ba); bot.K = n2;
    bot.A = Qin + (ba - r0) + (long long)mid * ld; bot.lda = ld;
    bot.B = w.U + mid + ucol * ldu; bot.ldb = ldu;
    bot.C = Qout + (ba - r0) + (long long)lo * ld; bot.ldc = ld;
  }
  w.probs[2 * i] = top;
  w.probs[2 * i + 1] = bot;
}

// Deflated (unrotated) columns: the merged eigenvector is the child's
// eigenvector, copied to its sorted output position (zeros in the other
// child's rows).  One warp per column.
__global__ void dc_copy_deflated_kernel(Level L, int n, StedcWork w, const double* Qin,
                                        double* Qout, long long ld, int w0, int w1) {
  int lo, mid, hi;
  node_range(L, n, blockIdx.y, lo, mid, hi);
  const int K = w.counts[3 * blockIdx.y], nr = w.counts[3 * blockIdx.y + 2];
  if (K < 0 || nr > 0) return;
  const int m = hi - lo, nd = m - K;
  const int c = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (c >= nd) return;
  const int lane = threadIdx.x & 31;
  const int jloc = w.perm[lo + w.defl[lo + c]];  // node-local original column
  const int outc = w.pos[lo + K + c];
  const bool first = (lo + jloc) < mid;
  const int r0 = first ? lo : mid, r1 = first ? mid : hi;
  const double* src = Qin + (long long)(lo + jloc) * ld - w0;
  double* dst = Qout + (long long)(lo + outc) * ld - w0;
  for (int r = max(lo, w0) + lane; r < min(hi, w1); r += 32)
    dst[r] = (r >= r0 && r < r1) ? src[r] : 0.0;
}

__global__ void dc_finish_kernel(int n, const double* D, double* wout, const double* scal) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) wout[i] = D[i] * (scal[0] > 0.0 ? scal[0] : 1.0);
}

__global__ void copy_matrix_kernel(int rows, int cols, const double* src, long long lds, double* dst,
                                   long long ldd) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)rows * cols) return;
  const int r = (int)(idx % rows), c = (int)(idx / rows);
  dst[r + (long long)c * ldd] = src[r + (long long)c * lds];
}

// Values only: the i-th smallest eigenvalue of the symmetric tridiagonal
// (d, e) by bisection on Sturm counts (one thread per eigenvalue), with the
// pivmin guard and convergence width of the reference's _bisect_values
// (kernels.py:275-299).
__global__ void sturm_bisect_kernel(int n, const double* __restrict__ d,
                                    const double* __restrict__ e, double* __restrict__ w,
                                    const double* __restrict__ bounds, int* fail) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double pivmin = bounds[2];
  double lo = bounds[0], hi = bounds[1];
  // like the reference (kernels.py:275-299, <= 160 halvings then the
  // midpoint), running out of halvings is not an error; a non-finite bracket
  // (NaN/Inf in d or e) is
  for (int it = 0; it < 200; ++it) {
    if (!(hi - lo > 2.0 * kEps * (fabs(lo) + fabs(hi)) + 2.0 * kSafmin)) break;
    const double x = 0.5 * (lo + hi);
    int cnt = 0;
    double q = d[0] - x;
    if (fabs(q) < pivmin) q = -pivmin;
    cnt += q < 0.0;
    for (int k = 1; k < n; ++k) {
      q = d[k] - x - (e[k - 1] * e[k - 1]) / q;
      if (fabs(q) < pivmin) q = -pivmin;
      cnt += q < 0.0;
    }
    if (cnt > i) hi = x; else lo = x;
  }
  if (fail && !(isfinite(lo) && isfinite(hi))) atomicOr(fail, 1);
  w[i] = 0.5 * (lo + hi);
}

__global__ void gershgorin_kernel(int n, const double* d, const double* e, double* bounds) {
  __shared__ double slo[32], shi[32], se[32];
  double lo = 1e300, hi = -1e300, emax2 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double r = 0.0;
    if (i > 0) r += fabs(e[i - 1]);
    if (i < n - 1) { r += fabs(e[i]); emax2 = fmax(emax2, e[i] * e[i]); }
    lo = fmin(lo, d[i] - r);
    hi = fmax(hi, d[i] + r);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    emax2 = fmax(emax2, __shfl_xor_sync(0xffffffffu, emax2, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { slo[w] = lo; shi[w] = hi; se[w] = emax2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      lo = fmin(lo, slo[k]); hi = fmax(hi, shi[k]); emax2 = fmax(emax2, se[k]);
    }
    lo = fmin(lo, slo[0]); hi = fmax(hi, shi[0]); emax2 = fmax(emax2, se[0]);
    const double pivmin = kSafmin * fmax(1.0, emax2);
    const double pad = 2.0 * kEps * fmax(fabs(lo), fabs(hi)) + 2.0 * pivmin;
    bounds[0] = lo - pad;
    bounds[1] = hi + pad;
    bounds[2] = pivmin;
  }
}

}  // namespace

cudaError_t tridiag_values(int n, const double* d, const double* e, double* w, double* scratch3,
                           cudaStream_t s, int* fail) {
  if (n <= 0) return cudaSuccess;
  gershgorin_kernel<<<1, 1024, 0, s>>>(n, d, e, scratch3);
  count_launch();
  sturm_bisect_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, s>>>(n, d, e, w, scratch3, fail);
  count_launch();
  return cudaGetLastError();
}

StedcWork stedc_carve(Arena& a, int n, int rows, int ucols) {
  StedcWork w;
  // rows >= 0: row-distributed mode, Qa/Qb hold `rows` rows of every block and
  // U has ucols columns (the caller sets row0/row1/zrow_reduce)
  const long long ld = pad_ld(rows >= 0 ? rows : n);
  w.ld = ld;
  w.Qa = a.take<double>((size_t)ld * n);
  w.Qb = a.take<double>((size_t)ld * n);
  if (rows >= 0) {
    w.ldu = pad_ld(n);
    w.ucols = std::max(64, std::min(n, ucols));
    w.U = a.take<double>((size_t)w.ldu * w.ucols);
    w.zrow = a.take<double>(n);
  } else {
    w.U = a.take<double>((size_t)ld * n);
  }
  w.Da = a.take<double>(n);
  w.Db = a.take<double>(n);
  w.ds = a.take<double>(n);
  w.zs = a.take<double>(n);
  w.dk = a.take<double>(n);
  w.zk = a.take<double>(n);
  w.zh = a.take<double>(n);
  w.zh2 = a.take<double>(n);
  w.tau = a.take<double>(n);
  w.val = a.take<double>(n);
  w.org = a.take<int>(n);
  w.perm = a.take<int>(n);
  w.keep = a.take<int>(n);
  w.defl = a.take<int>(n);
  w.pos = a.take<int>(n);
  w.rotp = a.take<int>(n);
  w.rotq = a.take<int>(n);
  w.rotc = a.take<double>(n);
  w.rots = a.take<double>(n);
  w.counts = a.take<int>(3 * (size_t)n + 3);
  w.probs = a.take<GemmProblem>(2 * (size_t)n + 2);
  w.scal = a.take<double>(4);
  w.fail = a.take<int>(4);
  w.dsan = a.take<double>(n);
  w.esan = a.take<double>(n);
  return w;
}

size_t stedc_bytes(int n) {
  Arena a;
  a.dry = true;
  stedc_carve(a, n);
  return a.used;
}

cudaError_t stedc(int n, double* d, double* e, double* wout, double* Q, long long ldq,
                  const StedcWork& ws, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err;
  const long long ld = ws.ld;
  if (ws.fail && (err = cudaMemsetAsync(ws.fail, 0, sizeof(int), s)) != cudaSuccess) return err;
  sanitize_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(n, d, e, ws.dsan, ws.esan, ws.fail);
  count_launch();
  d = ws.dsan;
  e = ws.esan;
  absmax_kernel<<<1, 1024, 0, s>>>(n, d, e, ws.scal);
  count_launch();
  // row window (row-distributed mode: dist.cu), U geometry
  const int r0 = ws.row1 >= 0 ? ws.row0 : 0, r1 = ws.row1 >= 0 ? ws.row1 : n;
  const long long ldu = ws.ldu ? ws.ldu : ld;
  const int ucols = ws.ucols ? ws.ucols : n;
  dc_init_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(n, d, e, ws.Da, ws.Qa, ld, ws.scal, r0, r1);
  count_launch();
  double* Din = ws.Da;
  double* Dout = ws.Db;
  double* Qin = ws.Qa;
  double* Qout = ws.Qb;
  for (int size = 2; size / 2 < n; size *= 2) {
    Level L{size, size / 2, (int)ceil_div(n, size)};
    const int maxm = std::min(size, n);
    stage_mark("dc_prepare", s);
    if (ws.zrow) {
      // the children's boundary rows (z of the rank-one tear), from their owners
      dc_zrow_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(L, n, Qin, ld, r0, r1, ws.zrow);
      count_launch();
      if (ws.zrow_reduce && (err = ws.zrow_reduce(ws.zrow_ctx, ws.zrow, n, s)) != cudaSuccess) return err;
    }
    dc_prepare_kernel<<<L.nnodes, kDcThreads, 0, s>>>(L, n, e, ws.scal, Din, Dout, Qin, Qout, ld, ws,
                                                      r0, r1, ws.zrow);
    count_launch();
    const dim3 g1((unsigned)ceil_div(maxm, 128), (unsigned)L.nnodes);
    stage_mark("dc_secular", s);
    const dim3 gs((unsigned)ceil_div((long long)maxm * kSecLanes, 128), (unsigned)L.nnodes);
    dc_secular_kernel<<<gs, 128, 0, s>>>(L, n, ws);
    count_launch();
    stage_mark("dc_vectors", s);
    dc_zhat_kernel<<<gs, 128, 0, s>>>(L, n, ws, ws.zh);
    count_launch();
    dc_order_kernel<<<g1, 128, 0, s>>>(L, n, ws, Dout);
    count_launch();
    // U (block diagonal: node i owns rows [lo, hi)) lives in a ldu x ucols
    // buffer of column slots cw wide; node i uses slot i % slots -- nodes
    // sharing a slot own disjoint rows.  A level whose nodes are wider than
    // the buffer (row-distributed mode keeps it at n x ucols) is processed in
    // column chunks of cw.
    const int cw = maxm <= ucols ? maxm : std::max(32, ucols / 32 * 32);
    if (cw > ucols) return cudaErrorInvalidValue;
    const int slots = std::max(1, ucols / cw);
    if (std::getenv("BSE_DC_STATS") && L.nnodes <= 4) {
      int hc[12];
      cudaMemcpyAsync(hc, ws.counts, sizeof(int) * 3 * L.nnodes, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      for (int q = 0; q < L.nnodes; ++q)
        std::fprintf(stderr, "[dc] level size %d node %d: K=%d deflated=%d rotations=%d\n", size, q,
                     hc[3 * q], hc[3 * q + 1], hc[3 * q + 2]);
    }
    for (int cc0 = 0; cc0 < maxm; cc0 += cw) {
      const int cwc = std::min(cw, maxm - cc0);
      const dim3 g2c((unsigned)ceil_div(cwc, kDcThreads / 32), (unsigned)L.nnodes);
      const dim3 g1c((unsigned)ceil_div(cwc, 128), (unsigned)L.nnodes);
      if (cc0 > 0) stage_mark("dc_vectors", s);
      dc_vectors_kernel<<<g2c, kDcThreads, 0, s>>>(L, n, ws, ldu, cc0, cw, slots);
      count_launch();
      dc_rotate_kernel<<<g1c, 128, 0, s>>>(L, n, ws, ldu, cc0, cw, slots);
      count_launch();
      dc_probs_kernel<<<(unsigned)ceil_div(L.nnodes, 128), 128, 0, s>>>(L, n, ws, Qin, Qout, ld, ldu,
                                                                        r0, r1, cc0, cw, slots);
      count_launch();
      if ((err = cudaGetLastError()) != cudaSuccess) return err;
      stage_mark("dc_gemm", s);
      static const int oz_nodes =
          std::getenv("BSE_DC_OZ_NODES") ? std::min(8, std::atoi(std::getenv("BSE_DC_OZ_NODES"))) : 2;
      if (ws.oz && L.nnodes <= oz_nodes && (double)L.half * L.half * maxm >= oz_min_work()) {
        // top merges: the problem shapes come back to the host (one sync per
        // level) and the large products run on the emulated-FP64 engine
        GemmProblem hp[16];
        if ((err = cudaMemcpyAsync(hp, ws.probs, sizeof(GemmProblem) * 2 * L.nnodes,
                                   cudaMemcpyDeviceToHost, s)) != cudaSuccess)
          return err;
        if ((err = cudaStreamSynchronize(s)) != cudaSuccess) return err;
        for (int q = 0; q < 2 * L.nnodes; ++q) {
          const GemmProblem& p = hp[q];
          if (p.M <= 0 || p.N <= 0) continue;
          err = (double)p.M * p.N * p.K >= oz_min_work()
                    ? ozgemm(false, false, p, ws.oz, ws.oz_bytes, 2048, s)
                    : gemm(false, false, p, s);
          if (err != cudaSuccess) return err;
        }
      } else {
        err = gemm_grouped(false, false, ws.probs, 2 * L.nnodes, std::min(L.half, r1 - r0), cwc, s,
                           L.half >= 2 && (r0 & 1) == 0, L.half >= 512 ? 3 : 1);
        if (err != cudaSuccess) return err;
      }
    }
    const dim3 g2((unsigned)ceil_div(maxm, kDcThreads / 32), (unsigned)L.nnodes);
    dc_copy_deflated_kernel<<<g2, kDcThreads, 0, s>>>(L, n, ws, Qin, Qout, ld, r0, r1);
    count_launch();
    std::swap(Din, Dout);
    std::swap(Qin, Qout);
  }
  dc_finish_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(n, Din, wout, ws.scal);
  count_launch();
  const long long tot = (long long)(r1 - r0) * n;
  if (Q && tot > 0) {
    copy_matrix_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(r1 - r0, n, Qin, ld, Q, ldq);
    count_launch();
  }
  return cudaGetLastError();
}

}  // namespace bse
