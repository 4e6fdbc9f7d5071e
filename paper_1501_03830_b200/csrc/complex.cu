// Complex Hermitian BSE on the device (the drop-in for solvers.solve_complex,
// solvers.py:29-77, on BASELINE cfg1/cfg3): real 2n x 2n embedding, the real
// product-form solve with column selection, and the complex extraction.
//
//   A' = [[Ar, -Ai], [Ai, Ar]],  B' = [[Br, Bi], [Bi, -Br]]   (D3)
//   M' = sym(A' + B'),  K' = sym(A' - B'),  sym(T) = (T + T^T) / 2
//
// Every complex eigenvalue appears twice in the real spectrum and any real
// eigenvector r of the pair gives the complex one x = r[:n] + i r[n:],
// y = w[:n] - i w[n:] (normalised in x1^H x1 - x2^H x2 already).  So after
// the divide and conquer only ONE column per simple pair is back-transformed
// (Q2, Q1 and the X recovery run on ~n of the 2n columns); clusters of
// (nearly) equal complex eigenvalues keep all their 2k columns and k vectors
// are chosen by pivoted Gram-Schmidt in the indefinite product
// <x, y> = x1^H y1 - x2^H y2, the analogue of the reference's
// _pivoted_orthonormal (kernels.py:659-674).
//
// Complex arrays are interleaved (re, im) complex128 in ROW-major order
// (numpy C order) with leading dimensions in complex elements.
#include <algorithm>
#include <cmath>
#include <vector>
#include "../../include/bse_b200.h"
#include "complex.cuh"
#include "eig.cuh"
#include "gemm.cuh"
#include "solver.cuh"

namespace bse {
namespace {

constexpr int kT = 32;

// M'(r, c), K'(r, c) (column-major, ld) for all r, c < N = 2n.  The tile of
// T(r, c) and the transposed tile T(c, r) are both read row-wise (coalesced
// along j of the row-major A, B) through shared memory.  Arithmetic is the
// host embedding's (solvers.real_embedding): t = a' + b' (M) or a' - b' (K),
// then 0.5 * (t_rc + t_cr) -- bitwise equal to numpy.
__global__ void __launch_bounds__(kT * 8) embed_kernel(int n, const double2* __restrict__ A,
                                                       long long lda, const double2* __restrict__ B,
                                                       long long ldb, double* M, double* K,
                                                       long long ld) {
  __shared__ double sa[2][kT][kT + 1], sb[2][kT][kT + 1];  // [0]: T(r, c) tile, [1]: T(c, r) tile
  const int N = 2 * n;
  const int r0 = blockIdx.y * kT, c0 = blockIdx.x * kT;
  const int tx = threadIdx.x, ty0 = threadIdx.y;
  // a'(r, c), b'(r, c) of the embedding
  auto load = [&](int r, int c, double& av, double& bv) {
    av = 0.0;
    bv = 0.0;
    if (r >= N || c >= N) return;
    const int p = r >= n, q = c >= n;
    const int i = r - p * n, j = c - q * n;
    const double2 a = A[(long long)i * lda + j];
    const double2 b = B[(long long)i * ldb + j];
    if (!p && !q) { av = a.x; bv = b.x; }
    else if (!p && q) { av = -a.y; bv = b.y; }
    else if (p && !q) { av = a.y; bv = b.y; }
    else { av = a.x; bv = -b.x; }
  };
  for (int ty = ty0; ty < kT; ty += blockDim.y) {
    load(r0 + ty, c0 + tx, sa[0][ty][tx], sb[0][ty][tx]);  // T(r0+ty, c0+tx)
    load(c0 + ty, r0 + tx, sa[1][ty][tx], sb[1][ty][tx]);  // T(c0+ty, r0+tx)
  }
  __syncthreads();
  for (int ty = ty0; ty < kT; ty += blockDim.y) {
    const int r = r0 + tx, c = c0 + ty;  // column-major write: r fastest
    if (r >= N || c >= N) continue;
    // T(r, c) = s?[0][tx][ty], T(c, r) = s?[1][ty][tx]
    const double a1 = sa[0][tx][ty], b1 = sb[0][tx][ty];
    const double a2 = sa[1][ty][tx], b2 = sb[1][ty][tx];
    const double m1 = a1 + b1, m2 = a2 + b2;
    const double k1 = a1 + (-b1), k2 = a2 + (-b2);
    M[r + (long long)c * ld] = 0.5 * (m1 + m2);
    K[r + (long long)c * ld] = 0.5 * (k1 + k2);
  }
}

// Simple pairs: output column dst takes selected real column src[dst]:
//   X1c(i, dst) = X1r(i, s) + i X1r(n + i, s),  X2c(i, dst) = X2r(i, s) - i X2r(n + i, s)
// into COLUMN-major complex scratch (ldc), coalesced on both sides.
__global__ void extract_simple_kernel(int n, const int* __restrict__ src,
                                      const double* __restrict__ X1r,
                                      const double* __restrict__ X2r, long long ld, double2* X1c,
                                      double2* X2c, long long ldc) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * n) return;
  const int i = (int)(idx % n), dst = (int)(idx / n);
  const int s = src[dst];
  if (s < 0) return;
  const double* c1 = X1r + (long long)s * ld;
  const double* c2 = X2r + (long long)s * ld;
  X1c[(long long)dst * ldc + i] = make_double2(c1[i], c1[n + i]);
  X2c[(long long)dst * ldc + i] = make_double2(c2[i], -c2[n + i]);
}

// Clusters: one CTA each.  Candidates = the cluster's selected real columns
// (as complex vectors, updated in place in X1r / X2r); k = size / 2 pivoted
// Gram-Schmidt steps in the indefinite product, deterministic reductions.
struct Cluster {
  int sc0, size, dst0;
};
constexpr int kMaxClusterCand = 1024;
constexpr int kClThreads = 512;

__device__ double cl_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(kClThreads) extract_cluster_kernel(
    int n, const Cluster* __restrict__ cls, double* X1r, double* X2r, long long ld, double2* X1c,
    double2* X2c, long long ldc) {
  __shared__ double red[33];
  __shared__ double nrm[kMaxClusterCand];
  __shared__ unsigned char used[kMaxClusterCand];
  __shared__ double coef_re, coef_im;
  const Cluster cl = cls[blockIdx.x];
  const int s = min(cl.size, kMaxClusterCand), k = cl.size / 2;
  for (int c = threadIdx.x; c < s; c += blockDim.x) used[c] = 0;
  __syncthreads();
  // complex view of candidate c: x1 = (p1[i], p1[n+i]), x2 = (p2[i], -p2[n+i])
  for (int t = 0; t < k; ++t) {
    for (int c = 0; c < s; ++c) {
      double v = 0.0;
      if (!used[c]) {
        const double* p1 = X1r + (long long)(cl.sc0 + c) * ld;
        const double* p2 = X2r + (long long)(cl.sc0 + c) * ld;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const double a = p1[i], b = p1[n + i], e = p2[i], f = p2[n + i];
          v += a * a + b * b - e * e - f * f;
        }
      }
      v = cl_block_sum(v, red);
      if (threadIdx.x == 0) nrm[c] = used[c] ? -HUGE_VAL : v;
    }
    __syncthreads();
    int j = 0;
    for (int c = 1; c < s; ++c)
      if (nrm[c] > nrm[j]) j = c;
    const double sc = sqrt(fmax(nrm[j], 1e-300));
    double* u1 = X1r + (long long)(cl.sc0 + j) * ld;
    double* u2 = X2r + (long long)(cl.sc0 + j) * ld;
    const int dst = cl.dst0 + t;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      u1[i] /= sc; u1[n + i] /= sc; u2[i] /= sc; u2[n + i] /= sc;
      X1c[(long long)dst * ldc + i] = make_double2(u1[i], u1[n + i]);
      X2c[(long long)dst * ldc + i] = make_double2(u2[i], -u2[n + i]);
    }
    __syncthreads();
    if (threadIdx.x == 0) used[j] = 1;
    __syncthreads();
    // w_c -= u * (u1^H w1_c - u2^H w2_c)
    for (int c = 0; c < s; ++c) {
      if (used[c]) continue;  // uniform across the block
      double* w1 = X1r + (long long)(cl.sc0 + c) * ld;
      double* w2 = X2r + (long long)(cl.sc0 + c) * ld;
      double re = 0.0, im = 0.0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        // conj(u) w for x1 = (a, b): (ua - i ub)(wa + i wb); x2 = (e, -f)
        const double ua = u1[i], ub = u1[n + i], wa = w1[i], wb = w1[n + i];
        const double ue = u2[i], uf = -u2[n + i], we = w2[i], wf = -w2[n + i];
        re += ua * wa + ub * wb - (ue * we + uf * wf);
        im += ua * wb - ub * wa - (ue * wf - uf * we);
      }
      re = cl_block_sum(re, red);
      im = cl_block_sum(im, red);
      if (threadIdx.x == 0) { coef_re = re; coef_im = im; }
      __syncthreads();
      const double cr = coef_re, ci = coef_im;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        // w1 -= u1 * coef ; w2 -= u2 * coef  (complex), stored back in the real layout
        const double ua = u1[i], ub = u1[n + i];
        w1[i] -= ua * cr - ub * ci;
        w1[n + i] -= ua * ci + ub * cr;
        // x2 = (e, -f) is stored as (e, f): the imaginary part flips sign
        const double ue = u2[i], uf = -u2[n + i];
        w2[i] -= ue * cr - uf * ci;
        w2[n + i] += ue * ci + uf * cr;
      }
      __syncthreads();
    }
  }
}


// Biorthogonality polish, banded.  Picking one real vector per doubled
// eigenvalue keeps the D&C's orthogonality only up to the mixing of nearby
// eigenpairs (x_j picks up O(eps |W| / gap) of its neighbours' partner
// vectors, which Z's orthogonality no longer cancels), so the indefinite Gram
// G = X1^H X1 - X2^H X2 deviates from I essentially on a band around the
// diagonal (sorted eigenvalues: close values are adjacent).  One Newton-Schulz
// step X <- X (1.5 I - 0.5 G) restricted to |j - k| <= kPolW removes it at
// O(n^2 kPolW) cost (the full-matrix polish is 32 n^3).
constexpr int kPolW = 16;  // band half-width
constexpr int kPolT = 32;  // output columns per CTA
constexpr int kPolR = 16;  // rows per shared-memory chunk (Gram)
constexpr int kPolRA = 8;  // rows per shared-memory chunk (apply; 48 KB static limit)
constexpr int kPolThreads = 256;

BSE_DEV double2 cmul_conj_a(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}

// G[d * (W+1) + o] = x_d^H x_{d+o} (indefinite product), o = 0..W
__global__ void __launch_bounds__(kPolThreads) band_gram_kernel(int n, const double2* __restrict__ X1,
                                                                const double2* __restrict__ X2,
                                                                long long ldc, double2* G) {
  constexpr int NC = kPolT + kPolW;
  constexpr int NP = kPolT * (kPolW + 1);
  constexpr int PPT = (NP + kPolThreads - 1) / kPolThreads;
  __shared__ double2 s1[kPolR][NC + 1], s2[kPolR][NC + 1];
  const int d0 = blockIdx.x * kPolT;
  double2 acc[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int r0 = 0; r0 < n; r0 += kPolR) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kPolR * NC; idx += blockDim.x) {
      const int i = idx % kPolR, c = idx / kPolR;
      const int col = d0 + c, row = r0 + i;
      const bool ok = col < n && row < n;
      s1[i][c] = ok ? X1[(long long)col * ldc + row] : make_double2(0.0, 0.0);
      s2[i][c] = ok ? X2[(long long)col * ldc + row] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int p = threadIdx.x + q * kPolThreads;
      if (p >= NP) break;
      const int dd = p / (kPolW + 1), o = p % (kPolW + 1);
#pragma unroll 4
      for (int i = 0; i < kPolR; ++i) {
        const double2 u = cmul_conj_a(s1[i][dd], s1[i][dd + o]);
        const double2 v = cmul_conj_a(s2[i][dd], s2[i][dd + o]);
        acc[q].x += u.x - v.x;
        acc[q].y += u.y - v.y;
      }
    }
  }
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int p = threadIdx.x + q * kPolThreads;
    if (p >= NP) break;
    const int d = d0 + p / (kPolW + 1), o = p % (kPolW + 1);
    if (d < n) G[(long long)d * (kPolW + 1) + o] = (d + o < n) ? acc[q] : make_double2(0.0, 0.0);
  }
}

// Out(i, d) = sum_{k = d-W}^{d+W} X(i, k) F_kd, F = 1.5 I - 0.5 G, written
// ROW-major (the caller's layout), coalesced along d.
__global__ void __launch_bounds__(kPolThreads) band_apply_kernel(
    int n, const double2* __restrict__ X1, const double2* __restrict__ X2, long long ldc,
    const double2* __restrict__ G, double2* O1, long long ldo1, double2* O2, long long ldo2) {
  constexpr int NC = kPolT + 2 * kPolW;
  constexpr int NO = 2 * kPolW + 1;
  __shared__ double2 F[NO][kPolT];  // F[o][dd]: coefficient of column d0 + dd + o - W
  __shared__ double2 s1[kPolRA][NC + 1], s2[kPolRA][NC + 1];
  const int d0 = blockIdx.x * kPolT;
  for (int idx = threadIdx.x; idx < NO * kPolT; idx += blockDim.x) {
    const int o = idx / kPolT, dd = idx % kPolT;
    const int d = d0 + dd, k = d + o - kPolW;
    double2 f = make_double2(0.0, 0.0);
    if (d < n && k >= 0 && k < n) {
      // G_kd = x_k^H x_d: stored as G[k][d - k] when k <= d, else conj(G[d][k - d])
      double2 g = k <= d ? G[(long long)k * (kPolW + 1) + (d - k)]
                         : G[(long long)d * (kPolW + 1) + (k - d)];
      if (k > d) g.y = -g.y;
      f = make_double2((k == d ? 1.5 : 0.0) - 0.5 * g.x, -0.5 * g.y);
    }
    F[o][dd] = f;
  }
  const int dd = threadIdx.x % kPolT;        // this thread's output column
  const int ig = threadIdx.x / kPolT;        // and rows ig, ig + 8, ...
  constexpr int RG = kPolThreads / kPolT;    // 8 row groups
  for (int r0 = 0; r0 < n; r0 += kPolRA) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kPolRA * NC; idx += blockDim.x) {
      const int i = idx % kPolRA, c = idx / kPolRA;
      const int col = d0 - kPolW + c, row = r0 + i;
      const bool ok = col >= 0 && col < n && row < n;
      s1[i][c] = ok ? X1[(long long)col * ldc + row] : make_double2(0.0, 0.0);
      s2[i][c] = ok ? X2[(long long)col * ldc + row] : make_double2(0.0, 0.0);
    }
    __syncthreads();
    const int d = d0 + dd;
    for (int i = ig; i < kPolRA; i += RG) {
      const int row = r0 + i;
      if (row >= n || d >= n) continue;
      double2 a1 = make_double2(0.0, 0.0), a2 = a1;
#pragma unroll
      for (int o = 0; o < NO; ++o) {
        const double2 f = F[o][dd];
        const double2 x1 = s1[i][dd + o], x2 = s2[i][dd + o];
        a1.x += x1.x * f.x - x1.y * f.y;
        a1.y += x1.x * f.y + x1.y * f.x;
        a2.x += x2.x * f.x - x2.y * f.y;
        a2.y += x2.x * f.y + x2.y * f.x;
      }
      O1[(long long)row * ldo1 + d] = a1;
      O2[(long long)row * ldo2 + d] = a2;
    }
  }
}

// Full biorthogonality polish (n <= kGlobalPolishMaxN): the same Newton-Schulz
// step with the whole indefinite Gram, as real DMMA GEMMs on the interleaved
// complex layout (a column-major n x n complex block is a real 2n x n matrix
// X with rows (Re, Im)); iX is the same block times i (rows (-Im, Re)).
//   Re G = X1^T X1 - X2^T X2,   Im G = X1^T (iX1) ... with signs as below,
//   X <- X Fr + (iX) Fi,  F = 1.5 I - 0.5 G.
constexpr int kGlobalPolishMaxN = 4096;

__global__ void times_i_kernel(long long count, const double2* X, double2* Y) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const double2 v = X[k];
  Y[k] = make_double2(-v.y, v.x);
}

// F (n x n, column-major real pair) = 1.5 I - 0.5 G
__global__ void polish_f_kernel(int n, double* Gr, double* Gi) {
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= (long long)n * n) return;
  const int r = (int)(k % n), c = (int)(k / n);
  Gr[k] = (r == c ? 1.5 : 0.0) - 0.5 * Gr[k];
  Gi[k] = -0.5 * Gi[k];
}

// row-major complex output from the column-major scratch (32 x 32 tiles)
__global__ void colmajor_to_rowmajor_kernel(int n, const double2* __restrict__ X, long long ldc,
                                            double2* O, long long ldo) {
  __shared__ double2 t[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int c = c0 + k, r = r0 + threadIdx.x;
    if (c < n && r < n) t[k][threadIdx.x] = X[(long long)c * ldc + r];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += blockDim.y) {
    const int r = r0 + k, c = c0 + threadIdx.x;
    if (c < n && r < n) O[(long long)r * ldo + c] = t[threadIdx.x][k];
  }
}

cudaError_t global_polish(int n, double2* S1, double2* S2, char* scratch, double2* O1,
                          long long ldo1, double2* O2, long long ldo2, cudaStream_t s) {
  cudaError_t e;
  const size_t cn = (size_t)n * n;
  double2* T1 = reinterpret_cast<double2*>(scratch);  // i X1, then X1 new
  double2* T2 = T1 + cn;                              // i X2, then X2 new
  double* Gr = reinterpret_cast<double*>(T2 + cn);
  double* Gi = Gr + cn;
  double2* N1 = reinterpret_cast<double2*>(Gi + cn);
  double2* N2 = N1 + cn;
  const unsigned g = (unsigned)ceil_div((long long)cn, 256);
  times_i_kernel<<<g, 256, 0, s>>>((long long)cn, S1, T1);
  times_i_kernel<<<g, 256, 0, s>>>((long long)cn, S2, T2);
  count_launch(2);
  const double* x1 = reinterpret_cast<const double*>(S1);
  const double* x2 = reinterpret_cast<const double*>(S2);
  const double* y1 = reinterpret_cast<const double*>(T1);
  const double* y2 = reinterpret_cast<const double*>(T2);
  const long long ld = 2LL * n;
  // G_jk = x1_j^H x1_k - x2_j^H x2_k:  Re G = X1^T X1 - X2^T X2 and, as
  // X^T (iX) = sum (re_j (-im_k) + im_j re_k) = -Im(x_j^H x_k),
  // Im G = -X1^T (iX1) + X2^T (iX2)   (K = 2n)
  const GemmProblem p[4] = {make_gemm(n, n, 2 * n, 1.0, x1, ld, x1, ld, 0.0, Gr, n),
                            make_gemm(n, n, 2 * n, -1.0, x2, ld, x2, ld, 1.0, Gr, n),
                            make_gemm(n, n, 2 * n, -1.0, x1, ld, y1, ld, 0.0, Gi, n),
                            make_gemm(n, n, 2 * n, 1.0, x2, ld, y2, ld, 1.0, Gi, n)};
  for (const GemmProblem& q : p)
    if ((e = gemm(true, false, q, s)) != cudaSuccess) return e;
  polish_f_kernel<<<g, 256, 0, s>>>(n, Gr, Gi);
  count_launch();
  // X_new = X Fr + (iX) Fi   (2n x n x n, interleaved rows)
  const GemmProblem u[4] = {
      make_gemm(2 * n, n, n, 1.0, x1, ld, Gr, n, 0.0, reinterpret_cast<double*>(N1), ld),
      make_gemm(2 * n, n, n, 1.0, y1, ld, Gi, n, 1.0, reinterpret_cast<double*>(N1), ld),
      make_gemm(2 * n, n, n, 1.0, x2, ld, Gr, n, 0.0, reinterpret_cast<double*>(N2), ld),
      make_gemm(2 * n, n, n, 1.0, y2, ld, Gi, n, 1.0, reinterpret_cast<double*>(N2), ld)};
  for (const GemmProblem& q : u)
    if ((e = gemm(false, false, q, s)) != cudaSuccess) return e;
  const dim3 grid((unsigned)ceil_div(n, 32), (unsigned)ceil_div(n, 32));
  colmajor_to_rowmajor_kernel<<<grid, dim3(32, 8), 0, s>>>(n, N1, n, O1, ldo1);
  colmajor_to_rowmajor_kernel<<<grid, dim3(32, 8), 0, s>>>(n, N2, n, O2, ldo2);
  count_launch(2);
  return cudaGetLastError();
}

size_t global_polish_bytes(int n) { return (size_t)n * n * (16 * 4 + 8 * 2) + 1024; }

// Host-side plan built by the column selector from the doubled spectrum.
struct ComplexPlan {
  int n = 0;
  std::vector<double> lam;      // n complex eigenvalues, descending
  std::vector<int> src;         // per output column: selected real column (simple pair) or -1
  std::vector<Cluster> cls;     // clusters (>= 4 real columns)
};

// ZSelect callback: w = the N = 2n eigenvalues lambda^2 of W' (ascending).
// Groups the descending spectrum by gaps in lambda^2 (the two copies of a
// doubled eigenvalue differ by O(eps |W|) absolute, so the grouping is
// absolute in lambda^2), merges odd-sized groups forward so that no pair is
// split, and selects one column per simple pair / all columns of a cluster.
// Returns -1 when some lambda^2 is not positive or not finite.
int complex_select(void* ctx, const double* w, int N, int* cols) {
  ComplexPlan& P = *static_cast<ComplexPlan*>(ctx);
  const int n = N / 2;
  for (int i = 0; i < N; ++i)
    if (!(w[i] > 0.0) || !std::isfinite(w[i])) return -1;
  auto d = [&](int i) { return w[N - 1 - i]; };  // descending lambda^2
  const double tol = kComplexGroupTol * N * kEps * d(0);
  std::vector<int> starts;
  for (int i = 0; i < N;) {
    int j = i + 1;
    while (j < N && d(j - 1) - d(j) <= tol) ++j;
    starts.push_back(i);
    i = j;
  }
  starts.push_back(N);
  P.n = n;
  P.lam.assign(n, 0.0);
  P.src.assign(n, -1);
  P.cls.clear();
  int nsel = 0, dst = 0;
  for (size_t g = 0; g + 1 < starts.size();) {
    const int start = starts[g];
    size_t h = g + 1;
    while ((starts[h] - start) % 2 != 0 && h + 1 < starts.size()) ++h;  // never split a pair
    const int size = starts[h] - start;
    g = h;
    if (size % 2 != 0 || dst + size / 2 > n) return -1;  // cannot happen for a doubled spectrum
    if (size == 2) {
      P.src[dst] = nsel;
      cols[nsel++] = N - 1 - start;
      P.lam[dst++] = 0.5 * (std::sqrt(d(start)) + std::sqrt(d(start + 1)));
    } else {
      P.cls.push_back(Cluster{nsel, size, dst});
      for (int t = 0; t < size; ++t) cols[nsel++] = N - 1 - (start + t);
      for (int t = 0; t < size / 2; ++t)
        P.lam[dst++] = 0.5 * (std::sqrt(d(start + 2 * t)) + std::sqrt(d(start + 2 * t + 1)));
    }
  }
  return dst == n ? nsel : -1;
}

}  // namespace

ComplexCarve carve_complex(Arena& a, int n, int flags) {
  ComplexCarve c{};
  const int N = 2 * n;
  c.ld = pad_ld(N);
  c.M = a.take<double>((size_t)c.ld * N);
  c.K = a.take<double>((size_t)c.ld * N);
  c.lam2 = a.take<double>(N);
  c.src = a.take<int>(n);
  c.cls = a.take<char>(sizeof(Cluster) * (size_t)(n + 1));
  // the solve workspace doubles as the extraction scratch once the solve is
  // done: two n x n complex column-major blocks and the band Gram, then (host
  // entry only) room for the outputs
  const size_t cb = 16 * (size_t)n * n;
  c.scratch_bytes = 2 * cb + std::max(16 * (size_t)n * (kPolW + 1),
                                      n <= kGlobalPolishMaxN ? global_polish_bytes(n) : 0) + 512;
  c.ws_bytes = std::max(solve_bytes(N, flags), c.scratch_bytes + 2 * cb + 512);
  c.ws = a.take<char>(c.ws_bytes);
  return c;
}

size_t complex_bytes(int n, int flags) {
  Arena a;
  a.dry = true;
  carve_complex(a, n, flags);
  return a.used + 4096;
}

cudaError_t solve_complex(int n, const double2* A, long long lda, const double2* B, long long ldb,
                          double* lam_dev, double* lam_host, double2* X1c, long long ldx1,
                          double2* X2c, long long ldx2, const ComplexCarve& c, int flags,
                          cudaStream_t s, SolveStatus* out) {
  const int N = 2 * n;
  cudaError_t e;
  stage_mark("embed", s);
  {
    const dim3 grid((unsigned)ceil_div(N, kT), (unsigned)ceil_div(N, kT));
    embed_kernel<<<grid, dim3(kT, 8), 0, s>>>(n, A, lda, B, ldb, c.M, c.K, c.ld);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  ComplexPlan plan;
  ZSelect zs;
  zs.fn = complex_select;
  zs.ctx = &plan;
  // real outputs X1r, X2r (N x nsel) overwrite K', M' (both dead by the
  // recovery: K' was copied into L, M' is only re-read before it)
  if ((e = solve_spd_pair(N, c.M, c.ld, c.K, c.ld, c.lam2, c.K, c.ld, c.M, c.ld, c.ws, c.ws_bytes,
                          flags, s, out, nullptr, nullptr, nullptr, nullptr, &zs)) != cudaSuccess)
    return e;
  if (out->code != 0) return cudaSuccess;
  stage_mark("extract", s);
  const int ncl = (int)plan.cls.size();
  if ((e = cudaMemcpyAsync(c.src, plan.src.data(), sizeof(int) * n, cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return e;
  if (ncl > 0 && (e = cudaMemcpyAsync(c.cls, plan.cls.data(), sizeof(Cluster) * ncl,
                                      cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  // scratch (column-major complex, ld n) and the band Gram in the dead solve
  // workspace
  double2* S1 = reinterpret_cast<double2*>(c.ws);
  double2* S2 = S1 + (size_t)n * n;
  double2* G = S2 + (size_t)n * n;
  {
    const long long tot = (long long)n * n;
    extract_simple_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(n, c.src, c.K, c.M, c.ld,
                                                                      S1, S2, n);
    count_launch();
  }
  if (ncl > 0) {
    extract_cluster_kernel<<<ncl, kClThreads, 0, s>>>(n, reinterpret_cast<const Cluster*>(c.cls),
                                                      c.K, c.M, c.ld, S1, S2, n);
    count_launch();
  }
  stage_mark("polish", s);
  if (n <= kGlobalPolishMaxN) {
    // the whole indefinite Gram (32 n^3 flops) on DMMA
    if ((e = global_polish(n, S1, S2, reinterpret_cast<char*>(G), X1c, ldx1, X2c, ldx2, s)) !=
        cudaSuccess)
      return e;
  } else {
    // banded: O(n^2 kPolW), the interactions that matter at this size
    const unsigned g = (unsigned)ceil_div(n, kPolT);
    band_gram_kernel<<<g, kPolThreads, 0, s>>>(n, S1, S2, n, G);
    band_apply_kernel<<<g, kPolThreads, 0, s>>>(n, S1, S2, n, G, X1c, ldx1, X2c, ldx2);
    count_launch(2);
  }
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (lam_dev &&
      (e = cudaMemcpyAsync(lam_dev, plan.lam.data(), sizeof(double) * n, cudaMemcpyHostToDevice,
                           s)) != cudaSuccess)
    return e;
  if (lam_host) std::copy(plan.lam.begin(), plan.lam.end(), lam_host);
  out->clusters = ncl;
  stage_mark("end", s);
  // plan's host vectors are read by the async copies above
  return cudaStreamSynchronize(s);
}

}  // namespace bse
