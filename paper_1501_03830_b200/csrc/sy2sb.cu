// Stage 1 of the two-stage symmetric reduction: full -> band (bandwidth b).
//
// The reference reduces its (skew-)symmetric matrix to tridiagonal form one
// Householder column at a time with BLAS-2 rank-2 updates
// (kernels.py:89-120, 39-46% of its runtime).  Here the first stage is
// blocked: each b-column panel is QR-factored by one cooperative kernel (the
// panel stays resident in shared memory across CTAs, one grid barrier per
// column) and the trailing matrix gets a two-sided compact-WY update made of
// DMMA GEMMs (SYMM as two triangular products, SYR2K on the lower triangle):
// 4/3 N^3 flops, all on the FP64 tensor pipe.
#include <cooperative_groups.h>
#include <algorithm>
#include "eig.cuh"

namespace bse {
namespace {

constexpr int kPanelThreads = 256;

BSE_DEV void grid_barrier(unsigned* ctr, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(ctr) : "memory");
      if (v >= target) break;
      __nanosleep(40);
    }
    __threadfence();
  }
  __syncthreads();
}

// Householder QR of the m x bw panel P (column-major, ldp), rows split over
// gridDim.x CTAs of R rows each (slab resident in smem).  Outputs:
//   P  <- R in its upper bw x bw triangle, zeros below
//   V  (ldv), V2 (ldv2): explicit unit-lower-trapezoidal reflectors
//   T  (bw x bw, ld bw): compact-WY factor, Q = I - V T V^T
// red: 2 * gridDim.x * (2 + 2*bw) doubles; bar: zeroed counter.
__global__ void __launch_bounds__(kPanelThreads) panel_qr_kernel(
    double* __restrict__ P, long long ldp, int m, int bw, double* __restrict__ V, long long ldv,
    double* __restrict__ V2, long long ldv2, double* __restrict__ T, double* __restrict__ red,
    unsigned* bar, int R) {
  extern __shared__ double smem[];
  double* S = smem;                    // slab, column-major [k*R + r]
  double* tot = S + (size_t)R * bw;    // 2 + 2*bw reduced values
  double* loc = tot + 2 + 2 * kMaxPanel;  // local partials
  double* wv = loc + 2 + 2 * kMaxPanel;   // w_k / y_i
  double* Ts = wv + kMaxPanel;             // T (CTA 0), [j*bw + i]
  __shared__ double sc[4];                 // tau, beta, scale

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int r0 = cta * R;                 // first panel row of this slab
  const int rows = max(0, min(R, m - r0));
  const int L = 2 + 2 * bw;

  for (int idx = tid; idx < R * bw; idx += blockDim.x) {
    const int r = idx % R, k = idx / R;
    S[idx] = (r < rows) ? P[(r0 + r) + (long long)k * ldp] : 0.0;
  }
  if (cta == 0)
    for (int idx = tid; idx < bw * bw; idx += blockDim.x) Ts[idx] = 0.0;
  __syncthreads();

  for (int j = 0; j < bw; ++j) {
    // ---- local partial sums over slab rows with global index >= j ----
    const int rbeg = max(0, j - r0);  // local row index of the first row >= j
    for (int k = warp; k < bw; k += nwarps) {
      double s = 0.0;
      const double* ck = S + (size_t)k * R;
      const double* cj = S + (size_t)j * R;
      for (int r = rbeg + lane; r < rows; r += 32) s += ck[r] * cj[r];
      s = warp_sum(s);
      if (lane == 0) loc[2 + k] = s;
    }
    if (warp == nwarps - 1) {
      double s = 0.0;
      const double* cj = S + (size_t)j * R;
      const int rb = max(0, j + 1 - r0);
      for (int r = rb + lane; r < rows; r += 32) s += cj[r] * cj[r];
      s = warp_sum(s);
      if (lane == 0) loc[0] = s;
    }
    const bool owner = (j >= r0 && j < r0 + rows);
    if (tid < bw) loc[2 + bw + tid] = owner ? S[(size_t)tid * R + (j - r0)] : 0.0;
    if (tid == 0) loc[1] = owner ? S[(size_t)j * R + (j - r0)] : 0.0;
    __syncthreads();

    if (G > 1) {
      double* slot = red + (size_t)(j & 1) * G * L;
      for (int t = tid; t < L; t += blockDim.x) slot[(size_t)cta * L + t] = loc[t];
      grid_barrier(bar, (unsigned)G * (unsigned)(j + 1));
      for (int t = tid; t < L; t += blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < G; ++c) s += __ldcg(slot + (size_t)c * L + t);
        tot[t] = s;
      }
    } else {
      for (int t = tid; t < L; t += blockDim.x) tot[t] = loc[t];
    }
    __syncthreads();

    if (tid == 0) {
      const double x0 = tot[1], st = tot[0];
      double tau = 0.0, beta = x0, scale = 0.0;
      if (st > 0.0) {
        beta = -copysign(sqrt(x0 * x0 + st), x0);
        tau = (beta - x0) / beta;
        scale = 1.0 / (x0 - beta);
      }
      sc[0] = tau; sc[1] = beta; sc[2] = scale;
    }
    __syncthreads();
    const double tau = sc[0], beta = sc[1], scale = sc[2];
    // w_k = v^T P[:,k] (k > j); y_i = V[:,i]^T v (i < j)
    if (tid < bw) wv[tid] = (tot[2 + tid] - beta * tot[2 + bw + tid]) * scale;
    __syncthreads();

    // ---- apply H_j to the slab (rows >= j, columns > j) and store v ----
    if (tau != 0.0) {
      const int cols = bw - j - 1;
      for (int idx = tid; idx < rows * cols; idx += blockDim.x) {
        const int r = idx % rows, k = j + 1 + idx / rows;
        const int gr = r0 + r;
        if (gr < j) continue;
        const double vr = (gr == j) ? 1.0 : S[(size_t)j * R + r] * scale;
        S[(size_t)k * R + r] -= tau * vr * wv[k];
      }
      __syncthreads();
      for (int r = tid; r < rows; r += blockDim.x) {
        const int gr = r0 + r;
        if (gr > j) S[(size_t)j * R + r] *= scale;
        else if (gr == j) S[(size_t)j * R + r] = beta;
      }
    } else {
      // identity reflector: v = e_j, the stored tail is zero
      for (int r = tid; r < rows; r += blockDim.x) {
        const int gr = r0 + r;
        if (gr > j) S[(size_t)j * R + r] = 0.0;
      }
    }
    // ---- T column j (CTA 0): T[j][j] = tau, T[i][j] = -tau sum_k T[i][k] y_k ----
    if (cta == 0 && tid < bw) {
      const int i = tid;
      if (i < j) {
        double s = 0.0;
        for (int k = i; k < j; ++k) s += Ts[k * bw + i] * wv[k];
        Ts[j * bw + i] = -tau * s;
      } else if (i == j) {
        Ts[j * bw + j] = tau;
      }
    }
    __syncthreads();
  }

  // ---- write back R (upper), explicit V (unit lower) ----
  for (int idx = tid; idx < rows * bw; idx += blockDim.x) {
    const int r = idx % rows, k = idx / rows;
    const int gr = r0 + r;
    const double s = S[(size_t)k * R + r];
    P[gr + (long long)k * ldp] = (gr <= k) ? s : 0.0;
    const double v = (gr > k) ? s : (gr == k ? 1.0 : 0.0);
    V[gr + (long long)k * ldv] = v;
    if (V2) V2[gr + (long long)k * ldv2] = v;
  }
  if (cta == 0)
    for (int idx = tid; idx < bw * bw; idx += blockDim.x) T[idx] = Ts[idx];
}

__global__ void extract_band_kernel(const double* __restrict__ A, long long lda, int n, int b,
                                    double* __restrict__ AB, int ldab) {
  const int j = blockIdx.x;
  for (int d = threadIdx.x; d < ldab; d += blockDim.x) {
    const int i = j + d;
    AB[(long long)j * ldab + d] = (d <= b && i < n) ? A[i + (long long)j * lda] : 0.0;
  }
}

}  // namespace

size_t panel_smem_bytes(int R, int bw) {
  return sizeof(double) * ((size_t)R * bw + 2 * (2 + 2 * kMaxPanel) + kMaxPanel +
                           (size_t)kMaxPanel * kMaxPanel);
}

int panel_rows_per_cta(int m, int bw, int max_ctas) {
  // as many CTAs as needed so that the slab fits in ~200 KB, >= 128 rows each
  int R = 128;
  while ((long long)R * max_ctas < m) R += 32;
  (void)bw;
  return R;
}

cudaError_t panel_qr(double* P, long long ldp, int m, int bw, double* V, long long ldv, double* V2,
                     long long ldv2, double* T, double* red, unsigned* bar, int num_sms,
                     cudaStream_t s) {
  const int R = panel_rows_per_cta(m, bw, num_sms);
  const int G = (int)ceil_div(m, R);
  const size_t smem = panel_smem_bytes(R, bw);
  static size_t attr = 0;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(panel_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  cudaError_t e = cudaMemsetAsync(bar, 0, sizeof(unsigned), s);
  if (e != cudaSuccess) return e;
  void* args[] = {&P, &ldp, &m, &bw, &V, &ldv, &V2, &ldv2, &T, &red, &bar, (void*)&R};
  count_launch();
  if (G == 1)
    return cudaLaunchKernel((void*)panel_qr_kernel, dim3(1), dim3(kPanelThreads), args, smem, s);
  return cudaLaunchCooperativeKernel((void*)panel_qr_kernel, dim3(G), dim3(kPanelThreads), args,
                                     smem, s);
}

cudaError_t extract_band(const double* A, long long lda, int n, int b, double* AB, int ldab,
                         cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  extract_band_kernel<<<n, 128, 0, s>>>(A, lda, n, b, AB, ldab);
  count_launch();
  return cudaGetLastError();
}

// Full -> band.  A (n x n, lower triangle referenced) is overwritten: its
// lower band holds the band matrix, panel regions hold R, rest is garbage.
// Vall (ldv): reflectors of panel p at rows k+b.., cols k..k+b-1 (k = p*b);
// Tall: bw x bw T factors, one per panel.
cudaError_t sy2sb(double* A, long long lda, int n, int b, double* Vall, long long ldv,
                  double* Tall, const Sy2sbScratch& w, int num_sms, cudaStream_t s) {
  cudaError_t e = cudaSuccess;
  for (int p = 0;; ++p) {
    const int k = p * b;
    const int m = n - k - b;
    if (m < 2) break;
    const int bw = b;
    double* P = A + (k + b) + (long long)k * lda;
    double* A2 = A + (k + b) + (long long)(k + b) * lda;
    double* Vp = Vall + (k + b) + (long long)k * ldv;
    double* Tp = Tall + (size_t)p * b * b;
    const long long lw = w.ldvwv;
    double* slot0 = w.vwv;
    double* slot1 = w.vwv + lw * bw;
    double* slot2 = w.vwv + 2 * lw * bw;
    stage_mark("sy2sb_panel", s);
    e = panel_qr(P, lda, m, bw, Vp, ldv, slot0, lw, Tp, w.red, w.bar, num_sms, s);
    if (e != cudaSuccess) return e;
    e = cudaMemcpy2DAsync(slot2, lw * sizeof(double), slot0, lw * sizeof(double),
                          (size_t)m * sizeof(double), bw, cudaMemcpyDeviceToDevice, s);
    if (e != cudaSuccess) return e;
    stage_mark("sy2sb_symm", s);
    // Y = tril(A2) V + tril(A2,-1)^T V
    // (split-K: the triangular masks give row blocks very different k-ranges;
    //  splitting K balances them and fills the GPU with thin m x b outputs)
    const int ssplit = (int)std::min<long long>(kSymmSplits, std::max<long long>(1, m / 1024));
    GemmProblem g1 = make_gemm(m, bw, m, 1.0, A2, lda, slot0, lw, 0.0, w.y, w.ldy);
    g1.ma = Mask::lower();
    if ((e = gemm_splitk(false, false, g1, ssplit, w.symm_ws, w.probs, s)) != cudaSuccess) return e;
    GemmProblem g2 = make_gemm(m, bw, m, 1.0, A2, lda, slot0, lw, 1.0, w.y, w.ldy);
    g2.ma = Mask::strict_lower();
    if ((e = gemm_splitk(true, false, g2, ssplit, w.symm_ws, w.probs + 32, s)) != cudaSuccess)
      return e;
    // X = Y T -> slot1
    GemmProblem g3 = make_gemm(m, bw, bw, 1.0, w.y, w.ldy, Tp, bw, 0.0, slot1, lw);
    g3.mb = Mask::upper();
    if ((e = gemm(false, false, g3, s)) != cudaSuccess) return e;
    stage_mark("sy2sb_small", s);
    // Zs = V^T X (bw x bw), split-K
    GemmProblem g4 = make_gemm(bw, bw, m, 1.0, slot0, lw, slot1, lw, 0.0, w.z, bw);
    const int splits = (int)std::min<long long>(48, std::max<long long>(1, m / 256));
    if ((e = gemm_splitk(true, false, g4, splits, w.splitk_ws, w.probs, s)) != cudaSuccess) return e;
    // Z2 = T^T Zs
    GemmProblem g5 = make_gemm(bw, bw, bw, 1.0, Tp, bw, w.z, bw, 0.0, w.z2, bw);
    g5.ma = Mask::upper();
    if ((e = gemm(true, false, g5, s)) != cudaSuccess) return e;
    // W = X - 0.5 V Z2 (in slot1)
    GemmProblem g6 = make_gemm(m, bw, bw, -0.5, slot0, lw, w.z2, bw, 1.0, slot1, lw);
    if ((e = gemm(false, false, g6, s)) != cudaSuccess) return e;
    stage_mark("sy2sb_syr2k", s);
    // A2 -= [V W][W V]^T (lower)
    GemmProblem g7 = make_gemm(m, m, 2 * bw, -1.0, slot0, lw, slot1, lw, 1.0, A2, lda);
    g7.mc = Mask::lower();
    if ((e = gemm(false, true, g7, s)) != cudaSuccess) return e;
  }
  return e;
}

}  // namespace bse
