// Eigenvector back-transforms Z <- Q1 Q2 Z.
//
// The reference applies its accumulated reflectors one rank-1 update at a
// time (kernels.py:123-137, 29-40% of its runtime).  Here:
//  * Q2 (bulge-chasing reflectors): g consecutive sweeps x one chase step form
//    a staircase compact-WY block (V, V*T); blocks are applied in a
//    dependency-respecting order (sweep groups descending, steps ascending)
//    by a column-slab kernel whose two small products run on DMMA.
//  * Q1 (SY2SB panels): plain compact-WY, three DMMA GEMMs per panel.
#include <algorithm>
#include "eig.cuh"

namespace bse {
namespace {

constexpr int kQ2G = 32;      // sweeps per block
constexpr int kQ2W = 64;      // Z columns per CTA
constexpr int kQ2Threads = 256;

BSE_HD int q2_hb(int b, int g) { return ((g + b + 1) / 2) * 2; }  // padded block height

BSE_DEV int refl_len(int n, int b, int s, int j) {
  const int r0 = s + 1 + j * b;
  if (s > n - 3 || r0 > n - 1) return 0;
  return min(b, n - r0);
}

// One CTA per (group, step): staircase V, T = larft(V), VT = V*T.
__global__ void __launch_bounds__(256) q2_build_kernel(int n, int b, int g, int maxsteps,
                                                       const double* __restrict__ V2,
                                                       const double* __restrict__ tau2,
                                                       double* __restrict__ Vblk,
                                                       double* __restrict__ VTblk) {
  extern __shared__ double sm[];
  const int HB = q2_hb(b, g);
  double* V = sm;                 // HB x g, [c*HB + r]
  double* G = V + HB * g;         // g x g gram
  double* T = G + g * g;          // g x g
  double* tau = T + g * g;        // g
  const int j = blockIdx.x, gi = blockIdx.y;
  const int s0 = gi * g;
  const int tid = threadIdx.x;
  const size_t blk = (size_t)gi * maxsteps + j;
  double* Vout = Vblk + blk * HB * g;
  double* VTout = VTblk + blk * HB * g;
  for (int idx = tid; idx < HB * g; idx += blockDim.x) {
    const int r = idx % HB, c = idx / HB;
    const int s = s0 + c;
    const int len = refl_len(n, b, s, j);
    double v = 0.0;
    if (len > 0 && r >= c && r < c + len) v = V2[((size_t)s * maxsteps + j) * b + (r - c)];
    V[idx] = v;
  }
  for (int c = tid; c < g; c += blockDim.x) {
    const int s = s0 + c;
    tau[c] = refl_len(n, b, s, j) > 0 ? tau2[(size_t)s * maxsteps + j] : 0.0;
  }
  __syncthreads();
  for (int idx = tid; idx < g * g; idx += blockDim.x) {
    const int a = idx % g, c = idx / g;
    double acc = 0.0;
    for (int r = 0; r < HB; ++r) acc += V[a * HB + r] * V[c * HB + r];
    G[idx] = acc;  // G[c*g + a] = v_a . v_c
    T[idx] = 0.0;
  }
  __syncthreads();
  for (int c = 0; c < g; ++c) {
    if (tid < c) {
      double acc = 0.0;
      for (int k = tid; k < c; ++k) acc += T[k * g + tid] * G[c * g + k];
      T[c * g + tid] = -tau[c] * acc;
    } else if (tid == c) {
      T[c * g + c] = tau[c];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < HB * g; idx += blockDim.x) {
    const int r = idx % HB, c = idx / HB;
    double acc = 0.0;
    for (int k = 0; k <= c; ++k) acc += V[k * HB + r] * T[c * g + k];
    Vout[idx] = V[idx];
    VTout[idx] = acc;
  }
}

// Column slab kernel: for each block in order, Z[r0:r0+HB, slab] -= VT (V^T Z).
// Y = V^T Z reuses V's shared memory, so two CTAs fit per SM and the 256
// slabs of an n = 16384 problem run as a single wave; Z rows are staged with
// 16-byte cp.async from the even row below r0.
template <int HB, int G>
__global__ void __launch_bounds__(kQ2Threads, 2) q2_apply_kernel(int n, int b, int maxsteps,
                                                                 const double* __restrict__ Vblk,
                                                                 const double* __restrict__ VTblk,
                                                                 double* __restrict__ Z,
                                                                 long long ldz, int ncols) {
  constexpr int LDV = HB + 4;   // == 4 mod 16: conflict-free fragment loads
  constexpr int LDZ = HB + 4;
  constexpr int LDY = G + 4;
  constexpr int W = kQ2W;
  static_assert(W * LDY <= G * LDV, "Y must fit in V's buffer");
  extern __shared__ __align__(16) double sm[];
  double* sV = sm;               // HB x G  [c*LDV + r]; later Y (G x W) [c*LDY + r]
  double* sVT = sV + G * LDV;    // HB x G
  double* sZ = sVT + G * LDV;    // (HB+2) x W  [c*LDZ + r]
  double* sY = sV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int c0 = blockIdx.x * W;
  const int wcols = min(W, ncols - c0);
  const int nsweeps = n - 2;
  const int ngroups = (int)ceil_div(nsweeps, G);
  const int kl = lane & 3, rl = lane >> 2;
  const int wm = warp & 1, wn = warp >> 1;

  for (int gi = ngroups - 1; gi >= 0; --gi) {
    const int s0 = gi * G;
    for (int j = 0; j < maxsteps; ++j) {
      const int r0 = s0 + 1 + j * b;
      if (r0 > n - 1) break;
      const size_t blk = (size_t)gi * maxsteps + j;
      const double* gV = Vblk + blk * HB * G;
      const double* gVT = VTblk + blk * HB * G;
      const int rows = min(HB, n - r0);
      const int off = r0 & 1;          // smem row of global row r0
      const int re = r0 - off;         // even start row
      const int rows_e = rows + off;   // rows staged
      for (int idx = tid; idx < HB * G / 2; idx += blockDim.x) {
        const int e = idx * 2;
        const int r = e % HB, c = e / HB;
        cp_async16(sV + c * LDV + r, gV + e, true);
        cp_async16(sVT + c * LDV + r, gVT + e, true);
      }
      constexpr int ZCH = (HB + 2) / 2;  // 16-byte chunks per column
      for (int idx = tid; idx < ZCH * W; idx += blockDim.x) {
        const int r = (idx % ZCH) * 2, c = idx / ZCH;
        const bool cok = c < wcols;
        const double* src = Z + re + r + (long long)(c0 + c) * ldz;
        double* dst = sZ + c * LDZ + r;
        const bool v0 = cok && r < rows_e, v1 = cok && r + 1 < rows_e;
        if (v0 && v1) cp_async16(dst, src, true);
        else { cp_async8(dst, v0 ? src : Z, v0); cp_async8(dst + 1, v1 ? src + 1 : Z, v1); }
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      // Y (G x W) = V^T Z : 8 warps as 2 (m) x 4 (n), warp tile (G/2) x 16
      {
        constexpr int WM = G / 2, MI = WM / 8;
        double acc[MI][2][2];
#pragma unroll
        for (int i = 0; i < MI; ++i) acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0.0;
        // reflector c of the block is nonzero on rows [c, c + b) only
        const int kbeg = wm * WM, kend = min(HB, wm * WM + WM + b);
#pragma unroll 4
        for (int k = kbeg; k < kend; k += 4) {
          double af[MI], bf[2];
#pragma unroll
          for (int i = 0; i < MI; ++i) af[i] = sV[(wm * WM + i * 8 + rl) * LDV + k + kl];
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) bf[jj] = sZ[(wn * 16 + jj * 8 + rl) * LDZ + off + k + kl];
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) dmma8x8x4(acc[i][jj], af[i], bf[jj]);
        }
        __syncthreads();  // V consumed: Y overwrites it
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int m = wm * WM + i * 8 + rl, c = wn * 16 + jj * 8 + kl * 2 + e;
              sY[c * LDY + m] = acc[i][jj][e];
            }
      }
      __syncthreads();
      // Z (HB x W) -= VT Y : 8 warps as 2 (m) x 4 (n), warp tile (HB/2) x 16
      {
        constexpr int WM = HB / 2, MI = WM / 8;
        double acc[MI][2][2];
#pragma unroll
        for (int i = 0; i < MI; ++i) acc[i][0][0] = acc[i][0][1] = acc[i][1][0] = acc[i][1][1] = 0.0;
#pragma unroll
        for (int k = 0; k < G; k += 4) {
          double af[MI], bf[2];
#pragma unroll
          for (int i = 0; i < MI; ++i) af[i] = sVT[(k + kl) * LDV + wm * WM + i * 8 + rl];
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) bf[jj] = sY[(wn * 16 + jj * 8 + rl) * LDY + k + kl];
#pragma unroll
          for (int i = 0; i < MI; ++i)
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) dmma8x8x4(acc[i][jj], af[i], bf[jj]);
        }
#pragma unroll
        for (int i = 0; i < MI; ++i)
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int r = wm * WM + i * 8 + rl, c = wn * 16 + jj * 8 + kl * 2 + e;
              if (r < rows && c < wcols)
                Z[(r0 + r) + (long long)(c0 + c) * ldz] = sZ[c * LDZ + off + r] - acc[i][jj][e];
            }
      }
      __syncthreads();
    }
  }
}

}  // namespace

size_t q2_block_doubles(int n, int b, int g) {
  const int maxsteps = sb2st_maxsteps(n, b);
  const int ngroups = (int)ceil_div(std::max(n - 2, 1), g);
  return (size_t)ngroups * maxsteps * q2_hb(b, g) * g;
}

cudaError_t q2_build(int n, int b, int g, const double* V2, const double* tau2, double* Vblk,
                     double* VTblk, cudaStream_t s) {
  if (n <= 2) return cudaSuccess;
  const int maxsteps = sb2st_maxsteps(n, b);
  const int ngroups = (int)ceil_div(n - 2, g);
  const int HB = q2_hb(b, g);
  const size_t smem = sizeof(double) * ((size_t)HB * g + 2 * (size_t)g * g + g);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(q2_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  q2_build_kernel<<<dim3(maxsteps, ngroups), 256, smem, s>>>(n, b, g, maxsteps, V2, tau2, Vblk, VTblk);
  count_launch();
  return cudaGetLastError();
}

cudaError_t q2_apply(int n, int b, int g, const double* Vblk, const double* VTblk, double* Z,
                     long long ldz, int ncols, cudaStream_t s) {
  if (n <= 2 || ncols <= 0) return cudaSuccess;
  if (b != 64 || g != kQ2G) return cudaErrorInvalidValue;
  constexpr int HB = 96, G = kQ2G;  // q2_hb(64, 32)
  const int maxsteps = sb2st_maxsteps(n, b);
  const size_t smem = sizeof(double) * (2 * (size_t)G * (HB + 4) + (size_t)kQ2W * (HB + 4));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(q2_apply_kernel<HB, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  q2_apply_kernel<HB, G><<<(unsigned)ceil_div(ncols, kQ2W), kQ2Threads, smem, s>>>(
      n, b, maxsteps, Vblk, VTblk, Z, ldz, ncols);
  count_launch();
  return cudaGetLastError();
}

cudaError_t q1_apply(int n, int b, const double* Vall, long long ldv, const double* Tall,
                     double* Z, long long ldz, int ncols, const Q1Scratch& w, cudaStream_t s) {
  // Panels are merged in groups of kQ1Group (compact-WY of the product,
  // T_g = [[T_A, -T_A (V_A^T V_B) T_B], [0, T_B]]) so the applying GEMMs run
  // with K = kQ1Group*b instead of b.  Vall must be zero outside the
  // reflectors (syevd memsets it before SY2SB).
  int np = 0;
  while (n - np * b - b >= 2) ++np;
  cudaError_t e = cudaSuccess;
  const int G = kQ1Group;
  for (int pend = np; pend > 0; pend -= G) {
    const int p0 = std::max(0, pend - G), k = pend - p0, kb = k * b;
    const int r0 = (p0 + 1) * b, m = n - r0;
    const double* V = Vall + r0 + (long long)(p0 * b) * ldv;  // m x kb
    double* Tg = w.tg;                                        // kb x kb (ld kb)
    stage_mark("q1_tg", s);
    // block-diagonal T_p, then the off-diagonal blocks column by column
    if ((e = cudaMemsetAsync(Tg, 0, sizeof(double) * kb * kb, s)) != cudaSuccess) return e;
    for (int j = 0; j < k; ++j) {
      if ((e = cudaMemcpy2DAsync(Tg + (long long)j * b + (long long)j * b * kb, kb * sizeof(double),
                                 Tall + (size_t)(p0 + j) * b * b, b * sizeof(double),
                                 b * sizeof(double), b, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
        return e;
    }
    for (int j = 1; j < k; ++j) {
      const int jb = j * b;
      // X = V[:, :jb]^T V[:, jb:jb+b]   (jb x b, K = m)
      GemmProblem gx = make_gemm(jb, b, m, 1.0, V, ldv, V + (long long)jb * ldv, ldv, 0.0, w.x, jb);
      if ((e = gemm_splitk(true, false, gx, 16, w.splitk_ws, w.probs, s)) != cudaSuccess) return e;
      // tmp = T_g[:jb,:jb] X ; T_g[:jb, jb:jb+b] = -tmp T_j
      GemmProblem g1 = make_gemm(jb, b, jb, 1.0, Tg, kb, w.x, jb, 0.0, w.tmp, jb);
      g1.ma = Mask::upper();
      if ((e = gemm(false, false, g1, s)) != cudaSuccess) return e;
      GemmProblem g2 = make_gemm(jb, b, b, -1.0, w.tmp, jb, Tg + jb + (long long)jb * kb, kb, 0.0,
                                 Tg + (long long)jb * kb, kb);
      g2.mb = Mask::upper();
      if ((e = gemm(false, false, g2, s)) != cudaSuccess) return e;
    }
    double* Zs = Z + r0;
    stage_mark("q1_gemm", s);
    // Y = V^T Zs (kb x ncols)
    GemmProblem g3 = make_gemm(kb, ncols, m, 1.0, V, ldv, Zs, ldz, 0.0, w.y, kb);
    if ((e = gemm(true, false, g3, s)) != cudaSuccess) return e;
    // Y2 = T_g Y
    GemmProblem g4 = make_gemm(kb, ncols, kb, 1.0, Tg, kb, w.y, kb, 0.0, w.y2, kb);
    g4.ma = Mask::upper();
    if ((e = gemm(false, false, g4, s)) != cudaSuccess) return e;
    // Zs -= V Y2
    GemmProblem g5 = make_gemm(m, ncols, kb, -1.0, V, ldv, w.y2, kb, 1.0, Zs, ldz);
    if ((e = gemm(false, false, g5, s)) != cudaSuccess) return e;
  }
  return e;
}

}  // namespace bse
