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
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "eig.cuh"
#include "ozgemm.cuh"

namespace bse {
namespace {

constexpr int kQ2G = 32;      // sweeps per block
// Z columns per CTA = 8 x warps.  14 warps (112 columns): 147 CTAs = one wave
// at n = 16384; narrower slabs (8/4/2 warps) keep >= 3/4 of the SMs busy when
// fewer columns are applied (a rank's column block, mid-size n).
constexpr int kQ2MaxWarps = 14;

BSE_HD int q2_hb(int b, int g) { return ((g + b + 1) / 2) * 2; }  // padded block height

// Stored block = the apply kernel's shared-memory stage, byte for byte, so one
// bulk copy moves it: V column-major (ld 96), then VT = V*T row-major (ld
// 32), both with the 16-byte units of odd columns (V) / odd rows (VT) XOR-ed
// by 4: the 128-bit fragment loads of a quarter warp (two consecutive
// columns / rows) then hit 8 distinct bank groups without padding.
constexpr int kQ2HB = 96;
constexpr int kQ2LDV = kQ2HB;  // sV[c * LDV + swz(r)]
constexpr int kQ2LDT = kQ2G;   // sVT[r * LDT + swz(c)]
constexpr int kQ2Stage = kQ2G * kQ2LDV + kQ2HB * kQ2LDT;
constexpr int kQ2Stages = 2;
// position of element k (row of V / column of VT) inside line `line`
BSE_HD int q2_swz(int k, int line) { return ((((k >> 1) ^ ((line & 1) << 2))) << 1) | (k & 1); }

BSE_DEV int refl_len(int n, int b, int s, int j) {
  const int r0 = s + 1 + j * b;
  if (s > n - 3 || r0 > n - 1) return 0;
  return min(b, n - r0);
}

// One CTA per (group, step): staircase V, T = larft(V), VT = V*T.  Shared
// arrays use odd strides (HB + 1, g + 1) so the column-indexed dot products
// are bank-conflict free; reflector c is nonzero only in rows [c, c + b).
__global__ void __launch_bounds__(256) q2_build_kernel(int n, int b, int g, int maxsteps,
                                                       const double* __restrict__ V2,
                                                       const double* __restrict__ tau2,
                                                       double* __restrict__ Vblk, int g_base) {
  extern __shared__ double sm[];
  const int HB = q2_hb(b, g);
  const int LV = HB + 1, LG = g + 1;
  double* V = sm;                 // HB x g, [c*LV + r]
  double* G = V + LV * g;         // g x g gram, [c*LG + a]
  double* T = G + LG * g;         // g x g, [c*LG + k]
  double* tau = T + LG * g;       // g
  // Vblk holds the blocks of groups g_base, g_base + 1, ... (all groups: 0)
  const int j = blockIdx.x, gi = g_base + blockIdx.y;
  const int s0 = gi * g;
  const int tid = threadIdx.x;
  const size_t blk = (size_t)blockIdx.y * maxsteps + j;
  double* Vout = Vblk + blk * kQ2Stage;
  for (int idx = tid; idx < HB * g; idx += blockDim.x) {
    const int r = idx % HB, c = idx / HB;
    const int s = s0 + c;
    const int len = refl_len(n, b, s, j);
    double v = 0.0;
    if (len > 0 && r >= c && r < c + len) v = V2[((size_t)s * maxsteps + j) * b + (r - c)];
    V[c * LV + r] = v;
  }
  for (int c = tid; c < g; c += blockDim.x) {
    const int s = s0 + c;
    tau[c] = refl_len(n, b, s, j) > 0 ? tau2[(size_t)s * maxsteps + j] : 0.0;
  }
  __syncthreads();
  // G[c][a] = v_a . v_c for a < c (rows where both are nonzero: [c, a + b))
  for (int idx = tid; idx < g * g; idx += blockDim.x) {
    const int a = idx % g, c = idx / g;
    double acc = 0.0;
    if (a < c) {
      const int r1 = min(a + b, HB);
      for (int r = c; r < r1; ++r) acc += V[a * LV + r] * V[c * LV + r];
    }
    G[c * LG + a] = acc;
    T[c * LG + a] = 0.0;
  }
  __syncthreads();
  for (int c = 0; c < g; ++c) {
    if (tid < c) {
      double acc = 0.0;
      for (int k = tid; k < c; ++k) acc += T[k * LG + tid] * G[c * LG + k];
      T[c * LG + tid] = -tau[c] * acc;
    } else if (tid == c) {
      T[c * LG + c] = tau[c];
    }
    __syncthreads();
  }
  double* VTo = Vout + (size_t)g * kQ2LDV;
  for (int idx = tid; idx < HB * g; idx += blockDim.x) {
    const int r = idx % HB, c = idx / HB;
    Vout[c * kQ2LDV + q2_swz(r, c)] = V[c * LV + r];
  }
  // VT[r][c] = sum_{k <= c} V[r][k] T[k][c], V[r][k] != 0 only for r - b < k <= r
  for (int idx = tid; idx < HB * g; idx += blockDim.x) {
    const int r = idx / g, c = idx % g;
    double acc = 0.0;
    const int k1 = min(c, r);
    for (int k = max(0, r - b + 1); k <= k1; ++k) acc += V[k * LV + r] * T[c * LG + k];
    VTo[r * kQ2LDT + q2_swz(c, r)] = acc;  // VT row-major (q2_apply's B-operand layout)
  }
}

// Column-slab apply kernel.  Each warp owns 8 columns of Z and keeps a
// window of Z rows in registers in the TRANSPOSED DMMA accumulator layout:
// lane (rl = lane/4, kl = lane%4) holds acc[i][e] = Z[W0 + 8i + 2kl + e][col rl].
// Both products are then computed transposed,
//   Y^T = Z^T V   (A = Z^T straight from acc, B = V from shared memory)
//   Z^T -= Y^T (V T)^T  (A = Y^T straight from its accumulators, B = VT)
// with the k-steps ordered as {2kl + e}, so no operand needs a warp shuffle;
// every shared-memory fragment pair is one conflict-free 128-bit load (V
// column-major with LDV = 104, VT row-major with LDT = 40: both == 8 mod 16).
// The zero corners of the staircase V (and of VT) are skipped at compile time.
constexpr int kQ2LDN = 64 + 8;     // prefetched rows, [col * LDN + row]

BSE_DEV double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

template <int OFF, int NT, int CG>
BSE_DEV void q2_block_t(double (&acc)[CG][NT][2], const double* sV, const double* sVT, int lane) {
  const int kl = lane & 3, rl = lane >> 2;
  // swizzle: this lane's line (column c = 8q + rl of V, row 8i + rl of VT)
  // has parity rl & 1, so 16-byte unit u moves to u ^ 4 on odd lines; with u
  // = 4t + kl (t a compile-time tile index) that is +-8 doubles by t's parity
  const int sw = (rl & 1) * 8;
  const double* pV0 = sV + rl * kQ2LDV + 2 * kl + sw;   // even tile
  const double* pV1 = sV + rl * kQ2LDV + 2 * kl - sw;   // odd tile
  const double* pT0 = sVT + rl * kQ2LDT + 2 * kl + sw;
  const double* pT1 = sVT + rl * kQ2LDT + 2 * kl - sw;
  // CG groups of 8 columns share every V / VT fragment load
  double yt[CG][4][2];
#pragma unroll
  for (int g = 0; g < CG; ++g)
#pragma unroll
    for (int q = 0; q < 4; ++q) yt[g][q][0] = yt[g][q][1] = 0.0;
  // Y^T (8 cols x 32 reflectors): reflector tile q meets row tiles q .. q+8
#pragma unroll
  for (int i = 0; i < 12; ++i) {
    double2 bv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (i >= q && i <= q + 8) bv[q] = lds2((i & 1 ? pV1 : pV0) + 8 * q * kQ2LDV + 8 * i);
#pragma unroll
    for (int g = 0; g < CG; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i >= q && i <= q + 8) dmma8x8x4(yt[g][q], acc[g][OFF + i][0], bv[q].x);
#pragma unroll
    for (int g = 0; g < CG; ++g)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (i >= q && i <= q + 8) dmma8x8x4(yt[g][q], acc[g][OFF + i][1], bv[q].y);
  }
#pragma unroll
  for (int g = 0; g < CG; ++g)
#pragma unroll
    for (int q = 0; q < 4; ++q) { yt[g][q][0] = -yt[g][q][0]; yt[g][q][1] = -yt[g][q][1]; }
  // Z^T -= Y^T VT^T: VT[r][c] = 0 for c < r - 63 (row tile i needs q >= i - 8)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
#pragma unroll
    for (int h = 0; h < 12; h += 6) {
      double2 bv[6];
#pragma unroll
      for (int i = h; i < h + 6; ++i)
        if (q >= i - 8) bv[i - h] = lds2((q & 1 ? pT1 : pT0) + 8 * i * kQ2LDT + 8 * q);
#pragma unroll
      for (int g = 0; g < CG; ++g)
#pragma unroll
        for (int i = h; i < h + 6; ++i)
          if (q >= i - 8) dmma8x8x4(acc[g][OFF + i], yt[g][q][0], bv[i - h].x);
#pragma unroll
      for (int g = 0; g < CG; ++g)
#pragma unroll
        for (int i = h; i < h + 6; ++i)
          if (q >= i - 8) dmma8x8x4(acc[g][OFF + i], yt[g][q][1], bv[i - h].y);
    }
  }
}

// Paired-group walk.  Two consecutive sweep groups (ga = gi, gb = gi - 1)
// walk down the rows together: at chase step j, block (ga, j) covers rows
// [B0 + 64j + 32, +96) and block (gb, j) rows [B0 + 64j, +96) (B0 = gb*G + 1).
// (gb, j) only overlaps (ga, j') for j' <= j, so the order (ga, 0), (gb, 0),
// (ga, 1), (gb, 1), ... respects Q2's application order.  The 128-row window
// stays in registers; 64 rows stream in (cp.async, one step ahead) and out
// per STEP instead of per block.

// V/VT blocks arrive by bulk async copy (TMA engine) into a 2-stage ring
// driven by mbarriers: a producer warp walks the same block order and issues
// each block's copy as soon as every consumer warp has released the stage
// (empty barrier, one arrival per warp); consumer warps wait only on the
// stage's full barrier.  No CTA-wide barrier in the loop: warps may drift up
// to one block apart.
template <int P, int NW, int CG>
__global__ void __launch_bounds__(32 * (NW + 1), 1) q2_apply_pair_kernel(
    int n, int b, int maxsteps, const double* __restrict__ Vblk, double* __restrict__ Z,
    long long ldz, int ncols, int g_hi, int g_lo) {
  // applies the blocks of sweep groups g_hi, g_hi - 1, ..., g_lo (a suffix of
  // the full walk when called range by range, top range first; Vblk holds the
  // blocks of group g_lo onwards).  The whole transform: g_hi = ngroups - 1,
  // g_lo = 0.
  constexpr int G = kQ2G;
  constexpr int STAGE = kQ2Stage;
  constexpr int LDN = kQ2LDN;
  constexpr int NT = 4 * P + 8;  // 8-row tiles in the window
  constexpr unsigned kStageBytes = STAGE * sizeof(double);
  extern __shared__ __align__(16) double sm[];
  constexpr int NS = kQ2Stages;
  double* sZn = sm + NS * STAGE;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(sZn + 8 * CG * NW * LDN);
  unsigned long long* full = bars;        // [NS]
  unsigned long long* empty = bars + NS;  // [NS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kl = lane & 3, rl = lane >> 2;
  constexpr int kQ2W = 8 * CG * NW;           // columns per CTA
  const int cw = blockIdx.x * kQ2W + warp * 8 * CG;  // this warp's first column
  const int nsweeps = n - 2;
  const int ngroups = (int)ceil_div(nsweeps, G);

  (void)b;  // == 64 (checked by the host)
  auto steps_of = [&](int gi) -> int {
    if (gi < 0) return 0;
    const int st = (n - 1 - gi * G + 63) >> 6;
    return st < maxsteps ? st : maxsteps;
  };
  // blocks of group ga - wh exist for j < steps; the earliest group of the
  // set (ga - P + 1) has the most steps
  auto smax_of = [&](int ga) { return steps_of(max(ga - P + 1, 0)); };
  // next existing block after (ga, j, wh); false when the walk is done
  auto advance = [&](int& ga, int& j, int& wh) -> bool {
    for (;;) {
      if (wh + 1 < P) ++wh;
      else { wh = 0; ++j; }
      if (j >= smax_of(ga)) {
        ga -= P;
        j = 0;
        wh = 0;
        return ga >= g_lo;
      }
      if (ga - wh >= 0 && j < steps_of(ga - wh)) return true;
    }
  };
  if (tid == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      mbar_init(&full[q], 1);
      mbar_init(&empty[q], NW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  if (ngroups <= 0 || g_hi < g_lo) return;
  if (warp == NW) {
    // producer: one bulk copy per block, in the consumers' order
    if (lane == 0) {
      int ga = g_hi, j = 0, wh = 0;
      for (unsigned blkno = 0, st = 0, use = 0;; ++blkno) {
        // stage st is being filled for the use-th time: wait for the
        // consumers' release of its (use-1)-th fill
        if (use > 0) mbar_wait(&empty[st], (use - 1) & 1);
        const size_t blk = (size_t)(ga - wh - g_lo) * maxsteps + j;
        mbar_arrive_expect_tx(&full[st], kStageBytes);
        bulk_g2s(sm + st * STAGE, Vblk + blk * STAGE, kStageBytes, &full[st]);
        if (!advance(ga, j, wh)) break;
        if (++st == NS) { st = 0; ++use; }
      }
    }
    return;
  }
  // this lane's columns of Z (one per group of 8; rows added per access)
  bool colok[CG];
  double* zc[CG];
#pragma unroll
  for (int g = 0; g < CG; ++g) {
    colok[g] = cw + 8 * g + rl < ncols;
    zc[g] = Z + (long long)(colok[g] ? cw + 8 * g + rl : 0) * ldz;
  }
  // row prefetch: every warp streams in its own 8 columns (lane l: rows l
  // and l + 32 of each column, so every copy instruction moves 256
  // contiguous bytes), and only a warp-level sync guards sZn

  double acc[CG][NT][2];
  int ga = g_hi, j = 0, wh = 0, stage = 0;
  unsigned use = 0;  // fills of `stage` consumed so far
  bool pair_start = true;
  for (;;) {
    const int B0 = (ga - P + 1) * G + 1;
    int nga = ga, nj = j, nwh = wh;
    const bool more = advance(nga, nj, nwh);
    const bool step_end = !more || nga != ga || nj != j;
    const bool pair_end = !more || nga != ga;
    if (pair_start) {
#pragma unroll
      for (int g = 0; g < CG; ++g)
#pragma unroll
        for (int i = 0; i < NT; ++i)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int row = B0 + 8 * i + 2 * kl + e;
            acc[g][i][e] = (colok[g] && row >= 0 && row < n) ? __ldcg(zc[g] + row) : 0.0;
          }
      pair_start = false;
    }
    // this block's V/VT have landed
    mbar_wait(&full[stage], use & 1);
    // first block of step j: prefetch the 64 rows step j+1 brings in
    bool step_first = true;
    for (int m = 0; m < wh; ++m)
      if (j < steps_of(ga - m)) step_first = false;
    if (step_first && j + 1 < smax_of(ga)) {
      const int row0 = B0 + 64 * j + 8 * NT;
#pragma unroll
      for (int c = 0; c < 8 * CG; ++c) {
        const int col = cw + c;
        const bool cok = col < ncols;
        const double* src = Z + (long long)(cok ? col : 0) * ldz;
        double* dst = sZn + (warp * 8 * CG + c) * LDN;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = row0 + lane + 32 * h;
          const bool ok = cok && row >= 0 && row < n;
          cp_async8(dst + lane + 32 * h, ok ? src + row : Z, ok);
        }
      }
      cp_async_commit();
    }
    const double* sV = sm + stage * STAGE;
    const double* sVT = sV + G * kQ2LDV;
    // group ga - wh's block sits 32 (P - 1 - wh) rows into the window
    if (P == 1 || wh == 0) q2_block_t<4 * (P - 1), NT, CG>(acc, sV, sVT, lane);
    else if (P == 2 || wh == 1) q2_block_t<4 * (P > 1 ? P - 2 : 0), NT, CG>(acc, sV, sVT, lane);
    else if (P == 3 || wh == 2) q2_block_t<4 * (P > 2 ? P - 3 : 0), NT, CG>(acc, sV, sVT, lane);
    else q2_block_t<4 * (P > 3 ? P - 4 : 0), NT, CG>(acc, sV, sVT, lane);
    // this warp is done with the stage
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (step_end) {
      const int nstore = pair_end ? NT : 8;
      const int rbase = B0 + 64 * j;
#pragma unroll
      for (int g = 0; g < CG; ++g)
#pragma unroll
        for (int i = 0; i < NT; ++i) {
          if (i < nstore) {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int row = rbase + 8 * i + 2 * kl + e;
              if (colok[g] && row >= 0 && row < n) zc[g][row] = acc[g][i][e];
            }
          }
        }
      if (!pair_end) {
        // the rows were streamed in by this warp only
        cp_async_wait<0>();
        __syncwarp();
#pragma unroll
        for (int g = 0; g < CG; ++g) {
          const int cl = warp * 8 * CG + 8 * g;
#pragma unroll
          for (int i = 0; i < NT - 8; ++i) {
            acc[g][i][0] = acc[g][8 + i][0];
            acc[g][i][1] = acc[g][8 + i][1];
          }
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const double2 z = lds2(sZn + (cl + rl) * LDN + 8 * i + 2 * kl);
            acc[g][NT - 8 + i][0] = z.x;
            acc[g][NT - 8 + i][1] = z.y;
          }
        }
      } else {
        // the next pair's row prefetches (other lanes) read rows stored here
        __syncwarp();
        pair_start = true;
      }
    }
    if (++stage == NS) { stage = 0; ++use; }
    if (!more) break;
    ga = nga;
    j = nj;
    wh = nwh;
  }
}

}  // namespace

size_t q2_block_doubles(int n, int b, int g) {
  const int maxsteps = sb2st_maxsteps(n, b);
  const int ngroups = (int)ceil_div(std::max(n - 2, 1), g);
  (void)b;
  return (size_t)ngroups * maxsteps * kQ2Stage;
}

int q2_groups(int n, int g) { return n <= 2 ? 0 : (int)ceil_div(n - 2, g); }

size_t q2_range_doubles(int n, int b, int ngr) {
  return (size_t)std::max(ngr, 1) * sb2st_maxsteps(n, b) * kQ2Stage;
}

cudaError_t q2_build(int n, int b, int g, const double* V2, const double* tau2, double* Vblk,
                     cudaStream_t s, int g_lo, int g_hi) {
  if (n <= 2) return cudaSuccess;
  if (b != 64 || g != kQ2G || q2_hb(b, g) != kQ2HB) return cudaErrorInvalidValue;
  const int maxsteps = sb2st_maxsteps(n, b);
  if (g_hi < 0) g_hi = (int)ceil_div(n - 2, g) - 1;
  if (g_hi < g_lo) return cudaSuccess;
  const int ngroups = g_hi - g_lo + 1;
  const int HB = q2_hb(b, g);
  const size_t smem = sizeof(double) * ((size_t)(HB + 1) * g + 2 * (size_t)(g + 1) * g + g);
  static PerDeviceOnce attr;
  cudaError_t ae = set_smem_limit(attr, q2_build_kernel, 200 * 1024);
  if (ae != cudaSuccess) return ae;
  q2_build_kernel<<<dim3(maxsteps, ngroups), 256, smem, s>>>(n, b, g, maxsteps, V2, tau2, Vblk, g_lo);
  count_launch();
  return cudaGetLastError();
}

cudaError_t q2_apply(int n, int b, int g, const double* Vblk, double* Z, long long ldz, int ncols,
                     cudaStream_t s, int g_lo, int g_hi) {
  if (n <= 2 || ncols <= 0) return cudaSuccess;
  if (b != 64 || g != kQ2G || q2_hb(b, g) != kQ2HB) return cudaErrorInvalidValue;
  const int maxsteps = sb2st_maxsteps(n, b);
  if (g_hi < 0) g_hi = (int)ceil_div(n - 2, g) - 1;
  if (g_hi < g_lo) return cudaSuccess;
  const int sms = device_sm_count();
  auto launch = [&](auto kern, int nw, int cg) {
    const size_t smem = sizeof(double) * (kQ2Stages * (size_t)kQ2Stage +
                                          (size_t)8 * cg * nw * kQ2LDN) +
                        2 * kQ2Stages * sizeof(unsigned long long);
    cudaError_t ae = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ae != cudaSuccess) return ae;
    kern<<<(unsigned)ceil_div(ncols, 8 * cg * nw), 32 * (nw + 1), smem, s>>>(
        n, b, maxsteps, Vblk, Z, ldz, ncols, g_hi, g_lo);
    count_launch();
    return cudaGetLastError();
  };
  auto enough = [&](int nw) { return 4 * ceil_div(ncols, 8 * nw) >= 3 * (long long)sms; };
  static const int cg2 = std::getenv("BSE_Q2_CG") ? std::atoi(std::getenv("BSE_Q2_CG")) : 1;
  if (cg2 == 2 && enough(kQ2MaxWarps))
    return launch(q2_apply_pair_kernel<2, kQ2MaxWarps / 2, 2>, kQ2MaxWarps / 2, 2);
  if (enough(kQ2MaxWarps)) return launch(q2_apply_pair_kernel<2, kQ2MaxWarps, 1>, kQ2MaxWarps, 1);
  if (enough(8)) return launch(q2_apply_pair_kernel<2, 8, 1>, 8, 1);
  if (enough(4)) return launch(q2_apply_pair_kernel<2, 4, 1>, 4, 1);
  return launch(q2_apply_pair_kernel<2, 2, 1>, 2, 1);
}

size_t q1_oz_bytes(int n, int b, int ncols, int group) {
  const int kb = group * b, c = std::min(ncols, kQ1OzChunk);
  // Y = V^T Zs (kb x c chunks, K = m <= n); Zs -= V Y2 (n x c chunks, K = kb)
  return std::max({ozgemm_bytes(kb, ncols, n, c), ozgemm_bytes(n, ncols, kb, c),
                   ozgemm_bytes(kb, ncols, kb, c)});
}

int q1_panels(int n, int b) {
  int np = 0;
  while (n - np * b - b >= 2) ++np;
  return np;
}

size_t q1_tg_doubles(int n, int b, int group) {
  const int np = q1_panels(n, b);
  size_t tot = 0;
  for (int pend = np; pend > 0; pend -= group) {
    const size_t kb = (size_t)(pend - std::max(0, pend - group)) * b;
    tot += kb * kb;
  }
  return std::max<size_t>(tot, 1);
}

size_t q1_vt_doubles(int n, int b, int group) {
  const int np = q1_panels(n, b);
  size_t tot = 0;
  for (int pend = np; pend > 0; pend -= group) {
    const int p0 = std::max(0, pend - group);
    const size_t kb = (size_t)(pend - p0) * b, m = (size_t)(n - (p0 + 1) * b);
    tot += m * kb;
  }
  return std::max<size_t>(tot, 1);
}

// T_g of one group of k panels (kb = k b columns of V, m rows; Tp = the
// panels' b x b factors back to back): T_g = [[T_A, -T_A (V_A^T V_B) T_B],
// [0, T_B]] by pairwise merging, bottom-up: blocks A = [a0, a0+h), B =
// [a0+h, a0+h+hb) of an already merged level combine as T_AB = -T_A X_AB T_B
// with X = V^T V (strict block-upper part, one product per group).  VT
// (optional, m x kb): V T_g.
cudaError_t q1_group_build(int k, int b, int m, const double* V, long long ldv, const double* Tp,
                           double* Tg, double* VT, const Q1Scratch& w, cudaStream_t s) {
  const int kb = k * b;
  cudaError_t e;
  if ((e = cudaMemsetAsync(Tg, 0, sizeof(double) * kb * kb, s)) != cudaSuccess) return e;
  for (int j = 0; j < k; ++j) {
    if ((e = cudaMemcpy2DAsync(Tg + (long long)j * b + (long long)j * b * kb, kb * sizeof(double),
                               Tp + (size_t)j * b * b, b * sizeof(double), b * sizeof(double), b,
                               cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return e;
  }
  if (k > 1) {
    GemmProblem gx = make_gemm(kb, kb, m, 1.0, V, ldv, V, ldv, 0.0, w.x, kb);
    gx.mc = Mask::strict_upper();  // covers every block above the diagonal blocks
    if (w.oz_side && (double)kb * kb * m >= oz_min_work())
      e = ozgemm(true, false, gx, w.oz_side, w.oz_side_bytes, kQ1OzChunk, s);
    else
      e = gemm(true, false, gx, s);
    if (e != cudaSuccess) return e;
  }
  for (int h = b; h < kb; h *= 2) {
    for (int a0 = 0; a0 + h < kb; a0 += 2 * h) {
      const int c0 = a0 + h, hb = std::min(h, kb - c0);
      // tmp = T_A X_AB   (h x hb)
      GemmProblem g1 = make_gemm(h, hb, h, 1.0, Tg + a0 + (long long)a0 * kb, kb,
                                 w.x + a0 + (long long)c0 * kb, kb, 0.0, w.tmp, h);
      g1.ma = Mask::upper();
      if ((e = gemm(false, false, g1, s)) != cudaSuccess) return e;
      // T_g[A, B] = -tmp T_B
      GemmProblem g2 = make_gemm(h, hb, hb, -1.0, w.tmp, h, Tg + c0 + (long long)c0 * kb, kb,
                                 0.0, Tg + a0 + (long long)c0 * kb, kb);
      g2.mb = Mask::upper();
      if ((e = gemm(false, false, g2, s)) != cudaSuccess) return e;
    }
  }
  if (VT) {
    // V T_g once per group here (off the critical path), so the apply is two
    // products instead of three
    GemmProblem gv = make_gemm(m, kb, kb, 1.0, V, ldv, Tg, kb, 0.0, VT, m);
    gv.mb = Mask::upper();
    if (w.oz_side && (double)m * kb * kb >= oz_min_work())
      e = ozgemm(false, false, gv, w.oz_side, w.oz_side_bytes, kQ1OzChunk, s);
    else
      e = gemm(false, false, gv, s);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Zs (m x ncols) <- (I - V T_g V^T) Zs for one group.
cudaError_t q1_group_apply(int kb, int m, const double* V, long long ldv, const double* Tg,
                           const double* VT, double* Zs, long long ldz, int ncols,
                           const Q1Scratch& w, cudaStream_t s) {
  cudaError_t e;
  // one product on the INT8 engine when it is large enough to pay for the
  // slicing and reconstruction passes
  auto mul = [&](bool ta, const GemmProblem& g) {
    if (w.oz && (double)g.M * g.N * g.K >= oz_min_work())
      return ozgemm(ta, false, g, w.oz, w.oz_bytes, kQ1OzChunk, s);
    return gemm(ta, false, g, s);
  };
  // Y = V^T Zs (kb x ncols)
  GemmProblem g3 = make_gemm(kb, ncols, m, 1.0, V, ldv, Zs, ldz, 0.0, w.y, kb);
  if ((e = mul(true, g3)) != cudaSuccess) return e;
  if (VT) {
    // Zs -= (V T_g) Y
    GemmProblem g5 = make_gemm(m, ncols, kb, -1.0, VT, m, w.y, kb, 1.0, Zs, ldz);
    return mul(false, g5);
  }
  // Y2 = T_g Y; Zs -= V Y2
  GemmProblem g4 = make_gemm(kb, ncols, kb, 1.0, Tg, kb, w.y, kb, 0.0, w.y2, kb);
  g4.ma = Mask::upper();
  if ((e = mul(false, g4)) != cudaSuccess) return e;
  GemmProblem g5 = make_gemm(m, ncols, kb, -1.0, V, ldv, w.y2, kb, 1.0, Zs, ldz);
  return mul(false, g5);
}

cudaError_t q1_build(int n, int b, const double* Vall, long long ldv, const double* Tall,
                     const Q1Scratch& w, cudaStream_t s) {
  // Panels are merged in groups of w.group (compact-WY of the product) so the
  // applying GEMMs run with K = group*b instead of b.  X = V^T V runs on the
  // emulated engine with its own workspace: this runs on a side stream next
  // to the divide and conquer, whose top merges use the shared one.
  // Vall must be zero outside the reflectors (syevd memsets it before SY2SB).
  const int np = q1_panels(n, b), G = w.group;
  cudaError_t e = cudaSuccess;
  double* Tg = w.tg;
  double* VT = w.vt;
  for (int pend = np; pend > 0; pend -= G) {
    const int p0 = std::max(0, pend - G), k = pend - p0, kb = k * b;
    const int r0 = (p0 + 1) * b, m = n - r0;
    const double* V = Vall + r0 + (long long)(p0 * b) * ldv;  // m x kb
    if ((e = q1_group_build(k, b, m, V, ldv, Tall + (size_t)p0 * b * b, Tg, w.vt ? VT : nullptr, w,
                            s)) != cudaSuccess)
      return e;
    if (w.vt) VT += (size_t)m * kb;
    Tg += (size_t)kb * kb;
  }
  return e;
}

cudaError_t q1_apply(int n, int b, const double* Vall, long long ldv, double* Z, long long ldz,
                     int ncols, const Q1Scratch& w, cudaStream_t s) {
  const int np = q1_panels(n, b), G = w.group;
  cudaError_t e = cudaSuccess;
  const double* Tg = w.tg;
  const double* VT = w.vt;
  for (int pend = np; pend > 0; pend -= G) {
    const int p0 = std::max(0, pend - G), k = pend - p0, kb = k * b;
    const int r0 = (p0 + 1) * b, m = n - r0;
    const double* V = Vall + r0 + (long long)(p0 * b) * ldv;  // m x kb
    if ((e = q1_group_apply(kb, m, V, ldv, Tg, w.vt ? VT : nullptr, Z + r0, ldz, ncols, w, s)) !=
        cudaSuccess)
      return e;
    if (w.vt) VT += (size_t)m * kb;
    Tg += (size_t)kb * kb;
  }
  return e;
}

}  // namespace bse
