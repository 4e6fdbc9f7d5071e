// Masked FP64 GEMM engine: DMMA.8x8x4 tiles fed by a multistage cp.async
// (LDGSTS) shared-memory pipeline.  See gemm.cuh for the contract.
#include <cstdio>
#include <cstdlib>
#include "gemm.cuh"

namespace bse {
namespace {

constexpr int kPad = 4;  // row pad (doubles): keeps half-warp fragment loads conflict-free

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB>
struct Cfg {
  static constexpr int WARPS_M = BM / WM;
  static constexpr int WARPS_N = BN / WN;
  static constexpr int NT = WARPS_M * WARPS_N * 32;
  // A: TA=false -> [BK][BM+pad] (m contiguous); TA=true -> [BM][BK+pad] (k contiguous)
  static constexpr int A_LDS = TA ? (BK + kPad) : (BM + kPad);
  static constexpr int A_ELEMS = TA ? BM * A_LDS : BK * A_LDS;
  // B: TB=true -> [BK][BN+pad] (n contiguous); TB=false -> [BN][BK+pad] (k contiguous)
  static constexpr int B_LDS = TB ? (BN + kPad) : (BK + kPad);
  static constexpr int B_ELEMS = TB ? BK * B_LDS : BN * B_LDS;
  static constexpr int STAGE = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double);
};

// Load a ROWS (contiguous) x COLS (strided) tile; element (r, c) lives at
// g[(r0 + r) + (c0 + c) * ld] and lands at s[c * LDS + r].  Out-of-range
// elements are zero-filled.
template <int ROWS, int COLS, int LDS, int VEC, int NT>
BSE_DEV void load_tile(double* s, const double* g, long long ld, int r0, int c0, int rmax,
                       int cmax, int tid) {
  constexpr int CPR = ROWS / VEC;  // chunks per strided line
  constexpr int CHUNKS = CPR * COLS;
#pragma unroll
  for (int id = tid; id < CHUNKS; id += NT) {
    const int c = id / CPR;
    const int r = (id % CPR) * VEC;
    const int gr = r0 + r, gc = c0 + c;
    double* sp = s + c * LDS + r;
    const bool cok = gc < cmax;
    const double* gp = g + (cok ? (long long)gc * ld : 0);
    if constexpr (VEC == 2) {
      const bool v0 = cok && gr < rmax, v1 = cok && gr + 1 < rmax;
      if (v0 && v1) {
        cp_async16(sp, gp + gr, true);
      } else {
        cp_async8(sp, v0 ? gp + gr : g, v0);
        cp_async8(sp + 1, v1 ? gp + gr + 1 : g, v1);
      }
    } else {
      const bool v0 = cok && gr < rmax;
      cp_async8(sp, v0 ? gp + gr : g, v0);
    }
  }
}

BSE_DEV double apply_mask(double v, int d, bool inb, const Mask& m) {
  if (m.unit && d == 0) return inb ? 1.0 : 0.0;
  return (d < m.lo || d > m.hi) ? 0.0 : v;
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB, int VEC,
          bool MASKED = true>
BSE_DEV void gemm_tile(const GemmProblem& p, int m0, int n0, double* smem) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>;
  const int M = p.M, N = p.N, K = p.K;
  if (m0 >= M || n0 >= N) return;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::WARPS_M, wn = warp / C::WARPS_M;
  const int mlast = min(m0 + BM, M) - 1, nlast = min(n0 + BN, N) - 1;

  // Output mask: skip tiles with no writable element.
  if (MASKED) {
    const long long dmin = (long long)n0 - mlast, dmax = (long long)nlast - m0;
    if (dmax < p.mc.lo || dmin > p.mc.hi) return;
  }

  // k-range implied by the operand masks.
  long long kb = 0, ke = K;
  if (MASKED) {
    const Mask& a = p.ma;
    const long long lo = a.unit ? min(a.lo, 0) : a.lo, hi = a.unit ? max(a.hi, 0) : a.hi;
    if (!TA) { kb = max(kb, (long long)m0 + lo); ke = min(ke, (long long)mlast + hi + 1); }
    else     { kb = max(kb, (long long)m0 - hi); ke = min(ke, (long long)mlast - lo + 1); }
    const Mask& b = p.mb;
    const long long blo = b.unit ? min(b.lo, 0) : b.lo, bhi = b.unit ? max(b.hi, 0) : b.hi;
    if (!TB) { kb = max(kb, (long long)n0 - bhi); ke = min(ke, (long long)nlast - blo + 1); }
    else     { kb = max(kb, (long long)n0 + blo); ke = min(ke, (long long)nlast + bhi + 1); }
  }
  kb = (kb / BK) * BK;
  const int k_begin = (int)kb;
  const int ntiles = ke > kb ? (int)ceil_div(ke - kb, BK) : 0;

  constexpr int MI = WM / 8, NJ = WN / 8;
  double acc[MI][NJ][2];
  // beta != 0 with alpha = +-1: start the accumulators at (beta/alpha) C so
  // the C read overlaps the pipeline prologue (exact for alpha = +-1)
  const bool cpre = p.beta != 0.0 && (p.alpha == 1.0 || p.alpha == -1.0) && K <= 512;
  {
    const int klq = (threadIdx.x & 31) & 3, rlq = (threadIdx.x & 31) >> 2;
    const int wmq = (threadIdx.x >> 5) % C::WARPS_M, wnq = (threadIdx.x >> 5) / C::WARPS_M;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          double v = 0.0;
          if (cpre) {
            const int gm = m0 + wmq * WM + i * 8 + rlq;
            const int gn = n0 + wnq * WN + j * 8 + klq * 2 + e;
            bool ok = gm < M && gn < N;
            if (MASKED && ok) {
              const int d = gn - gm;
              ok = d >= p.mc.lo && d <= p.mc.hi;
            }
            // raw load: the scaling by f waits until the prologue's copies
            // are in flight (below), so no warp stalls on C before them
            if (ok) v = p.C[gm + (long long)(p.ccol ? p.ccol[gn] : gn) * p.ldc];
          }
          acc[i][j][e] = v;
        }
  }
  const double cscale = cpre ? p.beta / p.alpha : 1.0;

  auto load_stage = [&](int st, int kt) {
    double* sA = smem + st * C::STAGE;
    double* sB = sA + C::A_ELEMS;
    const int k0 = k_begin + kt * BK;
    if constexpr (!TA) load_tile<BM, BK, C::A_LDS, VEC, C::NT>(sA, p.A, p.lda, m0, k0, M, K, tid);
    else               load_tile<BK, BM, C::A_LDS, VEC, C::NT>(sA, p.A, p.lda, k0, m0, K, M, tid);
    if constexpr (TB)  load_tile<BN, BK, C::B_LDS, VEC, C::NT>(sB, p.B, p.ldb, n0, k0, N, K, tid);
    else               load_tile<BK, BN, C::B_LDS, VEC, C::NT>(sB, p.B, p.ldb, k0, n0, K, N, tid);
  };

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ntiles) load_stage(s, s);
    cp_async_commit();
  }

  if (cpre && cscale != 1.0) {
    // acc = f C.  The empty volatile asm keeps these after the (volatile)
    // cp.async prologue; f = -1 (every trailing update of SY2SB / POTRF) flips
    // the sign bit on the integer pipe instead of a DMUL that would queue
    // behind the co-resident CTA's DMMAs on the FP64 pipe.
    const bool flip = cscale == -1.0;
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          asm volatile("" : "+d"(acc[i][j][e]));
          const double v = acc[i][j][e];
          acc[i][j][e] = flip ? __hiloint2double(__double2hiint(v) ^ (int)0x80000000, __double2loint(v))
                              : v * cscale;
        }
  }

  const bool maskA_on = MASKED && p.ma.active(), maskB_on = MASKED && p.mb.active();
  const int am_base = wm * WM + (lane >> 2);  // + i*8
  const int bn_base = wn * WN + (lane >> 2);  // + j*8
  const int kl = lane & 3;

  for (int kt = 0; kt < ntiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ntiles) load_stage(nk % STAGES, nk);
      cp_async_commit();
    }
    const double* sA = smem + (kt % STAGES) * C::STAGE;
    const double* sB = sA + C::A_ELEMS;
    const int k0 = k_begin + kt * BK;

    // Does this k-tile straddle a mask boundary?
    bool needA = false, needB = false;
    if (maskA_on) {
      const Mask& a = p.ma;
      long long dmin, dmax;
      if (!TA) { dmin = (long long)k0 - mlast; dmax = (long long)k0 + BK - 1 - m0; }
      else     { dmin = (long long)m0 - (k0 + BK - 1); dmax = (long long)mlast - k0; }
      needA = dmin < a.lo || dmax > a.hi || (a.unit && dmin <= 0 && dmax >= 0);
    }
    if (maskB_on) {
      const Mask& b = p.mb;
      long long dmin, dmax;
      if (!TB) { dmin = (long long)n0 - (k0 + BK - 1); dmax = (long long)nlast - k0; }
      else     { dmin = (long long)k0 - nlast; dmax = (long long)k0 + BK - 1 - n0; }
      needB = dmin < b.lo || dmax > b.hi || (b.unit && dmin <= 0 && dmax >= 0);
    }

#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[MI], bf[NJ];
#pragma unroll
      for (int i = 0; i < MI; ++i) {
        const int ml = am_base + i * 8, kq = kk + kl;
        af[i] = TA ? sA[ml * C::A_LDS + kq] : sA[kq * C::A_LDS + ml];
      }
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const int nl = bn_base + j * 8, kq = kk + kl;
        bf[j] = TB ? sB[kq * C::B_LDS + nl] : sB[nl * C::B_LDS + kq];
      }
      if (needA) {
#pragma unroll
        for (int i = 0; i < MI; ++i) {
          const int gm = m0 + am_base + i * 8, gk = k0 + kk + kl;
          const int d = TA ? gm - gk : gk - gm;
          af[i] = apply_mask(af[i], d, gm < M && gk < K, p.ma);
        }
      }
      if (needB) {
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          const int gn = n0 + bn_base + j * 8, gk = k0 + kk + kl;
          const int d = TB ? gk - gn : gn - gk;
          bf[j] = apply_mask(bf[j], d, gn < N && gk < K, p.mb);
        }
      }
#pragma unroll
      for (int i = 0; i < MI; ++i)
#pragma unroll
        for (int j = 0; j < NJ; ++j) dmma8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // Epilogue: C = alpha*acc + beta*C under the output mask.
  const double alpha = p.alpha, beta = p.beta;
#pragma unroll
  for (int i = 0; i < MI; ++i) {
    const int gm = m0 + wm * WM + i * 8 + (lane >> 2);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int gn = n0 + wn * WN + j * 8 + kl * 2 + e;
        if (gn >= N) continue;
        if (MASKED) {
          const int d = gn - gm;
          if (d < p.mc.lo || d > p.mc.hi) continue;
        }
        double* cp = p.C + gm + (long long)(p.ccol ? p.ccol[gn] : gn) * p.ldc;
        double v = alpha * acc[i][j][e];
        if (beta != 0.0 && !cpre) v += beta * *cp;
        *cp = v;
        if (p.mirror && gn < gm) p.C[gn + (long long)gm * p.ldc] = v;
      }
    }
  }
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB, int VEC,
          bool MASKED>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>::NT)
    gemm_single_kernel(const GemmProblem p) {
  extern __shared__ __align__(16) double smem[];
  gemm_tile<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC, MASKED>(p, blockIdx.x * BM, blockIdx.y * BN,
                                                             smem);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB, int VEC>
__global__ void __launch_bounds__(Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>::NT)
    gemm_grouped_kernel(const GemmProblem* __restrict__ probs) {
  extern __shared__ __align__(16) double smem[];
  const GemmProblem p = probs[blockIdx.z];
  gemm_tile<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC>(p, blockIdx.x * BM, blockIdx.y * BN, smem);
}

template <int BM, int BN, int BK, int WM, int WN, int STAGES, bool TA, bool TB, int VEC>
cudaError_t launch(const GemmProblem* single, const GemmProblem* grouped, int count, int maxM,
                   int maxN, cudaStream_t s) {
  using C = Cfg<BM, BN, BK, WM, WN, STAGES, TA, TB>;
  static PerDeviceOnce attr_once;  // per instantiation, per device
  if (attr_once.needed()) {
    cudaError_t e = cudaFuncSetAttribute(gemm_single_kernel<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm_single_kernel<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(gemm_grouped_kernel<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    attr_once.mark();
  }
  dim3 grid((unsigned)ceil_div(maxM, BM), (unsigned)ceil_div(maxN, BN), (unsigned)count);
  if (grid.x == 0 || grid.y == 0 || count == 0) return cudaSuccess;
  const bool masked = single && (single->ma.active() || single->mb.active() || single->mc.active());
  if (single && masked)
    gemm_single_kernel<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC, true><<<grid, C::NT, C::SMEM, s>>>(*single);
  else if (single)
    gemm_single_kernel<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC, false><<<grid, C::NT, C::SMEM, s>>>(*single);
  else
    gemm_grouped_kernel<BM, BN, BK, WM, WN, STAGES, TA, TB, VEC><<<grid, C::NT, C::SMEM, s>>>(grouped);
  count_launch();
  return cudaGetLastError();
}

template <bool TA, bool TB>
cudaError_t dispatch(int cfg, int vec, const GemmProblem* single, const GemmProblem* grouped,
                     int count, int maxM, int maxN, cudaStream_t s) {
  if (vec == 2) {
    if (cfg == 0) return launch<128, 128, 16, 64, 32, 4, TA, TB, 2>(single, grouped, count, maxM, maxN, s);
    if (cfg == 2) return launch<128, 128, 32, 64, 32, 3, TA, TB, 2>(single, grouped, count, maxM, maxN, s);
    if (cfg == 3) return launch<128, 64, 16, 32, 32, (TA ? 3 : 4), TA, TB, 2>(single, grouped, count, maxM, maxN, s);
    if (cfg == 4) return launch<128, 64, 32, 32, 32, 2, TA, TB, 2>(single, grouped, count, maxM, maxN, s);
    return launch<64, 64, 16, 32, 32, 4, TA, TB, 2>(single, grouped, count, maxM, maxN, s);
  }
  return launch<64, 64, 16, 32, 32, 4, TA, TB, 1>(single, grouped, count, maxM, maxN, s);
}

cudaError_t dispatch_all(bool ta, bool tb, int cfg, int vec, const GemmProblem* single,
                         const GemmProblem* grouped, int count, int maxM, int maxN, cudaStream_t s) {
  if (!ta && !tb) return dispatch<false, false>(cfg, vec, single, grouped, count, maxM, maxN, s);
  if (!ta && tb) return dispatch<false, true>(cfg, vec, single, grouped, count, maxM, maxN, s);
  if (ta && !tb) return dispatch<true, false>(cfg, vec, single, grouped, count, maxM, maxN, s);
  return dispatch<true, true>(cfg, vec, single, grouped, count, maxM, maxN, s);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__global__ void splitk_reduce_kernel(const double* __restrict__ ws, int splits, int M, int N,
                                     double alpha, double beta, double* C, long long ldc) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)M * N) return;
  const int r = (int)(idx % M), c = (int)(idx / M);
  double acc = 0.0;
  for (int s = 0; s < splits; ++s) acc += ws[(long long)s * M * N + idx];
  double* cp = C + r + (long long)c * ldc;
  *cp = alpha * acc + (beta != 0.0 ? beta * *cp : 0.0);
}

__global__ void splitk_setup_kernel(const GemmProblem p, bool transA, bool transB, int splits,
                                    int chunk, double* ws, GemmProblem* out) {
  const int i = threadIdx.x;
  if (i >= splits) return;
  GemmProblem q = p;
  const int k0 = i * chunk;
  q.K = min(chunk, p.K - k0);
  // op(A) is M x K -> advance along k; masks are in stored, view-relative coordinates
  q.A = transA ? p.A + k0 : p.A + (long long)k0 * p.lda;
  q.B = transB ? p.B + (long long)k0 * p.ldb : p.B + k0;
  const int da = transA ? k0 : -k0;   // shift of (c - r) for A's view
  const int db = transB ? -k0 : k0;   // ... and for B's
  if (p.ma.lo != kNoMaskLo) q.ma.lo = p.ma.lo + da;
  if (p.ma.hi != kNoMaskHi) q.ma.hi = p.ma.hi + da;
  if (p.mb.lo != kNoMaskLo) q.mb.lo = p.mb.lo + db;
  if (p.mb.hi != kNoMaskHi) q.mb.hi = p.mb.hi + db;
  q.C = ws + (long long)i * p.M * p.N;
  q.ldc = p.M;
  q.alpha = 1.0;
  q.beta = 0.0;
  q.mc = Mask{};
  out[i] = q;
}

}  // namespace

cudaError_t gemm_splitk(bool transA, bool transB, const GemmProblem& p, int splits, double* ws,
                        GemmProblem* probs_dev_scratch, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  if (splits <= 1 || p.K < 64 * splits) return gemm(transA, transB, p, s);
  if (p.ma.unit || p.mb.unit) return cudaErrorInvalidValue;  // unit diag not split-safe
  // chunk K in multiples of 16 so every slice keeps cp.async alignment
  int chunk = (int)ceil_div(p.K, splits);
  chunk = (int)ceil_div(chunk, 16) * 16;
  splits = (int)ceil_div(p.K, chunk);
  if (splits > 64) return cudaErrorInvalidValue;
  // descriptors are built on the device: no pageable H2D copy in the hot loop
  splitk_setup_kernel<<<1, 64, 0, s>>>(p, transA, transB, splits, chunk, ws, probs_dev_scratch);
  count_launch();
  const bool v2 = aligned16(p.A) && aligned16(p.B) && ((p.lda | p.ldb) & 1) == 0;
  // (64 x 64 tiles: measured faster than 128 x 64 for the thin split-K SYMM)
  static int cfg = -1;
  if (cfg < 0) {
    const char* v = std::getenv("BSE_SPLITK_CFG");  // tuning switch
    cfg = v ? std::atoi(v) : 1;
  }
  cudaError_t e = gemm_grouped(transA, transB, probs_dev_scratch, splits, p.M, p.N, s, v2, cfg);
  if (e != cudaSuccess) return e;
  const long long tot = (long long)p.M * p.N;
  splitk_reduce_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(ws, splits, p.M, p.N, p.alpha,
                                                                     p.beta, p.C, p.ldc);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gemm(bool transA, bool transB, const GemmProblem& p, cudaStream_t s) {
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  const bool v2 = aligned16(p.A) && aligned16(p.B) && ((p.lda | p.ldb) & 1) == 0;
  // 128x64 tiles, 8 warps of 32x32, 2 CTAs/SM (cfg 3) measured 32-33 TFLOP/s
  // on large FP64 GEMMs (86-90% of the DMMA peak); 64x64 for small outputs.
  // Transposed A: 128x64x32 tiles, 2 stages (measured 33.5 vs 30.7 TFLOP/s
  // for the k-contiguous A fragments of V^T Z / L^T B).
  const long long big_tiles = ceil_div(p.M, 128) * ceil_div(p.N, 64);
  int cfg = (v2 && big_tiles >= 148) ? (transA ? 4 : 3) : 1;
  static int forced = -2;
  if (forced == -2) {
    const char* v = std::getenv("BSE_GEMM_CFG");
    forced = v ? std::atoi(v) : -1;
  }
  if (forced >= 0 && (cfg == 3 || cfg == 4)) cfg = forced;
  return dispatch_all(transA, transB, cfg, v2 ? 2 : 1, &p, nullptr, 1, p.M, p.N, s);
}

cudaError_t gemm_grouped(bool transA, bool transB, const GemmProblem* probs_dev, int count,
                         int maxM, int maxN, cudaStream_t s, bool all_aligned16, int cfg) {
  // Grouped problems may mix alignments (e.g. D&C nodes at odd offsets): the
  // 8-byte path is always legal; callers that guarantee 16-byte alignment of
  // every operand and even leading dimensions get the vectorised loads.
  return dispatch_all(transA, transB, all_aligned16 ? cfg : 1, all_aligned16 ? 2 : 1, nullptr,
                      probs_dev, count, maxM, maxN, s);
}

}  // namespace bse
