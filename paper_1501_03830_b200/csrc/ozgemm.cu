// FP64 GEMM emulated on the INT8 tensor cores (Ozaki scheme II: integer
// slices + Chinese remaindering), for the large-K dense products of the solve.
//
//   C := alpha * op(A) * op(B) + beta * C       (FP64, column-major)
//
// 1. Each row i of op(A) and column j of op(B) is scaled by a power of two so
//    its largest entry lies in [2^(beta-1), 2^beta) and truncated to an
//    integer (beta <= 53 bits: exact in a double).  The integer product
//    C' = A' B' is then computed EXACTLY modulo 16 pairwise-coprime moduli
//    m_t <= 256 (product 2^125.4 > 2 |C'|):
// 2. residues A'_t, B'_t in [-128, 127] (int8, K-major), one batched
//    tcgen05 kind::i8 GEMM (CUTLASS sm_100 2-SM kernel, INT32 accumulators in
//    TMEM) gives C_t = A'_t B'_t exactly;
// 3. C' is rebuilt per element by the CRT (exact 32-bit-limb sums in FP64),
//    scaled back by 2^-(s_i + s_j) and written with alpha/beta and the output
//    mask.
// The truncation error per entry is below 2^-52 of its row (column) maximum,
// so the result is as accurate as a DGEMM for the operands it is used on
// (orthogonal / triangular factors with bounded row ranges); tests compare it
// against the DMMA engine and float64 numpy.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include "cutlass/cutlass.h"
#include "cute/tensor.hpp"
#include "cutlass/epilogue/collective/collective_builder.hpp"
#include "cutlass/gemm/collective/collective_builder.hpp"
#include "cutlass/gemm/device/gemm_universal_adapter.h"
#include "cutlass/gemm/dispatch_policy.hpp"
#include "cutlass/gemm/kernel/gemm_universal.hpp"
#include "cutlass/util/packed_stride.hpp"
#include "i8mma.cuh"
#include "ozgemm.cuh"

namespace bse {
namespace {

constexpr int kMods = 16;
// pairwise coprime (2^8, 3.5.17, 11.23, 251, 13.19, 241, 239, 233, 229, 227,
// 223, 7.31, 211, 199, 197, 193); compile-time after unrolling, so every
// "% m" below is a multiply-shift
BSE_HD constexpr int kMod(int t) {
  return t == 0 ? 256 : t == 1 ? 255 : t == 2 ? 253 : t == 3 ? 251 : t == 4 ? 247 : t == 5 ? 241
       : t == 6 ? 239 : t == 7 ? 233 : t == 8 ? 229 : t == 9 ? 227 : t == 10 ? 223
       : t == 11 ? 217 : t == 12 ? 211 : t == 13 ? 199 : t == 14 ? 197 : 193;
}

struct CrtConst {
  // Q_t = (M_t * (M_t^{-1} mod m_t)) mod P, M_t = P / m_t, as four 32-bit
  // limbs (Q_t = sum_k q[t][k] 2^(32 k)); P likewise; 1 / P
  double q[kMods][4];
  double p[4];
  double inv_p;
};
__constant__ CrtConst c_crt;

// ---------------------------------------------------------------------------
// CUTLASS sm_100 int8 x int8 -> int32, A row-major (K-major), B column-major
// (K-major), C column-major; 256x256x128 tiles on 2-SM clusters.
namespace cg = cutlass::gemm;
using namespace cute;
using MmaTile = Shape<_256, _256, _128>;
using ClusterShape = Shape<_2, _1, _1>;
using Epi = typename cutlass::epilogue::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, MmaTile, ClusterShape,
    cutlass::epilogue::collective::EpilogueTileAuto, int32_t, int32_t, int32_t,
    cutlass::layout::ColumnMajor, 4, int32_t, cutlass::layout::ColumnMajor, 4,
    cutlass::epilogue::TmaWarpSpecialized2Sm>::CollectiveOp;
using Main = typename cg::collective::CollectiveBuilder<
    cutlass::arch::Sm100, cutlass::arch::OpClassTensorOp, int8_t, cutlass::layout::RowMajor, 16,
    int8_t, cutlass::layout::ColumnMajor, 16, int32_t, MmaTile, ClusterShape,
    cg::collective::StageCountAutoCarveout<static_cast<int>(sizeof(typename Epi::SharedStorage))>,
    cg::KernelTmaWarpSpecialized2SmSm100>::CollectiveOp;
using Kernel = cg::kernel::GemmUniversal<Shape<int, int, int, int>, Main, Epi>;
using I8Gemm = cg::device::GemmUniversalAdapter<Kernel>;

cudaError_t i8_gemm_batched(int M, int N, int K, int L, const int8_t* A, const int8_t* B,
                            int32_t* C, cudaStream_t s) {
  auto sA = cutlass::make_cute_packed_stride(typename Kernel::StrideA{}, {M, K, L});
  auto sB = cutlass::make_cute_packed_stride(typename Kernel::StrideB{}, {N, K, L});
  auto sC = cutlass::make_cute_packed_stride(typename Kernel::StrideC{}, {M, N, L});
  auto sD = cutlass::make_cute_packed_stride(typename Kernel::StrideD{}, {M, N, L});
  typename I8Gemm::Arguments args{cg::GemmUniversalMode::kGemm, {M, N, K, L}, {A, sA, B, sB},
                                  {{1, 0}, C, sC, C, sD}};
  I8Gemm gemm;
  if (gemm.can_implement(args) != cutlass::Status::kSuccess) return cudaErrorInvalidValue;
  if (I8Gemm::get_workspace_size(args) != 0) return cudaErrorInvalidValue;
  if (gemm.initialize(args, nullptr, s) != cutlass::Status::kSuccess) return cudaErrorInvalidValue;
  if (gemm.run(s) != cutlass::Status::kSuccess) return cudaErrorLaunchFailure;
  count_launch();
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Slicing.  "Line" r of an operand is a row of op(A) or a column of op(B);
// it is written K-contiguous as 16 int8 residue rows out[t][r][0..Kp).
// Stored element of line r, position k:
//   contiguous: src[r * ld + k], stored coordinates (row, col) = (k, r)
//   strided:    src[r + k * ld], stored coordinates (row, col) = (r, k)

BSE_DEV double masked(double v, int row, int col, const Mask& m) {
  const int d = col - row;
  if (m.unit && d == 0) return 1.0;
  return (d < m.lo || d > m.hi) ? 0.0 : v;
}

// x * 2^k: one multiply by an exactly built power of two in the normal range
// (the common case), ldexp otherwise
BSE_DEV double scale2(double x, int k) {
  if (k >= -1020 && k <= 1020) return x * __longlong_as_double((long long)(k + 1023) << 52);
  return ldexp(x, k);
}

// scale exponent so that max |x| * 2^s lies in [2^(beta-1), 2^beta)
BSE_DEV int scale_exp(double mx, int beta) {
  if (!(mx > 0.0)) return 0;
  int e;
  frexp(mx, &e);  // mx = f 2^e, f in [0.5, 1)
  return beta - e;
}

// Residues of 4 integer-valued doubles (|x| < 2^53) for all 16 moduli,
// packed 4 per word (byte q = element q).  The moduli are reduced in pairs:
// r = x mod (m_a m_b) in FP64 (|r| < 1.5 m_a m_b < 2^17, exact), then both
// residues of the small non-negative integer r + 2 m_a m_b on the integer
// pipe (unsigned division by a constant), stored as int8 representatives
// centred in [-128, m - 128).
BSE_DEV uint32_t byte8(uint32_t u1, uint32_t m) {
  // u1 = u + 128 < 2^24: q = floor(u1 c / 2^32), c = ceil(2^32 / m), is exact
  // because u1 (c m - 2^32) < 2^24 m < 2^32.  (u1 mod m) - 128 is the
  // residue of u centred in [-128, m - 128) (no compare); as a byte that is
  // (u1 mod m) ^ 0x80.
  const uint32_t c = (uint32_t)((0x100000000ull + m - 1) / m);
  return (u1 - __umulhi(u1, c) * m) ^ 0x80u;
}

BSE_DEV void residues_all(const double (&x)[4], uint32_t (&w)[kMods]) {
#pragma unroll
  for (int t = 0; t < kMods; ++t) w[t] = 0;
#pragma unroll
  for (int pr = 0; pr < kMods / 2; ++pr) {
    constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
    const uint32_t ma = kMod(2 * pr), mb = kMod(2 * pr + 1);
    const double mp = (double)(ma * mb), inv = 1.0 / mp;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const double r = fma(-rint(x[q] * inv), mp, x[q]);
      const uint32_t u1 = (uint32_t)__double2loint(r + kMagic) + 2u * ma * mb + 128u;
      w[2 * pr] |= byte8(u1, ma) << (8 * q);
      w[2 * pr + 1] |= byte8(u1, mb) << (8 * q);
    }
  }
}

// Contiguous source: kSplitWPL warps per line (each a contiguous K range,
// so a line's loads are spread over several warps in flight), 256 / (32 *
// kSplitWPL) lines per CTA; the line maximum is combined in shared memory.
constexpr int kSplitWPL = 4;
constexpr int kSplitLPC = 256 / (32 * kSplitWPL);
__global__ void __launch_bounds__(256) split_contig_kernel(int lines, int K, int Kp,
                                                           const double* __restrict__ src,
                                                           long long ld, Mask mk, int beta,
                                                           int8_t* __restrict__ out,
                                                           long long mod_stride,
                                                           int* __restrict__ sexp) {
  __shared__ double smx[kSplitLPC][kSplitWPL];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ll = wid / kSplitWPL, part = wid % kSplitWPL;
  const int r = blockIdx.x * kSplitLPC + ll;
  const int rows_alloc = (int)(mod_stride / Kp);
  const bool alloc = r < rows_alloc;
  const bool live = r < lines;
  const double* row = src + (long long)(live ? r : 0) * ld;
  // this warp's K range: a multiple of 128 elements
  const int span = ((Kp + 128 * kSplitWPL - 1) / (128 * kSplitWPL)) * 128;
  const int kb = part * span, ke = min(Kp, kb + span);
  double mx = 0.0;
  if (live)
    for (int k = kb + lane; k < min(K, ke); k += 32) mx = fmax(mx, fabs(masked(row[k], k, r, mk)));
  mx = warp_max(mx);
  if (lane == 0) smx[ll][part] = mx;
  __syncthreads();
  if (!alloc) return;
  mx = smx[ll][0];
#pragma unroll
  for (int q = 1; q < kSplitWPL; ++q) mx = fmax(mx, smx[ll][q]);
  const int se = scale_exp(mx, beta);
  if (lane == 0 && part == 0) sexp[r] = se;
  uint32_t* o = reinterpret_cast<uint32_t*>(out + (long long)r * Kp);
  for (int k0 = kb + 4 * lane; k0 < ke; k0 += 128) {
    double x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = k0 + q;
      x[q] = (live && k < K) ? trunc(scale2(masked(row[k], k, r, mk), se)) : 0.0;
    }
    uint32_t w[kMods];
    residues_all(x, w);
#pragma unroll
    for (int t = 0; t < kMods; ++t) o[t * (mod_stride / 4) + k0 / 4] = w[t];
  }
}

// Strided source: line maxima first (thread per line, k split over gridDim.y).
__global__ void strided_max_kernel(int lines, int K, const double* __restrict__ src, long long ld,
                                   Mask mk, unsigned long long* __restrict__ mx_bits) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= lines) return;
  const int kc = (K + gridDim.y - 1) / gridDim.y;
  const int k0 = blockIdx.y * kc, k1 = min(K, k0 + kc);
  double mx = 0.0;
  for (int k = k0; k < k1; ++k) mx = fmax(mx, fabs(masked(src[r + (long long)k * ld], r, k, mk)));
  atomicMax(mx_bits + r, (unsigned long long)__double_as_longlong(mx));
}

// 64 lines x 64 k per CTA: coalesced loads along lines into shared memory,
// residues written K-contiguous.
__global__ void __launch_bounds__(256) split_strided_kernel(int lines, int K, int Kp,
                                                            const double* __restrict__ src,
                                                            long long ld, Mask mk, int beta,
                                                            const unsigned long long* __restrict__ mx_bits,
                                                            int8_t* __restrict__ out,
                                                            long long mod_stride,
                                                            int* __restrict__ sexp) {
  __shared__ double tile[64][65];  // [k][line]
  __shared__ int se_s[64];
  const int r0 = blockIdx.x * 64, k0 = blockIdx.y * 64, tid = threadIdx.x;
  if (tid < 64) {
    const int r = r0 + tid;
    const double mx = r < lines ? __longlong_as_double((long long)mx_bits[r]) : 0.0;
    se_s[tid] = scale_exp(mx, beta);
    if (blockIdx.y == 0 && (long long)r * Kp < mod_stride) sexp[r] = se_s[tid];
  }
  __syncthreads();
  for (int idx = tid; idx < 64 * 64; idx += 256) {
    const int rl = idx & 63, kl = idx >> 6;
    const int r = r0 + rl, k = k0 + kl;
    double v = 0.0;
    if (r < lines && k < K) v = trunc(scale2(masked(src[r + (long long)k * ld], r, k, mk), se_s[rl]));
    tile[kl][rl] = v;
  }
  __syncthreads();
  // thread -> (line, 4 consecutive k)
  for (int idx = tid; idx < 64 * 16; idx += 256) {
    const int rl = idx >> 4, kq = (idx & 15) * 4;
    const int r = r0 + rl, k = k0 + kq;
    if ((long long)r * Kp >= mod_stride || k >= Kp) continue;
    double x[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) x[q] = tile[kq + q][rl];
    uint32_t* o = reinterpret_cast<uint32_t*>(out + (long long)r * Kp + k);
    uint32_t w[kMods];
    residues_all(x, w);
#pragma unroll
    for (int t = 0; t < kMods; ++t) o[t * (mod_stride / 4)] = w[t];
  }
}

// ---------------------------------------------------------------------------
// CRT reconstruction.


// C' = sum_t v_t Q_t mod P with v_t = c_t mod m_t in [0, m_t): every
// v_t q[t][k] < 2^40, so the four limb sums A_k (< 2^44) are exact in FP64;
// the quotient q = rint(S / P) (|q| < 2^12) comes from the top limbs and
// R_k = A_k - q p_k is exact, leaving one rounding per limb addition.
// One thread per 4 consecutive rows of one column: 16-byte loads of every
// residue plane (Mp % 16 == 0 keeps them aligned), 4 independent CRTs.
__global__ void __launch_bounds__(256) crt_kernel(int M, int N, int Mp, const int32_t* __restrict__ c32,
                                                  long long batch, const int* __restrict__ sa,
                                                  const int* __restrict__ sb, double alpha,
                                                  double beta, double* __restrict__ C,
                                                  long long ldc, int col0, Mask mc,
                                                  const int* __restrict__ ccol) {
  const int M4 = (M + 3) >> 2;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)M4 * N) return;
  const int i0 = (int)(idx % M4) * 4, j = (int)(idx / M4);
  const int dj = col0 + j;
  // rows i0..i0+3 all outside the output band: nothing to do
  if (dj - (i0 + 3) > mc.hi || dj - i0 < mc.lo) return;
  const int4* p = reinterpret_cast<const int4*>(c32 + i0 + (long long)j * Mp);
  const long long b4 = batch >> 2;
  double a[4][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) a[e][0] = a[e][1] = a[e][2] = a[e][3] = 0.0;
#pragma unroll
  for (int t = 0; t < kMods; ++t) {
    const uint32_t m = kMod(t);
    // c_t + 2^31 - (2^31 mod m) >= 0 has the residue of c_t (|c_t| < 2^31 - 256)
    const uint32_t off = 0x80000000u - (0x80000000u % m);
    const int4 c4 = __ldcs(p + t * b4);
    const int cv[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t v = ((uint32_t)cv[e] + off) % m;
      const double dv = __hiloint2double(0x43300000, (int)v) - 4503599627370496.0;  // 2^52
      a[e][0] = fma(dv, c_crt.q[t][0], a[e][0]);
      a[e][1] = fma(dv, c_crt.q[t][1], a[e][1]);
      a[e][2] = fma(dv, c_crt.q[t][2], a[e][2]);
      a[e][3] = fma(dv, c_crt.q[t][3], a[e][3]);
    }
  }
  constexpr double k32 = 4294967296.0, k64 = k32 * k32, k96 = k64 * k32;
  double* cd = C + (long long)(ccol ? ccol[dj] : dj) * ldc;
  const int sj = sb[j];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int i = i0 + e;
    const int d = dj - i;
    if (i >= M || d < mc.lo || d > mc.hi) continue;
    const double q = rint(fma(a[e][3], k96, fma(a[e][2], k64, a[e][1] * k32)) * c_crt.inv_p);
    const double r0 = fma(-q, c_crt.p[0], a[e][0]), r1 = fma(-q, c_crt.p[1], a[e][1]);
    const double r2 = fma(-q, c_crt.p[2], a[e][2]), r3 = fma(-q, c_crt.p[3], a[e][3]);
    const double cp = ((r3 * k96 + r2 * k64) + r1 * k32) + r0;
    double v = alpha * scale2(cp, -(sa[i] + sj));
    if (beta != 0.0) v += beta * cd[i];
    cd[i] = v;
  }
}

// The same reconstruction from the byte planes written by the hand-written
// tcgen05 kernel (i8mma.cu): v_t = R[t][j][i] in [0, m_t) already reduced, one
// 32-bit word per plane holds rows i0..i0+3 of column j.
__global__ void __launch_bounds__(256) crt8_kernel(int M, int N, const uint8_t* __restrict__ r8,
                                                   long long ldr, long long plane,
                                                   const int* __restrict__ sa,
                                                   const int* __restrict__ sb, double alpha,
                                                   double beta, double* __restrict__ C,
                                                   long long ldc, int col0, Mask mc,
                                                   const int* __restrict__ ccol) {
  const int M4 = (M + 3) >> 2;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)M4 * N) return;
  const int i0 = (int)(idx % M4) * 4, j = (int)(idx / M4);
  const int dj = col0 + j;
  if (dj - (i0 + 3) > mc.hi || dj - i0 < mc.lo) return;
  const uint8_t* p = r8 + (long long)j * ldr + i0;
  double a[4][4];
#pragma unroll
  for (int e = 0; e < 4; ++e) a[e][0] = a[e][1] = a[e][2] = a[e][3] = 0.0;
#pragma unroll
  for (int t = 0; t < kMods; ++t) {
    const uint32_t w = __ldcs(reinterpret_cast<const uint32_t*>(p + t * plane));
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t v = (w >> (8 * e)) & 0xFFu;
      const double dv = __hiloint2double(0x43300000, (int)v) - 4503599627370496.0;  // 2^52
      a[e][0] = fma(dv, c_crt.q[t][0], a[e][0]);
      a[e][1] = fma(dv, c_crt.q[t][1], a[e][1]);
      a[e][2] = fma(dv, c_crt.q[t][2], a[e][2]);
      a[e][3] = fma(dv, c_crt.q[t][3], a[e][3]);
    }
  }
  constexpr double k32 = 4294967296.0, k64 = k32 * k32, k96 = k64 * k32;
  double* cd = C + (long long)(ccol ? ccol[dj] : dj) * ldc;
  const int sj = sb[j];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int i = i0 + e;
    const int d = dj - i;
    if (i >= M || d < mc.lo || d > mc.hi) continue;
    const double q = rint(fma(a[e][3], k96, fma(a[e][2], k64, a[e][1] * k32)) * c_crt.inv_p);
    const double r0 = fma(-q, c_crt.p[0], a[e][0]), r1 = fma(-q, c_crt.p[1], a[e][1]);
    const double r2 = fma(-q, c_crt.p[2], a[e][2]), r3 = fma(-q, c_crt.p[3], a[e][3]);
    const double cp = ((r3 * k96 + r2 * k64) + r1 * k32) + r0;
    double v = alpha * scale2(cp, -(sa[i] + sj));
    if (beta != 0.0) v += beta * cd[i];
    cd[i] = v;
  }
}

// Contraction engine: 0 = hand-written tcgen05 kernel on CTA pairs (default),
// 1 = the same on single CTAs, 2 = the CUTLASS kernel with INT32 planes (kept
// for A/B measurements: BSE_OZ_ENGINE).
std::atomic<int> g_oz_engine{-1};
int oz_engine() {
  int v = g_oz_engine.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("BSE_OZ_ENGINE");
    v = e ? std::atoi(e) : 0;
    if (v < 0 || v > 2) v = 0;
    g_oz_engine.store(v, std::memory_order_relaxed);
  }
  return v;
}

long long r16(long long x) { return (x + 15) / 16 * 16; }

bool g_const_ready[64] = {};

cudaError_t init_const() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && g_const_ready[dev]) return cudaSuccess;
  CrtConst h{};
  // exact integer arithmetic: P < 2^126 fits in 128 bits
  using u128 = unsigned __int128;
  auto limbs = [](u128 x, double (&out)[4]) {
    for (int k = 0; k < 4; ++k) out[k] = (double)(uint32_t)(x >> (32 * k));
  };
  u128 P = 1;
  for (int t = 0; t < kMods; ++t) P *= (u128)kMod(t);
  limbs(P, h.p);
  h.inv_p = 1.0 / (double)P;
  for (int t = 0; t < kMods; ++t) {
    const u128 m = (u128)kMod(t), Mt = P / m;
    const unsigned long long mt_mod = (unsigned long long)(Mt % m);
    unsigned long long y = 1;
    while ((mt_mod * y) % kMod(t) != 1) ++y;
    // Q_t = M_t y mod P = M_t (y mod m): y < m, so M_t y < P m fits in 128 bits
    limbs((Mt * (u128)y) % P, h.q[t]);
  }
  cudaError_t e = cudaMemcpyToSymbol(c_crt, &h, sizeof(h));
  if (e == cudaSuccess && dev >= 0 && dev < 64) g_const_ready[dev] = true;
  return e;
}

}  // namespace

double oz_min_work() {
  static const double v = [] {
    const char* e = std::getenv("BSE_OZ_MIN_WORK_LOG2");
    return std::ldexp(1.0, e ? std::atoi(e) : 34);
  }();
  return v;
}

int oz_set_engine(int engine) {
  const int prev = oz_engine();
  if (engine >= 0 && engine <= 2) g_oz_engine.store(engine, std::memory_order_relaxed);
  return prev;
}

// Residue planes of one column chunk: one byte per entry and modulus (row
// stride rounded to 32) from the hand-written kernel, INT32 for the CUTLASS
// A/B engine (the engine must not change between sizing and use).
static size_t plane_bytes(long long Mp, long long Np) {
  // sized for INT32 planes on every engine: the byte planes of the hand-written
  // kernel use a quarter of it.  (Shrinking it to the byte size changed the
  // layout of every workspace carved after an emulated-engine buffer, and
  // the cfg2 bench then hung in 3 of 10 runs -- some buffer downstream
  // evidently relies on this slack; not root-caused, so the size stays.)
  (void)oz_engine;
  return (size_t)kMods * Mp * Np * 4;
}

size_t ozgemm_bytes(int M, int N, int K, int chunk) {
  const long long Mp = r16(M), Kp = r16(K), Np = r16(std::min(N, chunk));
  const size_t a8 = (size_t)kMods * Mp * Kp, b8 = (size_t)kMods * Np * Kp;
  return a8 + b8 + plane_bytes(Mp, Np) + 8 * (size_t)(Mp + Np) * 2 + 4096;
}

namespace {
// BSE_OZ_TRACE=1: per-kernel CUDA-event times of every ozgemm call on stderr
// (synchronises the stream; diagnostics only).
struct OzTrace {
  bool on;
  cudaStream_t s;
  cudaEvent_t ev[64];
  const char* name[64];
  int n = 0;
  explicit OzTrace(cudaStream_t st) : s(st) {
    static const bool env = std::getenv("BSE_OZ_TRACE") != nullptr;
    on = env;
  }
  void mark(const char* what) {
    if (!on || n >= 64) return;
    cudaEventCreate(&ev[n]);
    cudaEventRecord(ev[n], s);
    name[n++] = what;
  }
  ~OzTrace() {
    if (!on || n == 0) return;
    cudaStreamSynchronize(s);
    std::fprintf(stderr, "[oz]");
    for (int i = 0; i + 1 < n; ++i) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
      std::fprintf(stderr, " %s %.3f", name[i], ms);
    }
    std::fprintf(stderr, "\n");
    for (int i = 0; i < n; ++i) cudaEventDestroy(ev[i]);
  }
};
}  // namespace

cudaError_t ozgemm(bool transA, bool transB, const GemmProblem& p, void* work, size_t work_bytes,
                   int chunk, cudaStream_t s, bool reuse_a) {
  OzTrace tr(s);
  if (p.M <= 0 || p.N <= 0) return cudaSuccess;
  cudaError_t e;
  if ((e = init_const()) != cudaSuccess) return e;
  const int M = p.M, K = p.K;
  const long long Mp = r16(M), Kp = r16(std::max(K, 1));
  const int nc_max = std::min(p.N, chunk);
  const long long Np = r16(nc_max);
  if (work_bytes < ozgemm_bytes(M, p.N, K, chunk)) return cudaErrorInvalidValue;
  // op(A)'s residues and row exponents first: their offsets depend on M and K
  // only, so a reuse_a call with a narrower last column chunk finds them
  char* w = static_cast<char*>(work);
  int8_t* a8 = reinterpret_cast<int8_t*>(w);
  w += (size_t)kMods * Mp * Kp;
  unsigned long long* mxa = reinterpret_cast<unsigned long long*>(w);
  w += 8 * (size_t)Mp;
  int* sa = reinterpret_cast<int*>(w);
  w += 8 * (size_t)Mp;
  int8_t* b8 = reinterpret_cast<int8_t*>(w);
  w += (size_t)kMods * Np * Kp;
  int32_t* c32 = reinterpret_cast<int32_t*>(w);
  w += plane_bytes(Mp, Np);
  unsigned long long* mxb = reinterpret_cast<unsigned long long*>(w);
  w += 8 * (size_t)Np;
  int* sb = reinterpret_cast<int*>(w);
  // fixed-point width: 2 beta + log2 K + 2 < log2 P (125.4)
  int lk = 0;
  while ((1LL << lk) < K) ++lk;
  const int beta = std::min(53, (123 - lk) / 2);
  auto split = [&](bool contiguous, int lines, const double* src, long long ld, Mask mk,
                   int8_t* out, long long rows_alloc, int* sexp, unsigned long long* mxbuf) {
    const long long mstride = rows_alloc * Kp;
    if (contiguous) {
      const unsigned blocks = (unsigned)ceil_div(rows_alloc, kSplitLPC);
      split_contig_kernel<<<blocks, 256, 0, s>>>(lines, K, (int)Kp, src, ld, mk, beta, out,
                                                 mstride, sexp);
      count_launch();
    } else {
      cudaMemsetAsync(mxbuf, 0, 8 * (size_t)rows_alloc, s);
      const int ysplit = (int)std::min<long long>(64, std::max<long long>(1, K / 256));
      strided_max_kernel<<<dim3((unsigned)ceil_div(lines, 256), ysplit), 256, 0, s>>>(
          lines, K, src, ld, mk, mxbuf);
      split_strided_kernel<<<dim3((unsigned)ceil_div(rows_alloc, 64), (unsigned)ceil_div(Kp, 64)),
                             256, 0, s>>>(lines, K, (int)Kp, src, ld, mk, beta, mxbuf, out, mstride,
                                          sexp);
      count_launch(2);
    }
    return cudaGetLastError();
  };
  // op(A) rows: stored A is M x K (transA false: strided lines) or K x M (contiguous)
  tr.mark("split_a");
  if (!reuse_a && (e = split(transA, M, p.A, p.lda, p.ma, a8, Mp, sa, mxa)) != cudaSuccess) return e;
  for (int j0 = 0; j0 < p.N; j0 += nc_max) {
    const int nc = std::min(nc_max, p.N - j0);
    const long long ncp = r16(nc);
    // op(B) columns: stored B is K x N (transB false: contiguous lines) or N x K.
    // Masks are view-relative to the stored matrix: shift by the chunk offset.
    Mask mb = p.mb;
    const double* bsrc;
    if (!transB) {
      bsrc = p.B + (long long)j0 * p.ldb;
      if (mb.lo != kNoMaskLo) mb.lo -= j0;
      if (mb.hi != kNoMaskHi) mb.hi -= j0;
    } else {
      bsrc = p.B + j0;
      if (mb.lo != kNoMaskLo) mb.lo += j0;
      if (mb.hi != kNoMaskHi) mb.hi += j0;
    }
    tr.mark("split_b");
    if ((e = split(!transB, nc, bsrc, p.ldb, mb, b8, ncp, sb, mxb)) != cudaSuccess) return e;
    tr.mark("mma");
    const long long tot = (long long)((M + 3) / 4) * nc;
    if (oz_engine() == 2) {
      if ((e = i8_gemm_batched((int)Mp, (int)ncp, (int)Kp, kMods, a8, b8, c32, s)) != cudaSuccess)
        return e;
      tr.mark("crt");
      crt_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(M, nc, (int)Mp, c32, Mp * ncp, sa, sb,
                                                             p.alpha, p.beta, p.C, p.ldc, j0, p.mc,
                                                             p.ccol);
    } else {
      // byte planes R[t][j][i] in the c32 region (a quarter of it)
      uint8_t* r8 = reinterpret_cast<uint8_t*>(c32);
      const long long ldr = (M + 31) / 32 * 32;
      if ((e = i8mma_residues(M, nc, (int)Kp, a8, Mp, b8, ncp, r8, ldr, j0, p.mc.lo, p.mc.hi,
                              oz_engine() == 0, s)) != cudaSuccess)
        return e;
      tr.mark("crt");
      crt8_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(M, nc, r8, ldr, ncp * ldr, sa, sb,
                                                              p.alpha, p.beta, p.C, p.ldc, j0, p.mc,
                                                              p.ccol);
    }
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  tr.mark("end");
  return cudaSuccess;
}

}  // namespace bse
