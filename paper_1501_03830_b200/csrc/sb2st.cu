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
__constant__ int c_sb_trace_s0;  // first traced sweep (BSE_SB2ST_TRACE)

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

// ---------------------------------------------------------------------------
// Fused step (default).  One step of sweep s works on the lq x lq symmetric
// block D at (q0, q0) and the lq x lp block O at (q0, p0) below the previous
// block, with v/tau the previous step's reflector:
//   A: w  = tau O v                          (right apply O' = O - w v^T)
//   B: vn = house(O'[:, 0])                   (every warp, redundantly)
//   C: t  = taun D vn, y = taun (O^T vn - v (w^T vn))
//   D: O'' = O - w v^T - vn y^T, D'' = D - vn w2^T - w2 vn^T, w2 = t - (taun/2)(t^T vn) vn
// Step 0 is the same step with O = column s (lp = 1) and tau = 0.
//
// Cross-sweep protocol (two counters per sweep).  Step j of sweep s reads,
// from sweep s-1, only D's last row and O(lq-1, lp-1) as written by its step
// j+1 -- exactly that step's row-0 outputs -- and everything else as left by
// its step j.  So each step publishes its row 0 first on `late` (warp 0),
// then every warp stores its share of the bulk and counts itself on `full`
// after its own fence.  A consumer issues
// the bulk staging as soon as `full` allows and overlaps it with the wait for
// `late`.
//
// Band layout: ldab = 2b + 1, so element (i, j) sits at linear 128 j + i and
// every block is a plain 2-D tile with a 1 KB stride: staging and stores use
// 16-byte accesses on rows with (q0 + r) even.  Shared blocks use an even
// leading dimension (66) shifted by q0 & 1 so the parities line up, and the
// matvec index patterns below are bank-conflict free for that stride.
constexpr int kLd2 = 66;
constexpr int kPairSlots = 34;  // 16-byte row-pair slots per column (33 used)
constexpr int kBulkWarps = kSbThreads / 32;  // every warp stores part of the bulk

struct SbfSmem {
  double D[2][kMaxPanel * kLd2 + 2];  // double-buffered: step j+1 stages while j computes
  double O[2][kMaxPanel * kLd2 + 2];
  double vbuf[2][kMaxPanel];
  double vnw[kSbThreads / 32][kMaxPanel];
  double w[kMaxPanel];
  double y[kMaxPanel];
  double tt[kMaxPanel];
};

// phase A (lanes: 4 rows x 4 quarters per half-warp) column pattern
BSE_DEV int colA(int q, int i) { return 8 * (i >> 1) + 2 * q + (i & 1); }
// phase C (lanes: 4 columns x 4 quarters per half-warp) row pattern
BSE_DEV int rowC(int q, int i) { return 16 * (i >> 2) + 2 * (i & 3) + (q & 1) + 8 * (q >> 1); }

// Acquire-poll one counter (thread 0).  No barrier.
BSE_DEV void poll_counter(const int* ctr, int need) {
  if (ld_relaxed(ctr) < need) {
    while (ld_relaxed(ctr) < need) {
    }
  }
  if (!(c_sb_flags & 32)) fence_acquire();
}

// 16-byte L2-only async copy of `bytes` (0, 8 or 16) with zero fill: band
// lines never enter L1, so no stale-L1 hazard across CTAs.
BSE_DEV void cp_async16_n(void* smem, const void* gmem, int bytes) {
  unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}

BSE_DEV void st_global_v2(double* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// Issue the bulk of a step's staging (everything but the late positions, which
// are loaded stale and overwritten after the late wait) into (Db, Ob), which
// are already shifted by q0 & 1.  Threads t0, t0 + nt, ... of a 256-slot grid.
BSE_DEV void stage_bulk(double* Db, double* Ob, const double* AB, int ldab, int q0, int lq, int p0,
                        int lp, int t0, int nt) {
  const int sh = q0 & 1;
  if (lq == kMaxPanel && lp == kMaxPanel) {
    // full blocks: 4 slots per column, 16-byte row pairs, no zero fill (D's
    // strict upper triangle is mirrored afterwards)
    for (int t = t0; t < kSbThreads; t += nt) {
      const int c = t >> 2, kq = t & 3;
      const double* osrc = AB + (long long)(p0 + c) * ldab + (q0 - p0 - c);
      const double* dsrc = AB + (long long)(q0 + c) * ldab - c;
      double* od = Ob + c * kLd2;
      double* dd = Db + c * kLd2;
#pragma unroll
      for (int i = 0; i < 9; ++i) {
        const int k = kq + 4 * i;
        if (k <= 32) {
          const int r0 = 2 * k - sh;
          const int bytes = k < 32 ? 16 : (sh ? 8 : 0);
          if (bytes) {
            cp_async16_n(od + r0, osrc + r0, bytes);
            if (r0 + 1 >= c) cp_async16_n(dd + r0, dsrc + r0, bytes);
          }
        }
      }
    }
  } else {
    constexpr int kTotal = 2 * kMaxPanel * kPairSlots;
    for (int t = t0; t < kTotal; t += nt) {
      const bool isO = t >= kMaxPanel * kPairSlots;
      const int u = isO ? t - kMaxPanel * kPairSlots : t;
      const int c = u / kPairSlots, k = u - kPairSlots * c;
      const int r0 = 2 * k - sh;
      if (r0 >= kMaxPanel) continue;
      double* dst = (isO ? Ob : Db) + c * kLd2 + r0;
      const double* src = isO ? AB + (long long)(p0 + c) * ldab + (q0 + r0 - p0 - c)
                              : AB + (long long)(q0 + c) * ldab + (r0 - c);
      // need: the row must come from this copy; zero: the row must read 0;
      // other rows (row -1/64 padding, D's upper triangle) are don't-care.
      const int r1 = r0 + 1;
      bool need0, need1, zero0, zero1;
      if (isO) {
        need0 = r0 >= 0 && r0 < lq && c < lp;
        need1 = r1 < kMaxPanel && r1 < lq && c < lp;
        zero0 = r0 >= 0 && !need0;
        zero1 = r1 < kMaxPanel && !need1;
      } else {
        need0 = r0 >= 0 && r0 >= c && r0 < lq;
        need1 = r1 < kMaxPanel && r1 >= c && r1 < lq;
        zero0 = r0 >= 0 && r0 >= c && !need0;
        zero1 = r1 < kMaxPanel && r1 >= c && !need1;
      }
      int bytes;
      if (need1) bytes = 16;
      else if (need0) bytes = 8;
      else if (zero0 || zero1) bytes = 0;
      else continue;
      cp_async16_n(dst, bytes ? src : AB, bytes);
    }
  }
}

// D's strict upper triangle from the lower one (except the late row lq - 1).
BSE_DEV void mirror_d(double* Db, int lq) {
  const int rl = lq - 1;
#pragma unroll 4
  for (int k = 0; k < kSlots; ++k) {
    const int idx = threadIdx.x + k * kSbThreads;
    const int r = idx & (kMaxPanel - 1), c = idx >> 6;
    if (r < c && c != rl) Db[c * kLd2 + r] = Db[r * kLd2 + c];
  }
}

// The late positions (D's last row and O(lq-1, lp-1)), after the late wait.
BSE_DEV void late_load(double* Db, double* Ob, const double* AB, int ldab, int q0, int lq, int p0,
                       int lp) {
  const int tid = threadIdx.x, rl = lq - 1;
  if (tid < kMaxPanel) {
    const int c = tid;
    const double x = c <= rl ? __ldcg(AB + (long long)(q0 + c) * ldab + (rl - c)) : 0.0;
    Db[c * kLd2 + rl] = x;
    Db[rl * kLd2 + c] = x;
  } else if (tid == kMaxPanel) {
    Ob[(lp - 1) * kLd2 + rl] = __ldcg(AB + (long long)(p0 + lp - 1) * ldab + (q0 + rl - p0 - lp + 1));
  }
}

BSE_DEV void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

__global__ void __launch_bounds__(kSbThreads) sb2st_fused_kernel(double* AB, int ldab, int n,
                                                                 int b, double* V2, double* tau2,
                                                                 int maxsteps, int* progress,
                                                                 unsigned long long* trace) {
  extern __shared__ __align__(16) unsigned char raw[];
  SbfSmem& sm = *reinterpret_cast<SbfSmem*>(raw);
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int mi = warp * 8 + (lane >> 2);  // row (A) / column (C) owned by this quarter-thread
  const int q = lane & 3;
  const int ts0 = c_sb_trace_s0;
  int tj = 0, ts = 0;
  auto T = [&](int slot) { trace[((long long)(ts - ts0) * maxsteps + tj) * 16 + slot] = gtimer(); };
  int* full = progress;
  int* late = progress + n;
  if (tid < kMaxPanel) sm.vbuf[0][tid] = sm.vbuf[1][tid] = 0.0;

  for (int s = blockIdx.x; s < n - 2; s += gridDim.x) {
    const bool trw = trace != nullptr && (s == ts0 || s == ts0 + 1);
    const bool trs = trw && tid == 0;
    const bool trs32 = trw && tid == 32;
    ts = s;
    const bool has_pred = s > 0;
    int p0 = s, lp = 1;
    double tau = 0.0;
    int q0 = s + 1, q1 = min(s + b, n - 1);
    int lq = q1 - q0 + 1;
    // prologue: step 0's bulk into buffer 0
    __syncthreads();  // the previous sweep is done with both buffers
    if (has_pred && tid == 0) poll_counter(full + s - 1, kBulkWarps);
    __syncthreads();
    stage_bulk(sm.D[0] + (q0 & 1), sm.O[0] + (q0 & 1), AB, ldab, q0, lq, p0, lp, tid, kSbThreads);
    cp_async_commit();
    for (int j = 0;; ++j) {
      const int cur = j & 1;
      const int sh = q0 & 1;
      double* Db = sm.D[cur] + sh;
      double* Ob = sm.O[cur] + sh;
      const double* v = sm.vbuf[j & 1];
      tj = j;
      if (trs) T(0);
      // late wait, overlapping the arrival of this step's staged bulk; then
      // mirror D and load the late row (disjoint positions, one barrier)
      if (has_pred && tid == 0) poll_counter(late + s - 1, j + 2);
      cp_async_wait<0>();
      __syncthreads();
      if (trs) T(1);
      mirror_d(Db, lq);
      late_load(Db, Ob, AB, ldab, q0, lq, p0, lp);
      __syncthreads();
      if (trs) T(2);
      // A: w = tau O v
      {
        double a = 0.0;
        if (tau != 0.0) {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = colA(q, i);
            a += Ob[c * kLd2 + mi] * v[c];
          }
          a += __shfl_xor_sync(0xffffffffu, a, 1);
          a += __shfl_xor_sync(0xffffffffu, a, 2);
        }
        if (q == 0) sm.w[mi] = tau * a;
      }
      __syncthreads();
      // B: vn = house(O[:, 0] - w), per warp
      double* vn = sm.vnw[warp];
      double taun = 0.0, betan;
      double swv;
      {
        const double x0 = lane < lq ? Ob[lane] - sm.w[lane] : 0.0;
        const double x1 = lane + 32 < lq ? Ob[lane + 32] - sm.w[lane + 32] : 0.0;
        const double ss = warp_sum((lane >= 1 ? x0 * x0 : 0.0) + x1 * x1);
        const double alpha = __shfl_sync(0xffffffffu, x0, 0);
        betan = alpha;
        double scale = 0.0;
        if (ss > 0.0) {
          betan = -copysign(sqrt(alpha * alpha + ss), alpha);
          taun = (betan - alpha) / betan;
          scale = 1.0 / (alpha - betan);
        }
        const double vn0 = lane == 0 ? 1.0 : x0 * scale;
        const double vn1 = x1 * scale;
        vn[lane] = vn0;
        vn[lane + 32] = vn1;
        swv = warp_sum(sm.w[lane] * vn0 + sm.w[lane + 32] * vn1);
        __syncwarp();
      }
      // C: t = taun D vn, y = taun (O^T vn - v swv)
      {
        double tc = 0.0, gc = 0.0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int r = rowC(q, i);
          const double vr = vn[r];
          tc += Db[mi * kLd2 + r] * vr;
          gc += Ob[mi * kLd2 + r] * vr;
        }
        tc += __shfl_xor_sync(0xffffffffu, tc, 1);
        tc += __shfl_xor_sync(0xffffffffu, tc, 2);
        gc += __shfl_xor_sync(0xffffffffu, gc, 1);
        gc += __shfl_xor_sync(0xffffffffu, gc, 2);
        if (q == 0) {
          sm.tt[mi] = taun * tc;
          sm.y[mi] = taun * (gc - v[mi] * swv);
        }
      }
      __syncthreads();
      if (trs) T(3);
      // next step's geometry
      const int nq0 = q1 + 1;
      const bool has_next = nq0 <= n - 1;
      const int nq1 = min(q1 + b, n - 1);
      const int nlq = nq1 - nq0 + 1;
      const double gm = warp_sum(sm.tt[lane] * vn[lane] + sm.tt[lane + 32] * vn[lane + 32]);
      const double al = -0.5 * taun * gm;
      if (warp == 0) {
        // publish the successor's late data: row 0 of O'' and D''(0, 0)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = lane + 32 * h;
          if (c < lp) {
            const double val = c == 0 ? betan : Ob[c * kLd2] - sm.w[0] * v[c] - sm.y[c];
            AB[(long long)(p0 + c) * ldab + (q0 - p0 - c)] = val;
          }
        }
        if (lane == 0) AB[(long long)q0 * ldab] = Db[0] - 2.0 * (sm.tt[0] + al);
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          st_release(late + s, j + 1);
          if (trs) T(4);
        }
      }
      if (warp == 1) {
        V2[((long long)s * maxsteps + j) * b + lane] = vn[lane];
        V2[((long long)s * maxsteps + j) * b + lane + 32] = vn[lane + 32];
        sm.vbuf[(j + 1) & 1][lane] = vn[lane];
        sm.vbuf[(j + 1) & 1][lane + 32] = vn[lane + 32];
        if (lane == 0) tau2[(long long)s * maxsteps + j] = taun;
      }
      // D: the bulk of O'' and D'' (rows >= 1)
      if (lq == kMaxPanel && lp == kMaxPanel) {
        const int c = kMaxPanel - 1 - (tid >> 2), kq = tid & 3;
        double* od = AB + (long long)(p0 + c) * ldab + (q0 - p0 - c);
        double* dd = AB + (long long)(q0 + c) * ldab - c;
        const double vc = v[c], yc = sm.y[c];
        const double vnc = vn[c], w2c = sm.tt[c] + al * vnc;
        const int dlo = c > 1 ? c : 1;
#pragma unroll
        for (int i = 0; i < 9; ++i) {
          const int k = kq + 4 * i;
          if (k <= 32) {
            const int r0 = 2 * k - sh, r1 = r0 + 1;
            const bool in0 = r0 >= 1 && r0 < kMaxPanel, in1 = r1 >= 1 && r1 < kMaxPanel;
            double o0 = 0.0, o1 = 0.0;
            if (c > 0) {
              if (in0) o0 = Ob[c * kLd2 + r0] - sm.w[r0] * vc - vn[r0] * yc;
              if (in1) o1 = Ob[c * kLd2 + r1] - sm.w[r1] * vc - vn[r1] * yc;
            }
            if (in0 && in1) st_global_v2(od + r0, o0, o1);
            else if (in0) od[r0] = o0;
            else if (in1) od[r1] = o1;
            const bool d0 = in0 && r0 >= dlo, d1 = in1 && r1 >= dlo;
            double e0 = 0.0, e1 = 0.0;
            if (d0) e0 = Db[c * kLd2 + r0] - (vn[r0] * w2c + (sm.tt[r0] + al * vn[r0]) * vnc);
            if (d1) e1 = Db[c * kLd2 + r1] - (vn[r1] * w2c + (sm.tt[r1] + al * vn[r1]) * vnc);
            if (d0 && d1) st_global_v2(dd + r0, e0, e1);
            else if (d0) dd[r0] = e0;
            else if (d1) dd[r1] = e1;
          }
        }
      } else {
        constexpr int kTotal = 2 * kMaxPanel * kPairSlots;
        for (int t = tid; t < kTotal; t += kSbThreads) {
          const bool isO = t >= kMaxPanel * kPairSlots;
          const int u = isO ? t - kMaxPanel * kPairSlots : t;
          const int c = u / kPairSlots, k = u - kPairSlots * c;
          const int r0 = 2 * k - sh, r1 = r0 + 1;
          if (r0 >= lq) continue;
          double val0 = 0.0, val1 = 0.0;
          bool ok0, ok1;
          double* dst;
          if (isO) {
            if (c >= lp) continue;
            ok0 = r0 >= 1;
            ok1 = r1 >= 1 && r1 < lq;
            dst = AB + (long long)(p0 + c) * ldab + (q0 + r0 - p0 - c);
            if (c > 0) {
              const double vc = v[c], yc = sm.y[c];
              if (ok0) val0 = Ob[c * kLd2 + r0] - sm.w[r0] * vc - vn[r0] * yc;
              if (ok1) val1 = Ob[c * kLd2 + r1] - sm.w[r1] * vc - vn[r1] * yc;
            }
          } else {
            ok0 = r0 >= 1 && r0 >= c;
            ok1 = r1 >= 1 && r1 >= c && r1 < lq;
            if (!ok0 && !ok1) continue;
            dst = AB + (long long)(q0 + c) * ldab + (r0 - c);
            const double vc = vn[c], w2c = sm.tt[c] + al * vc;
            if (ok0) val0 = Db[c * kLd2 + r0] - (vn[r0] * w2c + (sm.tt[r0] + al * vn[r0]) * vc);
            if (ok1) val1 = Db[c * kLd2 + r1] - (vn[r1] * w2c + (sm.tt[r1] + al * vn[r1]) * vc);
          }
          if (ok0 && ok1) st_global_v2(dst, val0, val1);
          else if (ok0) dst[0] = val0;
          else if (ok1) dst[1] = val1;
        }
      }
      // each warp publishes its own bulk stores: full[s] reaches
      // kBulkWarps * (j + 1) once step j is completely stored
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        atomicAdd(full + s, 1);
      }
      if (trs) T(5);
      if (warp != 0 && has_next) {
        // warps 1..7: stage step j+1's bulk into the other buffer (needs the
        // predecessor's step j+1 fully stored) -- after our own bulk, so our
        // `full` is never held back by our predecessor
        if (has_pred && tid == 32) poll_counter(full + s - 1, kBulkWarps * (j + 2));
        if (trs32) T(7);
        named_bar(1, kSbThreads - 32);
        const int nsh = nq0 & 1;
        stage_bulk(sm.D[cur ^ 1] + nsh, sm.O[cur ^ 1] + nsh, AB, ldab, nq0, nlq, q0, lq, tid - 32,
                   kSbThreads - 32);
        cp_async_commit();
        if (trs32) T(8);
      }
      tau = taun;
      if (!has_next) break;
      if (trs) T(6);
      p0 = q0;
      lp = lq;
      q0 = nq0;
      q1 = nq1;
      lq = nlq;
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      st_release(late + s, kDone);
      st_release(full + s, kDone);
    }
  }
}

// ---------------------------------------------------------------------------
// Pair kernel (default).  One CTA chases TWO consecutive sweeps, leader s
// (even) and follower s+1, interleaved step by step: round j = leader step
// j+1, then follower step j.  The follower's blocks are the leader's step-j
// blocks shifted by one row and column -- still in shared memory, updated in
// place by the leader -- plus one new row/column: the leader's step-(j+1)
// row 0 (also in shared memory) and 63 band entries already final in global
// memory.  So half of all cross-sweep hand-offs never leave the SM: no flag,
// no fence, no L2 round trip.  Only the follower publishes (late/full
// counters, as in the fused kernel) for the next pair's leader; the leader
// waits on the previous pair's follower.  Three shared block sets rotate:
// leader step J uses set J mod 3, the follower reuses it one round later,
// and the leader's step J+1 stages into the third.
constexpr int kLdc = kMaxPanel + 1;  // 65 columns: the follower's view reaches column 64
constexpr int kSetD = kLdc * kLd2 + 2;

struct SbpSmem {
  double D[3][kSetD];
  double O[3][kSetD];
  double vbuf[2][2][kMaxPanel];  // [leader / follower][parity]
  double vnw[kSbThreads / 32][kMaxPanel];
  double w[kMaxPanel];
  double y[kMaxPanel];
  double tt[kMaxPanel];
};

struct SbStep {
  int q0, lq, p0, lp;
};

// Phases A-C of one step on (Db, Ob): fills sm.w, sm.y, sm.tt and this warp's
// copy of vn; returns taun, betan and al = -taun (t^T vn) / 2.
BSE_DEV void sbp_abc(SbpSmem& sm, const double* Db, const double* Ob, int lq, const double* v,
                     double tau, double& taun, double& betan, double& al) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int mi = warp * 8 + (lane >> 2), q = lane & 3;
  {
    double a = 0.0;
    if (tau != 0.0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = colA(q, i);
        a += Ob[c * kLd2 + mi] * v[c];
      }
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
    }
    if (q == 0) sm.w[mi] = tau * a;
  }
  __syncthreads();
  double* vn = sm.vnw[warp];
  double swv;
  taun = 0.0;
  {
    const double x0 = lane < lq ? Ob[lane] - sm.w[lane] : 0.0;
    const double x1 = lane + 32 < lq ? Ob[lane + 32] - sm.w[lane + 32] : 0.0;
    const double ss = warp_sum((lane >= 1 ? x0 * x0 : 0.0) + x1 * x1);
    const double alpha = __shfl_sync(0xffffffffu, x0, 0);
    betan = alpha;
    double scale = 0.0;
    if (ss > 0.0) {
      betan = -copysign(sqrt(alpha * alpha + ss), alpha);
      taun = (betan - alpha) / betan;
      scale = 1.0 / (alpha - betan);
    }
    const double vn0 = lane == 0 ? 1.0 : x0 * scale;
    const double vn1 = x1 * scale;
    vn[lane] = vn0;
    vn[lane + 32] = vn1;
    swv = warp_sum(sm.w[lane] * vn0 + sm.w[lane + 32] * vn1);
    __syncwarp();
  }
  {
    double tc = 0.0, gc = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int r = rowC(q, i);
      const double vr = vn[r];
      tc += Db[mi * kLd2 + r] * vr;
      gc += Ob[mi * kLd2 + r] * vr;
    }
    tc += __shfl_xor_sync(0xffffffffu, tc, 1);
    tc += __shfl_xor_sync(0xffffffffu, tc, 2);
    gc += __shfl_xor_sync(0xffffffffu, gc, 1);
    gc += __shfl_xor_sync(0xffffffffu, gc, 2);
    if (q == 0) {
      sm.tt[mi] = taun * tc;
      sm.y[mi] = taun * (gc - v[mi] * swv);
    }
  }
  __syncthreads();
  al = -0.5 * taun * warp_sum(sm.tt[lane] * vn[lane] + sm.tt[lane + 32] * vn[lane + 32]);
}

// Phase D: O'' = O - w v^T - vn y^T, D'' = D - vn w2^T - w2 vn^T to the band;
// WB also writes them back into (Db, Ob) (the leader's blocks feed the
// follower).  Row 0 is done by warp 0 (and published on `late` when PUB).
template <bool WB, bool PUB>
BSE_DEV void sbp_store(SbpSmem& sm, double* AB, int ldab, const SbStep& g, double* Db, double* Ob,
                       const double* v, double betan, double al, int* late_s, int late_val) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* vn = sm.vnw[warp];
  const int sh = g.q0 & 1;
  const int q0 = g.q0, lq = g.lq, p0 = g.p0, lp = g.lp;
  if (warp == 0) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c < lp) {
        const double val = c == 0 ? betan : Ob[c * kLd2] - sm.w[0] * v[c] - sm.y[c];
        AB[(long long)(p0 + c) * ldab + (q0 - p0 - c)] = val;
        if (WB) Ob[c * kLd2] = val;
      }
    }
    if (lane == 0) {
      const double d00 = Db[0] - 2.0 * (sm.tt[0] + al);
      AB[(long long)q0 * ldab] = d00;
      if (WB) Db[0] = d00;
    }
    if (PUB) {
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        st_release(late_s, late_val);
      }
    }
  }
  auto put = [&](double* gp, double* sp, double* spm, bool ok0, bool ok1, double e0, double e1) {
    if (ok0 && ok1) st_global_v2(gp, e0, e1);
    else if (ok0) gp[0] = e0;
    else if (ok1) gp[1] = e1;
    if (WB) {
      if (ok0) { sp[0] = e0; if (spm) spm[0] = e0; }
      if (ok1) { sp[1] = e1; if (spm) spm[kLd2] = e1; }
    }
  };
  if (lq == kMaxPanel && lp == kMaxPanel) {
    const int c = kMaxPanel - 1 - (tid >> 2), kq = tid & 3;
    double* od = AB + (long long)(p0 + c) * ldab + (q0 - p0 - c);
    double* dd = AB + (long long)(q0 + c) * ldab - c;
    const double vc = v[c], yc = sm.y[c];
    const double vnc = vn[c], w2c = sm.tt[c] + al * vnc;
    const int dlo = c > 1 ? c : 1;
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      const int k = kq + 4 * i;
      if (k <= 32) {
        const int r0 = 2 * k - sh, r1 = r0 + 1;
        const bool in0 = r0 >= 1 && r0 < kMaxPanel, in1 = r1 >= 1 && r1 < kMaxPanel;
        double o0 = 0.0, o1 = 0.0;
        if (c > 0) {
          if (in0) o0 = Ob[c * kLd2 + r0] - sm.w[r0] * vc - vn[r0] * yc;
          if (in1) o1 = Ob[c * kLd2 + r1] - sm.w[r1] * vc - vn[r1] * yc;
        }
        put(od + r0, Ob + c * kLd2 + r0, nullptr, in0, in1, o0, o1);
        const bool d0 = in0 && r0 >= dlo, d1 = in1 && r1 >= dlo;
        double e0 = 0.0, e1 = 0.0;
        if (d0) e0 = Db[c * kLd2 + r0] - (vn[r0] * w2c + (sm.tt[r0] + al * vn[r0]) * vnc);
        if (d1) e1 = Db[c * kLd2 + r1] - (vn[r1] * w2c + (sm.tt[r1] + al * vn[r1]) * vnc);
        put(dd + r0, Db + c * kLd2 + r0, Db + r0 * kLd2 + c, d0, d1, e0, e1);
      }
    }
  } else {
    constexpr int kTotal = 2 * kMaxPanel * kPairSlots;
    for (int t = tid; t < kTotal; t += kSbThreads) {
      const bool isO = t >= kMaxPanel * kPairSlots;
      const int u = isO ? t - kMaxPanel * kPairSlots : t;
      const int c = u / kPairSlots, k = u - kPairSlots * c;
      const int r0 = 2 * k - sh, r1 = r0 + 1;
      if (r0 >= lq) continue;
      double val0 = 0.0, val1 = 0.0;
      bool ok0, ok1;
      if (isO) {
        if (c >= lp) continue;
        ok0 = r0 >= 1;
        ok1 = r1 >= 1 && r1 < lq;
        if (c > 0) {
          const double vc = v[c], yc = sm.y[c];
          if (ok0) val0 = Ob[c * kLd2 + r0] - sm.w[r0] * vc - vn[r0] * yc;
          if (ok1) val1 = Ob[c * kLd2 + r1] - sm.w[r1] * vc - vn[r1] * yc;
        }
        put(AB + (long long)(p0 + c) * ldab + (q0 + r0 - p0 - c), Ob + c * kLd2 + r0, nullptr, ok0,
            ok1, val0, val1);
      } else {
        ok0 = r0 >= 1 && r0 >= c;
        ok1 = r1 >= 1 && r1 >= c && r1 < lq;
        if (!ok0 && !ok1) continue;
        const double vc = vn[c], w2c = sm.tt[c] + al * vc;
        if (ok0) val0 = Db[c * kLd2 + r0] - (vn[r0] * w2c + (sm.tt[r0] + al * vn[r0]) * vc);
        if (ok1) val1 = Db[c * kLd2 + r1] - (vn[r1] * w2c + (sm.tt[r1] + al * vn[r1]) * vc);
        put(AB + (long long)(q0 + c) * ldab + (r0 - c), Db + c * kLd2 + r0, Db + r0 * kLd2 + c, ok0,
            ok1, val0, val1);
      }
    }
  }
}

__global__ void __launch_bounds__(kSbThreads) sb2st_pair_kernel(double* AB, int ldab, int n, int b,
                                                                double* V2, double* tau2,
                                                                int maxsteps, int* progress,
                                                                unsigned long long* trace) {
  (void)trace;
  extern __shared__ __align__(16) unsigned char raw[];
  SbpSmem& sm = *reinterpret_cast<SbpSmem*>(raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* full = progress;
  int* late = progress + n;
  const int nsweeps = n - 2;
  auto geo = [&](int s, int j) -> SbStep {  // step j of sweep s (q0 > n-1: none)
    SbStep g;
    g.q0 = s + 1 + j * b;
    g.lq = min(s + (j + 1) * b, n - 1) - g.q0 + 1;
    g.p0 = j == 0 ? s : s + 1 + (j - 1) * b;
    g.lp = j == 0 ? 1 : b;
    if (j > 0 && g.p0 + g.lp - 1 > n - 1) g.lp = n - g.p0;
    return g;
  };
  auto exists = [&](int s, int j) { return s < nsweeps && s + 1 + j * b <= n - 1; };

  for (int s = 2 * blockIdx.x; s < nsweeps; s += 2 * gridDim.x) {
    const int f = s + 1;
    const bool has_pred = s > 0;
    const bool has_f = f < nsweeps;
    double tauL = 0.0, tauF = 0.0;
    if (tid < kMaxPanel) {
      sm.vbuf[0][0][tid] = sm.vbuf[0][1][tid] = 0.0;
      sm.vbuf[1][0][tid] = sm.vbuf[1][1][tid] = 0.0;
    }
    // prologue: the leader's step-0 bulk into set 0
    __syncthreads();
    if (has_pred && tid == 0) poll_counter(full + s - 1, kBulkWarps);
    __syncthreads();
    {
      const SbStep g = geo(s, 0);
      stage_bulk(sm.D[0] + (g.q0 & 1), sm.O[0] + (g.q0 & 1), AB, ldab, g.q0, g.lq, g.p0, g.lp, tid,
                 kSbThreads);
      cp_async_commit();
      cp_async_wait<0>();
      __syncthreads();
      mirror_d(sm.D[0] + (g.q0 & 1), g.lq);
    }
    // round J: leader step J (set J % 3), then follower step J - 1 (set (J-1) % 3)
    for (int J = 0;; ++J) {
      const bool lead = exists(s, J);
      const bool foll = has_f && J >= 1 && exists(f, J - 1);
      if (!lead && !foll) break;
      if (lead) {
        const SbStep g = geo(s, J);
        const int set = J % 3;
        double* Db = sm.D[set] + (g.q0 & 1);
        double* Ob = sm.O[set] + (g.q0 & 1);
        const double* v = sm.vbuf[0][J & 1];
        if (has_pred && tid == 0) poll_counter(late + s - 1, J + 2);
        __syncthreads();  // also publishes the mirror writes
        late_load(Db, Ob, AB, ldab, g.q0, g.lq, g.p0, g.lp);
        __syncthreads();
        double taun, betan, al;
        sbp_abc(sm, Db, Ob, g.lq, v, tauL, taun, betan, al);
        if (warp == 1) {
          V2[((long long)s * maxsteps + J) * b + lane] = sm.vnw[1][lane];
          V2[((long long)s * maxsteps + J) * b + lane + 32] = sm.vnw[1][lane + 32];
          sm.vbuf[0][(J + 1) & 1][lane] = sm.vnw[1][lane];
          sm.vbuf[0][(J + 1) & 1][lane + 32] = sm.vnw[1][lane + 32];
          if (lane == 0) tau2[(long long)s * maxsteps + J] = taun;
        }
        sbp_store<true, false>(sm, AB, ldab, g, Db, Ob, v, betan, al, nullptr, 0);
        tauL = taun;
        // stage the leader's step J+1 into set (J+1) % 3 (free: the follower
        // finished with it last round), needs the predecessor's step J+1 stored
        if (exists(s, J + 1)) {
          const SbStep gn = geo(s, J + 1);
          if (has_pred && tid == 0) poll_counter(full + s - 1, kBulkWarps * (J + 2));
          __syncthreads();
          const int ns = (J + 1) % 3;
          stage_bulk(sm.D[ns] + (gn.q0 & 1), sm.O[ns] + (gn.q0 & 1), AB, ldab, gn.q0, gn.lq, gn.p0,
                     gn.lp, tid, kSbThreads);
          cp_async_commit();
        }
      }
      if (foll) {
        const int jf = J - 1;
        const SbStep g = geo(f, jf);
        const SbStep gl = geo(s, jf);  // the leader's step jf: its blocks, shifted, are ours
        const int set = jf % 3;
        double* Db = sm.D[set] + (gl.q0 & 1) + kLd2 + 1;
        double* Ob = sm.O[set] + (gl.q0 & 1) + kLd2 + 1;
        const double* DLb = sm.D[set] + (gl.q0 & 1);  // leader's step-jf block, unshifted
        const bool late_in = lead;  // the leader's step J produced our last row
        __syncthreads();            // the leader's write-back is complete
        const int rl = g.lq - 1;
        if (late_in) {
          const SbStep gn = geo(s, J);
          const double* DN = sm.D[J % 3] + (gn.q0 & 1);
          const double* ON = sm.O[J % 3] + (gn.q0 & 1);
          if (tid < kMaxPanel) {
            const int c = tid;
            double x;
            if (c < rl) x = ON[(c + 1) * kLd2];  // leader's O''(0, c+1)
            else if (c == rl) x = DN[0];           // leader's D''(0, 0)
            else x = 0.0;
            Db[c * kLd2 + rl] = x;
            Db[rl * kLd2 + c] = x;
          } else if (tid == kMaxPanel) {
            Ob[(g.lp - 1) * kLd2 + rl] = ON[0];  // leader's beta: O'(rl, lp-1)
          } else if (tid > kMaxPanel && tid - kMaxPanel - 1 < g.lp - 1) {
            const int c = tid - kMaxPanel - 1;  // O'(rl, c), c < lp-1: final in the band
            Ob[c * kLd2 + rl] = __ldcg(AB + (long long)(g.p0 + c) * ldab + (g.q0 + rl - g.p0 - c));
          }
        } else if (tid < kMaxPanel && g.lq < kMaxPanel) {
          // truncated block: clear the stale extra row / column of the set
          Db[tid * kLd2 + (kMaxPanel - 1)] = 0.0;
          Db[(kMaxPanel - 1) * kLd2 + tid] = 0.0;
          Ob[tid * kLd2 + (kMaxPanel - 1)] = 0.0;
        }
        // O'(r, lp-1) = leader's D''(r+1, 0) for r < lq (rl via beta when late_in)
        if (tid < kMaxPanel) {
          const int r = tid;
          if (!(late_in && r == rl)) Ob[(g.lp - 1) * kLd2 + r] = r < g.lq ? DLb[r + 1] : 0.0;
        }
        __syncthreads();
        const double* v = sm.vbuf[1][jf & 1];
        double taun, betan, al;
        sbp_abc(sm, Db, Ob, g.lq, v, tauF, taun, betan, al);
        if (warp == 1) {
          V2[((long long)f * maxsteps + jf) * b + lane] = sm.vnw[1][lane];
          V2[((long long)f * maxsteps + jf) * b + lane + 32] = sm.vnw[1][lane + 32];
          sm.vbuf[1][(jf + 1) & 1][lane] = sm.vnw[1][lane];
          sm.vbuf[1][(jf + 1) & 1][lane + 32] = sm.vnw[1][lane + 32];
          if (lane == 0) tau2[(long long)f * maxsteps + jf] = taun;
        }
        sbp_store<false, true>(sm, AB, ldab, g, Db, Ob, v, betan, al, late + f, jf + 1);
        // each warp publishes its bulk (and, by program order, the leader's
        // earlier stores) on `full`
        __syncwarp();
        if (lane == 0) {
          __threadfence();
          atomicAdd(full + f, 1);
        }
        tauF = taun;
      }
      // the leader's next set has landed: mirror its D
      if (exists(s, J + 1)) {
        const SbStep gn = geo(s, J + 1);
        cp_async_wait<0>();
        __syncthreads();
        mirror_d(sm.D[(J + 1) % 3] + (gn.q0 & 1), gn.lq);
      }
    }
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      if (has_f) {
        st_release(late + f, kDone);
        st_release(full + f, kDone);
      }
      st_release(late + s, kDone);
      st_release(full + s, kDone);
    }
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
    if ((err = cudaMemsetAsync(progress, 0, sizeof(int) * 2 * (size_t)n, s)) != cudaSuccess) return err;
    int flags = 0;
    if (const char* v = std::getenv("BSE_SB2ST_VARIANT")) flags = std::atoi(v);
    cudaMemcpyToSymbolAsync(c_sb_flags, &flags, sizeof(int), 0, cudaMemcpyHostToDevice, s);
    const bool legacy = (flags & 16) != 0;  // previous multi-phase step
    const bool single = (flags & 128) == 0;  // flag 128: sweep pairs per CTA (experimental)
    const void* kern = legacy ? (const void*)sb2st_kernel
                              : single ? (const void*)sb2st_fused_kernel : (const void*)sb2st_pair_kernel;
    const size_t smem = legacy ? sizeof(SbSmem) : single ? sizeof(SbfSmem) : sizeof(SbpSmem);
    static bool attr = false;
    if (!attr) {
      err = cudaFuncSetAttribute(sb2st_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)sizeof(SbSmem));
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(sb2st_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sizeof(SbfSmem));
      if (err == cudaSuccess)
        err = cudaFuncSetAttribute(sb2st_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sizeof(SbpSmem));
      if (err != cudaSuccess) return err;
      attr = true;
    }
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSbThreads, smem);
    if (!(flags & 8)) per_sm = 1;  // default 1 CTA/SM (flag 8 restores full occupancy)
    const int units = (legacy || single) ? n - 2 : (n - 1) / 2;  // sweeps or sweep pairs
    int grid = std::max(1, std::min(units, std::max(1, per_sm) * num_sms));
    int maxsteps = sb2st_maxsteps(n, b);
    unsigned long long* trace = nullptr;
    const char* tenv = std::getenv("BSE_SB2ST_TRACE");
    const bool want_trace = tenv != nullptr;
    int ts0 = want_trace ? std::atoi(tenv) : 0;
    ts0 = std::max(0, std::min(ts0, n - 4));
    cudaMemcpyToSymbolAsync(c_sb_trace_s0, &ts0, sizeof(int), 0, cudaMemcpyHostToDevice, s);
    const size_t tsz = (size_t)2 * maxsteps * 16;
    if (want_trace) {
      cudaMalloc(&trace, sizeof(unsigned long long) * tsz);
      cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * tsz, s);
    }
    void* args[] = {&AB, &ldab, &n, &b, &V2, &tau2, &maxsteps, &progress, &trace};
    count_launch();
    err = cudaLaunchCooperativeKernel(kern, dim3(grid), dim3(kSbThreads), args, smem, s);
    if (err != cudaSuccess) return err;
    if (want_trace && !legacy) {
      std::vector<unsigned long long> h(tsz);
      cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, s);
      cudaStreamSynchronize(s);
      // sweep ts0 + 1 (consumer) against sweep ts0 (producer): per-phase
      // averages, step period, and the hand-off gap = consumer's late-wait
      // exit of step j minus the producer's late release of step j + 1
      double acc[16] = {0}, period = 0.0, gap = 0.0;
      int cnt = 0;
      for (int j = 2; j < maxsteps - 2; ++j) {
        const unsigned long long* c = &h[((size_t)maxsteps + j) * 16];
        const unsigned long long* nx = &h[((size_t)maxsteps + j + 1) * 16];
        const unsigned long long* pr = &h[(size_t)(j + 1) * 16];
        if (!c[6] || !nx[0] || !pr[4]) break;
        for (int q = 1; q <= 6; ++q) acc[q] += (double)(c[q] - c[q - 1]);
        period += (double)(nx[0] - c[0]);
        gap += (double)c[1] - (double)pr[4];
        ++cnt;
      }
      double e7 = 0, e8 = 0, e9 = 0, e10 = 0;
      for (int j = 2; j < 2 + cnt; ++j) {
        const unsigned long long* c = &h[((size_t)maxsteps + j) * 16];
        e7 += (double)c[7] - (double)c[5];
        e8 += (double)c[8] - (double)c[7];
        e9 += (double)c[9] - (double)c[5];
        e10 += (double)c[10] - (double)c[9];
      }
      const double d = std::max(cnt, 1) * 1e3;
      std::fprintf(stderr, "[sb2st trace] after bulk(t0): poll %.2f issue %.2f | after own bulk: arrive(t32) %.2f sync %.2f\n",
                   e7 / d, e8 / d, e9 / d, e10 / d);
      std::fprintf(stderr, "[sb2st trace] sweep %d steps=%d us: latewait %.2f lateload %.2f ABC %.2f publish %.2f "
                   "bulk %.2f arrive+mirror %.2f | period %.2f handoff %.2f\n", ts0 + 1, cnt, acc[1] / d,
                   acc[2] / d, acc[3] / d, acc[4] / d, acc[5] / d, acc[6] / d, period / d, gap / d);
    }
    if (trace) cudaFree(trace);
  }
  band_to_tridiag_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(AB, ldab, n, d, e);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bse
