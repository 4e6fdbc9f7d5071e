// Stage 2: band -> tridiagonal by bulge chasing (Schwarz/Lang element
// annihilation, the task structure of LAPACK's SB2ST kernels), as one
// persistent cooperative kernel.  Sweep s is owned by CTA s mod G; step j of
// sweep s may start once sweep s-1 has published step j+1 (release/acquire
// counters per sweep), so ~N/(2b) sweeps are in flight at once.  The band
// (ldab = 2b + 1 doubles per column) stays L2-resident; every reflector is
// stored for the Q2 back-transform.
#include <cuda.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "eig.cuh"

namespace bse {
namespace {

constexpr int kSbThreads = 256;
constexpr int kDone = 0x7fffffff;
constexpr int kSlots = kMaxPanel * kMaxPanel / kSbThreads;  // 16 block slots per thread

__constant__ int c_sb_trace_s0;  // first traced sweep (BSE_SB2ST_TRACE)
__constant__ int c_sb_mode;      // diagnostics (BSE_SB2ST_MODE): 1 CTA-wide full publish, 2 acquire polls

BSE_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
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
//
// Hand-off mailboxes.  The late data of a step (b + 1 doubles) does not travel
// through the band and a release/acquire counter (store, fence, flag, poll,
// fence, load: two dependent L2 round trips plus two fences on the chain
// that paces the whole wavefront) but through a per-(sweep, step) mailbox of
// self-validating 16-byte slots {bits, bits ^ tag(sweep, step)}: the
// producer's warp 0 stores them without any fence, the consumer's threads
// poll their own slot until the two halves agree with the tag.  Each 8-byte
// half is written atomically, so a torn or stale slot never validates (tags
// are 64-bit hashes, unique per call; the ring is cleared per call).  Values
// handed over this way are NOT written to the band by the producer: the
// consumer's own bulk store rewrites exactly those positions (row lq - 1 of
// its blocks), so no store of the producer can race with it.  Steps without
// a consumer (step 0, the last sweep) publish to the band as before; a
// consumer whose predecessor has no step j + 1 waits for the predecessor to
// finish (`late` == kDone) and reads the band.
constexpr int kLd2 = 66;
constexpr int kBulkWarps = kSbThreads / 32;  // every warp stores part of the bulk
constexpr int kMailSlots = kMaxPanel + 2;    // slot 0: O(0, 0); 1..lp-1: O(0, c); lp: D(0, 0)
constexpr int kMailRing = 160;               // sweeps (> resident CTAs + 1)
constexpr int kSbMaxGrid = kMailRing - 4;

struct SbfSmem {
  // double-buffered: step j+1 stages while j computes; every buffer starts
  // 128-byte aligned (tensor-copy destination)
  alignas(128) double D[2][kMaxPanel * kLd2 + 16];
  alignas(128) double O[2][kMaxPanel * kLd2 + 16];
  double vbuf[2][kMaxPanel];
  double vnw[kSbThreads / 32][kMaxPanel];
  double w[kMaxPanel];
  double y[kMaxPanel];
  double tt[kMaxPanel];
  unsigned long long mbar[2];  // bulk-copy staging of full blocks, one per buffer
};

// phase A (lanes: 4 rows x 4 quarters per half-warp) column pattern
BSE_DEV int colA(int q, int i) { return 8 * (i >> 1) + 2 * q + (i & 1); }
// phase C (lanes: 4 columns x 4 quarters per half-warp) row pattern
BSE_DEV int rowC(int q, int i) { return 16 * (i >> 2) + 2 * (i & 3) + (q & 1) + 8 * (q >> 1); }

// Diagnostics (BSE_SB2ST_MODE bits 4/8/16/32): a pseudo-random delay of up to
// ~16 us keyed by (sweep, step, site) to perturb the hand-off timing.
template <bool kDiag>
BSE_DEV void dbg_delay(int bit, int s, int j) {
  if constexpr (!kDiag) return;
  if (!(c_sb_mode & bit)) return;
  unsigned h = (unsigned)(s * 2654435761u) ^ (unsigned)(j * 40503u) ^ (unsigned)(bit * 97u);
  h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
  if ((h & 7u) == 0) __nanosleep((h >> 8) & 0x3fffu);
}

// Acquire-poll one counter (thread 0).  No barrier.
template <bool kDiag>
BSE_DEV void poll_counter(const int* ctr, int need) {
  if (kDiag && (c_sb_mode & 2)) {
    while (ld_acquire(ctr) < need) {
    }
    return;
  }
  if (ld_relaxed(ctr) < need) {
    while (ld_relaxed(ctr) < need) {
    }
  }
  fence_acquire();
}

BSE_DEV void st_global_v2(double* p, double a, double b) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};\n" ::"l"(p), "d"(a), "d"(b) : "memory");
}

// Staging.  With ldab - 1 = 2b the band is a 2-D tensor T[j][x] at 2b j + x
// (rows overlap: x runs past 2b), in which a block is the box x in
// [q0 - sh, q0 - sh + kLd2), j in [c0, c0 + 64) -- exactly the shared-memory
// layout above (kLd2 doubles per column: the 16-byte aligned superset of its
// rows).  One thread issues two tensor copies per step that complete on the
// buffer's mbarrier: no per-thread copy instructions, no commit/wait groups.
// The box is always the full 64 x 64 block: ragged blocks (step 0's single
// column of O, the last steps of a sweep) bring in other finite band entries,
// or zeros past column n - 1, which only ever meet exact zeros of v / vn or
// land in rows and columns the stores mask out; D's strict upper triangle is
// never read.
constexpr unsigned kBlockBytes = kMaxPanel * kLd2 * sizeof(double);
BSE_DEV void tma_load_2d(void* dst, const CUtensorMap* map, unsigned long long* bar, int x, int j) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];\n" ::"r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(j)
      : "memory");
}
BSE_DEV void stage_tma(double* Dbuf, double* Obuf, unsigned long long* bar, const CUtensorMap* map,
                       int nq0, int q0) {
  const int x = nq0 - (nq0 & 1);
  mbar_arrive_expect_tx(bar, 2 * kBlockBytes);
  tma_load_2d(Obuf, map, bar, x, q0);
  tma_load_2d(Dbuf, map, bar, x, nq0);
}

// The late positions (D's last row and O(lq-1, lp-1)), after the late wait.
//
// One more position of a FULL block's last row is not covered by the two
// counters: O(lq-1, lp-2).  It is column 0, row 1 of the O block of sweep
// s-2's step j+1 -- an entry that sweep annihilates, so its bulk store writes
// 0 there -- and sweep s-1 never touches it.  Sweep s-1's step j only waits
// for sweep s-2's step j+1 ROW 0 (`late`), not for its bulk, so the staged
// copy of that entry may still hold the fill-in that sweep s-3 left there
// when sweep s-2 is descheduled between its two stores (observed under
// time-sliced GPU sharing, and reproduced by delaying the bulk stores).  Its
// final value is exactly 0 by construction, so it is set here instead of read.
// (The entries further left in that row were zeroed by sweeps s-3, s-4, ...,
// whose bulk stores are ordered before this step through `full`.)
BSE_DEV void late_load(double* Db, double* Ob, const double* AB, int ldab, int q0, int lq, int p0,
                       int lp, int b) {
  const int tid = threadIdx.x, rl = lq - 1;
  if (tid < kMaxPanel) {
    const int c = tid;
    if (c <= rl) Db[c * kLd2 + rl] = __ldcg(AB + (long long)(q0 + c) * ldab + (rl - c));
  } else if (tid == kMaxPanel) {
    Ob[(lp - 1) * kLd2 + rl] = __ldcg(AB + (long long)(p0 + lp - 1) * ldab + (q0 + rl - p0 - lp + 1));
  } else if (tid == kMaxPanel + 1) {
    if (lq == b && lp >= 2) Ob[(lp - 2) * kLd2 + rl] = 0.0;
  }
}

BSE_DEV void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
BSE_DEV void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
// barrier of the 8 compute warps (the staging warp never joins it)
BSE_DEV void cta_sync() { named_bar(3, kSbThreads); }

// kDiag: the BSE_SB2ST_MODE diagnostics (delay injection, alternative
// publication / polls) are compiled into a separate instance, so the
// production kernel carries none of their checks.
template <bool kDiag>
__global__ void __launch_bounds__(kSbThreads + 32) sb2st_fused_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                 double* AB, int ldab, int n,
                                                                 int b, double* V2, double* tau2,
                                                                 int maxsteps, int* progress,
                                                                 unsigned long long* mail,
                                                                 unsigned long long* trace) {
  extern __shared__ __align__(128) unsigned char raw[];
  SbfSmem& sm = *reinterpret_cast<SbfSmem*>(raw + ((128u - (smem_u32(raw) & 127u)) & 127u));
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
  if (tid == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    mbar_fence_init();
  }
  unsigned phb = 0u;  // mbarrier phase bits, one per buffer (CTA-uniform; a bit mask stays in a register)
  __syncthreads();  // all nine warps: the mbarriers are initialised

  // Staging warp.  The blocks of step j+1 can be fetched as soon as the
  // predecessor has stored its step j+1 and this sweep is done with step
  // j-1's buffer -- usually in the middle of step j's bulk store.  None of the
  // compute warps can poll for that moment without holding up its share of the
  // step, so a ninth warp does: it replays the step geometry, takes one
  // named-barrier arrival per staging from the compute warps (buffer free),
  // polls the predecessor's `full` counter and issues the two tensor copies.
  if (warp == kSbThreads / 32) {
    for (int s = blockIdx.x; s < n - 2; s += gridDim.x) {
      const bool trp = trace != nullptr && (s == ts0 || s == ts0 + 1) && lane == 0;
      ts = s;
      const bool has_pred = s > 0;
      int p0 = s, q0 = s + 1, q1 = min(s + b, n - 1);
      for (int j = 0;; ++j) {
        // stage step j into buffer j & 1: O at columns p0.., D at columns q0..
        tj = j > 0 ? j - 1 : 0;
        named_bar(2, kSbThreads + 32);
        if (lane == 0) {
          dbg_delay<kDiag>(16, s, j);
          if (has_pred) poll_counter<kDiag>(full + s - 1, kBulkWarps * (j + 1));
          fence_proxy_async();
          if (trp && j > 0) T(7);
          stage_tma(sm.D[j & 1], sm.O[j & 1], &sm.mbar[j & 1], &tmap, q0, p0);
          if (trp && j > 0) T(8);
        }
        __syncwarp();
        if (q1 + 1 > n - 1) break;
        p0 = q0;
        q0 = q1 + 1;
        q1 = min(q1 + b, n - 1);
      }
    }
    return;
  }

  for (int s = blockIdx.x; s < n - 2; s += gridDim.x) {
    const bool trw = trace != nullptr && (s == ts0 || s == ts0 + 1);
    const bool trs = trw && tid == 0;
    ts = s;
    const bool has_pred = s > 0;
    int p0 = s, lp = 1;
    double tau = 0.0;
    int q0 = s + 1, q1 = min(s + b, n - 1);
    int lq = q1 - q0 + 1;
    cta_sync();  // the previous sweep is done with both buffers
    named_bar_arrive(2, kSbThreads + 32);  // stage step 0
    for (int j = 0;; ++j) {
      const int cur = j & 1;
      const int sh = q0 & 1;
      // next step's geometry
      const int nq0 = q1 + 1;
      const bool has_next = nq0 <= n - 1;
      const int nq1 = min(q1 + b, n - 1);
      const int nlq = nq1 - nq0 + 1;

      double* Db = sm.D[cur] + sh;
      double* Ob = sm.O[cur] + sh;
      const double* v = sm.vbuf[j & 1];
      tj = j;
      if (trs) T(0);
      // late wait, overlapping the arrival of this step's staged bulk; then
      // mirror D and load the late row (disjoint positions, one barrier)
      // the predecessor has a step j + 1 exactly when this block is full
      const bool mailed = has_pred && lq == b;
      double lx = 0.0;
      if (mailed) {
        const unsigned long long* box =
            mail + ((size_t)((s - 1) % kMailRing) * maxsteps + (j + 1)) * (2 * kMailSlots);
        const unsigned long long tag = mail_tag(s - 1, j + 1);
        if (tid < b) lx = mail_get(box + 2 * (tid + 1), tag);          // D(lq-1, tid)
        else if (tid == kMaxPanel) lx = mail_get(box, tag);            // O(lq-1, lp-1)
      } else if (has_pred && tid == 0) {
        poll_counter<kDiag>(late + s - 1, kDone);
      }
      if (tid == 0) dbg_delay<kDiag>(32, s, j);
      mbar_wait(&sm.mbar[cur], (phb >> cur) & 1u);  // this step's blocks have landed
      phb ^= 1u << cur;
      cta_sync();
      // every compute warp is past step j-1: its buffer may be refilled
      if (has_next) named_bar_arrive(2, kSbThreads + 32);
      if (trs) T(1);
      if (mailed) {
        const int rl = lq - 1;
        if (tid < b) Db[tid * kLd2 + rl] = lx;
        else if (tid == kMaxPanel) Ob[(lp - 1) * kLd2 + rl] = lx;
        else if (tid == kMaxPanel + 1 && lp >= 2) Ob[(lp - 2) * kLd2 + rl] = 0.0;
      } else {
        late_load(Db, Ob, AB, ldab, q0, lq, p0, lp, b);
      }
      cta_sync();
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
      cta_sync();
      // B: vn = house(O[:, 0] - w), per warp
      double* vn = sm.vnw[warp];
      double taun = 0.0, betan;
      double swv;
      {
        const double wl0 = sm.w[lane], wl1 = sm.w[lane + 32];
        const double x0 = lane < lq ? Ob[lane] - wl0 : 0.0;
        const double x1 = lane + 32 < lq ? Ob[lane + 32] - wl1 : 0.0;
        // ||x[1:]||^2 and w[1:] . x[1:] reduced together (one shuffle latency chain)
        double ss = (lane >= 1 ? x0 * x0 : 0.0) + x1 * x1;
        double wx = (lane >= 1 ? wl0 * x0 : 0.0) + wl1 * x1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          ss += __shfl_xor_sync(0xffffffffu, ss, o);
          wx += __shfl_xor_sync(0xffffffffu, wx, o);
        }
        const double alpha = __shfl_sync(0xffffffffu, x0, 0);
        const double w00 = __shfl_sync(0xffffffffu, wl0, 0);
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
        swv = w00 + scale * wx;  // w . vn with vn = [1; scale x[1:]]
        __syncwarp();
      }
      // C: t = taun D vn, y = taun (O^T vn - v swv)
      {
        // D holds its lower triangle only: column mi from the diagonal down
        // (this phase's pattern) plus row mi left of the diagonal (phase A's
        // pattern) -- both conflict-free, no mirrored copy needed
        double tc = 0.0, gc = 0.0, ta = 0.0, tc1 = 0.0, gc1 = 0.0, ta1 = 0.0;
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const int r = rowC(q, i), r2 = rowC(q, i + 1);
          const double vr = vn[r], vr2 = vn[r2];
          const double dl = r >= mi ? Db[mi * kLd2 + r] : 0.0;
          const double dl2 = r2 >= mi ? Db[mi * kLd2 + r2] : 0.0;
          tc += dl * vr;
          tc1 += dl2 * vr2;
          gc += Ob[mi * kLd2 + r] * vr;
          gc1 += Ob[mi * kLd2 + r2] * vr2;
          const int c = colA(q, i), c2 = colA(q, i + 1);
          const double du = c < mi ? Db[c * kLd2 + mi] : 0.0;
          const double du2 = c2 < mi ? Db[c2 * kLd2 + mi] : 0.0;
          ta += du * vn[c];
          ta1 += du2 * vn[c2];
        }
        tc = (tc + tc1) + (ta + ta1);
        gc += gc1;
        tc += __shfl_xor_sync(0xffffffffu, tc, 1);
        tc += __shfl_xor_sync(0xffffffffu, tc, 2);
        gc += __shfl_xor_sync(0xffffffffu, gc, 1);
        gc += __shfl_xor_sync(0xffffffffu, gc, 2);
        if (q == 0) {
          sm.tt[mi] = taun * tc;
          sm.y[mi] = taun * (gc - v[mi] * swv);
        }
      }
      cta_sync();
      if (trs) T(3);
      const double gm = warp_sum(sm.tt[lane] * vn[lane] + sm.tt[lane + 32] * vn[lane + 32]);
      const double al = -0.5 * taun * gm;
      if (warp == 0) {
        if (lane == 0) dbg_delay<kDiag>(4, s, j);
        __syncwarp();
        // the successor's late data: row 0 of O'' and D''(0, 0) -- into the
        // mailbox when sweep s + 1 has a step j - 1 to consume it, else into
        // the band (ordered by this warp's `full` arrival below)
        const bool tomail = j >= 1 && s + 1 <= n - 3;
        unsigned long long* box = mail + ((size_t)(s % kMailRing) * maxsteps + j) * (2 * kMailSlots);
        const unsigned long long tag = mail_tag(s, j);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = lane + 32 * h;
          if (c < lp) {
            const double val = c == 0 ? betan : Ob[c * kLd2] - sm.w[0] * v[c] - sm.y[c];
            if (tomail) mail_put(box + 2 * c, val, tag);
            else AB[(long long)(p0 + c) * ldab + (q0 - p0 - c)] = val;
          }
        }
        if (lane == 0) {
          const double val = Db[0] - 2.0 * (sm.tt[0] + al);
          if (tomail) mail_put(box + 2 * lp, val, tag);
          else AB[(long long)q0 * ldab] = val;
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
      // D: the bulk of O'' and D'' (rows >= 1).  Lane l owns the 16-byte row
      // pair k = l + sh (rows 2k - sh, 2k - sh + 1: with the parity shift the
      // 32 pairs cover rows 1 .. 63) and keeps its row terms in registers;
      // warp w walks the columns w, 8 + w, ... (every warp the same share of
      // D's triangle), whose terms are broadcast loads.  One store instruction
      // writes 512 contiguous bytes of a band column.
      if constexpr (kDiag) {
        if (lane == 0 && (!(c_sb_mode & 128) || warp == 0) && (!(c_sb_mode & 256) || warp != 0))
          dbg_delay<kDiag>(8, s, (c_sb_mode & 64) ? j : j + warp);
        __syncwarp();
      }
      {
        const int r0 = 2 * lane + sh, r1 = r0 + 1;  // r0 >= 0, r1 <= 64
        const bool in0 = r0 >= 1 && r0 < lq, in1 = r1 < lq;
        const int r1c = r1 < kMaxPanel ? r1 : kMaxPanel - 1;
        const double w0 = sm.w[r0], w1 = sm.w[r1c];
        const double vn0 = vn[r0], vn1 = vn[r1c];
        const double u0 = sm.tt[r0] + al * vn0, u1 = sm.tt[r1c] + al * vn1;
#pragma unroll
        for (int i = 0; i < kMaxPanel / kBulkWarps; ++i) {
          const int c = kBulkWarps * i + warp;
          if (c < lp) {
            double o0 = 0.0, o1 = 0.0;
            if (c > 0) {
              const double2 ov = *reinterpret_cast<const double2*>(Ob + c * kLd2 + r0);
              const double vc = v[c], yc = sm.y[c];
              o0 = ov.x - w0 * vc - vn0 * yc;
              o1 = ov.y - w1 * vc - vn1 * yc;
            }
            double* od = AB + (long long)(p0 + c) * ldab + (q0 - p0 - c);
            if (in0 && in1) st_global_v2(od + r0, o0, o1);
            else if (in0) od[r0] = o0;
            else if (in1) od[r1] = o1;
          }
          if (c < lq) {
            const bool d0 = in0 && r0 >= c, d1 = in1 && r1 >= c;
            if (d0 || d1) {
              const double2 dv = *reinterpret_cast<const double2*>(Db + c * kLd2 + r0);
              const double vnc = vn[c], w2c = sm.tt[c] + al * vnc;
              const double e0 = dv.x - (vn0 * w2c + u0 * vnc);
              const double e1 = dv.y - (vn1 * w2c + u1 * vnc);
              double* dd = AB + (long long)(q0 + c) * ldab - c;
              if (d0 && d1) st_global_v2(dd + r0, e0, e1);
              else if (d0) dd[r0] = e0;
              else dd[r1] = e1;
            }
          }
        }
      }
      // each warp publishes its own bulk stores: full[s] reaches
      // kBulkWarps * (j + 1) once step j is completely stored
      if (kDiag && (c_sb_mode & 1)) {
        cta_sync();
        if (tid == 0) {
          __threadfence();
          atomicAdd(full + s, kBulkWarps);
        }
      } else {
        __syncwarp();
        if (lane == 0) red_release_add(full + s, 1);
      }
      if (trs) T(5);
      tau = taun;
      if (!has_next) break;
      if (trs) T(6);
      p0 = q0;
      lp = lq;
      q0 = nq0;
      q1 = nq1;
      lq = nlq;
    }
    cta_sync();
    if (tid == 0) {
      __threadfence();
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

// The band as the 2-D tensor T[j][x] = AB[(ldab - 1) j + x] (see stage_tma).
static bool band_map(CUtensorMap* map, double* AB, int ldab, int n) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr) != cudaSuccess ||
        qr != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<EncodeFn>(fn);
  }();
  if (!encode) return false;
  // x never exceeds n + kLd2; the boxes issued stay inside the allocation
  const cuuint64_t dims[2] = {(cuuint64_t)n + 2 * kMaxPanel, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)(ldab - 1) * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)kLd2, (cuuint32_t)kMaxPanel};
  const cuuint32_t estr[2] = {1u, 1u};
  const CUresult r = encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, AB, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  static bool warned = false;
  if (r != CUDA_SUCCESS && !warned) {
    warned = true;
    std::fprintf(stderr, "[bse] sb2st: tensor map rejected (%d), staging with per-thread copies\n", (int)r);
  }
  return r == CUDA_SUCCESS;
}

static size_t mail_offset_ints(int n) { return ((2 * (size_t)n + 3) / 4) * 4; }

size_t sb2st_progress_ints(int n, int b) {
  const size_t sweeps = (size_t)std::min(std::max(n, 1), kMailRing);
  return mail_offset_ints(n) + sweeps * sb2st_maxsteps(n, b) * kMailSlots * 4;
}

cudaError_t sb2st(double* AB, int ldab, int n, int b, double* d, double* e, double* V2,
                  double* tau2, int* progress, int num_sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t err;
  if (n > 2) {
    if ((err = cudaMemsetAsync(progress, 0, sizeof(int) * sb2st_progress_ints(n, b), s)) != cudaSuccess)
      return err;
    // mailboxes: 16-byte aligned, behind the 2n counters
    unsigned long long* mail = reinterpret_cast<unsigned long long*>(progress + mail_offset_ints(n));
    const size_t smem = sizeof(SbfSmem) + 128;
    static PerDeviceOnce attr, attr_diag;
    static const int sb_mode = std::getenv("BSE_SB2ST_MODE") ? std::atoi(std::getenv("BSE_SB2ST_MODE")) : 0;
    if ((err = sb_mode ? set_smem_limit(attr_diag, sb2st_fused_kernel<true>, (int)smem)
                       : set_smem_limit(attr, sb2st_fused_kernel<false>, (int)smem)) != cudaSuccess)
      return err;
    // one CTA per SM: the kernel is latency-bound and one resident step per
    // SM keeps every hand-off on an otherwise idle SM
    const int grid = std::max(1, std::min(n - 2, std::min(num_sms, kSbMaxGrid)));
    int maxsteps = sb2st_maxsteps(n, b);
    unsigned long long* trace = nullptr;
    const char* tenv = std::getenv("BSE_SB2ST_TRACE");
    const bool want_trace = tenv != nullptr;
    int ts0 = want_trace ? std::atoi(tenv) : 0;
    ts0 = std::max(0, std::min(ts0, n - 4));
    cudaMemcpyToSymbolAsync(c_sb_trace_s0, &ts0, sizeof(int), 0, cudaMemcpyHostToDevice, s);
    if (sb_mode) cudaMemcpyToSymbolAsync(c_sb_mode, &sb_mode, sizeof(int), 0, cudaMemcpyHostToDevice, s);
    const size_t tsz = (size_t)2 * maxsteps * 16;
    if (want_trace) {
      cudaMalloc(&trace, sizeof(unsigned long long) * tsz);
      cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * tsz, s);
    }
    CUtensorMap tmap;
    if (b != kMaxPanel || !band_map(&tmap, AB, ldab, n)) return cudaErrorNotSupported;
    void* args[] = {&tmap, &AB, &ldab, &n, &b, &V2, &tau2, &maxsteps, &progress, &mail, &trace};
    count_launch();
    err = cudaLaunchCooperativeKernel(sb_mode ? (const void*)sb2st_fused_kernel<true>
                                              : (const void*)sb2st_fused_kernel<false>,
                                      dim3(grid), dim3(kSbThreads + 32),
                                      args, smem, s);
    if (err != cudaSuccess) return err;
    if (want_trace) {
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
