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
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include "eig.cuh"

namespace bse {
namespace {

constexpr int kPanelThreads = 256;

// Householder QR of the m x bw panel P (column-major, ldp), rows split over
// gridDim.x CTAs; CTA c owns rows [c*R, c*R + R) with R = RPT * 256 and
// thread t owns rows t, t + 256, ... (row-major slab in smem, stride bw+1:
// a warp touching one column of 32 consecutive rows is conflict-free).
// Per column j: one fused CTA reduction (products of every column with x_j,
// ||tail||^2, the owner's row j) -> mailbox exchange -> a fixed-order sum of
// the G partials -> rank-1 update of the thread's own rows.  Outputs:
//   P  <- R in its upper bw x bw triangle, zeros below
//   V  (ldv), V2 (ldv2): explicit unit-lower-trapezoidal reflectors
//   T  (bw x bw, ld bw): compact-WY factor, Q = I - V T V^T
template <int RPT>
__global__ void __launch_bounds__(kPanelThreads) panel_qr_kernel(
    double* __restrict__ P, long long ldp, int m, int bw, double* __restrict__ V, long long ldv,
    double* __restrict__ V2, long long ldv2, double* __restrict__ T, double* __restrict__ red,
    unsigned epoch, unsigned long long* trace) {
  constexpr int R = RPT * kPanelThreads;
  constexpr int LS = kMaxPanel + 1;   // row stride
  constexpr int L = 2 + 2 * kMaxPanel;
  extern __shared__ double smem[];
  double* S = smem;                       // [r*LS + k]
  double* wpart = S + (size_t)R * LS;     // [warp][L] per-warp partials
  double* tot = wpart + 8 * L;            // reduced values
  double* wv = tot + L;                   // w_k / y_i
  double* Ts = wv + kMaxPanel;            // T (CTA 0), [j*bw + i]
  __shared__ double sc[4];
  __shared__ double gsum[3][2 + kMaxPanel];  // part sums of the exchange
  const bool tr = trace != nullptr && blockIdx.x == 0 && threadIdx.x == 0;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, cta = blockIdx.x;
  const int r0 = cta * R;
  const int rows = max(0, min(R, m - r0));

  for (int q = 0; q < RPT; ++q) {
    const int r = tid + q * kPanelThreads;
    for (int k = 0; k < kMaxPanel; ++k)
      S[r * LS + k] = (r < rows && k < bw) ? P[(r0 + r) + (long long)k * ldp] : 0.0;
  }
  if (cta == 0)
    for (int idx = tid; idx < bw * bw; idx += blockDim.x) Ts[idx] = 0.0;
  __syncthreads();

  for (int j = 0; j < bw; ++j) {
    unsigned long long t0 = 0, t1 = 0, t2 = 0, t3 = 0;
    if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    // ---- per-thread products over owned rows with global index >= j ----
    double pk[kMaxPanel];
    double tail = 0.0;
#pragma unroll
    for (int k = 0; k < kMaxPanel; ++k) pk[k] = 0.0;
    for (int q = 0; q < RPT; ++q) {
      const int r = tid + q * kPanelThreads;
      const int gr = r0 + r;
      if (r < rows && gr >= j) {
        const double* row = S + r * LS;
        const double xj = row[j];
#pragma unroll
        for (int k = 0; k < kMaxPanel; ++k) pk[k] += row[k] * xj;
        if (gr > j) tail += xj * xj;
      }
    }
    // warp reduce-scatter butterfly over the 64 products (62 shuffles per
    // lane instead of 64 full reductions): after step o the lanes with bit o
    // set keep the upper half of the remaining values
#pragma unroll
    for (int h = kMaxPanel / 2, o = 16; o >= 1; h >>= 1, o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < h; ++i) {
        const double send = up ? pk[i] : pk[i + h];
        const double keep = up ? pk[i + h] : pk[i];
        pk[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    tail = warp_sum(tail);
    {
      const int base = ((lane >> 4) & 1) * 32 + ((lane >> 3) & 1) * 16 + ((lane >> 2) & 1) * 8 +
                       ((lane >> 1) & 1) * 4 + (lane & 1) * 2;
      wpart[warp * L + 2 + base] = pk[0];
      wpart[warp * L + 2 + base + 1] = pk[1];
      if (lane == 0) wpart[warp * L] = tail;
    }
    __syncthreads();
    // CTA partial: [0] tail, [1] x0 (owner), [2+k] dots, [2+bw+k] owner's row j
    const bool owner = (j >= r0 && j < r0 + rows);
    // The exchange across CTAs goes through self-validating mailbox slots
    // (common.cuh), double-buffered by column parity: every CTA stores its L
    // partials and then polls the others' -- no grid barrier, no fences, one
    // L2 round trip.  A CTA can only be two columns ahead of another after
    // that one has read the buffer being reused.
    unsigned long long* box = reinterpret_cast<unsigned long long*>(red) + (size_t)(j & 1) * G * L * 2;
    const unsigned long long tag = mail_tag((int)epoch, j);
    for (int t = tid; t < L; t += blockDim.x) {
      double v;
      if (t == 1) {
        v = owner ? S[(j - r0) * LS + j] : 0.0;
      } else if (t >= 2 + kMaxPanel) {
        v = owner ? S[(j - r0) * LS + (t - 2 - kMaxPanel)] : 0.0;
      } else {
        v = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) v += wpart[w * L + t];
      }
      if (G > 1) mail_put(box + 2 * ((size_t)cta * L + t), v, tag);
      else tot[t] = v;
    }
    if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (G > 1) {
      // sums over the CTAs (fixed order): values [0, NV) by three threads each
      // (a third of the CTAs, up to 24 loads in flight); the first 64 of these
      // threads also fetch the owner's row (one more load in the same batch)
      constexpr int NV = 2 + kMaxPanel;
      constexpr int NP = 3, CH = 24;
      auto ld2 = [](unsigned long long& a, unsigned long long& b, const unsigned long long* sl) {
        asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(a), "=l"(b) : "l"(sl) : "memory");
      };
      if (tid < NP * NV) {
        const int t = tid % NV, part = tid / NV;
        const int per = (G + NP - 1) / NP;
        const int lo = part * per, hi = min(G, lo + per);
        const bool own = tid < kMaxPanel;
        const unsigned long long* osl = box + 2 * ((size_t)(j / R) * L + NV + tid);
        unsigned long long ol = 0, oh = 0;
        if (own) ld2(ol, oh, osl);
        double acc = 0.0;
        for (int c0 = lo; c0 < hi; c0 += CH) {
          unsigned long long l[CH], h[CH];
          bool ok;
          do {
            ok = true;
#pragma unroll
            for (int u = 0; u < CH; ++u)
              if (c0 + u < hi) ld2(l[u], h[u], box + 2 * ((size_t)(c0 + u) * L + t));
#pragma unroll
            for (int u = 0; u < CH; ++u)
              if (c0 + u < hi) ok = ok && ((l[u] ^ h[u]) == tag);
          } while (!ok);
#pragma unroll
          for (int u = 0; u < CH; ++u)
            if (c0 + u < hi) acc += __longlong_as_double((long long)l[u]);
        }
        gsum[part][t] = acc;
        if (own) {
          while ((ol ^ oh) != tag) ld2(ol, oh, osl);
          tot[NV + tid] = __longlong_as_double((long long)ol);
        }
      }
      if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t2));
      __syncthreads();
      if (tid < NV) tot[tid] = (gsum[0][tid] + gsum[1][tid]) + gsum[2][tid];
    }
    __syncthreads();
    if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t3));
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
    if (tid < bw) {
      // provisional; scaled below once tau/beta are known (same thread order)
    }
    __syncthreads();
    const double tau = sc[0], beta = sc[1], scale = sc[2];
    if (tid < bw) wv[tid] = (tot[2 + tid] - beta * tot[2 + kMaxPanel + tid]) * scale;
    __syncthreads();
    // ---- rank-1 update of the owned rows (columns > j), store v_j ----
    for (int q = 0; q < RPT; ++q) {
      const int r = tid + q * kPanelThreads;
      const int gr = r0 + r;
      if (r < rows && gr >= j) {
        double* row = S + r * LS;
        if (tau != 0.0) {
          const double vr = (gr == j) ? 1.0 : row[j] * scale;
          const double tv = tau * vr;
          for (int k = j + 1; k < bw; ++k) row[k] -= tv * wv[k];
          row[j] = (gr == j) ? beta : vr;
        } else if (gr > j) {
          row[j] = 0.0;
        }
      }
    }
    // ---- T column j (CTA 0): T[j][j] = tau, T[i][j] = -tau sum_k T[i][k] y_k ----
    if (cta == 0 && tid < bw) {
      const int i = tid;
      if (i < j) {
        double sacc = 0.0;
        for (int k = i; k < j; ++k) sacc += Ts[k * bw + i] * wv[k];
        Ts[j * bw + i] = -tau * sacc;
      } else if (i == j) {
        Ts[j * bw + j] = tau;
      }
    }
    __syncthreads();
    if (tr) {
      unsigned long long t4;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t4));
      trace[5 * j + 0] = t1 - t0; trace[5 * j + 1] = t2 ? t2 - t1 : 0;
      trace[5 * j + 2] = t3 - (t2 ? t2 : t1); trace[5 * j + 3] = t4 - t3; trace[5 * j + 4] = 1;
    }
  }

  // ---- write back R (upper), explicit V (unit lower) ----
  for (int idx = tid; idx < rows * bw; idx += blockDim.x) {
    const int r = idx % rows, k = idx / rows;
    const int gr = r0 + r;
    const double sv = S[r * LS + k];
    P[gr + (long long)k * ldp] = (gr <= k) ? sv : 0.0;
    const double v = (gr > k) ? sv : (gr == k ? 1.0 : 0.0);
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
  (void)bw;
  constexpr int L = 2 + 2 * kMaxPanel;
  return sizeof(double) * ((size_t)R * (kMaxPanel + 1) + 8 * L + L + kMaxPanel +
                           (size_t)kMaxPanel * kMaxPanel);
}

cudaError_t panel_qr(double* P, long long ldp, int m, int bw, double* V, long long ldv, double* V2,
                     long long ldv2, double* T, double* red, unsigned* bar, int num_sms,
                     cudaStream_t s) {
  // one slab row per thread (RPT = 1) while that keeps G <= #SMs, else two
  const int rpt = ((long long)kPanelThreads * num_sms >= m) ? 1 : 2;
  const int R = rpt * kPanelThreads;
  const int G = (int)ceil_div(m, R);
  if (G > num_sms) return cudaErrorInvalidValue;
  const size_t smem = panel_smem_bytes(R, bw);
  // largest limit set so far, per (variant, device): the attribute is per device
  static std::atomic<size_t> attr[3][64];
  void* fn = rpt == 1 ? (void*)panel_qr_kernel<1> : (void*)panel_qr_kernel<2>;
  std::atomic<size_t>& lim = attr[rpt][PerDeviceOnce::ordinal()];
  if (smem > lim.load()) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    lim.store(smem);
  }
  (void)bar;  // the exchange needs no barrier counter
  // tags are unique per launch: the mailbox buffer is reused without clearing
  static std::atomic<unsigned> epoch_ctr{1};
  unsigned epoch = epoch_ctr.fetch_add(1);
  static unsigned long long* trace = nullptr;
  static int traced = 0;
  const bool want = std::getenv("BSE_PANEL_TRACE") != nullptr && traced == 0 && m > 8000;
  unsigned long long* tptr = nullptr;
  if (want) {
    cudaMalloc(&trace, sizeof(unsigned long long) * 5 * 64);
    cudaMemsetAsync(trace, 0, sizeof(unsigned long long) * 5 * 64, s);
    tptr = trace;
  }
  void* args[] = {&P, &ldp, &m, &bw, &V, &ldv, &V2, &ldv2, &T, &red, &epoch, &tptr};
  count_launch();
  cudaError_t le;
  if (G == 1)
    le = cudaLaunchKernel(fn, dim3(1), dim3(kPanelThreads), args, smem, s);
  else
    le = cudaLaunchCooperativeKernel(fn, dim3(G), dim3(kPanelThreads), args, smem, s);
  if (want) {
    traced = 1;
    unsigned long long h[5 * 64];
    cudaMemcpyAsync(h, trace, sizeof(h), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    double a[4] = {0};
    for (int j = 0; j < 64; ++j)
      for (int q = 0; q < 4; ++q) a[q] += h[5 * j + q];
    std::fprintf(stderr, "[panel trace] m=%d G=%d R=%d per column us: local %.2f barrier %.2f "
                 "reduce %.2f update %.2f\n", m, G, R, a[0] / 64e3, a[1] / 64e3, a[2] / 64e3,
                 a[3] / 64e3);
  }
  return le;
}

cudaError_t extract_band(const double* A, long long lda, int n, int b, double* AB, int ldab,
                         cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  extract_band_kernel<<<n, 128, 0, s>>>(A, lda, n, b, AB, ldab);
  count_launch();
  return cudaGetLastError();
}

namespace {

// Y (m x b, in w.y) = A2 V with A2 symmetric (lower triangle referenced),
// as two masked split-K GEMMs (the triangular masks give row blocks very
// different k-ranges; splitting K balances them and fills the GPU).
cudaError_t symm_panel(const double* A2, long long lda, int m, int bw, const double* V,
                       long long ldv, const Sy2sbScratch& w, cudaStream_t s, bool full = false) {
  const int ssplit = (int)std::min<long long>(kSymmSplits, std::max<long long>(1, m / 1024));
  if (full) {
    // A2 holds both triangles (symmetrised once per pair): one unmasked product
    GemmProblem g = make_gemm(m, bw, m, 1.0, A2, lda, V, ldv, 0.0, w.y, w.ldy);
    return gemm_splitk(false, false, g, ssplit, w.symm_ws, w.probs, s);
  }
  GemmProblem g1 = make_gemm(m, bw, m, 1.0, A2, lda, V, ldv, 0.0, w.y, w.ldy);
  g1.ma = Mask::lower();
  cudaError_t e = gemm_splitk(false, false, g1, ssplit, w.symm_ws, w.probs, s);
  if (e != cudaSuccess) return e;
  GemmProblem g2 = make_gemm(m, bw, m, 1.0, A2, lda, V, ldv, 1.0, w.y, w.ldy);
  g2.ma = Mask::strict_lower();
  return gemm_splitk(true, false, g2, ssplit, w.symm_ws, w.probs + 32, s);
}

}  // namespace

// W = X - 1/2 V (T^T (V^T X)), X = Y T  (Y in w.y): the two-sided update
// A - V W^T - W V^T of one panel (compact WY, LAPACK dsytrd's LATRD form).
cudaError_t panel_w(int m, int bw, const double* V, long long ldv, const double* Tp, double* W,
                    long long ldw, const Sy2sbScratch& w, cudaStream_t s) {
  cudaError_t e;
  GemmProblem g3 = make_gemm(m, bw, bw, 1.0, w.y, w.ldy, Tp, bw, 0.0, W, ldw);
  g3.mb = Mask::upper();
  if ((e = gemm(false, false, g3, s)) != cudaSuccess) return e;
  stage_mark("sy2sb_small", s);
  GemmProblem g4 = make_gemm(bw, bw, m, 1.0, V, ldv, W, ldw, 0.0, w.z, bw);
  const int splits = (int)std::min<long long>(48, std::max<long long>(1, m / 256));
  if ((e = gemm_splitk(true, false, g4, splits, w.splitk_ws, w.probs + 64, s)) != cudaSuccess) return e;
  GemmProblem g5 = make_gemm(bw, bw, bw, 1.0, Tp, bw, w.z, bw, 0.0, w.z2, bw);
  g5.ma = Mask::upper();
  if ((e = gemm(true, false, g5, s)) != cudaSuccess) return e;
  GemmProblem g6 = make_gemm(m, bw, bw, -0.5, V, ldv, w.z2, bw, 1.0, W, ldw);
  return gemm(false, false, g6, s);
}

// Full -> band.  A (n x n, lower triangle referenced) is overwritten: its
// lower band holds the band matrix, panel regions hold R, rest is garbage.
// Vall (ldv): reflectors of panel p at rows k+b.., cols k..k+b-1 (k = p*b);
// Tall: bw x bw T factors, one per panel.
//
// Panels are processed in PAIRS with one aggregated rank-4b trailing update
// (the band analogue of LAPACK's LATRD look-ahead): after panel p only the
// next panel's b columns are updated; panel p+1's SYMM runs on the stale
// trailing matrix and is corrected with two thin products,
//   A3_true V2 = A3 V2 - V1' (W1'^T V2) - W1' (V1'^T V2),
// and the trailing matrix is then updated once,
//   A3 -= [V1' V2 W1' W2] [W1' W2 V1' V2]^T   (lower, K = 4b),
// halving the read-modify-write passes of the SYR2K and doubling its depth.
// Scratch slots (ld lw, b columns each): V1 W1 V2 W2 | W1c V1c W2c V2c (the
// right half copies the left in swapped pairs), the second panel's columns
// sit b rows down so every slot shares the trailing row index.  Then
// [V1 W1] [W1c V1c]^T, [W1c V1c]^T V2 and [V1 W1 V2 W2] [W1c V1c W2c V2c]^T
// are single GEMMs.
bool sy2sb_full_symm() {
  static const bool off = std::getenv("BSE_SY2SB_TRI_SYMM") != nullptr;  // A/B timing switch
  return !off;
}

cudaError_t sy2sb(double* A, long long lda, int n, int b, double* Vall, long long ldv,
                  double* Tall, const Sy2sbScratch& w, int num_sms, cudaStream_t s,
                  cudaStream_t la, cudaEvent_t ev_cols, cudaEvent_t ev_panel) {
  cudaError_t e = cudaSuccess;
  const int bw = b;
  const long long lw = w.ldvwv;
  // two sets of 8 slots: the look-ahead panel of the next pair writes its V
  // into the other set while this pair's trailing update still reads V1/W1
  double* slots[2][8];
  for (int q = 0; q < 2; ++q)
    for (int i = 0; i < 8; ++i) slots[q][i] = w.vwv + (q * 8 + i) * lw * bw;
  auto copy_cols = [&](double* dst, const double* src, int rows) {
    return cudaMemcpy2DAsync(dst, lw * sizeof(double), src, lw * sizeof(double),
                             (size_t)rows * sizeof(double), bw, cudaMemcpyDeviceToDevice, s);
  };
  bool panel_ready = false;  // this pair's first panel was factored by the look-ahead
  for (int p = 0, set = 0;; p += 2, set ^= 1) {
    double *sV1 = slots[set][0], *sW1 = slots[set][1], *sV2 = slots[set][2], *sW2 = slots[set][3];
    double *sW1c = slots[set][4], *sV1c = slots[set][5], *sW2c = slots[set][6], *sV2c = slots[set][7];
    const int k = p * b;
    const int m = n - k - b;
    if (m < 2) break;
    double* P1 = A + (k + b) + (long long)k * lda;
    double* A2 = A + (k + b) + (long long)(k + b) * lda;
    double* Tp1 = Tall + (size_t)p * b * b;
    stage_mark("sy2sb_panel", s);
    if (panel_ready) {
      if ((e = cudaStreamWaitEvent(s, ev_panel, 0)) != cudaSuccess) return e;
    } else {
      e = panel_qr(P1, lda, m, bw, Vall + (k + b) + (long long)k * ldv, ldv, sV1, lw, Tp1, w.red,
                   w.bar, num_sms, s);
      if (e != cudaSuccess) return e;
    }
    panel_ready = false;
    stage_mark("sy2sb_symm", s);
    // both SYMMs of the pair read the trailing matrix as it stands now (the
    // second one on its stale sub-block A3): mirror its lower triangle once
    // (mirrored once for the first pair; afterwards the trailing update's
    // epilogue stores both triangles of the next pair's A2)
    const bool full = sy2sb_full_symm();
    static const bool epi_mirror = std::getenv("BSE_SY2SB_NO_EPI_MIRROR") == nullptr;  // A/B switch
    if (full && (p == 0 || !epi_mirror) && (e = symmetrize_from_lower(A2, lda, m, s)) != cudaSuccess)
      return e;
    if ((e = symm_panel(A2, lda, m, bw, sV1, lw, w, s, full)) != cudaSuccess) return e;
    if ((e = panel_w(m, bw, sV1, lw, Tp1, sW1, lw, w, s)) != cudaSuccess) return e;
    if ((e = copy_cols(sW1c, sW1, m)) != cudaSuccess) return e;
    if ((e = copy_cols(sV1c, sV1, m)) != cudaSuccess) return e;
    const int m2 = m - b;
    if (m2 < 2) {
      // last panel: plain rank-2b update A2 -= [V1 W1] [W1 V1]^T
      stage_mark("sy2sb_syr2k", s);
      GemmProblem g = make_gemm(m, m, 2 * bw, -1.0, sV1, lw, sW1c, lw, 1.0, A2, lda);
      g.mc = Mask::lower();
      if ((e = gemm(false, true, g, s)) != cudaSuccess) return e;
      break;
    }
    stage_mark("sy2sb_small", s);
    // next panel block (and the diagonal block above it):
    // A2[:, 0:b] -= [V1 W1] [W1 V1][0:b, :]^T
    {
      GemmProblem g = make_gemm(m, bw, 2 * bw, -1.0, sV1, lw, sW1c, lw, 1.0, A2, lda);
      g.mc = Mask::lower();
      if ((e = gemm(false, true, g, s)) != cudaSuccess) return e;
    }
    // panel p+1 on the updated columns
    double* P2 = A2 + b;  // rows k+2b.., cols k+b..k+2b-1
    double* A3 = A2 + b + (long long)b * lda;
    double* Tp2 = Tall + (size_t)(p + 1) * b * b;
    stage_mark("sy2sb_panel", s);
    e = panel_qr(P2, lda, m2, bw, Vall + (k + 2 * b) + (long long)(k + b) * ldv, ldv, sV2 + b, lw,
                 Tp2, w.red, w.bar, num_sms, s);
    if (e != cudaSuccess) return e;
    stage_mark("sy2sb_symm", s);
    if ((e = symm_panel(A3, lda, m2, bw, sV2 + b, lw, w, s, full)) != cudaSuccess) return e;
    stage_mark("sy2sb_small", s);
    {
      // Y2 -= [V1' W1'] S,  S = [W1' V1']^T V2  (2b x b, split-K into z:z2)
      const int splits = (int)std::min<long long>(48, std::max<long long>(1, m2 / 256));
      GemmProblem g = make_gemm(2 * bw, bw, m2, 1.0, sW1c + b, lw, sV2 + b, lw, 0.0, w.z, 2 * bw);
      if ((e = gemm_splitk(true, false, g, splits, w.splitk_ws, w.probs + 64, s)) != cudaSuccess)
        return e;
      GemmProblem c = make_gemm(m2, bw, 2 * bw, -1.0, sV1 + b, lw, w.z, 2 * bw, 1.0, w.y, w.ldy);
      if ((e = gemm(false, false, c, s)) != cudaSuccess) return e;
    }
    if ((e = panel_w(m2, bw, sV2 + b, lw, Tp2, sW2 + b, lw, w, s)) != cudaSuccess) return e;
    if ((e = copy_cols(sW2c + b, sW2 + b, m2)) != cudaSuccess) return e;
    if ((e = copy_cols(sV2c + b, sV2 + b, m2)) != cudaSuccess) return e;
    // one rank-4b trailing update: A3 -= [V1' W1' V2 W2] [W1' V1' W2 V2]^T (lower)
    stage_mark("sy2sb_syr2k", s);
    // Look-ahead: the next pair's first panel lives in A3's first b columns.
    // Update those first, factor the panel on the (high-priority) look-ahead
    // stream -- the panel kernel needs at most m/256 SMs -- while the rest of
    // the trailing update runs here.
    const int kn = k + 2 * b, mn = n - kn - b;
    const bool ahead = la && mn >= 2 && (long long)kPanelThreads * num_sms >= mn;
    if (ahead) {
      GemmProblem ga = make_gemm(m2, bw, 4 * bw, -1.0, sV1 + b, lw, sW1c + b, lw, 1.0, A3, lda);
      ga.mc = Mask::lower();
      if ((e = gemm(false, true, ga, s)) != cudaSuccess) return e;
      if ((e = cudaEventRecord(ev_cols, s)) != cudaSuccess) return e;
      if ((e = cudaStreamWaitEvent(la, ev_cols, 0)) != cudaSuccess) return e;
      double* Pn = A + (kn + b) + (long long)kn * lda;
      e = panel_qr(Pn, lda, mn, bw, Vall + (kn + b) + (long long)kn * ldv, ldv, slots[set ^ 1][0],
                   lw, Tall + (size_t)(p + 2) * b * b, w.red, w.bar, num_sms, la);
      if (e != cudaSuccess) return e;
      if ((e = cudaEventRecord(ev_panel, la)) != cudaSuccess) return e;
      panel_ready = true;
      // rest: rows b.., columns b.. of A3 (lower)
      GemmProblem gb = make_gemm(m2 - b, m2 - b, 4 * bw, -1.0, sV1 + 2 * b, lw, sW1c + 2 * b, lw,
                                 1.0, A3 + b + (long long)b * lda, lda);
      gb.mc = Mask::lower();
      gb.mirror = full && epi_mirror;
      if ((e = gemm(false, true, gb, s)) != cudaSuccess) return e;
    } else {
      GemmProblem g7 = make_gemm(m2, m2, 4 * bw, -1.0, sV1 + b, lw, sW1c + b, lw, 1.0, A3, lda);
      g7.mc = Mask::lower();
      g7.mirror = full && epi_mirror;
      if ((e = gemm(false, true, g7, s)) != cudaSuccess) return e;
    }
  }
  return e;
}

}  // namespace bse
