// Recursive POTRF / TRSM built from 64-wide in-CTA leaves and the masked DMMA
// GEMM.  Recursion halves the problem so every off-diagonal update is one
// large GEMM (the blocked right-looking counterpart of the reference's
// left-looking GEMV loop, kernels.py:43-65).
#include <cstdlib>
#include "dense.cuh"
#include "ozgemm.cuh"

namespace bse {
namespace {

constexpr int kLeaf = 64;
constexpr int kLds = kLeaf + 1;

// --- POTF2: in-place lower Cholesky of an n x n (n <= 64) diagonal block ---
// A single-CTA leaf sits on the critical path of every recursion level, so it
// is written for latency with a small, rolled instruction stream: two threads
// per row keep its column halves in registers; the current column is always
// register 0 (the owning half shifts its registers once per column), so no
// register array is ever indexed dynamically.  Column j is broadcast through
// a double-buffered shared vector (one barrier per column) and the
// elimination runs unscaled (T_rc -= T_rj T_cj / T_jj; L_rc = T_rc / sqrt(T_cc)
// at the end).  The leaf inverse (cached for every TRSM leaf of the solve) is
// formed in the same loop by elimination of the identity.
constexpr int kHalf = kLeaf / 2;
__global__ void __launch_bounds__(2 * kLeaf) potf2_kernel(double* A, long long lda, int n, int off,
                                                          DevStatus* st, double* inv) {
  extern __shared__ double dyn[];
  double* Ls = dyn;                    // row-major, Ls[i * kLds + k]
  __shared__ double colj[2][kLeaf];
  __shared__ double rowj[2][kLeaf];    // row j of the unit-lower inverse
  __shared__ double dsq[kLeaf];
  if (st->info >= 0) return;           // an earlier block already failed
  const int r = threadIdx.x & (kLeaf - 1), h = threadIdx.x >> 6;
  const int cb = h * kHalf;            // this thread's columns: cb .. cb + 31
  double t[kHalf];
  // Y = (L diag(L)^-1)^-1 by forward elimination of the identity, in the same
  // column loop (row j of Y is final once column j is eliminated), so the
  // leaf inverse costs no extra barriers: L^-1 = diag(1/L_rr) Y.
  double y[kHalf];
#pragma unroll
  for (int q = 0; q < kHalf; ++q) {
    const int c = cb + q;
    t[q] = (r < n && c < n && c <= r) ? A[r + c * lda] : 0.0;
    y[q] = (c == r) ? 1.0 : 0.0;
  }
  for (int j = 0; j < n; ++j) {
    const int owner = j / kHalf;
    double* cj = colj[j & 1];
    double* yj = rowj[j & 1];
    if (h == owner) {
      cj[r] = t[0];
      Ls[r * kLds + j] = t[0];
    }
    if (inv && r == j) {
#pragma unroll
      for (int q = 0; q < kHalf; ++q) yj[cb + q] = y[q];
    }
    __syncthreads();
    const double piv = cj[j];
    if (!(piv > 0.0)) {  // uniform: every thread read the same value
      if (threadIdx.x == 0) { st->info = off + j; st->value = piv; }
      return;
    }
    if (threadIdx.x == 0) dsq[j] = sqrt(piv);
    // T_rj / T_jj = L_rj / L_jj
    const double a = (r > j) ? cj[r] * (1.0 / piv) : 0.0;
    // register q holds column base + q (base advances once per owned column)
    const int base = cb + (h == 0 ? j : max(0, j - kHalf));
#pragma unroll
    for (int q = 0; q < kHalf; ++q) {
      const int c = base + q;
      if (c > j && c <= r && c < cb + kHalf) t[q] -= a * cj[c];
    }
    if (inv) {
#pragma unroll
      for (int q = 0; q < kHalf; ++q)
        if (cb + q <= j) y[q] -= a * yj[cb + q];
    }
    if (h == owner) {
#pragma unroll
      for (int q = 0; q + 1 < kHalf; ++q) t[q] = t[q + 1];
      t[kHalf - 1] = 0.0;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && n > 0) {
    // smallest pivot L_jj^2 of this leaf -> st->aux (positive doubles order
    // like their bit patterns, so an integer atomicMin is a double min)
    double mn = dsq[0] * dsq[0];
    for (int j = 1; j < n; ++j) mn = fmin(mn, dsq[j] * dsq[j]);
    atomicMin(reinterpret_cast<unsigned long long*>(&st->aux),
              (unsigned long long)__double_as_longlong(mn));
  }
  // scale: L_rc = T_rc / sqrt(T_cc), write back
  for (int idx = threadIdx.x; idx < kLeaf * kLeaf; idx += blockDim.x) {
    const int i = idx & (kLeaf - 1), c = idx >> 6;  // i fastest: coalesced
    double l = 0.0;
    if (i < n && c < n) l = i > c ? Ls[i * kLds + c] / dsq[c] : (i == c ? dsq[c] : 0.0);
    if (i < n && c < n) A[i + c * lda] = l;
  }
  if (!inv) return;
  const double rd = (r < n) ? 1.0 / dsq[r] : 0.0;
#pragma unroll
  for (int q = 0; q < kHalf; ++q) {
    const int c = cb + q;
    inv[r + c * kLeaf] = (r < n && c < n) ? y[q] * rd : 0.0;
  }
}

// --- X L^T = A for a 64-row slab of A, L n x n (n <= 64) lower ---
__global__ void __launch_bounds__(kLeaf) trsm_rlt_leaf(const double* __restrict__ L, long long ldl,
                                                       int n, double* A, long long lda, int m) {
  extern __shared__ double dyn[];
  double* Ls = dyn;                  // row-major: Ls[j*kLds + i] = L[j][i]
  double* As = dyn + kLeaf * kLds;   // row-major: As[r*kLds + j]
  const int tid = threadIdx.x;
  const int r0 = blockIdx.x * kLeaf;
  for (int idx = tid; idx < n * n; idx += blockDim.x) {
    const int j = idx % n, i = idx / n;  // coalesced along j (rows of L)
    Ls[j * kLds + i] = (j >= i) ? L[j + i * ldl] : 0.0;
  }
  for (int j = 0; j < n; ++j) {
    const int r = r0 + tid;
    As[tid * kLds + j] = r < m ? A[r + j * lda] : 0.0;
  }
  __syncthreads();
  double* x = As + tid * kLds;
  for (int j = 0; j < n; ++j) {
    double s = x[j];
    const double* lj = Ls + j * kLds;
    for (int i = 0; i < j; ++i) s -= x[i] * lj[i];
    x[j] = s / lj[j];
  }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const int r = r0 + tid;
    if (r < m) A[r + j * lda] = As[tid * kLds + j];
  }
}

// --- L^T X = B (backward) or L X = B (forward) for a 64-column slab of B ---
template <bool TRANS>
__global__ void __launch_bounds__(kLeaf) trsm_left_leaf(const double* __restrict__ L, long long ldl,
                                                        int n, double* B, long long ldb, int ncols) {
  extern __shared__ double dyn[];
  double* Ls = dyn;                  // column-major: Ls[c*kLds + r] = L[r][c]
  double* Bs = dyn + kLeaf * kLds;   // per-column: Bs[c*kLds + i]
  const int tid = threadIdx.x;
  const int c0 = blockIdx.x * kLeaf;
  for (int idx = tid; idx < n * n; idx += blockDim.x) {
    const int r = idx % n, c = idx / n;
    Ls[c * kLds + r] = (r >= c) ? L[r + c * ldl] : 0.0;
  }
  for (int c = 0; c < kLeaf; ++c) {
    const int gc = c0 + c;
    for (int i = tid; i < n; i += blockDim.x) Bs[c * kLds + i] = gc < ncols ? B[i + gc * ldb] : 0.0;
  }
  __syncthreads();
  double* x = Bs + tid * kLds;
  if (TRANS) {  // L^T x = b: x_j = (b_j - sum_{i>j} L[i][j] x_i) / L[j][j]
    for (int j = n - 1; j >= 0; --j) {
      double s = x[j];
      const double* lc = Ls + j * kLds;  // column j of L
      for (int i = j + 1; i < n; ++i) s -= lc[i] * x[i];
      x[j] = s / lc[j];
    }
  } else {  // L x = b: x_j = (b_j - sum_{i<j} L[j][i] x_i) / L[j][j]
    for (int j = 0; j < n; ++j) {
      double s = x[j];
      for (int i = 0; i < j; ++i) s -= Ls[i * kLds + j] * x[i];
      x[j] = s / Ls[j * kLds + j];
    }
  }
  __syncthreads();
  for (int c = 0; c < kLeaf; ++c) {
    const int gc = c0 + c;
    if (gc >= ncols) break;
    for (int i = tid; i < n; i += blockDim.x) B[i + gc * ldb] = Bs[c * kLds + i];
  }
}

// --- inverse of an n x n (n <= 64) lower-triangular block: Y = L^{-1} ---
// One thread per column j: L y = e_j by forward substitution (exact zeros above j).
__global__ void __launch_bounds__(kLeaf) trtri_leaf(const double* __restrict__ L, long long ldl,
                                                    int n, double* __restrict__ Y) {
  __shared__ double Ls[kLeaf * kLds];  // column-major
  const int tid = threadIdx.x;
  for (int idx = tid; idx < n * n; idx += blockDim.x) {
    const int r = idx % n, c = idx / n;
    Ls[c * kLds + r] = (r >= c) ? L[r + c * ldl] : 0.0;
  }
  __syncthreads();
  const int j = tid;
  if (j < n) {
    double y[kLeaf];
#pragma unroll
    for (int i = 0; i < kLeaf; ++i) y[i] = 0.0;
#pragma unroll
    for (int i = 0; i < kLeaf; ++i) {
      if (i < j || i >= n) continue;
      double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < kLeaf; ++k)
        if (k >= j && k < i) s -= Ls[k * kLds + i] * y[k];
      y[i] = s / Ls[i * kLds + i];
    }
#pragma unroll
    for (int i = 0; i < kLeaf; ++i)
      if (i < n) Y[i + j * kLeaf] = y[i];
  }
}

__global__ void zero_upper_kernel(double* A, long long lda, int n) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y;
  if (r < n && r < c) A[r + (long long)c * lda] = 0.0;
}

__global__ void symmetrize_kernel(double* A, long long lda, int n) {
  // tile transpose of the lower triangle into the upper one; one CTA per
  // lower tile (bi >= bj), linear index k = bi (bi + 1) / 2 + bj
  __shared__ double t[32][33];
  const long long k = blockIdx.x;
  int bi = (int)((sqrt(8.0 * (double)k + 1.0) - 1.0) * 0.5);
  while ((long long)(bi + 1) * (bi + 2) / 2 <= k) ++bi;
  while ((long long)bi * (bi + 1) / 2 > k) --bi;
  const int bj = (int)(k - (long long)bi * (bi + 1) / 2);
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int q = ty; q < 32; q += 8) {
    const int r = bi * 32 + tx, c = bj * 32 + q;
    t[q][tx] = (r < n && c < n) ? A[r + (long long)c * lda] : 0.0;
  }
  __syncthreads();
  // write A[c][r] = A[r][c] for r > c
  for (int q = ty; q < 32; q += 8) {
    const int rr = bj * 32 + tx;  // destination row (= source col)
    const int cc = bi * 32 + q;   // destination col (= source row)
    if (rr < n && cc < n && cc > rr) A[rr + (long long)cc * lda] = t[tx][q];
  }
}

constexpr size_t kLeafSmem = 2 * kLeaf * kLds * sizeof(double);

template <auto Kern>
cudaError_t ensure_smem() {
  static PerDeviceOnce once;  // one flag set per kernel, one bit per device
  return set_smem_limit(once, Kern, (int)kLeafSmem);
}

// Per-device scratch for leaf inverses (64 x 64), allocated once.
double* leaf_scratch() {
  static double* bufs[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!bufs[dev]) cudaMalloc(&bufs[dev], sizeof(double) * kLeaf * kLeaf);
  return bufs[dev];
}

int split_point(int n) {
  int n1 = ((n / 2 + kLeaf - 1) / kLeaf) * kLeaf;
  if (n1 >= n) n1 = n - kLeaf;
  return n1;
}

}  // namespace

size_t potrf_inv_cache_doubles(int n) { return (size_t)ceil_div(n, kLeaf) * kLeaf * kLeaf; }

// C-block update on the emulated-FP64 engine when it is given and the
// product is large enough, else on the DMMA engine
static cudaError_t update(bool ta, bool tb, const GemmProblem& p, const OzWork* oz, cudaStream_t s) {
  if (oz && oz->p && (double)p.M * p.N * p.K >= oz_min_work())
    return ozgemm(ta, tb, p, oz->p, oz->bytes, oz->chunk, s);
  return gemm(ta, tb, p, s);
}

cudaError_t trsm_rlt(const double* L, long long ldl, int n, double* A, long long lda, int m,
                     cudaStream_t s, const double* inv, const OzWork* oz) {
  if (n <= 0 || m <= 0) return cudaSuccess;
  if (n <= kLeaf) {
    // A <- A * (L^{-1})^T : (cached) inverse of the block, then one in-place
    // DMMA GEMM (N = K = n <= BN: every CTA reads its full row slab first).
    const double* Y = inv;
    if (!Y) {
      double* Yw = leaf_scratch();
      trtri_leaf<<<1, kLeaf, 0, s>>>(L, ldl, n, Yw);
      count_launch();
      Y = Yw;
    }
    GemmProblem p = make_gemm(m, n, n, 1.0, A, lda, Y, kLeaf, 0.0, A, lda);
    p.mb = Mask::lower();
    return gemm(false, true, p, s);
  }
  const int n1 = split_point(n), n2 = n - n1;
  cudaError_t e = trsm_rlt(L, ldl, n1, A, lda, m, s, inv, oz);
  if (e != cudaSuccess) return e;
  // A2 -= X1 * L21^T
  GemmProblem p = make_gemm(m, n2, n1, -1.0, A, lda, L + n1, ldl, 1.0, A + n1 * lda, lda);
  e = update(false, true, p, oz, s);
  if (e != cudaSuccess) return e;
  return trsm_rlt(L + n1 + n1 * ldl, ldl, n2, A + n1 * lda, lda, m, s,
                  inv ? inv + (size_t)(n1 / kLeaf) * kLeaf * kLeaf : nullptr, oz);
}

size_t trsm_llt_oz_bytes(int n, int ncols, int chunk) {
  if (n <= kLeaf) return 0;
  const int n1 = split_point(n), n2 = n - n1;
  // the top-level update is the largest; deeper ones fit in its workspace
  return ozgemm_bytes(n1, ncols, n2, std::min(ncols, chunk));
}

cudaError_t trsm_llt(const double* L, long long ldl, int n, double* B, long long ldb, int ncols,
                     cudaStream_t s, const double* inv, const OzWork* oz, const RowHook* hook) {
  if (n <= 0 || ncols <= 0) return cudaSuccess;
  cudaError_t e;
  if (hook && (hook->depth <= 0 || n <= kLeaf)) {
    // report this whole row range once it is solved
    if ((e = trsm_llt(L, ldl, n, B, ldb, ncols, s, inv, oz, nullptr)) != cudaSuccess) return e;
    return hook->fn(hook->ctx, hook->base, hook->base + n, s);
  }
  if (n <= kLeaf) {
    const double* Y = inv;
    if (!Y) {
      double* Yw = leaf_scratch();
      trtri_leaf<<<1, kLeaf, 0, s>>>(L, ldl, n, Yw);
      count_launch();
      Y = Yw;
    }
    GemmProblem p = make_gemm(n, ncols, n, 1.0, Y, kLeaf, B, ldb, 0.0, B, ldb);
    p.ma = Mask::lower();
    return gemm(true, false, p, s);
  }
  const int n1 = split_point(n), n2 = n - n1;
  // rows [n1, n) are final after the first call (L^T is upper triangular)
  RowHook hb{}, ht{};
  if (hook) {
    hb = *hook; hb.depth -= 1; hb.base = hook->base + n1;
    ht = *hook; ht.depth -= 1;
  }
  e = trsm_llt(L + n1 + n1 * ldl, ldl, n2, B + n1, ldb, ncols, s,
               inv ? inv + (size_t)(n1 / kLeaf) * kLeaf * kLeaf : nullptr, oz, hook ? &hb : nullptr);
  if (e != cudaSuccess) return e;
  // B1 -= L21^T X2
  GemmProblem p = make_gemm(n1, ncols, n2, -1.0, L + n1, ldl, B + n1, ldb, 1.0, B, ldb);
  e = update(true, false, p, oz, s);
  if (e != cudaSuccess) return e;
  return trsm_llt(L, ldl, n1, B, ldb, ncols, s, inv, oz, hook ? &ht : nullptr);
}

cudaError_t trsm_lln(const double* L, long long ldl, int n, double* B, long long ldb, int ncols,
                     cudaStream_t s) {
  if (n <= 0 || ncols <= 0) return cudaSuccess;
  if (n <= kLeaf) {
    double* Y = leaf_scratch();
    trtri_leaf<<<1, kLeaf, 0, s>>>(L, ldl, n, Y);
    count_launch();
    GemmProblem p = make_gemm(n, ncols, n, 1.0, Y, kLeaf, B, ldb, 0.0, B, ldb);
    p.ma = Mask::lower();
    return gemm(false, false, p, s);
  }
  const int n1 = split_point(n), n2 = n - n1;
  cudaError_t e = trsm_lln(L, ldl, n1, B, ldb, ncols, s);
  if (e != cudaSuccess) return e;
  // B2 -= L21 X1
  GemmProblem p = make_gemm(n2, ncols, n1, -1.0, L + n1, ldl, B, ldb, 1.0, B + n1, ldb);
  e = gemm(false, false, p, s);
  if (e != cudaSuccess) return e;
  return trsm_lln(L + n1 + n1 * ldl, ldl, n2, B + n1, ldb, ncols, s);
}

int potrf_top_split(int n) { return n <= kLeaf ? n : split_point(n); }

static cudaError_t potrf_rec(double* A, long long lda, int n, int off, DevStatus* st,
                             cudaStream_t s, double* inv, const OzWork* oz,
                             const PotrfHook* hook = nullptr) {
  cudaError_t e;
  if (n <= kLeaf) {
    // a leaf still owing pieces: deliver them (in column order) first
    for (int L = 1; hook && L <= hook->depth; ++L)
      if ((e = hook->fn(hook->ctx, L, s)) != cudaSuccess) return e;
    if ((e = ensure_smem<potf2_kernel>()) != cudaSuccess) return e;
    potf2_kernel<<<1, 2 * kLeaf, kLeafSmem, s>>>(A, lda, n, off, st, inv);
    count_launch();
    return cudaGetLastError();
  }
  const int n1 = split_point(n), n2 = n - n1;
  // the top-left recursion owes the pieces below this level's
  PotrfHook inner{};
  const PotrfHook* ih = nullptr;
  if (hook && hook->depth > 1) {
    inner = *hook;
    inner.depth -= 1;
    ih = &inner;
  }
  e = potrf_rec(A, lda, n1, off, st, s, inv, oz, ih);
  if (e != cudaSuccess) return e;
  e = trsm_rlt(A, lda, n1, A + n1, lda, n2, s, inv, oz);  // A21 <- A21 L11^{-T}
  if (e != cudaSuccess) return e;
  // columns [n1, n) are first touched here (the host entry streams them in)
  if (hook && (e = hook->fn(hook->ctx, hook->depth, s)) != cudaSuccess) return e;
  // A22 -= A21 A21^T (lower triangle only)
  double* A21 = A + n1;
  double* A22 = A + n1 + n1 * lda;
  {
    // lower triangle only: the DMMA engine skips masked tiles, and so does the
    // emulated engine's contraction kernel (256-wide tiles above the diagonal
    // are never issued; the CRT pass skips masked entries)
    GemmProblem p = make_gemm(n2, n2, n1, -1.0, A21, lda, A21, lda, 1.0, A22, lda);
    p.mc = Mask::lower();
    static const bool half_rule = std::getenv("BSE_POTRF_OZ_OLD") == nullptr;
    const bool big = (double)n2 * n2 * n1 >= (half_rule ? 2.0 : 4.0) * oz_min_work();
    if ((e = big ? update(false, true, p, oz, s) : gemm(false, true, p, s)) != cudaSuccess) return e;
  }
  return potrf_rec(A + n1 + n1 * lda, lda, n2, off + n1, st, s,
                   inv ? inv + (size_t)(n1 / kLeaf) * kLeaf * kLeaf : nullptr, oz);
}

cudaError_t potrf_lower(double* A, long long lda, int n, DevStatus* st, cudaStream_t s,
                        double* inv_cache, const OzWork* oz, const PotrfHook* hook) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = potrf_rec(A, lda, n, 0, st, s, inv_cache, oz, hook);
  if (e != cudaSuccess) return e;
  return zero_strict_upper(A, lda, n, s);
}

cudaError_t potrf_lower_at(double* A, long long lda, int n, int off, DevStatus* st, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  cudaError_t e = potrf_rec(A, lda, n, off, st, s, nullptr, nullptr, nullptr);
  if (e != cudaSuccess) return e;
  return zero_strict_upper(A, lda, n, s);
}

cudaError_t zero_strict_upper(double* A, long long lda, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  zero_upper_kernel<<<dim3((unsigned)ceil_div(n, 256), (unsigned)n), 256, 0, s>>>(A, lda, n);
  count_launch();
  return cudaGetLastError();
}

cudaError_t symmetrize_from_lower(double* A, long long lda, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const unsigned t = (unsigned)ceil_div(n, 32);
  symmetrize_kernel<<<(unsigned)((long long)t * (t + 1) / 2), dim3(32, 8), 0, s>>>(A, lda, n);
  count_launch();
  return cudaGetLastError();
}

}  // namespace bse
