// Memory-distributed product-form BSE solve over a 1 x Q block-cyclic column
// layout (dist.cuh).  Same step order as the single-GPU pipeline and the
// reference's solvers (solvers.py:97-104): Cholesky -> congruence ->
// eigendecomposition -> back-transform -> scale; the paper's own distributed
// algorithm uses the same block-cyclic building blocks on
// a CPU cluster.
#include <algorithm>
#include <cmath>
#include <vector>
#include "dist.cuh"
#include "eig.cuh"
#include "ozgemm.cuh"

namespace bse {
namespace {

constexpr int kBand = 64;
constexpr int kQ2Group = 32;
constexpr int kQ2RangeGroups = 64;  // sweep groups per Q2 block range (even)
constexpr int kQ1Cols = 4096;       // columns of V per Q1 group on the emulated engine

constexpr int kDistOzChunk = 2048;   // output columns per emulated-engine pass

int q1_group_tiles(int nb, bool oz) { return oz ? std::max(1, kQ1Cols / nb) : 1; }

// Large products of the distributed stages go to the emulated-FP64 engine
// (same rule as the single-GPU pipeline: at least oz_min_work multiply-adds
// and a workspace that holds the call), the rest to the DMMA engine.
struct OzBuf {
  void* p = nullptr;
  size_t bytes = 0;
};
cudaError_t mm(bool ta, bool tb, const GemmProblem& g, const OzBuf& oz, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (oz.p && g.K > 0 && (double)g.M * g.N * g.K >= oz_min_work() &&
      ozgemm_bytes(g.M, g.N, g.K, kDistOzChunk) <= oz.bytes)
    return ozgemm(ta, tb, g, oz.p, oz.bytes, kDistOzChunk, s);
  return gemm(ta, tb, g, s);
}
// workspace for every panel product of shape (n x cols x nb) or (nb x cols x n)
size_t panel_oz_bytes(int n, int nb, int cols) {
  return std::max(ozgemm_bytes(n, cols, nb, kDistOzChunk), ozgemm_bytes(nb, cols, n, kDistOzChunk));
}
bool dist_oz(int n, int flags) { return !(flags & kFlagNativeFp64) && n >= kOzMinN; }

// ---------------------------------------------------------------------------
// small kernels

// L(:, lc) = tril(K)(:, g(lc)) for this rank's columns
__global__ void copy_lower_bc_kernel(BcLayout lay, int nloc, const double* K, long long ldk,
                                     double* L, long long ld) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)lay.n * nloc) return;
  const int r = (int)(idx % lay.n), lc = (int)(idx / lay.n);
  const int g = lay.global_col(lc, lay.rank);
  L[r + (long long)lc * ld] = r >= g ? K[r + (long long)lc * ldk] : 0.0;
}

// red[rank] = failing pivot index (or 4e18), red[world + rank] = its value,
// red[2 world + rank] = min pivot; zeros elsewhere (summed over the ranks)
__global__ void status_pack_kernel(const DevStatus* st, int world, int rank, double* red) {
  const int t = threadIdx.x;
  if (t >= 3 * world) return;
  double v = 0.0;
  if (t == rank) v = st->info >= 0 ? (double)st->info : 4e18;
  if (t == world + rank) v = st->info >= 0 ? st->value : 0.0;
  if (t == 2 * world + rank) v = st->aux;
  red[t] = v;
}

// Per-panel GEMM descriptors of the distributed band reduction, one thread
// per local tile lt (global tile lt * world + rank): the tile's trailing
// columns [c0, c1) = [max(tile start, k + b), tile end).
//   y1[lt]: slot_lt[roff:, :]   = tril(A[c0:, c0:c1]) V[roff:roff+cw, :]
//   y2[lt]: Y2[roff:roff+cw, :] = stril(A[c0:, c0:c1])^T V[roff:, :]
//   up[lt]: A[c0:, c0:c1]      -= [V W][roff:, :] ([W V][roff:roff+cw, :])^T  (lower)
// (roff = c0 - (k + b): row index in the panel's coordinates)
__global__ void sy2sb_probs_kernel(BcLayout lay, int k, int b, int lt0, int nlt, double* A,
                                   long long ld, const double* V, const double* VW,
                                   const double* WV, long long ldv, double* slots, double* Y2,
                                   GemmProblem* y1, GemmProblem* y2, GemmProblem* up) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nlt) return;
  const int lt = lt0 + i;
  const int gt = lt * lay.world + lay.rank;
  const int c0 = max(gt * lay.nb, k + b), c1 = min((gt + 1) * lay.nb, lay.n);
  const int cw = max(0, c1 - c0);
  const int roff = c0 - (k + b), mt = lay.n - c0;
  const long long lc0 = (long long)lt * lay.nb + (c0 - gt * lay.nb);
  double* At = A + c0 + lc0 * ld;
  GemmProblem p1, p2, p3;
  p1.M = cw > 0 ? mt : 0; p1.N = b; p1.K = cw;
  p1.A = At; p1.lda = ld; p1.ma = Mask::lower();
  p1.B = V + roff; p1.ldb = ldv;
  p1.C = slots + (size_t)lt * ldv * b + roff; p1.ldc = ldv;
  p1.alpha = 1.0; p1.beta = 0.0;
  p2.M = cw; p2.N = b; p2.K = cw > 0 ? mt : 0;
  p2.A = At; p2.lda = ld; p2.ma = Mask::strict_lower();
  p2.B = V + roff; p2.ldb = ldv;
  p2.C = Y2 + roff; p2.ldc = ldv;
  p2.alpha = 1.0; p2.beta = 0.0;
  p3.M = cw > 0 ? mt : 0; p3.N = cw; p3.K = 2 * b;
  p3.A = VW + roff; p3.lda = ldv;
  p3.B = WV + roff; p3.ldb = ldv;
  p3.C = At; p3.ldc = ld; p3.mc = Mask::lower();
  p3.alpha = -1.0; p3.beta = 1.0;
  y1[i] = p1;
  y2[i] = p2;
  up[i] = p3;
}

// This rank's part of Y = A22 V: the slots of its tiles in fixed order plus
// the transposed term on its own rows; rows >= m are zero.
__global__ void y_reduce_kernel(BcLayout lay, int k, int b, int m, int lt0, int nlt,
                                const double* slots, const double* Y2, long long ldv,
                                double* Y) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= ldv * b) return;
  const int r = (int)(idx % ldv), c = (int)(idx / ldv);
  double acc = 0.0;
  if (r < m) {
    for (int i = 0; i < nlt; ++i) {
      const int lt = lt0 + i;
      const int gt = lt * lay.world + lay.rank;
      const int c0 = max(gt * lay.nb, k + b), c1 = min((gt + 1) * lay.nb, lay.n);
      if (c1 <= c0) continue;
      const int roff = c0 - (k + b);
      if (r >= roff) acc += slots[(size_t)lt * ldv * b + r + (long long)c * ldv];
      if (r >= roff && r < roff + (c1 - c0)) acc += Y2[r + (long long)c * ldv];
    }
  }
  Y[idx] = acc;
}

// Band of this rank's columns into the (zeroed) replicated band store.
__global__ void band_bc_kernel(BcLayout lay, int nloc, int b, const double* A, long long ld,
                               double* AB, int ldab) {
  const int lc = blockIdx.x;
  if (lc >= nloc) return;
  const int j = lay.global_col(lc, lay.rank);
  for (int d = threadIdx.x; d <= b; d += blockDim.x) {
    const int i = j + d;
    if (i < lay.n) AB[(long long)j * ldab + d] = A[i + (long long)lc * ld];
  }
}

// Row block [rr0, rr0 + nr) of the tridiagonal eigenvectors (ascending
// columns, src nr x n) into this rank's solution columns: local column lc
// is eigenpair c = g(lc) in descending order = ascending column n - 1 - c.
__global__ void zcol_scatter_kernel(BcLayout lay, int nloc, int rr0, int nr, const double* src,
                                    long long lds, double* Z, long long ld) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)nr * nloc) return;
  const int i = (int)(idx % nr), lc = (int)(idx / nr);
  const int c = lay.global_col(lc, lay.rank);
  Z[(rr0 + i) + (long long)lc * ld] = src[i + (long long)(lay.n - 1 - c) * lds];
}

// lam (descending, all n) and this rank's lam per local column; *bad set when
// some lam^2 <= 0
__global__ void lam_bc_kernel(BcLayout lay, int nloc, const double* lam2, double* lam,
                              double* lamloc, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < lay.n) {
    const double l2 = lam2[lay.n - 1 - i];
    lam[i] = l2 > 0.0 ? sqrt(l2) : 0.0;
    if (!(l2 > 0.0)) atomicExch(bad, 1);
  }
  if (i < nloc) {
    const double l2 = lam2[lay.n - 1 - lay.global_col(i, lay.rank)];
    lamloc[i] = l2 > 0.0 ? sqrt(l2) : 0.0;
  }
}

// V = Z diag(lamloc)
__global__ void scale_cols_kernel(int n, int nloc, const double* Z, long long ld,
                                  const double* lamloc, double* V, long long ldv) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * nloc) return;
  const int r = (int)(idx % n), c = (int)(idx / n);
  V[r + (long long)c * ldv] = Z[r + (long long)c * ld] * lamloc[c];
}

// X1 = (u + v) / (2 sqrt(lam)), X2 = (u - v) / (2 sqrt(lam))
__global__ void recover_bc_kernel(int n, int nloc, const double* U, const double* V, long long ld,
                                  const double* lamloc, double* X1, long long ldx1, double* X2,
                                  long long ldx2) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * nloc) return;
  const int r = (int)(idx % n), c = (int)(idx / n);
  const double l = lamloc[c];
  const double sc = l > 0.0 ? 0.5 / sqrt(l) : 0.0;
  const double u = U[r + (long long)c * ld], v = V[r + (long long)c * ld];
  X1[r + (long long)c * ldx1] = (u + v) * sc;
  X2[r + (long long)c * ldx2] = (u - v) * sc;
}

unsigned blocks_for(long long cnt, int t = 256) { return (unsigned)std::max<long long>(1, ceil_div(cnt, t)); }

cudaError_t copy2d(double* dst, long long ldd, const double* src, long long lds, int rows, int cols,
                   cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  return cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double),
                           (size_t)rows * sizeof(double), cols, cudaMemcpyDeviceToDevice, s);
}

// ---------------------------------------------------------------------------
// workspace

struct DistWork {
  long long ld = 0;      // pad(n): rows of every column-distributed matrix
  int nloc = 0;          // this rank's columns
  int nlmax = 0;         // max over ranks (buffer sizes are rank independent)
  int nrmax = 0;         // max rows of a row block
  // persistent
  double* L = nullptr;   // K -> L
  double* TV = nullptr;  // T1 = M L, then the SY2SB reflectors of the owned panels
  double* WZ = nullptr;  // W, then the eigenvector columns Z
  double* Tall = nullptr;
  double* lam2 = nullptr;
  double* lamloc = nullptr;
  double* d = nullptr;
  double* e = nullptr;
  double* red = nullptr;  // status reduction (3 * world)
  DevStatus* st = nullptr;
  double* AB = nullptr; int ldab = 0;
  double* V2 = nullptr; double* tau2 = nullptr; int* progress = nullptr;
  char* scratch = nullptr; size_t scratch_bytes = 0;
  size_t replicated = 0;
};

// scratch layouts of the phases (dry arenas give the sizes)
struct PhaseA { double* P; OzBuf oz; };                       // Cholesky, congruence, recovery panels
struct PhaseB {                                     // SY2SB
  double* TVW;   // [T (b^2) | V (ldv b) | W (ldv b)]
  double* WV;    // [W | V]
  double* Y; double* Y2; double* slots;
  Sy2sbScratch sc;
  GemmProblem* probs;  // 3 * local tiles
};
struct PhaseD { StedcWork dc; double* Zrow; long long ldzr; };
struct PhaseE1 { double* TB; };
struct PhaseE2 { double* Vblk; };
struct PhaseE3 { double* Vg; double* Tg; Q1Scratch q1; };
struct PhaseE4 { double* P; double* Bu; double* Bv; OzBuf oz; };

PhaseA carve_a(Arena& a, int n, int nb, int nlmax = 0, bool oz = false) {
  PhaseA p{};
  p.P = a.take<double>((size_t)pad_ld(n) * nb);
  if (oz && nlmax > 0) {
    p.oz.bytes = panel_oz_bytes(n, nb, nlmax);
    p.oz.p = a.take<char>(p.oz.bytes);
  }
  return p;
}

PhaseB carve_b(Arena& a, int n, int nb, int ntl) {
  PhaseB p{};
  const int b = kBand;
  const long long ldv = pad_ld(n);
  p.TVW = a.take<double>((size_t)b * b + 2 * (size_t)ldv * b);
  p.WV = a.take<double>(2 * (size_t)ldv * b);
  p.Y = a.take<double>((size_t)ldv * b);
  p.Y2 = a.take<double>((size_t)ldv * b);
  p.slots = a.take<double>((size_t)std::max(ntl, 1) * ldv * b);
  p.sc.ldy = ldv;
  p.sc.y = p.Y;
  p.sc.z = a.take<double>(2 * (size_t)b * b);
  p.sc.z2 = a.take<double>((size_t)b * b);
  p.sc.red = a.take<double>(4 * 192 * (2 + 2 * (size_t)b));  // 2 x 16-byte mailbox slots
  p.sc.bar = a.take<unsigned>(4);
  p.sc.splitk_ws = a.take<double>(64 * (size_t)b * b);
  p.sc.probs = a.take<GemmProblem>(128);
  p.probs = a.take<GemmProblem>(3 * (size_t)std::max(ntl, 1));
  (void)nb;
  return p;
}

PhaseD carve_d(Arena& a, int n, int nrmax, int ucols, bool oz = false) {
  PhaseD p{};
  p.dc = stedc_carve(a, n, nrmax, ucols);
  if (oz) {
    // top merges on the emulated engine: (rows of this rank) x (U chunk) x n/2
    p.dc.oz_bytes = ozgemm_bytes(std::max(nrmax, 1), p.dc.ucols, (n + 1) / 2, 2048);
    p.dc.oz = a.take<char>(p.dc.oz_bytes);
  }
  p.ldzr = pad_ld(nrmax);
  p.Zrow = a.take<double>((size_t)p.ldzr * n);
  return p;
}

PhaseE1 carve_e1(Arena& a, int n, int nrmax) {
  PhaseE1 p{};
  p.TB = a.take<double>((size_t)pad_ld(nrmax) * n);
  return p;
}

PhaseE2 carve_e2(Arena& a, int n) {
  PhaseE2 p{};
  p.Vblk = a.take<double>(q2_range_doubles(n, kBand, kQ2RangeGroups));
  return p;
}

PhaseE3 carve_e3(Arena& a, int n, int nb, int nlmax, bool oz) {
  PhaseE3 p{};
  const int b = kBand;
  const size_t kb = (size_t)q1_group_tiles(nb, oz) * nb;
  p.Vg = a.take<double>((size_t)pad_ld(n) * kb);
  p.Tg = a.take<double>(kb * kb);
  p.q1.group = (int)(kb / b);
  p.q1.x = a.take<double>(kb * kb);
  p.q1.tmp = a.take<double>(kb * kb / 2 + kb * b);
  p.q1.y = a.take<double>(kb * (size_t)std::max(nlmax, 1));
  p.q1.y2 = a.take<double>(kb * (size_t)std::max(nlmax, 1));
  p.q1.probs = a.take<GemmProblem>(64);
  if (oz) {
    p.q1.oz_bytes = q1_oz_bytes(n, b, std::max(nlmax, 1), (int)(kb / b));
    p.q1.oz = a.take<char>(p.q1.oz_bytes);
    p.q1.oz_side_bytes = std::max(ozgemm_bytes((int)kb, (int)kb, n, kQ1OzChunk),
                                  ozgemm_bytes(n, (int)kb, (int)kb, kQ1OzChunk));
    p.q1.oz_side = a.take<char>(p.q1.oz_side_bytes);
  }
  return p;
}

PhaseE4 carve_e4(Arena& a, int n, int nb, int nlmax, bool oz = false) {
  PhaseE4 p{};
  const long long ld = pad_ld(n);
  p.P = a.take<double>((size_t)ld * nb);
  p.Bu = a.take<double>((size_t)ld * std::max(nlmax, 1));
  p.Bv = a.take<double>((size_t)ld * std::max(nlmax, 1));
  if (oz && nlmax > 0) {
    p.oz.bytes = panel_oz_bytes(n, nb, nlmax);
    p.oz.p = a.take<char>(p.oz.bytes);
  }
  return p;
}

template <class F>
size_t dry_bytes(F&& f) {
  Arena a;
  a.dry = true;
  f(a);
  return a.used;
}

DistWork carve_dist(Arena& a, const BcLayout& lay, int flags) {
  DistWork w{};
  const int n = lay.n, b = kBand, world = lay.world;
  w.ld = pad_ld(n);
  w.nloc = lay.ncols_of(lay.rank);
  for (int r = 0; r < world; ++r) w.nlmax = std::max(w.nlmax, lay.ncols_of(r));
  for (int r = 0; r < world; ++r) {
    long long c0, c1;
    shard_range(n, world, r, &c0, &c1);
    w.nrmax = std::max(w.nrmax, (int)(c1 - c0));
  }
  const size_t mat = (size_t)w.ld * std::max(w.nlmax, 1);
  w.L = a.take<double>(mat);
  w.TV = a.take<double>(mat);
  w.WZ = a.take<double>(mat);
  const size_t rep0 = a.used;
  const int np = std::max(1, n / b + 1);
  w.Tall = a.take<double>((size_t)np * b * b);
  w.lam2 = a.take<double>(n);
  w.lamloc = a.take<double>(std::max(w.nlmax, 1));
  w.d = a.take<double>(n);
  w.e = a.take<double>(n);
  w.red = a.take<double>(3 * (size_t)world + 4);
  w.st = a.take<DevStatus>(2);
  w.ldab = 2 * b + 1;
  w.AB = a.take<double>((size_t)w.ldab * n);
  const int maxsteps = sb2st_maxsteps(n, b);
  w.V2 = a.take<double>((size_t)n * maxsteps * b);
  w.tau2 = a.take<double>((size_t)n * maxsteps);
  w.progress = a.take<int>(sb2st_progress_ints(n, b));  // sweep counters + hand-off mailboxes (sb2st)
  w.replicated = a.used - rep0;
  const bool oz = dist_oz(n, flags);
  int ntlmax = 0;
  for (int r = 0; r < world; ++r) ntlmax = std::max(ntlmax, lay.ntiles_of(r));
  size_t sb = 0;
  sb = std::max(sb, dry_bytes([&](Arena& x) { carve_a(x, n, lay.nb, w.nlmax, oz); }));
  sb = std::max(sb, dry_bytes([&](Arena& x) { carve_b(x, n, lay.nb, ntlmax); }));
  sb = std::max(sb, dry_bytes([&](Arena& x) {
    carve_d(x, n, w.nrmax, w.nlmax, oz);
    carve_e1(x, n, w.nrmax);  // the transposition reads Zrow (phase D) through TB
  }));
  sb = std::max(sb, dry_bytes([&](Arena& x) { carve_e2(x, n); }));
  sb = std::max(sb, dry_bytes([&](Arena& x) { carve_e3(x, n, lay.nb, w.nlmax, oz); }));
  sb = std::max(sb, dry_bytes([&](Arena& x) { carve_e4(x, n, lay.nb, w.nlmax, oz); }));
  w.scratch_bytes = sb + 4096;
  w.scratch = a.take<char>(w.scratch_bytes);
  return w;
}

#define BSE_TRY(x)                         \
  do {                                     \
    cudaError_t e_ = (x);                  \
    if (e_ != cudaSuccess) return e_;      \
  } while (0)

// ---------------------------------------------------------------------------
// A = L L^T, right-looking over column tiles: the owner factors the tile
// (diagonal block, then the panel below it), broadcasts it, and every rank
// updates its own trailing tiles.  P: (pad(n) x nb) panel buffer.
cudaError_t potrf_bc(Comm& comm, const BcLayout& lay, double* A, long long ld, double* P,
                     DevStatus* st, cudaStream_t s) {
  const int T = lay.ntiles(), n = lay.n, nb = lay.nb;
  for (int k = 0; k < T; ++k) {
    const int kb = lay.tile_cols(k), r0 = k * nb, m = n - r0;
    const long long ldp = pad_ld(m);
    if (lay.owner(k) == lay.rank) {
      double* Ak = A + r0 + (long long)lay.local_col(r0) * ld;
      BSE_TRY(potrf_lower_at(Ak, ld, kb, r0, st, s));
      if (m > kb) BSE_TRY(trsm_rlt(Ak, ld, kb, Ak + kb, ld, m - kb, s));
      BSE_TRY(copy2d(P, ldp, Ak, ld, m, kb, s));
    }
    if (lay.world > 1) BSE_TRY(comm.bcast(P, (size_t)ldp * kb, lay.owner(k), s));
    int j = k + 1;
    while (j < T && lay.owner(j) != lay.rank) ++j;
    for (; j < T; j += lay.world) {
      const int jb = lay.tile_cols(j), rj = j * nb, mj = n - rj;
      double* C = A + rj + (long long)lay.local_col(rj) * ld;
      GemmProblem g = make_gemm(mj, jb, kb, -1.0, P + (rj - r0), ldp, P + (rj - r0), ldp, 1.0, C, ld);
      g.mc = Mask::lower();
      BSE_TRY(gemm(false, true, g, s));
    }
  }
  return cudaSuccess;
}

// Combined factorization status of all ranks: first failing pivot (smallest
// global index), its value, and the smallest pivot.
cudaError_t reduce_status(Comm& comm, const BcLayout& lay, const DevStatus* st, double* red,
                          cudaStream_t s, long long* info, double* value, double* minpiv) {
  const int world = lay.world;
  status_pack_kernel<<<1, std::max(32, 3 * world), 0, s>>>(st, world, lay.rank, red);
  count_launch();
  if (world > 1) BSE_TRY(comm.allreduce_sum(red, 3 * (size_t)world, s));
  std::vector<double> h(3 * (size_t)world);
  BSE_TRY(cudaMemcpyAsync(h.data(), red, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s));
  BSE_TRY(cudaStreamSynchronize(s));
  *info = -1;
  *value = 0.0;
  *minpiv = HUGE_VAL;
  double best = 4e18;
  for (int r = 0; r < world; ++r) {
    if (h[r] < best) { best = h[r]; *info = (long long)h[r]; *value = h[world + r]; }
    *minpiv = std::min(*minpiv, h[2 * world + r]);
  }
  return cudaSuccess;
}

// W = L^T M L (lower) in two SUMMA passes over broadcast column tiles:
// T1 = M L from M's lower triangle (tile k of M contributes tril(M_k) L[k, :]
// to rows >= k and stril(M_k)^T L to rows of tile k), then W[i, :] = L_i^T T1.
cudaError_t congruence_bc(Comm& comm, const BcLayout& lay, const double* M, long long ldm,
                          const double* L, double* T1, double* W, long long ld, int nloc,
                          double* P, const OzBuf& oz, cudaStream_t s) {
  const int T = lay.ntiles(), n = lay.n, nb = lay.nb;
  if (nloc > 0) BSE_TRY(cudaMemsetAsync(T1, 0, sizeof(double) * ld * nloc, s));
  for (int k = 0; k < T; ++k) {
    const int kb = lay.tile_cols(k), r0 = k * nb, m = n - r0;
    const long long ldp = pad_ld(m);
    if (lay.owner(k) == lay.rank)
      BSE_TRY(copy2d(P, ldp, M + r0 + (long long)lay.local_col(r0) * ldm, ldm, m, kb, s));
    if (lay.world > 1) BSE_TRY(comm.bcast(P, (size_t)ldp * kb, lay.owner(k), s));
    const int nc = lay.ncols_upto(k, lay.rank);
    if (nc == 0) continue;
    GemmProblem ga = make_gemm(m, nc, kb, 1.0, P, ldp, L + r0, ld, 1.0, T1 + r0, ld);
    ga.ma = Mask::lower();
    BSE_TRY(mm(false, false, ga, oz, s));
    GemmProblem gb = make_gemm(kb, nc, m, 1.0, P, ldp, L + r0, ld, 1.0, T1 + r0, ld);
    gb.ma = Mask::strict_lower();
    BSE_TRY(mm(true, false, gb, oz, s));
  }
  if (nloc > 0) BSE_TRY(cudaMemsetAsync(W, 0, sizeof(double) * ld * nloc, s));
  for (int i = 0; i < T; ++i) {
    const int ib = lay.tile_cols(i), r0 = i * nb, m = n - r0;
    const long long ldp = pad_ld(m);
    if (lay.owner(i) == lay.rank)
      BSE_TRY(copy2d(P, ldp, L + r0 + (long long)lay.local_col(r0) * ld, ld, m, ib, s));
    if (lay.world > 1) BSE_TRY(comm.bcast(P, (size_t)ldp * ib, lay.owner(i), s));
    const int nc = lay.ncols_upto(i, lay.rank);
    if (nc == 0) continue;
    GemmProblem g = make_gemm(ib, nc, m, 1.0, P, ldp, T1 + r0, ld, 0.0, W + r0, ld);
    g.ma = Mask::lower();
    BSE_TRY(mm(true, false, g, oz, s));
  }
  return cudaSuccess;
}

// Full -> band on the column-distributed W (lower).  Per panel: the owner
// factors it (cooperative panel QR) and broadcasts (T, V); every rank forms
// the part of Y = A22 V its own tiles contribute (grouped DMMA GEMMs, one
// problem per local tile), the parts are summed over the ranks, W = Y T -
// 1/2 V (T^T V^T Y T) is formed redundantly (O(m b^2)) and every rank applies
// the rank-2b update to its own tiles.  Vown keeps the reflectors of the
// owned panels (zero elsewhere), Tall every panel's T.
cudaError_t sy2sb_bc(Comm& comm, const BcLayout& lay, double* A, double* Vown, long long ld,
                     int nloc, double* Tall, PhaseB& w, int sms, cudaStream_t s) {
  const int n = lay.n, b = kBand;
  const long long ldv = ld;
  double* Tbuf = w.TVW;
  double* V = w.TVW + (size_t)b * b;
  double* Wp = V + (size_t)ldv * b;
  const int ntl = lay.ntiles_of(lay.rank);
  if (nloc > 0) BSE_TRY(cudaMemsetAsync(Vown, 0, sizeof(double) * ld * nloc, s));
  for (int p = 0;; ++p) {
    const int k = p * b, m = n - k - b;
    if (m < 2) break;
    const int owner = lay.owner(k / lay.nb);
    stage_mark("sy2sb_panel", s);
    if (owner == lay.rank) {
      const long long lc = lay.local_col(k);
      BSE_TRY(panel_qr(A + (k + b) + lc * ld, ld, m, b, V, ldv, Vown + (k + b) + lc * ld, ld, Tbuf,
                       w.sc.red, w.sc.bar, sms, s));
    }
    if (lay.world > 1) BSE_TRY(comm.bcast(Tbuf, (size_t)b * b + (size_t)ldv * b, owner, s));
    BSE_TRY(cudaMemcpyAsync(Tall + (size_t)p * b * b, Tbuf, sizeof(double) * b * b,
                            cudaMemcpyDeviceToDevice, s));
    stage_mark("sy2sb_symm", s);
    // local tiles holding trailing columns (>= k + b)
    int lt0 = 0;
    while (lt0 < ntl && (lt0 * lay.world + lay.rank + 1) * lay.nb <= k + b) ++lt0;
    const int nlt = ntl - lt0;
    GemmProblem* y1 = w.probs;
    GemmProblem* y2 = w.probs + std::max(ntl, 1);
    GemmProblem* up = w.probs + 2 * (size_t)std::max(ntl, 1);
    if (nlt > 0) {
      sy2sb_probs_kernel<<<blocks_for(nlt, 64), 64, 0, s>>>(lay, k, b, lt0, nlt, A, ld, V, V, w.WV,
                                                            ldv, w.slots, w.Y2, y1, y2, up);
      count_launch();
      BSE_TRY(cudaGetLastError());
      BSE_TRY(gemm_grouped(false, false, y1, nlt, m, b, s, true));
      BSE_TRY(gemm_grouped(true, false, y2, nlt, lay.nb, b, s, true));
    }
    y_reduce_kernel<<<blocks_for(ldv * b), 256, 0, s>>>(lay, k, b, m, lt0, nlt, w.slots, w.Y2, ldv,
                                                        w.Y);
    count_launch();
    if (lay.world > 1) BSE_TRY(comm.allreduce_sum(w.Y, (size_t)ldv * b, s));
    BSE_TRY(panel_w(m, b, V, ldv, Tbuf, Wp, ldv, w.sc, s));
    stage_mark("sy2sb_syr2k", s);
    if (nlt > 0) {
      // [W | V] next to [V | W]
      BSE_TRY(copy2d(w.WV, ldv, Wp, ldv, m, b, s));
      BSE_TRY(copy2d(w.WV + (size_t)ldv * b, ldv, V, ldv, m, b, s));
      BSE_TRY(gemm_grouped(false, true, up, nlt, m, lay.nb, s, true));
    }
  }
  return cudaGetLastError();
}

cudaError_t zrow_reduce_cb(void* ctx, double* zrow, int n, cudaStream_t s) {
  return static_cast<Comm*>(ctx)->allreduce_sum(zrow, (size_t)n, s);
}

}  // namespace

DistBytes dist_solve_bytes(int n, int nb, int world, int rank, int flags) {
  DistBytes out;
  if (n <= 0) return out;
  BcLayout lay;
  lay.n = n; lay.nb = nb; lay.world = world; lay.rank = rank;
  Arena a;
  a.dry = true;
  DistWork w = carve_dist(a, lay, flags);
  out.total = a.used + 4096;
  out.replicated = w.replicated;
  out.distributed = out.total - out.replicated;
  return out;
}

cudaError_t solve_spd_pair_bc(Comm& comm, int n, int nb, const double* Mloc, long long ldm,
                              const double* Kloc, long long ldk, double* lam, double* X1loc,
                              long long ldx1, double* X2loc, long long ldx2, void* work,
                              size_t work_bytes, int flags, cudaStream_t s, SolveStatus* out) {
  out->code = 0;
  out->pivot_index = -1;
  out->pivot_value = 0.0;
  out->failed_factor = -1;
  out->min_pivot = 0.0;
  out->clusters = 0;
  out->native_lm = false;
  if (n <= 0) return cudaSuccess;
  if (nb < kBand || nb % kBand != 0) return cudaErrorInvalidValue;
  BcLayout lay;
  lay.n = n; lay.nb = nb; lay.world = comm.world; lay.rank = comm.rank;
  Arena a{static_cast<char*>(work), work_bytes, 0, false};
  DistWork w = carve_dist(a, lay, flags);
  if (!w.scratch) return cudaErrorMemoryAllocation;
  const int b = kBand, nloc = w.nloc, world = lay.world;
  const long long ld = w.ld;
  const int sms = device_sm_count();
  const bool oz = dist_oz(n, flags);
  auto scratch = [&]() { return Arena{w.scratch, w.scratch_bytes, 0, false}; };
  const DevStatus h0[2] = {{-1, 0, 0.0, HUGE_VAL}, {-1, 0, 0.0, HUGE_VAL}};
  BSE_TRY(cudaMemcpyAsync(w.st, h0, sizeof(h0), cudaMemcpyHostToDevice, s));

  // 1. K = L L^T
  stage_mark("potrf", s);
  {
    Arena sa = scratch();
    PhaseA pa = carve_a(sa, n, nb, w.nlmax, oz);
    if (nloc > 0) {
      copy_lower_bc_kernel<<<blocks_for((long long)n * nloc), 256, 0, s>>>(lay, nloc, Kloc, ldk, w.L, ld);
      count_launch();
    }
    BSE_TRY(potrf_bc(comm, lay, w.L, ld, pa.P, &w.st[0], s));
    long long info;
    double value, minpiv;
    BSE_TRY(reduce_status(comm, lay, &w.st[0], w.red, s, &info, &value, &minpiv));
    out->min_pivot = minpiv;
    if (info >= 0) {
      // the reference factors A+B first (solvers.py:97-98): probe M and
      // report it if it fails too
      if (nloc > 0) {
        copy_lower_bc_kernel<<<blocks_for((long long)n * nloc), 256, 0, s>>>(lay, nloc, Mloc, ldm, w.TV, ld);
        count_launch();
      }
      BSE_TRY(potrf_bc(comm, lay, w.TV, ld, pa.P, &w.st[1], s));
      long long minfo;
      double mvalue, mminpiv;
      BSE_TRY(reduce_status(comm, lay, &w.st[1], w.red, s, &minfo, &mvalue, &mminpiv));
      out->code = 1;
      if (minfo >= 0) { out->failed_factor = 1; out->pivot_index = minfo; out->pivot_value = mvalue; }
      else { out->failed_factor = 0; out->pivot_index = info; out->pivot_value = value; }
      return cudaSuccess;
    }
    // 2. W = L^T M L
    stage_mark("congruence", s);
    BSE_TRY(congruence_bc(comm, lay, Mloc, ldm, w.L, w.TV, w.WZ, ld, nloc, pa.P, pa.oz, s));
  }
  // 3a. full -> band
  stage_mark("sy2sb", s);
  {
    Arena sa = scratch();
    PhaseB pb = carve_b(sa, n, nb, lay.ntiles_of(lay.rank));
    BSE_TRY(sy2sb_bc(comm, lay, w.WZ, w.TV, ld, nloc, w.Tall, pb, sms, s));
  }
  // 3b. band -> tridiagonal on the gathered band: rank 0 chases the bulges and
  // broadcasts d, e and the reflectors
  stage_mark("sb2st", s);
  BSE_TRY(cudaMemsetAsync(w.AB, 0, sizeof(double) * w.ldab * n, s));
  if (nloc > 0) {
    band_bc_kernel<<<nloc, 128, 0, s>>>(lay, nloc, b, w.WZ, ld, w.AB, w.ldab);
    count_launch();
  }
  if (world > 1) BSE_TRY(comm.allreduce_sum(w.AB, (size_t)w.ldab * n, s));
  BSE_TRY(sb2st_shared(&comm, w.AB, w.ldab, n, b, w.d, w.e, w.V2, w.tau2, w.progress, sms, s));
  // 3c. tridiagonal divide and conquer on row blocks, then the transposition
  // into this rank's solution columns (into WZ: W is dead)
  stage_mark("stedc", s);
  {
    long long r0, r1;
    shard_range(n, world, lay.rank, &r0, &r1);
    Arena sa = scratch();
    PhaseD pd = carve_d(sa, n, w.nrmax, w.nlmax, oz);
    PhaseE1 pe = carve_e1(sa, n, w.nrmax);
    if (!pe.TB) return cudaErrorMemoryAllocation;
    pd.dc.row0 = (int)r0;
    pd.dc.row1 = (int)r1;
    if (world > 1) {
      pd.dc.zrow_reduce = zrow_reduce_cb;
      pd.dc.zrow_ctx = &comm;
    }
    BSE_TRY(stedc(n, w.d, w.e, w.lam2, pd.Zrow, pd.ldzr, pd.dc, s));
    BSE_TRY(cudaMemcpyAsync(&w.st[0].conv_fail, pd.dc.fail, sizeof(int), cudaMemcpyDeviceToDevice, s));
    stage_mark("z_transpose", s);
    for (int r = 0; r < world; ++r) {
      long long q0, q1;
      shard_range(n, world, r, &q0, &q1);
      const int nr = (int)(q1 - q0);
      if (nr <= 0) continue;
      double* src = (r == lay.rank) ? pd.Zrow : pe.TB;
      if (world > 1) BSE_TRY(comm.bcast(src, (size_t)pd.ldzr * n, r, s));
      if (nloc > 0) {
        zcol_scatter_kernel<<<blocks_for((long long)nr * nloc), 256, 0, s>>>(lay, nloc, (int)q0, nr, src,
                                                                            pd.ldzr, w.WZ, ld);
        count_launch();
      }
    }
  }
  int* bad = &w.st[1].conv_fail;
  lam_bc_kernel<<<blocks_for(std::max(n, nloc)), 256, 0, s>>>(lay, nloc, w.lam2, lam, w.lamloc, bad);
  count_launch();
  // 3d. Z <- Q2 Z on this rank's columns, block range by block range
  stage_mark("q2_apply", s);
  {
    Arena sa = scratch();
    PhaseE2 pe = carve_e2(sa, n);
    const int ng = q2_groups(n, kQ2Group);
    for (int g_hi = ng - 1; g_hi >= 0; g_hi -= kQ2RangeGroups) {
      const int g_lo = std::max(0, g_hi - kQ2RangeGroups + 1);
      BSE_TRY(q2_build(n, b, kQ2Group, w.V2, w.tau2, pe.Vblk, s, g_lo, g_hi));
      if (nloc > 0) BSE_TRY(q2_apply(n, b, kQ2Group, pe.Vblk, w.WZ, ld, nloc, s, g_lo, g_hi));
    }
  }
  // 3e. Z <- Q1 Z: panel groups gathered from their owners, last group first
  stage_mark("q1_apply", s);
  {
    Arena sa = scratch();
    PhaseE3 pe = carve_e3(sa, n, nb, w.nlmax, oz);
    const int np = q1_panels(n, b), gt = q1_group_tiles(nb, oz), T = lay.ntiles();
    const int ppt = nb / b;  // panels per tile
    for (int gi = (T - 1) / gt; gi >= 0; --gi) {
      const int t0 = gi * gt, t1 = std::min(T, t0 + gt);
      const int p0 = t0 * ppt, pend = std::min(np, t1 * ppt);
      if (pend <= p0) continue;
      for (int t = t0; t < t1 && t * ppt < pend; ++t) {
        const int tc = lay.tile_cols(t);
        double* dst = pe.Vg + (long long)(t - t0) * nb * ld;
        if (lay.owner(t) == lay.rank)
          BSE_TRY(cudaMemcpyAsync(dst, w.TV + (long long)lay.local_col(t * nb) * ld,
                                  sizeof(double) * ld * tc, cudaMemcpyDeviceToDevice, s));
        if (world > 1) BSE_TRY(comm.bcast(dst, (size_t)ld * tc, lay.owner(t), s));
      }
      const int k = pend - p0, kb = k * b, r0 = (p0 + 1) * b, m = n - r0;
      const double* Vp = pe.Vg + r0;  // column 0 of Vg is global column p0 * b
      BSE_TRY(q1_group_build(k, b, m, Vp, ld, w.Tall + (size_t)p0 * b * b, pe.Tg, nullptr, pe.q1, s));
      if (nloc > 0)
        BSE_TRY(q1_group_apply(kb, m, Vp, ld, pe.Tg, nullptr, w.WZ + r0, ld, nloc, pe.q1, s));
    }
  }
  // 4. u = L Z, v = L^{-T} Z Lam over L's column tiles (last first: the back
  // substitution's order), X1,2 = (u +- v) / (2 sqrt(lam))
  stage_mark("recover", s);
  {
    Arena sa = scratch();
    PhaseE4 pe = carve_e4(sa, n, nb, w.nlmax, oz);
    const int T = lay.ntiles();
    if (nloc > 0) {
      BSE_TRY(cudaMemsetAsync(pe.Bu, 0, sizeof(double) * ld * nloc, s));
      scale_cols_kernel<<<blocks_for((long long)n * nloc), 256, 0, s>>>(n, nloc, w.WZ, ld, w.lamloc,
                                                                        pe.Bv, ld);
      count_launch();
    }
    for (int k = T - 1; k >= 0; --k) {
      const int kb = lay.tile_cols(k), r0 = k * nb, m = n - r0;
      const long long ldp = pad_ld(m);
      if (lay.owner(k) == lay.rank)
        BSE_TRY(copy2d(pe.P, ldp, w.L + r0 + (long long)lay.local_col(r0) * ld, ld, m, kb, s));
      if (world > 1) BSE_TRY(comm.bcast(pe.P, (size_t)ldp * kb, lay.owner(k), s));
      if (nloc == 0) continue;
      GemmProblem gu = make_gemm(m, nloc, kb, 1.0, pe.P, ldp, w.WZ + r0, ld, 1.0, pe.Bu + r0, ld);
      gu.ma = Mask::lower();
      BSE_TRY(mm(false, false, gu, pe.oz, s));
      if (m > kb) {
        GemmProblem gv = make_gemm(kb, nloc, m - kb, -1.0, pe.P + kb, ldp, pe.Bv + r0 + kb, ld, 1.0,
                                   pe.Bv + r0, ld);
        BSE_TRY(mm(true, false, gv, pe.oz, s));
      }
      BSE_TRY(trsm_llt(pe.P, ldp, kb, pe.Bv + r0, ld, nloc, s));
    }
    if (nloc > 0) {
      recover_bc_kernel<<<blocks_for((long long)n * nloc), 256, 0, s>>>(
          n, nloc, pe.Bu, pe.Bv, ld, w.lamloc, X1loc, ldx1, X2loc, ldx2);
      count_launch();
    }
  }
  stage_mark("end", s);
  BSE_TRY(cudaGetLastError());
  DevStatus hs[2];
  BSE_TRY(cudaMemcpyAsync(hs, w.st, sizeof(hs), cudaMemcpyDeviceToHost, s));
  BSE_TRY(cudaStreamSynchronize(s));
  if (hs[0].conv_fail) {
    out->code = 2;  // a secular root missed its bound (kernels.ConvergenceError)
    return cudaSuccess;
  }
  if (hs[1].conv_fail) {
    // W = L^T M L lost definiteness: probe M (the reference factors A+B
    // first, solvers.py:97-98); if it factors, the spectrum itself is not
    // positive (code 5)
    Arena sa = scratch();
    PhaseA pa = carve_a(sa, n, nb);
    BSE_TRY(cudaMemcpyAsync(&w.st[1], &h0[1], sizeof(DevStatus), cudaMemcpyHostToDevice, s));
    if (nloc > 0) {
      copy_lower_bc_kernel<<<blocks_for((long long)n * nloc), 256, 0, s>>>(lay, nloc, Mloc, ldm, w.TV, ld);
      count_launch();
    }
    BSE_TRY(potrf_bc(comm, lay, w.TV, ld, pa.P, &w.st[1], s));
    long long minfo;
    double mvalue, mminpiv;
    BSE_TRY(reduce_status(comm, lay, &w.st[1], w.red, s, &minfo, &mvalue, &mminpiv));
    if (minfo >= 0) {
      out->code = 1;
      out->failed_factor = 1;
      out->pivot_index = minfo;
      out->pivot_value = mvalue;
    } else {
      out->code = 5;
    }
    return cudaSuccess;
  }
  return cudaSuccess;
}

}  // namespace bse
