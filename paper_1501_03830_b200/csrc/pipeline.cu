// Pipelines: the two-stage symmetric eigensolver and the BSE product-form
// solve (north-star path: K = L L^T, W = L^T M L = Z Lam^2 Z^T, recover X, Y).
//
// Step order follows the reference's solvers (solvers.py:46-77 / :97-104):
// Cholesky -> congruence -> eigendecomposition -> back-transform -> scale.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unistd.h>
#include <vector>
#include "eig.cuh"
#include "comm.cuh"
#include "ozgemm.cuh"
#include "solver.cuh"

namespace bse {

StageLog& stage_log() {
  static StageLog log;
  return log;
}

void stage_mark(const char* name, cudaStream_t s) {
  StageLog& L = stage_log();
  if (!L.on) return;
  if (L.used >= (int)L.ev.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    L.ev.push_back(e);
    L.names.emplace_back();
  }
  cudaEventRecord(L.ev[L.used], s);
  L.names[L.used] = name;
  ++L.used;
}

SideStream& side_stream() {
  // one per device (the solve may run on any current device)
  static SideStream per_dev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  SideStream& ss = per_dev[dev & 63];
  if (!ss.s) {
    int least = 0, greatest = 0;
    cudaDeviceGetStreamPriorityRange(&least, &greatest);
    cudaStreamCreateWithPriority(&ss.s, cudaStreamNonBlocking, least);
    cudaStreamCreateWithPriority(&ss.hp, cudaStreamNonBlocking, greatest);
    cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss.hp_fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss.hp_join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss.la_cols, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ss.la_panel, cudaEventDisableTiming);
  }
  return ss;
}

int device_sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

namespace {

constexpr int kBand = 64;
constexpr int kQ2Group = 32;

struct SyevdWork {
  double* Vall; long long ldv;
  double* Tall;
  Sy2sbScratch sc;
  double* AB; int ldab;
  double* d; double* e;
  double* V2; double* tau2; int* progress;
  double* Vblk;  // Q2 blocks in the apply kernel's stage layout
  Q1Scratch q1;
  StedcWork dc;
};

SyevdWork carve_syevd(Arena& a, int n, int flags) {
  SyevdWork w{};
  const int b = kBand;
  const long long ld = pad_ld(n);
  const int np = std::max(1, n / b + 1);
  w.ldv = ld;
  w.Vall = a.take<double>((size_t)ld * n);
  w.Tall = a.take<double>((size_t)np * b * b);
  w.sc.ldvwv = ld;
  w.sc.vwv = a.take<double>((size_t)ld * 16 * b);  // 2 x (V1 W1 V2 W2 | W1c V1c W2c V2c)
  w.sc.ldy = ld;
  w.sc.y = a.take<double>((size_t)ld * b);
  w.sc.z = a.take<double>(2 * (size_t)b * b);
  w.sc.z2 = a.take<double>((size_t)b * b);
  w.sc.red = a.take<double>(4 * 192 * (2 + 2 * (size_t)b));  // 2 x 16-byte mailbox slots
  w.sc.bar = a.take<unsigned>(4);
  w.sc.splitk_ws = a.take<double>(64 * (size_t)b * b);
  w.sc.symm_ws = a.take<double>((size_t)kSymmSplits * ld * b);
  w.sc.probs = a.take<GemmProblem>(128);
  w.ldab = 2 * b + 1;  // element (i, j) at 128 j + i: 2-D tiles with a 1 KB stride
  w.AB = a.take<double>((size_t)w.ldab * n);
  w.d = a.take<double>(n);
  w.e = a.take<double>(n);
  const int maxsteps = sb2st_maxsteps(n, b);
  w.V2 = a.take<double>((size_t)n * maxsteps * b);
  w.tau2 = a.take<double>((size_t)n * maxsteps);
  w.progress = a.take<int>(sb2st_progress_ints(n, b));  // sweep counters + hand-off mailboxes (sb2st)
  const size_t qb = q2_block_doubles(n, b, kQ2Group);
  w.Vblk = a.take<double>(qb);
  const bool oz = !(flags & kFlagNativeFp64) && !(flags & 0x1) && n >= kOzMinN;
  w.q1.group = oz ? kQ1GroupOz : kQ1Group;
  if (const char* g = std::getenv("BSE_Q1_GROUP")) w.q1.group = std::max(1, std::atoi(g));  // tuning
  const size_t gb = (size_t)w.q1.group * b;
  w.q1.tg = a.take<double>(q1_tg_doubles(n, b, w.q1.group));
  w.q1.x = a.take<double>(gb * gb);
  w.q1.tmp = a.take<double>(gb * gb / 2 + gb * b);
  w.q1.y = a.take<double>(gb * n);
  w.q1.y2 = a.take<double>(gb * n);
  w.q1.splitk_ws = a.take<double>(16 * gb * b);
  w.q1.probs = a.take<GemmProblem>(64);
  w.dc = stedc_carve(a, n);
  if (oz) {
    // shared by the top D&C merges and Q1 (never live at the same time)
    const int h = (n + 1) / 2;
    w.q1.oz_bytes = std::max(q1_oz_bytes(n, b, n, w.q1.group), ozgemm_bytes(h, n, h, 2048));
    w.q1.oz = a.take<char>(w.q1.oz_bytes);
    w.dc.oz = w.q1.oz;
    w.dc.oz_bytes = w.q1.oz_bytes;
    const int kb = w.q1.group * b;
    // V^T V (kb x kb, K = m) and V T_g (m x kb, K = kb) of q1_build
    w.q1.oz_side_bytes = std::max(ozgemm_bytes(kb, kb, n, kQ1OzChunk),
                                  ozgemm_bytes(n, kb, kb, kQ1OzChunk));
    w.q1.oz_side = a.take<char>(w.q1.oz_side_bytes);
    w.q1.vt = a.take<double>(q1_vt_doubles(n, b, w.q1.group));
  }
  return w;
}

}  // namespace

namespace {
// dst(:, c) = Z(:, cols[c])  (n rows, nsel columns)
__global__ void gather_cols_kernel(int n, int nsel, const double* Z, long long ldz,
                                   const int* cols, double* dst, long long ldd) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * nsel) return;
  const int r = (int)(idx % n), c = (int)(idx / n);
  dst[r + (long long)c * ldd] = Z[r + (long long)cols[c] * ldz];
}
}  // namespace

namespace {
// BSE_DEBUG_HASH=1: checksum of an intermediate on stderr (synchronises; the
// determinism probe compares them between repetitions to find the first
// stage whose output differs)
void debug_hash(const char* name, const void* dptr, size_t bytes, cudaStream_t s) {
  static const bool on = std::getenv("BSE_DEBUG_HASH") != nullptr;
  if (!on || bytes == 0) return;
  std::vector<unsigned char> h(bytes);
  cudaMemcpyAsync(h.data(), dptr, bytes, cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  unsigned long long x = 1469598103934665603ull;
  const unsigned long long* q = reinterpret_cast<const unsigned long long*>(h.data());
  for (size_t i = 0; i < bytes / 8; ++i) x = (x ^ q[i]) * 1099511628211ull;
  std::fprintf(stderr, "[hash %d] %s %016llx\n", (int)getpid(), name, x);
  if (const char* dir = std::getenv("BSE_DEBUG_DUMP")) {
    if (bytes <= (1u << 22)) {  // small arrays only (d, e, w)
      static int counter = 0;
      const std::string path = std::string(dir) + "/" + name + "_" + std::to_string((int)getpid()) +
                               "_" + std::to_string(counter++) + ".bin";
      if (FILE* f = std::fopen(path.c_str(), "wb")) {
        std::fwrite(h.data(), 1, bytes, f);
        std::fclose(f);
      }
    }
  }
}
}  // namespace

cudaError_t sb2st_shared(Comm* comm, double* AB, int ldab, int n, int b, double* d, double* e,
                         double* V2, double* tau2, int* progress, int num_sms, cudaStream_t s) {
  cudaError_t err;
  if (!comm || comm->world <= 1) return sb2st(AB, ldab, n, b, d, e, V2, tau2, progress, num_sms, s);
  if (comm->rank == 0 &&
      (err = sb2st(AB, ldab, n, b, d, e, V2, tau2, progress, num_sms, s)) != cudaSuccess)
    return err;
  const size_t steps = (size_t)sb2st_maxsteps(n, b);
  if ((err = comm->group_begin()) != cudaSuccess) return err;
  if ((err = comm->bcast(d, (size_t)n, 0, s)) != cudaSuccess) return err;
  if ((err = comm->bcast(e, (size_t)n, 0, s)) != cudaSuccess) return err;
  if ((err = comm->bcast(tau2, (size_t)n * steps, 0, s)) != cudaSuccess) return err;
  if ((err = comm->bcast(V2, (size_t)n * steps * b, 0, s)) != cudaSuccess) return err;
  return comm->group_end(s);
}

size_t syevd_bytes(int n, int flags) {
  Arena a;
  a.dry = true;
  carve_syevd(a, n, flags);
  return a.used + 4096;
}

cudaError_t syevd(int n, double* A, long long lda, double* w, double* Z, long long ldz,
                  void* work, size_t work_bytes, int flags, cudaStream_t s, int zc0, int zc1,
                  int* conv_out, ZSelect* sel, Comm* comm) {
  if (n <= 0) return cudaSuccess;
  Arena a{static_cast<char*>(work), work_bytes, 0, false};
  SyevdWork ws = carve_syevd(a, n, flags);
  if (!ws.dc.scal) return cudaErrorMemoryAllocation;
  const int b = kBand;
  const int sms = device_sm_count();
  cudaError_t e;
  stage_mark("sy2sb", s);
  if ((e = cudaMemsetAsync(ws.Vall, 0, sizeof(double) * ws.ldv * n, s)) != cudaSuccess) return e;
  SideStream& side = side_stream();
  if ((e = sy2sb(A, lda, n, b, ws.Vall, ws.ldv, ws.Tall, ws.sc, sms, s, side.hp, side.la_cols,
                 side.la_panel)) != cudaSuccess)
    return e;
  stage_mark("sb2st", s);
  if ((e = extract_band(A, lda, n, b, ws.AB, ws.ldab, s)) != cudaSuccess) return e;
  debug_hash("band", ws.AB, sizeof(double) * ws.ldab * n, s);
  debug_hash("Tall", ws.Tall, sizeof(double) * (size_t)(n / b) * b * b, s);
  debug_hash("Vall", ws.Vall, sizeof(double) * ws.ldv * n, s);
  if ((e = sb2st_shared(comm, ws.AB, ws.ldab, n, b, ws.d, ws.e, ws.V2, ws.tau2, ws.progress, sms, s)) !=
      cudaSuccess)
    return e;
  debug_hash("d", ws.d, sizeof(double) * n, s);
  debug_hash("e", ws.e, sizeof(double) * (n - 1), s);
  debug_hash("tau2", ws.tau2, sizeof(double) * (size_t)n * sb2st_maxsteps(n, b), s);
  if (flags & 0x1) {  // BSE_FLAG_VALUES_ONLY: no vectors, no back-transforms
    stage_mark("values", s);
    if (conv_out && (e = cudaMemsetAsync(conv_out, 0, sizeof(int), s)) != cudaSuccess) return e;
    return tridiag_values(n, ws.d, ws.e, w, ws.dc.scal, s, conv_out);
  }
  // The Q2 blocks (from the bulge-chasing reflectors) and the Q1 group T
  // factors (from the SY2SB panels) do not depend on the divide and conquer:
  // they are built on a side stream while the latency-bound D&C runs.
  // A/B timing switch: 0 both builds on the side stream, 1 both serial before
  // the D&C, 2 Q2 build on the side stream and the Q1 build after the D&C
  static const int mode = std::getenv("BSE_BUILD_MODE") ? std::atoi(std::getenv("BSE_BUILD_MODE")) : 0;
  cudaStream_t sb = mode == 1 ? s : side.s;
  if (mode == 1) stage_mark("q_builds", s);
  if ((e = cudaEventRecord(side.fork, s)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(sb, side.fork, 0)) != cudaSuccess) return e;
  if ((e = q2_build(n, b, kQ2Group, ws.V2, ws.tau2, ws.Vblk, sb)) != cudaSuccess)
    return e;
  if (mode != 2 && (e = q1_build(n, b, ws.Vall, ws.ldv, ws.Tall, ws.q1, sb)) != cudaSuccess) return e;
  if ((e = cudaEventRecord(side.join, sb)) != cudaSuccess) return e;
  // the D&C chain of small latency-bound kernels runs on a high-priority
  // stream so the side stream's CTAs never delay its next launch
  static const bool dc_main = std::getenv("BSE_DC_MAIN") != nullptr;  // diagnostics: D&C on s
  cudaStream_t sdc = dc_main ? s : side.hp;
  if ((e = cudaEventRecord(side.hp_fork, s)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(sdc, side.hp_fork, 0)) != cudaSuccess) return e;
  stage_mark("stedc", sdc);
  if ((e = stedc(n, ws.d, ws.e, w, Z, ldz, ws.dc, sdc)) != cudaSuccess) return e;
  if (conv_out && (e = cudaMemcpyAsync(conv_out, ws.dc.fail, sizeof(int), cudaMemcpyDeviceToDevice,
                                       sdc)) != cudaSuccess)
    return e;
  if ((e = cudaEventRecord(side.hp_join, sdc)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(s, side.hp_join, 0)) != cudaSuccess) return e;
  debug_hash("w", w, sizeof(double) * n, s);
  if (mode == 2) {
    stage_mark("q1_build", s);
    if ((e = q1_build(n, b, ws.Vall, ws.ldv, ws.Tall, ws.q1, s)) != cudaSuccess) return e;
  }
  if (sel) {
    // eigenvalues to the host, choose the columns, gather them into sel->dst
    stage_mark("z_select", s);
    std::vector<double> wh(n);
    std::vector<int> cols(n);
    if ((e = cudaMemcpyAsync(wh.data(), w, sizeof(double) * n, cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    sel->nsel = sel->fn(sel->ctx, wh.data(), n, cols.data());
    if (sel->nsel <= 0) return cudaSuccess;
    if ((e = cudaMemcpyAsync(sel->dcols, cols.data(), sizeof(int) * sel->nsel,
                             cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return e;
    const long long cnt = (long long)n * sel->nsel;
    gather_cols_kernel<<<(unsigned)ceil_div(cnt, 256), 256, 0, s>>>(n, sel->nsel, Z, ldz,
                                                                    sel->dcols, sel->dst,
                                                                    sel->lddst);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // the host vectors must outlive the async copy: wait for it here (the
    // gather is queued behind it, so this costs no bubble on the device)
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    Z = sel->dst;
    ldz = sel->lddst;
    zc0 = 0;
    zc1 = sel->nsel;
  }
  stage_mark("q2_build_wait", s);
  if ((e = cudaStreamWaitEvent(s, side.join, 0)) != cudaSuccess) return e;
  if (zc1 < 0) zc1 = n;
  double* Zs = Z + (long long)zc0 * ldz;
  const int nz = zc1 - zc0;
  stage_mark("q2_apply", s);
  if ((e = q2_apply(n, b, kQ2Group, ws.Vblk, Zs, ldz, nz, s)) != cudaSuccess) return e;
  stage_mark("q1_apply", s);
  if (nz <= 0) return cudaSuccess;
  return q1_apply(n, b, ws.Vall, ws.ldv, Zs, ldz, nz, ws.q1, s);
}

// ---------------------------------------------------------------------------
// BSE product-form solve

namespace {

struct SolveWork {
  double* L; double* T1; double* W; double* Zr; long long ld;
  double* lam2;
  double* linv;
  DevStatus* st;
  int* cols;  // ZSelect column indices
  void* eig; size_t eig_bytes;
  void* oz; size_t oz_bytes;  // emulated-FP64 workspace (aliases eig when it fits)
  OzWork oz_trsm;             // separate: the TRMM's L slices stay live across blocks
};

bool use_oz(int n, int flags) { return !(flags & kFlagNativeFp64) && n >= kOzMinN; }

SolveWork carve_solve(Arena& a, int n, int flags) {
  SolveWork w{};
  w.ld = pad_ld(n);
  w.L = a.take<double>((size_t)w.ld * n);
  w.T1 = a.take<double>((size_t)w.ld * n);
  w.W = a.take<double>((size_t)w.ld * n);
  w.Zr = a.take<double>((size_t)w.ld * n);
  w.lam2 = a.take<double>(n);
  w.linv = a.take<double>(potrf_inv_cache_doubles(n));
  w.st = a.take<DevStatus>(2);
  w.cols = a.take<int>(n);
  w.eig_bytes = syevd_bytes(n, flags);
  w.eig = a.take<char>(w.eig_bytes);
  w.oz_bytes = use_oz(n, flags) ? ozgemm_bytes(n, n, n, kRecoverBlock) : 0;
  w.oz = w.oz_bytes <= w.eig_bytes ? w.eig : a.take<char>(w.oz_bytes);
  if (use_oz(n, flags)) {
    w.oz_trsm.chunk = kRecoverBlock;
    w.oz_trsm.bytes = trsm_llt_oz_bytes(n, n, kRecoverBlock);
    w.oz_trsm.p = a.take<char>(w.oz_trsm.bytes);
  }
  return w;
}

// dst(:, c0:c1) = tril(src)(:, c0:c1)  (n rows)
__global__ void copy_lower_kernel(int n, const double* src, long long lds, double* dst, long long ldd,
                                  int c0 = 0, int c1 = -1) {
  if (c1 < 0) c1 = n;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * (c1 - c0)) return;
  const int r = (int)(idx % n), c = c0 + (int)(idx / n);
  dst[r + (long long)c * ldd] = (r >= c) ? src[r + (long long)c * lds] : 0.0;
}

// min / max of the diagonals of M and K (graded-input guard): out = {min M,
// max M, min K, max K}; one CTA, deterministic.
__global__ void diag_range_kernel(int n, const double* M, long long ldm, const double* K,
                                  long long ldk, double* out) {
  __shared__ double red[4][32];
  double v[4] = {HUGE_VAL, -HUGE_VAL, HUGE_VAL, -HUGE_VAL};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double m = M[i + (long long)i * ldm], k = K[i + (long long)i * ldk];
    v[0] = fmin(v[0], m); v[1] = fmax(v[1], m);
    v[2] = fmin(v[2], k); v[3] = fmax(v[3], k);
  }
  for (int o = 16; o > 0; o >>= 1) {
    v[0] = fmin(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
    v[1] = fmax(v[1], __shfl_xor_sync(0xffffffffu, v[1], o));
    v[2] = fmin(v[2], __shfl_xor_sync(0xffffffffu, v[2], o));
    v[3] = fmax(v[3], __shfl_xor_sync(0xffffffffu, v[3], o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0)
    for (int q = 0; q < 4; ++q) red[q][w] = v[q];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = blockDim.x >> 5;
    for (int q = 0; q < 4; ++q) {
      double r = red[q][0];
      for (int k = 1; k < nw; ++k) r = (q & 1) ? fmax(r, red[q][k]) : fmin(r, red[q][k]);
      out[q] = r;
    }
  }
}

// Later column pieces of the host entry's K upload: wait for piece L, then
// copy it into L's buffer (potrf hook, see PotrfHook).
struct KTail {
  int n;
  const double* K; long long ldk;
  double* L; long long ld;
  int depth;
  int c0[kKPieces], c1[kKPieces];
  cudaEvent_t ready[kKPieces];
};

cudaError_t k_tail_hook(void* ctx, int level, cudaStream_t s) {
  const KTail& t = *static_cast<const KTail*>(ctx);
  if (level < 1 || level > t.depth) return cudaSuccess;
  cudaError_t e = cudaStreamWaitEvent(s, t.ready[level], 0);
  if (e != cudaSuccess) return e;
  const long long cnt = (long long)t.n * (t.c1[level] - t.c0[level]);
  if (cnt > 0) {
    copy_lower_kernel<<<(unsigned)ceil_div(cnt, 256), 256, 0, s>>>(t.n, t.K, t.ldk, t.L, t.ld,
                                                                   t.c0[level], t.c1[level]);
    count_launch();
  }
  return cudaGetLastError();
}

// Output columns [c0, c0 + nc): v <- Z(:, n-1-c) * lam_c, Zr(:, c) <- Z(:, n-1-c)
// (descending lam).  lam_out and the definiteness flag cover all n columns.
__global__ void scale_reverse_kernel(int n, int c0, int nc, const double* Z, long long ldz,
                                     const double* lam2, double* Zr, double* V, long long ld,
                                     double* lam_out, int* bad) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx < n) {
    const double l2 = lam2[n - 1 - idx];
    lam_out[idx] = l2 > 0.0 ? sqrt(l2) : 0.0;
    if (!(l2 > 0.0)) atomicExch(bad, 1);
  }
  if (idx >= (long long)n * nc) return;
  const int r = (int)(idx % n), c = c0 + (int)(idx / n);
  const int src = n - 1 - c;
  const double l2 = lam2[src];
  const double lam = l2 > 0.0 ? sqrt(l2) : 0.0;
  const double z = Z[r + (long long)src * ldz];
  Zr[r + (long long)c * ld] = z;
  V[r + (long long)c * ld] = z * lam;
}

// Selected columns: V(:, c) = Zr(:, c) * lam_c, lam_out[c] = lam_c with
// lam_c = sqrt(lam2[cols[c]]) (> 0, checked by the selector).
__global__ void scale_selected_kernel(int n, int nsel, const double* Zr, long long ld,
                                      const double* lam2, const int* cols, double* V,
                                      double* lam_out) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * nsel) return;
  const int r = (int)(idx % n), c = (int)(idx / n);
  const double lm = sqrt(lam2[cols[c]]);
  if (r == 0) lam_out[c] = lm;
  V[r + (long long)c * ld] = Zr[r + (long long)c * ld] * lm;
}

// X1 = (u + v) / (2 sqrt(lam)), X2 = (u - v) / (2 sqrt(lam))  (n rows, ncols columns)
__global__ void recover_kernel(int n, int ncols, const double* U, const double* V, long long ld,
                               const double* lam, double* X1, long long ldx1, double* X2,
                               long long ldx2) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)n * ncols) return;
  const int r = (int)(idx % n), c = (int)(idx / n);
  const double sc = 0.5 / sqrt(lam[c]);
  const double u = U[r + (long long)c * ld], v = V[r + (long long)c * ld];
  X1[r + (long long)c * ldx1] = (u + v) * sc;
  X2[r + (long long)c * ldx2] = (u - v) * sc;
}

unsigned nb_all(int n) { return (unsigned)ceil_div((long long)n * n, 256); }

// Rows [r0, r1) of X1, X2 (all ncols columns) from u (U) and v (V).
__global__ void recover_rows_kernel(int r0, int r1, int ncols, const double* U, const double* V,
                                    long long ld, const double* lam, double* X1, long long ldx1,
                                    double* X2, long long ldx2) {
  const int h = r1 - r0;
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)h * ncols) return;
  const int r = r0 + (int)(idx % h), c = (int)(idx / h);
  const double sc = 0.5 / sqrt(lam[c]);
  const double u = U[r + (long long)c * ld], v = V[r + (long long)c * ld];
  X1[r + (long long)c * ldx1] = (u + v) * sc;
  X2[r + (long long)c * ldx2] = (u - v) * sc;
}

// Host-entry recovery: as each row range of v = L^{-T} Z Lam is final, its
// rows of X1, X2 are formed and copied back on the copy stream.
struct RowsOut {
  int ncols;
  const double* U; const double* V; long long ld;
  const double* lam;
  double* X1; long long ldx1;
  double* X2; long long ldx2;
  const HostOut* hout;
  std::vector<cudaEvent_t>* evs;
};

cudaError_t rows_out_hook(void* ctx, int r0, int r1, cudaStream_t s) {
  const RowsOut& o = *static_cast<const RowsOut*>(ctx);
  if (r1 <= r0) return cudaSuccess;
  const long long tot = (long long)(r1 - r0) * o.ncols;
  recover_rows_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(
      r0, r1, o.ncols, o.U, o.V, o.ld, o.lam, o.X1, o.ldx1, o.X2, o.ldx2);
  count_launch();
  cudaError_t e;
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  cudaEvent_t ev;
  if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return e;
  o.evs->push_back(ev);
  if ((e = cudaEventRecord(ev, s)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(o.hout->stream, ev, 0)) != cudaSuccess) return e;
  const size_t w = sizeof(double) * (size_t)(r1 - r0);
  if ((e = cudaMemcpy2DAsync(o.hout->X1 + r0, o.hout->ldx1 * 8, o.X1 + r0, o.ldx1 * 8, w, o.ncols,
                             cudaMemcpyDeviceToHost, o.hout->stream)) != cudaSuccess)
    return e;
  return cudaMemcpy2DAsync(o.hout->X2 + r0, o.hout->ldx2 * 8, o.X2 + r0, o.ldx2 * 8, w, o.ncols,
                           cudaMemcpyDeviceToHost, o.hout->stream);
}

// Definiteness failure report (after K's Cholesky failed, or after W lost
// definiteness): the reference factors A+B first (solvers.py:97-98), so M is
// probed and reported if it fails; else K's failure, else a non-positive
// spectrum of W with both factors definite (code 5).
cudaError_t definiteness_failure(int n, const double* M, long long ldm, const SolveWork& w,
                                 const DevStatus& hk, cudaStream_t s, SolveStatus* out) {
  cudaError_t e;
  const long long ld = w.ld;
  copy_lower_kernel<<<nb_all(n), 256, 0, s>>>(n, M, ldm, w.W, ld);
  count_launch();
  DevStatus* stm = &w.st[1];
  const DevStatus h0{-1, 0, 0.0, HUGE_VAL};
  if ((e = cudaMemcpyAsync(stm, &h0, sizeof(DevStatus), cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  if ((e = potrf_lower(w.W, ld, n, stm, s)) != cudaSuccess) return e;
  DevStatus hm;
  if ((e = cudaMemcpyAsync(&hm, stm, sizeof(hm), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  out->code = 1;
  if (hm.info >= 0) {
    out->failed_factor = 1;
    out->pivot_index = hm.info;
    out->pivot_value = hm.value;
  } else if (hk.info >= 0) {
    out->failed_factor = 0;
    out->pivot_index = hk.info;
    out->pivot_value = hk.value;
  } else {
    out->code = 5;  // M and K definite, but some lambda^2 <= 0 in floating point
    out->failed_factor = -1;
    out->pivot_index = -1;
    out->pivot_value = 0.0;
  }
  return cudaSuccess;
}

}  // namespace

void kpieces_plan(int n, int depth, KPieces* kp) {
  int sp[kKPieces + 1];
  sp[0] = n;
  int d = 0;
  while (d < depth && d + 1 < kKPieces && sp[d] > 64) {
    sp[d + 1] = potrf_top_split(sp[d]);
    ++d;
  }
  kp->depth = d;
  // piece L = [s_{d-L+1}, s_{d-L}), piece 0 = [0, s_d)
  kp->c0[0] = 0;
  kp->c1[0] = sp[d];
  for (int L = 1; L <= d; ++L) {
    kp->c0[L] = sp[d - L + 1];
    kp->c1[L] = sp[d - L];
    kp->ready[L] = nullptr;
  }
}

size_t solve_bytes(int n, int flags) {
  Arena a;
  a.dry = true;
  carve_solve(a, n, flags);
  return a.used + 4096;
}

// Returns cudaSuccess and fills *status_host with {info, value, failed_factor}.
cudaError_t solve_spd_pair(int n, const double* M, long long ldm, const double* K, long long ldk,
                           double* lam, double* X1, long long ldx1, double* X2, long long ldx2,
                           void* work, size_t work_bytes, int flags, cudaStream_t s,
                           SolveStatus* out, cudaEvent_t m_ready, const HostOut* hout,
                           Comm* comm, const KPieces* k_pieces, ZSelect* zsel) {
  out->code = 0;
  out->pivot_index = -1;
  out->pivot_value = 0.0;
  out->failed_factor = -1;
  out->min_pivot = 0.0;
  out->clusters = 0;
  out->native_lm = false;
  if (n <= 0) return cudaSuccess;
  Arena a{static_cast<char*>(work), work_bytes, 0, false};
  SolveWork w = carve_solve(a, n, flags);
  if (!w.eig) return cudaErrorMemoryAllocation;
  const long long ld = w.ld;
  const long long tot = (long long)n * n;
  const unsigned nb = (unsigned)ceil_div(tot, 256);
  cudaError_t e;
  // Graded-input guard.  The emulated-FP64 engine scales each row of op(A)
  // and column of op(B) by one power of two, so an entry far below its
  // line's maximum keeps fewer bits than in a DGEMM; for the products with
  // L and M (Cholesky, congruence, recovery) that only matters when their
  // rows span many binades, which their diagonals reveal.  Above
  // kGradedDiagRatio those products run on the DMMA engine; the orthogonal
  // factors (D&C merges, Q1) stay emulated.
  bool oz_lm = w.oz_bytes != 0;
  if (oz_lm && (flags & kFlagGraded)) {
    oz_lm = false;
  } else if (oz_lm && !(flags & kFlagNotGraded)) {
    double hr[4];
    double* dr = reinterpret_cast<double*>(w.st);  // 48-byte scratch, re-initialised below
    diag_range_kernel<<<1, 1024, 0, s>>>(n, M, ldm, K, ldk, dr);
    count_launch();
    if ((e = cudaMemcpyAsync(hr, dr, sizeof(hr), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    oz_lm = !diag_graded(hr[0], hr[1]) && !diag_graded(hr[2], hr[3]);
  }
  out->native_lm = !oz_lm && w.oz_bytes != 0;
  DevStatus h0[2] = {{-1, 0, 0.0, HUGE_VAL}, {-1, 0, 0.0, HUGE_VAL}};
  if ((e = cudaMemcpyAsync(w.st, h0, sizeof(h0), cudaMemcpyHostToDevice, s)) != cudaSuccess) return e;
  // 1. K = L L^T
  stage_mark("potrf", s);
  {
    // with k_pieces (host entry), only K's piece 0 has landed: the Cholesky
    // factors it while the later pieces stream in
    KTail tail{};
    tail.n = n; tail.K = K; tail.ldk = ldk; tail.L = w.L; tail.ld = ld;
    int p0 = n;
    if (k_pieces) {
      tail.depth = k_pieces->depth;
      for (int L = 1; L <= tail.depth; ++L) {
        tail.c0[L] = k_pieces->c0[L];
        tail.c1[L] = k_pieces->c1[L];
        tail.ready[L] = k_pieces->ready[L];
      }
      p0 = k_pieces->c1[0];
    }
    const long long cnt = (long long)n * p0;
    copy_lower_kernel<<<(unsigned)ceil_div(cnt, 256), 256, 0, s>>>(n, K, ldk, w.L, ld, 0, p0);
    count_launch();
    PotrfHook hook{k_tail_hook, &tail, tail.depth};
    // the emulated engine's workspace aliases the (still idle) eigensolver's
    OzWork ozp{w.oz, w.oz_bytes, kRecoverBlock};
    if ((e = potrf_lower(w.L, ld, n, &w.st[0], s, w.linv, oz_lm ? &ozp : nullptr,
                         k_pieces ? &hook : nullptr)) != cudaSuccess)
      return e;
  }
  if (m_ready && (e = cudaStreamWaitEvent(s, m_ready, 0)) != cudaSuccess) return e;
  {
    // K's definiteness is known now: stop before any further O(n^3) work
    // (one host sync; the reference raises from cholesky() at this point,
    // solvers.py:97-98, after probing A+B first)
    DevStatus hk;
    if ((e = cudaMemcpyAsync(&hk, &w.st[0], sizeof(hk), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (hk.info >= 0) return definiteness_failure(n, M, ldm, w, hk, s, out);
  }
  stage_mark("congruence", s);
  // Distributed: this rank forms the column block [c0, c1) of T1 and W, then
  // every block is broadcast from its owner (the only exchange before the
  // replicated reduction).  Masks are view-relative, so a block starting at
  // column c0 shifts the diagonal of L, T1 and W by -c0.
  const int world = comm ? comm->world : 1;
  long long c0 = 0, c1 = n;
  if (world > 1) shard_range(n, world, comm->rank, &c0, &c1);
  const int nc = (int)(c1 - c0);
  const int sh = (int)c0;
  // 2. W = L^T M L  (T1 = M L from the lower triangle of M, then W = L^T T1, lower)
  if (oz_lm) {
    // Emulated-FP64 engine: column blocks [j0, j1) of W need only rows >= j0
    // of T1 and of L^T, so each block is two dense products on the trailing
    // square: T1_j = Msym[j0:, j0:] L[j0:, j0:j1], W[j0:, j0:j1] =
    // L[j0:, j0:]^T T1_j (lower part).  Msym (full symmetric M) lives in Zr
    // until the recovery needs it.
    const int nb = kRecoverBlock;
    copy_lower_kernel<<<nb_all(n), 256, 0, s>>>(n, M, ldm, w.Zr, ld);
    count_launch();
    if ((e = symmetrize_from_lower(w.Zr, ld, n, s)) != cudaSuccess) return e;
    for (int j0 = (int)c0; j0 < (int)c1; j0 += nb) {
      const int wj = std::min(nb, (int)c1 - j0), mt = n - j0;
      const long long o = j0 + (long long)j0 * ld;
      GemmProblem t1 = make_gemm(mt, wj, mt, 1.0, w.Zr + o, ld, w.L + o, ld, 0.0, w.T1 + o, ld);
      t1.mb = Mask::lower();
      if ((e = ozgemm(false, false, t1, w.oz, w.oz_bytes, nb, s)) != cudaSuccess) return e;
      GemmProblem t2 = make_gemm(mt, wj, mt, 1.0, w.L + o, ld, w.T1 + o, ld, 0.0, w.W + o, ld);
      t2.ma = Mask::lower();
      t2.mc = Mask::lower();
      if ((e = ozgemm(true, false, t2, w.oz, w.oz_bytes, nb, s)) != cudaSuccess) return e;
    }
  } else {
    GemmProblem g1 = make_gemm(n, nc, n, 1.0, M, ldm, w.L + c0 * ld, ld, 0.0, w.T1 + c0 * ld, ld);
    g1.ma = Mask::lower();
    g1.mb = Mask{kNoMaskLo, -sh, 0};
    if (nc > 0 && (e = gemm(false, false, g1, s)) != cudaSuccess) return e;
    // only T1's lower triangle feeds W = L^T T1 (lower): the strictly-upper
    // half of M's contribution is needed for rows k >= j only (N^3/3 flops
    // saved); g1 has already zeroed T1's upper triangle (k-range empty there)
    GemmProblem g2 = make_gemm(n, nc, n, 1.0, M, ldm, w.L + c0 * ld, ld, 1.0, w.T1 + c0 * ld, ld);
    g2.ma = Mask::strict_lower();
    g2.mb = Mask{kNoMaskLo, -sh, 0};
    g2.mc = Mask{kNoMaskLo, -sh, 0};
    if (nc > 0 && (e = gemm(true, false, g2, s)) != cudaSuccess) return e;
    GemmProblem g3 = make_gemm(n, nc, n, 1.0, w.L, ld, w.T1 + c0 * ld, ld, 0.0, w.W + c0 * ld, ld);
    g3.ma = Mask::lower();
    g3.mc = Mask{kNoMaskLo, -sh, 0};
    if (nc > 0 && (e = gemm(true, false, g3, s)) != cudaSuccess) return e;
  }
  if (world > 1) {
    stage_mark("allgather_w", s);
    if ((e = allgather_cols(*comm, w.W, ld, n, s)) != cudaSuccess) return e;
  }
  // 3. W = Z diag(lam^2) Z^T (ascending lam^2); Z into T1.  The reduction and
  // D&C are replicated; only this rank's eigenvector columns (output columns
  // [c0, c1) = Z columns [n - c1, n - c0)) are back-transformed.
  if (zsel) {
    if (world > 1) return cudaErrorInvalidValue;  // selection is a single-GPU mode
    zsel->dst = w.Zr;
    zsel->lddst = ld;
    zsel->dcols = w.cols;
  }
  if ((e = syevd(n, w.W, ld, w.lam2, w.T1, ld, w.eig, w.eig_bytes, flags, s, (int)(n - c1),
                 (int)(n - c0), &w.st[0].conv_fail, zsel, world > 1 ? comm : nullptr)) != cudaSuccess)
    return e;
  if (zsel && zsel->nsel <= 0) {
    // the selector refused the spectrum (non-positive or non-finite lambda^2):
    // a D&C convergence failure, else the definiteness report (M is intact)
    DevStatus hs[2];
    if ((e = cudaMemcpyAsync(hs, w.st, sizeof(hs), cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    out->min_pivot = hs[0].aux;
    if (hs[0].conv_fail) {
      out->code = 2;
      return cudaSuccess;
    }
    return definiteness_failure(n, M, ldm, w, hs[0], s, out);
  }
  stage_mark("recover", s);
  int* bad = reinterpret_cast<int*>(&w.st[1].conv_fail);
  if (zsel) {
    // selected columns (already in output order in Zr): v = Zr Lam into W
    c0 = 0;
    c1 = zsel->nsel;
    const long long tot_sh = (long long)n * zsel->nsel;
    scale_selected_kernel<<<(unsigned)ceil_div(tot_sh, 256), 256, 0, s>>>(
        n, zsel->nsel, w.Zr, ld, w.lam2, w.cols, w.W, lam);
    count_launch();
  } else {
    // 4. descending order; v = Z Lam into W, Z reversed into Zr
    const long long tot_sh = std::max<long long>((long long)n * nc, n);
    scale_reverse_kernel<<<(unsigned)ceil_div(tot_sh, 256), 256, 0, s>>>(
        n, (int)c0, nc, w.T1, ld, w.lam2, w.Zr, w.W, ld, lam, bad);
    count_launch();
  }
  // u = L Zr (into T1), v = L^{-T} (Zr Lam) (in W).  With host outputs, v's
  // rows finalise bottom-up inside the TRSM recursion: each eighth of the rows of
  // X1, X2 are formed and their D2H copy overlaps the rest of the solve.
  std::vector<cudaEvent_t> evs;
  // destroyed on every exit path (the copies they gate are on hout->stream;
  // destroying a recorded event is safe)
  struct EvGuard {
    std::vector<cudaEvent_t>& v;
    ~EvGuard() { for (auto ev : v) cudaEventDestroy(ev); }
  } guard{evs};
  const int nc_all = (int)(c1 - c0);
  if (nc_all > 0) {
    stage_mark("recover_trmm", s);
    if (oz_lm) {
      // row blocks: u[r0:r1, :] = L[r0:r1, 0:r1] Zr[0:r1, :] -- the emulated
      // engine cannot skip L's zero triangle, so trim K per block (1.25 N^3
      // executed instead of 2 N^3 with four blocks)
      const int rb = (int)((ceil_div(n, 4) + 63) / 64 * 64);
      for (int r0 = 0; r0 < n; r0 += rb) {
        const int r1 = std::min(n, r0 + rb);
        GemmProblem g4 = make_gemm(r1 - r0, nc_all, r1, 1.0, w.L + r0, ld, w.Zr + c0 * ld, ld, 0.0,
                                   w.T1 + r0 + c0 * ld, ld);
        g4.ma = Mask{kNoMaskLo, r0, 0};  // view-relative: L[r0 + i][k] for k <= r0 + i
        if ((e = ozgemm(false, false, g4, w.oz, w.oz_bytes, kRecoverBlock, s)) != cudaSuccess)
          return e;
      }
    } else {
      GemmProblem g4 = make_gemm(n, nc_all, n, 1.0, w.L, ld, w.Zr + c0 * ld, ld, 0.0,
                                 w.T1 + c0 * ld, ld);
      g4.ma = Mask::lower();
      if ((e = gemm(false, false, g4, s)) != cudaSuccess) return e;
    }
    stage_mark("recover_trsm", s);
    const bool host_rows = hout && world == 1;
    RowsOut ro{nc_all, w.T1 + c0 * ld, w.W + c0 * ld, ld, lam + c0, X1 + c0 * ldx1, ldx1,
               X2 + c0 * ldx2, ldx2, hout, &evs};
    RowHook hk{rows_out_hook, &ro, 3, 0};  // eighths: the last D2H is rows [0, n/8)
    if ((e = trsm_llt(w.L, ld, n, w.W + c0 * ld, ld, nc_all, s, w.linv,
                      (w.oz_trsm.p && oz_lm) ? &w.oz_trsm : nullptr, host_rows ? &hk : nullptr)) != cudaSuccess)
      return e;
    if (!host_rows) {
      const long long tb = (long long)n * nc_all;
      recover_kernel<<<(unsigned)ceil_div(tb, 256), 256, 0, s>>>(
          n, nc_all, w.T1 + c0 * ld, w.W + c0 * ld, ld, lam + c0, X1 + c0 * ldx1, ldx1,
          X2 + c0 * ldx2, ldx2);
      count_launch();
    }
  }
  if (world > 1) {
    stage_mark("allgather_x", s);
    if ((e = allgather_cols(*comm, X1, ldx1, n, s)) != cudaSuccess) return e;
    if ((e = allgather_cols(*comm, X2, ldx2, n, s)) != cudaSuccess) return e;
  }
  if (hout) {
    if ((e = cudaMemcpyAsync(hout->lam, lam, sizeof(double) * n, cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      return e;
  }
  stage_mark("end", s);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // status
  DevStatus hs[2];

  if ((e = cudaMemcpyAsync(hs, w.st, sizeof(hs), cudaMemcpyDeviceToHost, s)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  out->min_pivot = hs[0].aux;
  if (hs[0].conv_fail) {
    // a secular root of the divide and conquer missed its bound
    // (kernels.ConvergenceError, kernels.py:403-419)
    out->code = 2;
    return cudaSuccess;
  }
  if (hs[1].conv_fail) {
    // W = L^T M L lost definiteness: M is probed (A+B first, as the
    // reference); if M factors, the spectrum itself is not positive
    return definiteness_failure(n, M, ldm, w, hs[0], s, out);
  }
  return cudaSuccess;
}

}  // namespace bse
