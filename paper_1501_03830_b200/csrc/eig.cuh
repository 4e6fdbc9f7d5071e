// Two-stage symmetric eigensolver (full -> band -> tridiagonal -> divide and
// conquer -> WY back-transforms).  Replaces the reference's tridiagonal route
// (kernels.py:89-137 Householder reduction, :460-535 bisection + inverse
// iteration, :123-137 reflector-by-reflector back-transform).
#pragma once
#include <cuda_runtime.h>
#include "dense.cuh"
#include "workspace.cuh"

namespace bse {

constexpr int kMaxPanel = 64;  // SY2SB bandwidth b (<= 64)

struct Sy2sbScratch {
  double* vwv = nullptr;  // 2 x 8 slots of b columns: V1 W1 V2 W2 | W1c V1c W2c V2c (sy2sb)
  long long ldvwv = 0;
  double* y = nullptr;    // m x b
  long long ldy = 0;
  double* z = nullptr;    // 2b x b
  double* z2 = nullptr;   // b x b
  double* red = nullptr;  // panel-QR grid reduction (2 * 148 * (2 + 2b))
  unsigned* bar = nullptr;
  double* splitk_ws = nullptr;  // 48 * b * b
  double* symm_ws = nullptr;    // kSymmSplits * ld * b
  GemmProblem* probs = nullptr; // 128 problems (split-K descriptors at +0, +32, +64)
};
constexpr int kSymmSplits = 16;

// la (optional): look-ahead stream for the next pair's first panel, with two
// events (trailing columns ready, panel done).
cudaError_t sy2sb(double* A, long long lda, int n, int b, double* Vall, long long ldv,
                  double* Tall, const Sy2sbScratch& w, int num_sms, cudaStream_t s,
                  cudaStream_t la = nullptr, cudaEvent_t ev_cols = nullptr,
                  cudaEvent_t ev_panel = nullptr);
cudaError_t extract_band(const double* A, long long lda, int n, int b, double* AB, int ldab,
                         cudaStream_t s);
// SY2SB building blocks (also driven panel by panel by the distributed solve):
// Householder QR of an m x bw panel (P <- R, explicit V and optional copy V2,
// T), and W = X - 1/2 V (T^T (V^T X)), X = Y T with Y = A2 V in w.y.
cudaError_t panel_qr(double* P, long long ldp, int m, int bw, double* V, long long ldv, double* V2,
                     long long ldv2, double* T, double* red, unsigned* bar, int num_sms,
                     cudaStream_t s);
cudaError_t panel_w(int m, int bw, const double* V, long long ldv, const double* Tp, double* W,
                    long long ldw, const Sy2sbScratch& w, cudaStream_t s);

// Bulge chasing on the band (lower storage, ldab = 2b + 1): d, e out; reflectors
// of sweep s, step j stored at V2[(s*maxsteps + j) * b], tau2[s*maxsteps + j].
int sb2st_maxsteps(int n, int b);
// ints behind `progress`: two counters per sweep + the hand-off mailbox ring
size_t sb2st_progress_ints(int n, int b);
cudaError_t sb2st(double* AB, int ldab, int n, int b, double* d, double* e, double* V2,
                  double* tau2, int* progress, int num_sms, cudaStream_t s);

// Q2 back-transform: Z <- Q2 Z (Z n x ncols).  Groups of g sweeps form
// compact-WY blocks (V and V*T, stored in q2_apply's shared-memory stage
// layout); Vblk sized by q2_block_doubles().
size_t q2_block_doubles(int n, int b, int g);
// g_lo/g_hi: only the sweep groups [g_lo, g_hi] (g_hi < 0: the last group);
// Vblk then holds that range's blocks (q2_range_doubles).  Applying the
// ranges top range first, each of even length, equals the whole transform --
// the distributed solve bounds its block storage that way.
int q2_groups(int n, int g);
size_t q2_range_doubles(int n, int b, int ngr);
cudaError_t q2_build(int n, int b, int g, const double* V2, const double* tau2, double* Vblk,
                     cudaStream_t s, int g_lo = 0, int g_hi = -1);
cudaError_t q2_apply(int n, int b, int g, const double* Vblk, double* Z, long long ldz, int ncols,
                     cudaStream_t s, int g_lo = 0, int g_hi = -1);

// Q1 back-transform: Z <- Q1 Z using the SY2SB panels, merged `group` at a
// time into one compact-WY block (kQ1Group on the DMMA engine; kQ1GroupOz
// when the large products run on the emulated-FP64 INT8 engine, whose
// efficiency needs K = group * b in the thousands).
constexpr int kQ1Group = 8;
constexpr int kQ1GroupOz = 64;
constexpr int kQ1OzChunk = 2048;
struct Q1Scratch {
  int group = kQ1Group;
  double* tg = nullptr;    // every group's T_g, back to back (q1_tg_doubles)
  double* vt = nullptr;    // every group's V_g T_g (m_g x kb), back to back (q1_vt_doubles)
  double* x = nullptr;     // (G b) x (G b): V^T V of the group
  double* tmp = nullptr;   // (G b)^2 / 2
  double* y = nullptr;     // (G b) x ncols
  double* y2 = nullptr;    // (G b) x ncols
  double* splitk_ws = nullptr;  // 16 * (G b) * b
  GemmProblem* probs = nullptr; // 64
  void* oz = nullptr;      // emulated-FP64 workspace (null: DMMA only)
  size_t oz_bytes = 0;
  void* oz_side = nullptr; // q1_build's own emulated workspace (it overlaps the D&C)
  size_t oz_side_bytes = 0;
};
size_t q1_oz_bytes(int n, int b, int ncols, int group);
size_t q1_tg_doubles(int n, int b, int group);
size_t q1_vt_doubles(int n, int b, int group);
// One group of k panels: T_g (kb x kb, kb = k b) from the panels' T factors Tp
// and V (m x kb), optionally VT = V T_g; and its application to Zs (m x ncols).
int q1_panels(int n, int b);
cudaError_t q1_group_build(int k, int b, int m, const double* V, long long ldv, const double* Tp,
                           double* Tg, double* VT, const Q1Scratch& w, cudaStream_t s);
cudaError_t q1_group_apply(int kb, int m, const double* V, long long ldv, const double* Tg,
                           const double* VT, double* Zs, long long ldz, int ncols,
                           const Q1Scratch& w, cudaStream_t s);
// T_g of every panel group (may run on a side stream; own emulated workspace).
cudaError_t q1_build(int n, int b, const double* Vall, long long ldv, const double* Tall,
                     const Q1Scratch& w, cudaStream_t s);
// Z <- Q1 Z with the T_g from q1_build.
cudaError_t q1_apply(int n, int b, const double* Vall, long long ldv, double* Z, long long ldz,
                     int ncols, const Q1Scratch& w, cudaStream_t s);

// Tridiagonal divide and conquer.
struct StedcWork {
  double* Qa = nullptr;  // n x n (ld)
  double* Qb = nullptr;
  double* U = nullptr;
  long long ld = 0;
  double* Da = nullptr;  // n
  double* Db = nullptr;
  double* ds = nullptr;   // sorted poles (n)
  double* zs = nullptr;   // sorted z (n)
  double* dk = nullptr;   // kept poles (n)
  double* zk = nullptr;   // kept z (n)
  double* zh = nullptr;   // per-node rho stash at [lo]
  double* zh2 = nullptr;  // zhat (n)
  double* val = nullptr;  // roots [0,K) and deflated values (from the back)
  double* tau = nullptr;  // secular offsets (n)
  int* org = nullptr;     // secular origins (n)
  int* perm = nullptr;    // sorted -> local original (n)
  int* keep = nullptr;    // kept sorted indices (n)
  int* defl = nullptr;    // deflated sorted indices (n)
  int* pos = nullptr;     // output column for each (roots then deflated) (n)
  int* rotp = nullptr;    // rotation pairs (n)
  int* rotq = nullptr;
  double* rotc = nullptr;
  double* rots = nullptr;
  int* counts = nullptr;  // per node: K, ndefl, nrot (3 * n)
  GemmProblem* probs = nullptr;  // 2 * n
  void* oz = nullptr;            // emulated-FP64 workspace for the top merges (optional)
  size_t oz_bytes = 0;
  double* scal = nullptr;  // scaling scalar(s)
  int* fail = nullptr;     // set nonzero when a secular root misses its bound (reset per stedc)
  double* dsan = nullptr;  // finite copies of d, e (non-finite input -> 0, fail set)
  double* esan = nullptr;
  // Row-distributed mode (dist.cu): this rank holds rows [row0, row1) of every
  // eigenvector block (Qa, Qb are (row1 - row0) x n with leading dimension
  // ld); U is ldu x ucols and a level whose U is wider is processed in column
  // chunks; the children's boundary rows come through zrow, summed over the
  // ranks by zrow_reduce.  Defaults: all rows, ldu = ld, ucols = n.
  int row0 = 0, row1 = -1;
  long long ldu = 0;
  int ucols = 0;
  double* zrow = nullptr;
  cudaError_t (*zrow_reduce)(void* ctx, double* zrow, int n, cudaStream_t s) = nullptr;
  void* zrow_ctx = nullptr;
};
size_t stedc_bytes(int n);
StedcWork stedc_carve(Arena& a, int n, int rows = -1, int ucols = 0);
// Eigenvalues ascending into w (may alias d), vectors into Q (ldq).
cudaError_t stedc(int n, double* d, double* e, double* w, double* Q, long long ldq,
                  const StedcWork& ws, cudaStream_t s);

// Values only: ascending eigenvalues of the tridiagonal by Sturm bisection.
// *fail (device int, may be null) is set nonzero when a value's bracket does
// not reach the convergence width of kernels.py:275-299 or is not finite.
cudaError_t tridiag_values(int n, const double* d, const double* e, double* w, double* scratch3,
                           cudaStream_t s, int* fail = nullptr);

// Column selection between the divide and conquer and the back-transforms
// (the complex path: one eigenvector per doubled eigenvalue of the real
// embedding is all the complex solution needs, so Q2/Q1 and the recovery run
// on about half the columns).  After the D&C, syevd synchronises, copies the
// ascending eigenvalues to the host and calls fn; fn returns the number of
// selected columns (their Z indices in output order written to cols,
// capacity n), or < 0 to skip the back-transforms (nsel is set to it).  The
// selected columns are gathered into dst[:, 0:nsel] and back-transformed
// there; Z keeps the D&C vectors.
struct ZSelect {
  int (*fn)(void* ctx, const double* w_host, int n, int* cols) = nullptr;
  void* ctx = nullptr;
  double* dst = nullptr;
  long long lddst = 0;
  int* dcols = nullptr;  // device copy of cols (n ints)
  int nsel = 0;          // out
};

// Full pipeline on a symmetric matrix (lower triangle of A read, destroyed).
size_t syevd_bytes(int n, int flags);
// zc0/zc1: back-transform only Z columns [zc0, zc1) (the column shard of a
// distributed solve; D&C still produces every column).  zc1 < 0 means n.
// conv_out (device int, may be null): nonzero after the call completes when
// the tridiagonal eigensolver did not converge (maps to BSE_NO_CONVERGENCE,
// the analogue of kernels.ConvergenceError, kernels.py:403-419).
// comm (replicated multi-rank callers): the bulge chasing runs on rank 0 only
// and d, e and its reflectors are broadcast, so every rank back-transforms
// with the same bits (and ranks sharing one GPU in tests never time-slice the
// persistent SB2ST kernel).
struct Comm;
cudaError_t syevd(int n, double* A, long long lda, double* w, double* Z, long long ldz,
                  void* work, size_t work_bytes, int flags, cudaStream_t s, int zc0 = 0,
                  int zc1 = -1, int* conv_out = nullptr, ZSelect* sel = nullptr,
                  Comm* comm = nullptr);
// Band -> tridiagonal on rank 0 of comm (all ranks when comm is null or has
// one rank), then d, e, V2, tau2 broadcast.
cudaError_t sb2st_shared(Comm* comm, double* AB, int ldab, int n, int b, double* d, double* e,
                         double* V2, double* tau2, int* progress, int num_sms, cudaStream_t s);

int device_sm_count();

}  // namespace bse
