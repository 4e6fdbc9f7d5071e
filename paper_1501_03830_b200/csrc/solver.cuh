// Pipeline-level declarations shared by the C ABI.
#pragma once
#include <cuda_runtime.h>
#include "comm.cuh"
#include "eig.cuh"

#include <string>
#include <vector>

namespace bse {

struct StageLog {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  std::vector<std::string> names;
  int used = 0;
};
StageLog& stage_log();

// Per-device auxiliary stream (+ fork/join events) for work that overlaps the
// main solve stream.
struct SideStream {
  cudaStream_t s = nullptr;   // lowest priority: work that overlaps the solve stream
  cudaStream_t hp = nullptr;  // highest priority: latency-bound chains next to it
  cudaEvent_t fork = nullptr, join = nullptr, hp_fork = nullptr, hp_join = nullptr;
  cudaEvent_t la_cols = nullptr, la_panel = nullptr;  // SY2SB panel look-ahead
};
SideStream& side_stream();

double launch_peak(int which, int blocks, int iters, double* sink, cudaStream_t s);

struct SolveStatus {
  int code;            // 0 ok, 1 not positive definite, 2 no convergence,
                       // 5 spectrum not positive (M, K definite; some lambda^2 <= 0)
  long long pivot_index;
  double pivot_value;
  int failed_factor;   // 0: K (A-B), 1: M (A+B)
  double min_pivot;    // min_j L_jj^2 of K's factor (code 0)
  int clusters;        // complex path: clusters resolved by pivoted Gram-Schmidt
  bool native_lm;      // graded-input guard moved the L / M products to DMMA
};

// Host-entry upload of K by column pieces (see PotrfHook): piece 0 =
// [c0[0], c1[0]) is on the device at the call, piece L lands when ready[L]
// fires.  kpieces_plan() fills the boundaries for n.
constexpr int kKPieces = 4;  // pieces 0..3 (depth <= 3)
struct KPieces {
  int depth;
  int c0[kKPieces], c1[kKPieces];
  cudaEvent_t ready[kKPieces];
};
void kpieces_plan(int n, int depth, KPieces* kp);
// Optional host destination for the e2e path: X1/X2 column blocks are copied
// on `stream` as soon as they are recovered.
struct HostOut {
  double* X1; long long ldx1;
  double* X2; long long ldx2;
  double* lam;
  cudaStream_t stream;
};
constexpr int kRecoverBlock = 2048;      // emulated-engine column chunk
// BSE_FLAG_NATIVE_FP64: every product on the DMMA engine (no INT8 emulation)
constexpr int kFlagNativeFp64 = 0x4;
// the emulated-FP64 engine is used for the large products from this n up
constexpr int kOzMinN = 4096;
// internal flags (not in the C ABI): the caller already knows whether the
// inputs are graded (host entry: diagonals read on the host)
constexpr int kFlagGraded = 0x100;
constexpr int kFlagNotGraded = 0x200;
// graded-input guard: diagonal max/min ratio above which L / M products use DMMA
constexpr double kGradedDiagRatio = 65536.0;
inline bool diag_graded(double lo, double hi) {
  return lo > 0.0 && hi > 0.0 && hi > kGradedDiagRatio * lo;
}

size_t solve_bytes(int n, int flags);
cudaError_t solve_spd_pair(int n, const double* M, long long ldm, const double* K, long long ldk,
                           double* lam, double* X1, long long ldx1, double* X2, long long ldx2,
                           void* work, size_t work_bytes, int flags, cudaStream_t s,
                           SolveStatus* out, cudaEvent_t m_ready = nullptr,
                           const HostOut* hout = nullptr, Comm* comm = nullptr,
                           const KPieces* k_pieces = nullptr, ZSelect* zsel = nullptr);

cudaError_t absorption(int n, const double* lam, const double* X1c, long long ldx1,
                       const double* X2c, long long ldx2, const double* dr, const double* dl,
                       int ngrid, const double* grid, double sigma, double* weights,
                       double* values, double* defect, double* minpair, cudaStream_t s);

// Per-pair residuals / biorthogonality defect of a real product-form solution
// (verify.cu).
size_t verify_bytes(int n);
cudaError_t pair_residuals(int n, const double* M, long long ldm, const double* K, long long ldk,
                           const double* lam, const double* X1, long long ldx1, const double* X2,
                           long long ldx2, double* res, double* xn, double* bio, void* work,
                           size_t work_bytes, cudaStream_t s);

}  // namespace bse
