/*
 * bse_b200.h -- C ABI of the B200-native (sm_100a) structure-preserving
 * Bethe-Salpeter eigensolver.
 *
 * The reference package (bse-solver 0.1.0, pure Python/numpy) has no FFI
 * layer; these entry points sit *under* its Python solver API and replace
 * the numerical core of each call, one-for-one:
 *
 *   bse_solve_spd_pair_*   solvers.solve_real      pkg/src/bse/solvers.py:80-109
 *                          solvers.solve_complex   pkg/src/bse/solvers.py:29-77
 *                          (real path; the complex path calls it on the
 *                          2n x 2n real embedding, D3)
 *   bse_potrf_dev          kernels.cholesky         pkg/src/bse/kernels.py:43-65
 *   bse_syevd_dev          kernels.skew_tridiagonalize + phase_fold +
 *                          tridiag_eig + SkewTridiagonal.apply_q
 *                                                   pkg/src/bse/kernels.py:194-213,
 *                                                   :231-240, :460-535, :154-158
 *   bse_stedc_dev          kernels.tridiag_eig      pkg/src/bse/kernels.py:460-535
 *   bse_absorption_dev     spectra.absorption_spectrum
 *                                                   pkg/src/bse/spectra.py:120-151
 *   bse_pair_residuals_dev core.residual_metrics    pkg/src/bse/core.py:281-294
 *                          (per-pair form, no dense H / Y: SURVEY 8c(8))
 *
 * Conventions: all matrices are column-major FP64 with explicit leading
 * dimensions; "_dev" functions take device pointers and a cudaStream_t passed
 * as void*; "_host" functions take host pointers and do the copies.  No
 * function throws; each returns a bse_status and never frees caller memory.
 */
#ifndef BSE_B200_H
#define BSE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  BSE_OK = 0,
  BSE_NOT_POSITIVE_DEFINITE = 1, /* maps to kernels.NotPositiveDefinite */
  BSE_NO_CONVERGENCE = 2,        /* maps to kernels.ConvergenceError */
  BSE_BAD_ARGUMENT = 3,          /* maps to ValueError */
  BSE_CUDA_ERROR = 4,            /* message in bse_last_error() */
  BSE_SPECTRUM_NOT_POSITIVE = 5  /* A+B, A-B definite but some lambda^2 <= 0 in floating
                                    point: maps to the ValueError the reference's
                                    PositiveEigensystem raises (core.py:159-160) */
} bse_status;

/* Flags.  Solve entries accept BSE_FLAG_NATIVE_FP64 only (any other bit is
 * BSE_BAD_ARGUMENT); bse_syevd_dev also accepts BSE_FLAG_VALUES_ONLY. */
#define BSE_FLAG_VALUES_ONLY 0x1 /* bse_syevd_dev: eigenvalues only (TDA / validation); Z untouched */
#define BSE_FLAG_NATIVE_FP64 0x4 /* all products on FP64 DMMA (no INT8-emulated GEMMs) */

typedef struct bse_info {
  int64_t pivot_index;  /* first non-positive Cholesky pivot (status 1), else -1 */
  double pivot_value;   /* its value */
  int32_t failed_factor;/* 0: K = A - B, 1: M = A + B, -1: none */
  int32_t clusters;     /* complex solves: clusters resolved by pivoted Gram-Schmidt */
  double min_pivot;     /* status 0: min_j L_jj^2 of the factor of K (bse_potrf_dev: of A) */
} bse_info;

int bse_version(void);
const char* bse_last_error(void);

/* Workspace (bytes) needed by bse_solve_spd_pair_dev for dimension n. */
size_t bse_solve_workspace_bytes(int64_t n, int flags);

/*
 * Real symmetric-definite product pair (M = A + B, K = A - B, both SPD):
 *   K = L L^T, W = L^T M L = Z diag(lam^2) Z^T,
 *   X1 = (L Z + L^{-T} Z Lam) Lam^{-1/2} / 2,  X2 = (L Z - L^{-T} Z Lam) Lam^{-1/2} / 2
 * lam is returned DESCENDING and strictly positive (core.py:159-162).
 * M and K are read-only; only their lower triangles are referenced.
 * Work is ordered on `stream`; internally the solve forks per-device
 * auxiliary streams (panel look-ahead, block builds under the divide and
 * conquer) and joins them back into `stream` before the last kernel, so
 * events recorded on `stream` bracket the whole solve.  One solve at a time
 * per device and process (the auxiliary streams are shared).
 */
int bse_solve_spd_pair_dev(int64_t n, const double* dM, int64_t ldm, const double* dK,
                           int64_t ldk, double* dLam, double* dX1, int64_t ldx1, double* dX2,
                           int64_t ldx2, void* dWork, size_t work_bytes, int flags, void* stream,
                           bse_info* info);

/* Same contract with host buffers (copies inside; the e2e path). */
int bse_solve_spd_pair_host(int64_t n, const double* M, int64_t ldm, const double* K,
                            int64_t ldk, double* lam, double* X1, int64_t ldx1, double* X2,
                            int64_t ldx2, int flags, bse_info* info);

/*
 * Complex Hermitian BSE: the drop-in for solvers.solve_complex
 * (pkg/src/bse/solvers.py:29-77) on complex operators.  A (Hermitian) and
 * B (complex symmetric) are n x n complex128, interleaved (re, im), ROW-major
 * (numpy C order) with leading dimensions in complex elements; X1, X2 are
 * returned in the same layout, lam (n) descending and strictly positive, with
 * X1^H X1 - X2^H X2 = I.  Internally: the real 2n x 2n embedding
 * M' = A' + B', K' = A' - B' (D3), the product-form solve with one
 * eigenvector per doubled eigenvalue back-transformed, and the complex
 * extraction (pivoted Gram-Schmidt in x1^H y1 - x2^H y2 inside clusters of
 * equal complex eigenvalues).  Definiteness failures report the pivots of
 * the reference's cholesky(build_m) (status 1).
 */
size_t bse_solve_complex_workspace_bytes(int64_t n, int flags);
int bse_solve_complex_dev(int64_t n, const double* dA, int64_t lda, const double* dB,
                          int64_t ldb, double* dLam, double* dX1, int64_t ldx1, double* dX2,
                          int64_t ldx2, void* dWork, size_t work_bytes, int flags, void* stream,
                          bse_info* info);
/* Same with host buffers (uploads, solve and downloads inside). */
int bse_solve_complex_host(int64_t n, const double* A, int64_t lda, const double* B, int64_t ldb,
                           double* lam, double* X1, int64_t ldx1, double* X2, int64_t ldx2,
                           int flags, bse_info* info);

/* In-place lower Cholesky (strict upper zeroed). */
int bse_potrf_dev(int64_t n, double* dA, int64_t lda, void* stream, bse_info* info);

/* Workspace for bse_syevd_dev. */
size_t bse_syevd_workspace_bytes(int64_t n, int flags);

/* All eigenpairs of a real symmetric matrix (lower triangle of dA is read and
 * destroyed): two-stage reduction (full -> band -> tridiagonal), divide and
 * conquer, WY back-transforms.  w ascending; Z columns orthonormal. */
int bse_syevd_dev(int64_t n, double* dA, int64_t lda, double* dW, double* dZ, int64_t ldz,
                  void* dWork, size_t work_bytes, int flags, void* stream);

/* Symmetric tridiagonal divide and conquer: d (n), e (n-1) -> w ascending,
 * Q (n x n) orthonormal eigenvectors.  d and e are overwritten. */
size_t bse_stedc_workspace_bytes(int64_t n);
int bse_stedc_dev(int64_t n, double* dD, double* dE, double* dQ, int64_t ldq, void* dWork,
                  size_t work_bytes, void* stream);

/* Absorption weights and broadened curve (spectra.py:120-151):
 *   p_j = y_j^H x_j,  w_j = Re[(d_r^H x_j)(y_j^H d_l) / p_j],
 *   eps(omega_g) = sum_j w_j N(omega_g - lam_j; sigma), |omega - lam| <= 8 sigma,
 * accumulated in eigenvalue order.  Complex data are interleaved (re, im).
 * X1, X2: n x n complex (ld in complex elements); dr, dl: 2n complex.
 * Outputs: weights (n), pairing defect max|p_j - 1| (1), values (ngrid). */
int bse_absorption_dev(int64_t n, const double* dLam, const double* dX1c, int64_t ldx1,
                       const double* dX2c, int64_t ldx2, const double* dDr, const double* dDl,
                       int64_t ngrid, const double* dGrid, double sigma, double* dWeights,
                       double* dValues, double* dDefect, double* dMinPair, void* stream);

/* Verification without the 2n x 2n H or Y (core.residual_metrics,
 * core.py:281-294, in the per-pair form of SURVEY 8c(8)).  For a real
 * solution of (M, K) (lower triangles referenced):
 *   dRes[j]   = || H [x1_j; x2_j] - lam_j [x1_j; x2_j] ||_2,  H = [[A, B], [-B, -A]]
 *   dXnorm[j] = || [x1_j; x2_j] ||_2
 *   *dBio     = || X1^T X1 - X2^T X2 - I ||_F
 * Cost 6 n^3 flops (two SYMMs and one GEMM); workspace from
 * bse_residual_workspace_bytes. */
size_t bse_residual_workspace_bytes(int64_t n);
int bse_pair_residuals_dev(int64_t n, const double* dM, int64_t ldm, const double* dK, int64_t ldk,
                           const double* dLam, const double* dX1, int64_t ldx1, const double* dX2,
                           int64_t ldx2, double* dRes, double* dXnorm, double* dBio, void* dWork,
                           size_t work_bytes, void* stream);

/* Building blocks exposed for tests. */
int bse_gemm_dev(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                 const double* dA, int64_t lda, const double* dB, int64_t ldb, double beta,
                 double* dC, int64_t ldc, const int32_t* masks /* 9 ints or NULL */,
                 void* stream);
/* Same contract on the emulated-FP64 engine: Ozaki scheme II, 16 int8
 * residue products on the tcgen05 tensor cores + CRT reconstruction
 * (csrc/ozgemm.cu).  chunk: output columns per pass (<= 0: all N). */
int bse_ozgemm_dev(int transA, int transB, int64_t M, int64_t N, int64_t K, double alpha,
                   const double* dA, int64_t lda, const double* dB, int64_t ldb, double beta,
                   double* dC, int64_t ldc, const int32_t* masks, int64_t chunk, void* stream);
/* Contraction kernel of the emulated engine: 0 = hand-written tcgen05 kind::i8
 * kernel on CTA pairs with the residue-reducing epilogue (csrc/i8mma.cu, the
 * default), 1 = the same on single CTAs, 2 = CUTLASS kernel with INT32 residue
 * planes (kept for A/B measurements).  Returns the previous setting; out of
 * range values only query. */
int bse_oz_set_engine(int engine);
/* kind: 0 = A L^{-T} (right), 1 = L^{-T} B (left, trans), 2 = L^{-1} B (left) */
int bse_trsm_dev(int kind, int64_t n, const double* dL, int64_t ldl, double* dB, int64_t ldb,
                 int64_t m, void* stream);

/* Large host <-> device copies of PAGEABLE host memory (numpy arrays) through
 * the library's pinned staging ring with multi-threaded host copies; 2-D with
 * byte pitches.  to_device != 0: host -> device (returns once the data is on
 * the device), else device -> host (returns once dst is complete). */
int bse_memcpy2d_staged(int to_device, void* dst, size_t dpitch, const void* src, size_t spitch,
                        size_t width_bytes, size_t rows, void* stream);

/* Instrumentation (bench/profiling): stage timing with CUDA events recorded
 * on the solve stream, and the number of kernels this library has launched. */
int bse_profile_enable(int on);
/* Number of stage intervals recorded since bse_profile_enable (size the
 * buffers of bse_profile_read with it: one solve records ~1300). */
int bse_profile_count(void);
/* Fills up to max_stages durations (ms) and 32-byte names; returns the count
 * and resets the log. */
int bse_profile_read(int max_stages, double* ms, char* names);
long long bse_launch_count(void);
/* Returns the host entries' cached device memory (library-owned pool; the
 * device's default pool is never modified) to the driver. */
int bse_release_cached_memory(void);

/* FP64 peak probe: which 0 = DMMA, 1 = DFMA.  Returns flops of one launch in
 * *flops and the mean device time over `reps` launches in *ms. */
int bse_peak_fp64(int which, int blocks, int iters, int reps, double* flops, double* ms);

/*
 * Column-sharded multi-GPU solve (one process per GPU).
 * Same contract as bse_solve_spd_pair_dev -- the sharded form of
 * solvers.solve_real / solve_complex (pkg/src/bse/solvers.py:80-109,
 * :29-77) -- called collectively by every rank with identical M, K.  Rank r
 * forms the column block [c0_r, c1_r) (bse_shard_range) of the congruence
 * W = L^T M L and of the back-transformed eigenvectors and X1/X2; the blocks
 * are broadcast from their owners (one NCCL group of per-root broadcasts),
 * so on return every rank holds lam, X1 and X2 in full.  The Cholesky, the
 * band reduction, bulge chasing and D&C are replicated (bitwise identical on
 * every rank: no kernel on the path reduces in a data-dependent order).
 */
typedef struct bse_comm bse_comm;
/* Host broadcast used by the host-staged transport: broadcast `bytes` at
 * host_buf from rank `root` to every rank; return 0 on success. */
typedef int (*bse_host_bcast_fn)(void* ctx, void* host_buf, size_t bytes, int root);

/* 128-byte ncclUniqueId (rank 0 creates it; the caller distributes it). */
int bse_comm_nccl_unique_id(void* id128);
/* NCCL communicator over libnccl.so.2 (resolved at run time). */
int bse_comm_create_nccl(int rank, int world, const void* id128, bse_comm** out);
/* Host-staged transport (device block -> host -> fn -> device). */
int bse_comm_create_host(int rank, int world, bse_host_bcast_fn fn, void* ctx, bse_comm** out);
/* Measurement only: acts as rank `rank` of `world` but exchanges nothing, so
 * one GPU can time the kernels of one rank of a world-GPU solve
 * (tools/dist_projection.py).  Its results are NOT a solution. */
int bse_comm_create_solo(int rank, int world, bse_comm** out);
int bse_comm_destroy(bse_comm* comm);
/* This rank's column block [c0, c1) of an n-column matrix. */
int bse_shard_range(int64_t n, int world, int rank, int64_t* c0, int64_t* c1);
/* Every rank's column block of dA (n columns, ld) broadcast to all ranks. */
int bse_comm_allgather_cols_dev(bse_comm* comm, double* dA, int64_t ld, int64_t n, void* stream);
int bse_solve_spd_pair_dist_dev(bse_comm* comm, int64_t n, const double* dM, int64_t ldm,
                                const double* dK, int64_t ldk, double* dLam, double* dX1,
                                int64_t ldx1, double* dX2, int64_t ldx2, void* dWork,
                                size_t work_bytes, int flags, void* stream, bse_info* info);


/*
 * Memory-distributed multi-GPU solve (csrc/dist.cu).
 * Same contract as bse_solve_spd_pair_dev -- the sharded form of
 * solvers.solve_real (pkg/src/bse/solvers.py:80-109) and of the paper's
 * distributed algorithm -- but no rank ever holds an
 * N x N matrix: M, K -> L, T1 = M L, W = L^T M L, the SY2SB reflectors and
 * X1, X2 are laid out block-cyclically by COLUMN TILES of width nb (the
 * 1 x Q grid of the 2-D block-cyclic family: global column tile J lives on
 * rank J mod Q with all its rows), and the divide and conquer's eigenvector
 * matrix by contiguous ROW blocks (bse_shard_range).  Per-rank dense storage
 * is O(n^2 / Q); the band, the tridiagonal data and the bulge-chasing
 * reflectors (n^2 doubles) are replicated (the bulge chasing itself runs on
 * rank 0, which broadcasts its output).
 *
 * Called collectively.  dMloc, dKloc: this rank's bse_bc_local_cols columns
 * (n rows each; lower triangle of the global matrices referenced; local
 * column lc is global column bse_bc_global_col(lc)).  dLam: all n eigenvalues
 * (descending) on every rank.  dX1loc, dX2loc: this rank's columns of X1, X2
 * in the same layout (solution column c pairs with dLam[c]).  nb: a multiple
 * of 64 (BASELINE: 512 for cfg2/cfg3, 1024 for cfg4).  Exchanges: panel
 * broadcasts (Cholesky, SUMMA congruence, SY2SB reflectors, Q1 panel groups,
 * recovery), sums (each SY2SB panel's A22 V; band; D&C boundary rows) and
 * one transposition of the tridiagonal eigenvectors.
 */
int64_t bse_bc_local_cols(int64_t n, int nb, int world, int rank);
int64_t bse_bc_global_col(int64_t local_col, int nb, int world, int rank);
/* Workspace of one rank; *distributed / *replicated (may be NULL) split it
 * into the O(n^2 / Q) part and the replicated part. */
size_t bse_solve_bc_workspace_bytes(int64_t n, int nb, int world, int rank, int flags,
                                    size_t* distributed, size_t* replicated);
int bse_solve_spd_pair_bc_dev(bse_comm* comm, int64_t n, int nb, const double* dMloc, int64_t ldm,
                              const double* dKloc, int64_t ldk, double* dLam, double* dX1loc,
                              int64_t ldx1, double* dX2loc, int64_t ldx2, void* dWork,
                              size_t work_bytes, int flags, void* stream, bse_info* info);
/* Sum of `count` doubles at dptr over all ranks, in place (exposed for tests
 * of the transports). */
int bse_comm_allreduce_sum_dev(bse_comm* comm, double* dptr, size_t count, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BSE_B200_H */
