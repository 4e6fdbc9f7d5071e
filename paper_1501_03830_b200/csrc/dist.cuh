// Memory-distributed multi-GPU solve.
//
// One process per GPU.  Every N x N matrix of the product-form solve is
// distributed: M, K -> L, T1 = M L, W = L^T M L, the SY2SB reflectors and the
// outputs X1, X2 live in a block-cyclic column layout with tile nb (the 1 x Q
// member of the 2-D block-cyclic P x Q family: global column tile J belongs
// to rank J mod Q, all rows local), the divide-and-conquer eigenvectors in
// contiguous row blocks.  Per-rank dense storage is O(N^2 / Q); only the
// band, the tridiagonal data and the bulge-chasing reflectors are replicated.
//
// Exchanges (NCCL over NVLink / NVSwitch; all on the solve stream):
//   * panel broadcasts: the factored column tile of the right-looking
//     Cholesky, the column tiles of M and L in the two SUMMA passes of the
//     congruence, each SY2SB panel's reflectors (V, T), the panel groups of
//     the Q1 back-transform, L's column tiles in the recovery;
//   * reductions: each SY2SB panel's product A22 V (every rank sums the
//     contributions of its own column tiles), the band, the boundary rows of
//     the divide and conquer's rank-one tears (disjoint pieces, zero padded);
//   * one transposition of the tridiagonal eigenvectors from row blocks to
//     column tiles.
#pragma once
#include <cuda_runtime.h>
#include "comm.cuh"
#include "solver.cuh"

namespace bse {

// 1 x Q block-cyclic column layout of an n-column matrix with tile nb.
struct BcLayout {
  int n = 0, nb = 512, world = 1, rank = 0;
  BSE_HD int ntiles() const { return (n + nb - 1) / nb; }
  BSE_HD int owner(int tile) const { return tile % world; }
  BSE_HD int tile_cols(int tile) const { return min_i(nb, n - tile * nb); }
  // tiles / columns owned by rank r
  BSE_HD int ntiles_of(int r) const {
    const int t = ntiles();
    return r < t ? (t - r + world - 1) / world : 0;
  }
  BSE_HD int ncols_of(int r) const {
    const int lt = ntiles_of(r);
    if (lt == 0) return 0;
    const int last = (lt - 1) * world + r;  // this rank's last global tile
    return (lt - 1) * nb + tile_cols(last);
  }
  // local column of global column g (on its owner) and back
  BSE_HD int local_col(int g) const { return (g / nb / world) * nb + g % nb; }
  BSE_HD int global_col(int lc, int r) const { return ((lc / nb) * world + r) * nb + lc % nb; }
  // number of this rank's columns that lie in global tiles <= tile
  BSE_HD int ncols_upto(int tile, int r) const {
    if (tile < r) return 0;
    const int lt = (tile - r) / world + 1;  // local tiles with global index <= tile
    const int last = (lt - 1) * world + r;
    return (lt - 1) * nb + tile_cols(last);
  }
  BSE_HD static int min_i(int a, int b) { return a < b ? a : b; }
};

// Workspace of one rank (bytes) and its split into distributed (O(N^2 / Q))
// and replicated parts, for reporting.
struct DistBytes {
  size_t total = 0;
  size_t distributed = 0;  // block-cyclic / row-block matrices and their scratch
  size_t replicated = 0;   // band, tridiagonal data, bulge-chasing reflectors
};
DistBytes dist_solve_bytes(int n, int nb, int world, int rank, int flags);

// Collective.  Mloc, Kloc: this rank's columns (n rows, lower triangle of the
// global matrices referenced); lam: all n eigenvalues (descending) on every
// rank; X1loc, X2loc: this rank's columns of X1, X2 (column c of the solution
// pairs with lam[c]; same block-cyclic layout).
cudaError_t solve_spd_pair_bc(Comm& comm, int n, int nb, const double* Mloc, long long ldm,
                              const double* Kloc, long long ldk, double* lam, double* X1loc,
                              long long ldx1, double* X2loc, long long ldx2, void* work,
                              size_t work_bytes, int flags, cudaStream_t s, SolveStatus* out);

}  // namespace bse
