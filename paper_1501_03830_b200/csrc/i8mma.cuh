// Hand-written tcgen05 kind::i8 batched GEMM with a residue-reducing epilogue
// for the emulated-FP64 engine (see i8mma.cu, ozgemm.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace bse {

constexpr int kI8Mods = 16;

// For every modulus t < 16:
//   R[t][j][i] = (sum_k A8[t][i][k] * B8[t][j][k]) mod m_t   in [0, m_t), one byte,
// A8: 16 planes of rows_a x Kp int8 (K contiguous), B8: 16 planes of rows_b x Kp,
// R: 16 planes of rows_b x ldr bytes (i contiguous; ldr % 32 == 0, ldr >= M).
// Only entries with i < M, j < N are meaningful; tiles entirely outside the
// output band lo <= (col0 + j) - i <= hi are skipped (their bytes are not
// written).  Kp % 16 == 0, all base pointers 16-byte aligned, K <= 65536.
// two_sm: CTA pairs (cta_group::2, 256 x 256 tiles) instead of single CTAs
// (128 x 256).
cudaError_t i8mma_residues(int M, int N, int Kp, const int8_t* A8, long long rows_a,
                           const int8_t* B8, long long rows_b, uint8_t* R, long long ldr,
                           int col0, int lo, int hi, bool two_sm, cudaStream_t s);

// Modulus t of the engine (pairwise coprime, <= 256).
constexpr int i8_modulus(int t) {
  return t == 0 ? 256 : t == 1 ? 255 : t == 2 ? 253 : t == 3 ? 251 : t == 4 ? 247 : t == 5 ? 241
       : t == 6 ? 239 : t == 7 ? 233 : t == 8 ? 229 : t == 9 ? 227 : t == 10 ? 223
       : t == 11 ? 217 : t == 12 ? 211 : t == 13 ? 199 : t == 14 ? 197 : 193;
}

}  // namespace bse
