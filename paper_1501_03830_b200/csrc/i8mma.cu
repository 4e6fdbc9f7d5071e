// Hand-written tcgen05 int8 contraction for the emulated-FP64 engine.
//
// For each of the 16 moduli m_t the engine needs C_t = A'_t B'_t^T mod m_t,
// where A'_t (rows i) and B'_t (rows j) are int8 residue planes with K
// contiguous.  This kernel computes all 16 products as one persistent,
// warp-specialised launch:
//
//   warp 0      TMA producer: cp.async.bulk.tensor (3-D maps: k, row, modulus),
//               128-byte swizzled 128-deep K slabs into a 4/6-stage smem ring
//   warp 1      one elected thread issues tcgen05.mma kind::i8 (INT32
//               accumulators in TMEM, two 256-column accumulator stages) and
//               tcgen05.commit's the smem slots / the finished accumulator
//   warps 2-9   epilogue: tcgen05.ld the accumulator, reduce every entry
//               modulo m_t in registers and store ONE BYTE per entry -- the
//               INT32 products never reach HBM (16 B instead of 64 B per
//               output across the 16 moduli); the CRT kernel reads the bytes.
//
// The accumulator is laid out with the OUTPUT COLUMN j on the TMEM lanes (the
// MMA's M side is B'_t) and the output row i on the TMEM columns (N side is
// A'_t), so a thread holds 32 consecutive rows of one output column and
// writes them as two 16-byte stores into the column-major byte plane.
//
// two_sm: a CTA pair shares one 256 (j) x 256 (i) tile through
// tcgen05.mma.cta_group::2 -- each CTA stages its own 128 lanes of B'_t and
// half of A'_t, the leader CTA issues the MMAs, tcgen05.commit multicasts the
// slot / accumulator barriers to both CTAs.  Halves the shared-memory and L2
// operand traffic per MAC against the single-CTA 128 x 256 tile.
#include <cuda.h>
#include <algorithm>
#include <cstdio>
#include "common.cuh"
#include "i8mma.cuh"

namespace bse {
namespace {

constexpr int kBK = 128;     // K bytes per stage = one 128-byte swizzle row
constexpr int kLanes = 128;  // TMEM lanes per CTA: output columns j
constexpr int kCols = 256;   // TMEM columns per accumulator stage: output rows i
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kGroupJ = 8;   // rasterisation: j tiles per group (L2 reuse of both operands)

struct ModTab {
  uint32_t m[kI8Mods], c2[kI8Mods], off[kI8Mods];
};
__constant__ ModTab c_mod;

template <int CG>
struct Cfg {
  static constexpr int kBytesL = kLanes * kBK;        // this CTA's lane-operand rows
  static constexpr int kBytesC = (kCols / CG) * kBK;  // this CTA's share of the column operand
  static constexpr int kStageBytes = kBytesL + kBytesC;
  static constexpr int kStages = (192 * 1024) / kStageBytes;  // 4 (CG 1) or 6 (CG 2)
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  // kind::i8, S32 accumulate, signed A and B, both K-major, N = 256, M = 128 CG
  static constexpr uint32_t kIdesc = (2u << 4) | (1u << 7) | (1u << 10) |
                                     ((uint32_t)(kCols >> 3) << 17) |
                                     ((uint32_t)((kLanes * CG) >> 4) << 24);
};

struct I8Params {
  uint8_t* R;
  long long plane, ldr;
  int M, N, num_kb, tiles_j, tiles_i, total, col0, lo, hi;
};

// ---- PTX wrappers (addresses are 32-bit shared-window addresses) ----------
BSE_DEV uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
BSE_DEV uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
BSE_DEV void bar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
BSE_DEV void bar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes)
               : "memory");
}
BSE_DEV void bar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
// Bounded wait: a protocol error traps (the launch fails) instead of hanging.
BSE_DEV void bar_wait(uint32_t a, uint32_t parity) {
  uint32_t done = 0;
  unsigned long long t0 = 0;
  for (uint32_t it = 0;; ++it) {
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity), "r"(0x989680u)  // suspend-time hint: the waiter sleeps in hardware
        : "memory");
    if (done) return;
    if ((it & 4095u) == 4095u) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      if (t - t0 > 20000000000ull) __trap();  // 20 s
    }
  }
}
BSE_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
BSE_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
BSE_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n"
               "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG>
BSE_DEV void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2) {
  if constexpr (CG == 1) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  } else {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  }
}

template <int CG>
BSE_DEV void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  if constexpr (CG == 1) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  } else {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
  }
}

// arrive on the barrier at this smem offset (in both CTAs of a pair) once all
// MMAs issued so far by this thread have completed
template <int CG>
BSE_DEV void mma_commit(uint32_t bar) {
  if constexpr (CG == 1) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                 : "memory");
  } else {
    const uint16_t mask = 3;
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(bar),
        "h"(mask)
        : "memory");
  }
}

// K-major operand tile, rows of 128 bytes, 128-byte swizzle (8-row atoms of
// 1024 bytes): start address, SBO = 1024 B, descriptor version 1 (sm_100).
BSE_DEV uint64_t smem_desc_sw128(uint32_t addr) {
  return (uint64_t)((addr & 0x3FFFFu) >> 4) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}

struct Tile {
  int t, tj, ti;
  bool skip;
};
template <int CG>
BSE_DEV Tile decode_tile(const I8Params& p, int tile) {
  Tile q;
  const int per = p.tiles_j * p.tiles_i;
  q.t = tile / per;
  const int rem = tile - q.t * per;
  const int grp = rem / (kGroupJ * p.tiles_i);
  const int gj0 = grp * kGroupJ;
  const int gsz = min(kGroupJ, p.tiles_j - gj0);
  const int loc = rem - grp * kGroupJ * p.tiles_i;
  q.tj = gj0 + loc % gsz;
  q.ti = loc / gsz;
  // output band: keep the tile if some (i, j) has lo <= col0 + j - i <= hi
  const int j0 = p.col0 + q.tj * (kLanes * CG), i0 = q.ti * kCols;
  const int j1 = min(p.col0 + p.N, j0 + kLanes * CG) - 1, i1 = min(p.M, i0 + kCols) - 1;
  q.skip = (j1 - i0 < p.lo) || (j0 - i1 > p.hi);
  return q;
}

template <int CG>
__global__ void __launch_bounds__(kThreads, 1)
i8mma_kernel(const __grid_constant__ CUtensorMap tmL, const __grid_constant__ CUtensorMap tmC,
             const I8Params p) {
  using C = Cfg<CG>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  const uint32_t bars = base + C::kStages * C::kStageBytes;
  auto full_bar = [&](int s) { return bars + 8u * s; };
  auto empty_bar = [&](int s) { return bars + 8u * (C::kStages + s); };
  auto tfull_bar = [&](int a) { return bars + 8u * (2 * C::kStages + a); };
  auto tempty_bar = [&](int a) { return bars + 8u * (2 * C::kStages + 2 + a); };
  const uint32_t tmem_slot = bars + 8u * (2 * C::kStages + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 1 ? 0u : cluster_ctarank();
  const int cluster_id = blockIdx.x / CG, num_clusters = gridDim.x / CG;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmL) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmC) : "memory");
    for (int s = 0; s < C::kStages; ++s) {
      bar_init(full_bar(s), 1);
      bar_init(empty_bar(s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      bar_init(tfull_bar(a), 1);
      bar_init(tempty_bar(a), kEpiWarps * CG);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tmem_slot),
                   "r"(512)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if constexpr (CG == 1) __syncthreads(); else cluster_sync_all();
  tc_fence_after();
  uint32_t tmem_base;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(tmem_base) : "r"(tmem_slot) : "memory");

  if (warp == 0) {
    // ===== TMA producer =====
    if (lane == 0) {
      const uint32_t full0 = CG == 1 ? full_bar(0) : mapa_rank(full_bar(0), 0);  // the leader's
      int st = 0;
      uint32_t ph = 0;
      for (int tile = cluster_id; tile < p.total; tile += num_clusters) {
        const Tile q = decode_tile<CG>(p, tile);
        if (q.skip) continue;
        const int rowL = q.tj * (kLanes * CG) + (int)rank * kLanes;
        const int rowC = q.ti * kCols + (int)rank * (kCols / CG);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          bar_wait(empty_bar(st), ph ^ 1u);
          if (rank == 0) bar_expect_tx(full_bar(st), (uint32_t)(CG * C::kStageBytes));
          const uint32_t dst = base + st * C::kStageBytes;
          tma_load_3d<CG>(dst, &tmL, full0 + 8u * st, kb * kBK, rowL, q.t);
          tma_load_3d<CG>(dst + C::kBytesL, &tmC, full0 + 8u * st, kb * kBK, rowC, q.t);
          if (++st == C::kStages) { st = 0; ph ^= 1u; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (leader CTA) =====
    if (lane == 0 && rank == 0) {
      int st = 0, as = 0;
      uint32_t ph = 0, aph = 0;
      for (int tile = cluster_id; tile < p.total; tile += num_clusters) {
        const Tile q = decode_tile<CG>(p, tile);
        if (q.skip) continue;
        bar_wait(tempty_bar(as), aph ^ 1u);
        tc_fence_after();
        const uint32_t tacc = tmem_base + (uint32_t)(as * kCols);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          bar_wait(full_bar(st), ph);
          tc_fence_after();
          const uint32_t sL = base + st * C::kStageBytes, sC = sL + C::kBytesL;
          const uint64_t dL = smem_desc_sw128(sL), dC = smem_desc_sw128(sC);
#pragma unroll
          for (int k = 0; k < kBK / 32; ++k)
            mma_i8<CG>(tacc, dL + (uint64_t)(2 * k), dC + (uint64_t)(2 * k), C::kIdesc,
                       (uint32_t)((kb | k) != 0));
          mma_commit<CG>(empty_bar(st));
          if (++st == C::kStages) { st = 0; ph ^= 1u; }
        }
        mma_commit<CG>(tfull_bar(as));
        if (++as == 2) { as = 0; aph ^= 1u; }
      }
    }
    __syncwarp();
  } else {
    // ===== epilogue: accumulator -> residues mod m_t -> bytes =====
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const uint32_t tempty0 = CG == 1 ? tempty_bar(0) : mapa_rank(tempty_bar(0), 0);
    int as = 0;
    uint32_t aph = 0;
    for (int tile = cluster_id; tile < p.total; tile += num_clusters) {
      const Tile q = decode_tile<CG>(p, tile);
      if (q.skip) continue;
      const uint32_t m = c_mod.m[q.t], c2 = c_mod.c2[q.t], off = c_mod.off[q.t];
      const int j = q.tj * (kLanes * CG) + (int)rank * kLanes + quad * 32 + lane;
      uint8_t* rowp = p.R + q.t * p.plane + (long long)j * p.ldr;
      bar_wait(tfull_bar(as), aph);
      tc_fence_after();
      const uint32_t taddr =
          tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(as * kCols + half * 128);
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
            "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
              "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
              "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
              "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
              "=r"(r[31])
            : "r"(taddr + (uint32_t)(c * 32))
            : "memory");
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        uint32_t w[8];
#pragma unroll
        for (int g = 0; g < 8; ++g) {
          uint32_t word = 0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            // u = c + off >= 0 with off = 0 mod m; floor(u / m) = (u c2) >> 39 exactly
            const uint32_t u = r[4 * g + e] + off;
            const uint32_t v = u - (__umulhi(u, c2) >> 7) * m;
            word |= v << (8 * e);
          }
          w[g] = word;
        }
        const int i0 = q.ti * kCols + half * 128 + c * 32;
        if (j < p.N && i0 < p.ldr) {
          uint4* dst = reinterpret_cast<uint4*>(rowp + i0);
          dst[0] = make_uint4(w[0], w[1], w[2], w[3]);
          dst[1] = make_uint4(w[4], w[5], w[6], w[7]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) bar_arrive_cluster(tempty0 + 8u * as);
      if (++as == 2) { as = 0; aph ^= 1u; }
    }
  }

  // ===== teardown =====
  tc_fence_before();
  if constexpr (CG == 1) __syncthreads(); else cluster_sync_all();
  if (warp == 1) {
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512)
                   : "memory");
  }
}

// ---------------------------------------------------------------------------
struct DevState {
  bool ready = false;
  int clusters[3] = {0, 0, 0};  // persistent grid size (in clusters) per CG
};
DevState g_dev[64];

template <int CG>
cudaError_t prepare(DevState& d) {
  using C = Cfg<CG>;
  cudaError_t e = cudaFuncSetAttribute(i8mma_kernel<CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       C::kSmem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int n = sms / CG;
  if (CG > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(sms / CG * CG));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = C::kSmem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int nc = 0;
    e = cudaOccupancyMaxActiveClusters(&nc, i8mma_kernel<CG>, &cfg);
    if (e != cudaSuccess) return e;
    if (nc > 0) n = std::min(n, nc);
  }
  d.clusters[CG] = std::max(1, n);
  return cudaSuccess;
}

cudaError_t init_device(DevState*& out) {
  int dev = 0;
  cudaGetDevice(&dev);
  DevState& d = g_dev[dev & 63];
  out = &d;
  if (d.ready) return cudaSuccess;
  ModTab h{};
  for (int t = 0; t < kI8Mods; ++t) {
    const uint64_t m = (uint64_t)i8_modulus(t);
    h.m[t] = (uint32_t)m;
    h.c2[t] = (uint32_t)(((1ull << 39) + m - 1) / m);
    h.off[t] = (uint32_t)((((1ull << 30) + m - 1) / m) * m);
  }
  cudaError_t e = cudaMemcpyToSymbol(c_mod, &h, sizeof(h));
  if (e != cudaSuccess) return e;
  if ((e = prepare<1>(d)) != cudaSuccess) return e;
  if ((e = prepare<2>(d)) != cudaSuccess) return e;
  d.ready = true;
  return cudaSuccess;
}

// 3-D map over 16 planes of rows x Kp int8: (k, row, modulus), box 128 x box_rows x 1
cudaError_t make_map(CUtensorMap* map, const int8_t* base, long long rows, int Kp, int box_rows) {
  const cuuint64_t dims[3] = {(cuuint64_t)Kp, (cuuint64_t)rows, (cuuint64_t)kI8Mods};
  const cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)rows * (cuuint64_t)Kp};
  const cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)box_rows, 1u};
  const cuuint32_t estr[3] = {1u, 1u, 1u};
  // resolved through the runtime (no link-time dependency on libcuda: the
  // library must load on a machine without a driver)
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
  if (!encode) return cudaErrorNotSupported;
  const CUresult r = encode(
      map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int CG>
cudaError_t launch(const DevState& d, const CUtensorMap& tmL, const CUtensorMap& tmC, const I8Params& p,
                   cudaStream_t s) {
  using C = Cfg<CG>;
  const int clusters = std::min(d.clusters[CG], p.total);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(clusters * CG));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, i8mma_kernel<CG>, tmL, tmC, p);
}

}  // namespace

cudaError_t i8mma_residues(int M, int N, int Kp, const int8_t* A8, long long rows_a,
                           const int8_t* B8, long long rows_b, uint8_t* R, long long ldr, int col0,
                           int lo, int hi, bool two_sm, cudaStream_t s) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  if (Kp <= 0 || Kp % 16 != 0 || Kp > 65536 || ldr % 32 != 0 || ldr < M || rows_a < M || rows_b < N)
    return cudaErrorInvalidValue;
  DevState* d = nullptr;
  cudaError_t e = init_device(d);
  if (e != cudaSuccess) return e;
  const int cg = two_sm ? 2 : 1;
  I8Params p;
  p.R = R;
  p.plane = rows_b * ldr;
  p.ldr = ldr;
  p.M = M;
  p.N = N;
  p.num_kb = (Kp + kBK - 1) / kBK;
  p.tiles_j = (N + kLanes * cg - 1) / (kLanes * cg);
  p.tiles_i = (M + kCols - 1) / kCols;
  p.total = kI8Mods * p.tiles_j * p.tiles_i;
  p.col0 = col0;
  p.lo = lo;
  p.hi = hi;
  CUtensorMap tmL, tmC;
  if ((e = make_map(&tmL, B8, rows_b, Kp, kLanes)) != cudaSuccess) return e;
  if ((e = make_map(&tmC, A8, rows_a, Kp, kCols / cg)) != cudaSuccess) return e;
  e = two_sm ? launch<2>(*d, tmL, tmC, p, s) : launch<1>(*d, tmL, tmC, p, s);
  if (e != cudaSuccess) return e;
  count_launch();
  return cudaGetLastError();
}

}  // namespace bse
