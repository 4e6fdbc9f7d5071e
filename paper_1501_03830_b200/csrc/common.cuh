// Shared device helpers for the B200 (sm_100a) FP64 BSE eigensolver.
//
// FP64 math on sm_100a: tcgen05 has no f64 kind, so dense contractions use the
// warp-level DMMA path (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4) fed from
// shared memory staged with cp.async (LDGSTS).  Everything here is FP64.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#define BSE_HD __host__ __device__ __forceinline__
#define BSE_DEV __device__ __forceinline__

namespace bse {

constexpr double kEps = 2.220446049250313e-16;     // DBL_EPSILON (numpy finfo eps)
constexpr double kSafmin = 2.2250738585072014e-308; // DBL_MIN (numpy finfo tiny)
constexpr int kNoMaskLo = -(1 << 30);
constexpr int kNoMaskHi = (1 << 30);

// ---------------------------------------------------------------------------
// DMMA: D(8x8) += A(8x4, row) * B(4x8, col), FP64.
//   a: A[lane>>2][lane&3]   b: B[lane&3][lane>>2]   d: D[lane>>2][2*(lane&3)+{0,1}]
BSE_DEV void dmma8x8x4(double (&d)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// cp.async (LDGSTS).  src-size 0 zero-fills the destination.
BSE_DEV void cp_async16(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
BSE_DEV void cp_async8(void* smem, const void* gmem, bool pred) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  int sz = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
BSE_DEV void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BSE_DEV void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---------------------------------------------------------------------------
// mbarrier + bulk async copy (TMA engine, non-tensor form)
BSE_DEV unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
BSE_DEV void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
BSE_DEV void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
BSE_DEV void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
BSE_DEV void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
BSE_DEV void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy (bytes % 16 == 0, 16-byte aligned), completion
// counted on `bar` as transaction bytes
BSE_DEV void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

// orders this thread's earlier generic-proxy accesses (here: an acquire of
// data other CTAs stored) before its later async-proxy (bulk copy) accesses
BSE_DEV void fence_proxy_async() { asm volatile("fence.proxy.async;\n" ::: "memory"); }

// ---------------------------------------------------------------------------
// Self-validating 16-byte mailbox slots {bits, bits ^ tag}: a value handed
// from one CTA to another without fences or a separate flag.  Each 8-byte
// half is written atomically, so a torn or stale slot never validates
// against the reader's tag (64-bit hashes of the slot's use); readers poll.
BSE_DEV unsigned long long mail_tag(int s, int j) {
  unsigned long long x = ((unsigned long long)(unsigned)s << 24) ^ (unsigned long long)(unsigned)j;
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return (x ^ (x >> 31)) | 1ull;
}
BSE_DEV void mail_put(unsigned long long* slot, double v, unsigned long long tag) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  asm volatile("st.global.v2.u64 [%0], {%1, %2};\n" ::"l"(slot), "l"(bits), "l"(bits ^ tag) : "memory");
}
BSE_DEV double mail_get(const unsigned long long* slot, unsigned long long tag) {
  unsigned long long lo, hi;
  do {
    asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];\n" : "=l"(lo), "=l"(hi) : "l"(slot) : "memory");
  } while ((lo ^ hi) != tag);
  return __longlong_as_double((long long)lo);
}

// ---------------------------------------------------------------------------
// Reductions
BSE_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
BSE_DEV double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum in fixed order (deterministic).  `red` needs >= 32 doubles.
BSE_DEV double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// L2-coherent loads for data written by other CTAs of the same launch.
BSE_DEV double ld_cg(const double* p) { return __ldcg(p); }

// Acquire / release flag helpers for inter-CTA pipelines.
BSE_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
BSE_DEV int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
BSE_DEV void fence_acquire() { asm volatile("fence.acq_rel.gpu;\n" ::: "memory"); }
BSE_DEV void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// release increment: orders this thread's earlier writes (and, through a
// preceding warp barrier, its warp's) before the add, without the acquire half
// of a full fence (no L1 invalidate)
BSE_DEV void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

BSE_HD long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

// One-time per-kernel setup that applies to the CURRENT device only
// (cudaFuncSetAttribute): one bit per device ordinal, so a process that later
// solves on another device repeats the setup there.
struct PerDeviceOnce {
  std::atomic<unsigned long long> bits{0};
  static int ordinal() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  bool needed() const { return !((bits.load(std::memory_order_acquire) >> ordinal()) & 1ull); }
  void mark() { bits.fetch_or(1ull << ordinal(), std::memory_order_acq_rel); }
};

// Raise a kernel's dynamic shared-memory limit once per device; returns the
// runtime's error (not swallowed).
template <class F>
inline cudaError_t set_smem_limit(PerDeviceOnce& once, F* kern, int bytes) {
  if (!once.needed()) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) once.mark();
  return e;
}

// Host-side count of kernel launches issued by this library (bench evidence).
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
inline void count_launch(long long k = 1) { launch_counter().fetch_add(k, std::memory_order_relaxed); }

// Stage timing with CUDA events (enabled by bse_profile_enable).
void stage_mark(const char* name, cudaStream_t s);

}  // namespace bse
