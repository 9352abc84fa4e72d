// Shared device helpers for the SlabLU B200 engine (sm_100a).
//
// FP64 tensor math on sm_100a is the warp-level mma.sync f64 path, which
// lowers to SASS DMMA.8x8x4 (tcgen05 has no f64 kind).  Everything here is
// written for that pipe: m8n8k4 fragments, cp.async staging, padded shared
// tiles (row stride == 4 mod 16 doubles so a fragment load is 2 wavefronts).
#pragma once
#include <cstdlib>
#include <utility>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define SLB_CUDA_CHECK(expr)                                                        \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) throw ::slb::CudaFailure(_e, #expr, __FILE__, __LINE__); \
  } while (0)

namespace slb {

struct CudaFailure {
  cudaError_t err;
  const char* expr;
  const char* file;
  int line;
  CudaFailure(cudaError_t e, const char* x, const char* f, int l) : err(e), expr(x), file(f), line(l) {}
};

// D(8x8) += A(8x4) * B(4x8).  Fragments (lane = 4*g + t):
//   a = A[g][t], b = B[t][g], d0/d1 = D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async copy global -> shared; zero-fills when !pred.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
  const int bytes = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes));
}
// 16-byte async copy (both addresses 16-byte aligned); zero-fills when !pred.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
  const int bytes = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return cdiv(a, b) * b; }

}  // namespace slb

namespace slb {
// Kernels launched by the engine (every launch site calls count_launch(); reported as
// gpu_launches / solve_launches).
extern std::atomic<long long> g_kernel_count;
inline void count_launch() { g_kernel_count.fetch_add(1, std::memory_order_relaxed); }

// Launch with programmatic stream serialization (the kernel may begin before the previous grid
// of the stream completes; it calls pdl_wait() before reading that grid's results).
// SLB_NO_PDL=1 launches it plainly.
template <class... P, class... A>
inline void launch_pdl(void (*k)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  static const bool off = getenv("SLB_NO_PDL") != nullptr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = off ? 0 : 1;
  SLB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...));
  count_launch();
}
// ---- mbarrier + TMA bulk copy (cp.async.bulk) helpers ----------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// Non-blocking probe of a phase (mbarrier.test_wait): true once the phase with this parity completed.
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, P1;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(phase)
      : "memory");
  return ok != 0;
}
// Same with a suspend-time hint: the waiting thread sleeps in hardware until the phase completes
// (or the hint, in ns, expires) instead of re-polling; spinning warps otherwise take issue slots
// from the warps doing the work on the same sub-partition.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(1000000u)
      : "memory");
}
// Distributed shared memory: address of `local` in CTA `rank` of the cluster, and 32-bit loads
// through the shared::cluster window (cheaper than generic loads of a mapped pointer).
// Programmatic dependent launch: wait for the preceding grid's completion (a no-op for a grid
// launched without the attribute) / let the next grid of the stream start launching.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t dsmem_map(const void* local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
__device__ __forceinline__ double dsmem_ld_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];\n" : "=d"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void dsmem_st_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(addr), "d"(v) : "memory");
}
__device__ __forceinline__ void dsmem_st_s32(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int dsmem_ld_s32(uint32_t addr) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];\n" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
// idx / d for small quotients (idx < 2^20, idx / d <= 4096) via a float reciprocal: the hot
// index loops of the chain kernels otherwise spend their issue slots on integer division.
// (idx + 0.5) / d stays >= 0.5 / d away from the next integer, far above the float error.
__device__ __forceinline__ int qdiv(int idx, float inv_d) { return (int)(((float)idx + 0.5f) * inv_d); }

// 16-byte store into a peer CTA's shared memory, completion counted (bytes) on the peer's mbarrier
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
               "d"(a), "d"(b), "r"(rbar)
               : "memory");
}
// 1-D TMA bulk copy global -> shared, completion signalled on bar (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
}  // namespace slb
