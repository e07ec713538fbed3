// tg_ptx.cuh — sm_100a inline-PTX wrappers: mbarrier, TMA, tcgen05 / TMEM,
// system-scope flags.  Used only by the product kernels (not by the oracle).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace tg {

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Timeout for every device-side wait: a hung wait traps instead of hanging the GPU.
constexpr uint64_t kWaitTimeoutNs = 4000000000ull;

__device__ __forceinline__ void device_fail(int *err, int code) {
  if (err) atomicExch(err, code);
  __threadfence_system();
  asm volatile("trap;");
}

// ------------------------------------------------------------------ mbarrier
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, P1;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Blocking wait on an mbarrier phase, bounded by kWaitTimeoutNs.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity, int *err) {
  if (mbar_try_wait(bar, parity)) return;
  uint64_t t0 = globaltimer_ns();
  while (!mbar_try_wait(bar, parity)) {
    if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, 0x1001);
  }
}

// ---------------------------------------------------------------------- TMA
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap *map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// 2D tiled load global -> shared, completes tx bytes on `bar`.  c0 = inner (column) coordinate.
__device__ __forceinline__ void tma_load_2d(void *smem_dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, uint64_t cache_policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(cache_policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// Bulk L2 prefetch of a contiguous global range (size % 16 == 0).
__device__ __forceinline__ void prefetch_l2_bulk(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(p)), "r"(bytes)
               : "memory");
}
// Generic-proxy writes (st.global) -> visible to later async-proxy (TMA) reads.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------ tcgen05 / TMEM
__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// D[tmem] (+)= A[smem] * B[smem]^T, bf16 x bf16 -> fp32, cta_group::1.
__device__ __forceinline__ void umma_bf16_ss(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive on `bar` when all previously issued tcgen05.mma of this thread complete.
__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns: thread i gets lane (base+i), columns col..col+31.
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}

// Shared-memory matrix descriptor, K-major operand staged by TMA with 128-byte
// swizzle: rows of 128 B (64 bf16 of K), 8-row core groups 1024 B apart (SBO).
__device__ __forceinline__ uint64_t desc_sw128_kmajor(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr & 0x3FFFFu) >> 4);  // [0,14) start address >> 4
  d |= static_cast<uint64_t>(1) << 16;                       // [16,30) LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;               // [32,46) SBO = 1024 B
  d |= static_cast<uint64_t>(1) << 46;                       // [46,48) descriptor version 1 (sm100)
  d |= static_cast<uint64_t>(2) << 61;                       // [61,64) SWIZZLE_128B
  return d;
}

// Instruction descriptor, kind::f16: A = B = bf16, D = fp32, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16_f32(int M, int N) {
  return (1u << 4)                                   // D format f32
         | (1u << 7)                                 // A format bf16
         | (1u << 10)                                // B format bf16
         | (static_cast<uint32_t>(N >> 3) << 17)     // N >> 3
         | (static_cast<uint32_t>(M >> 4) << 24);    // M >> 4
}

// ------------------------------------------------------- cross-GPU flags
__device__ __forceinline__ void st_release_sys(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acquire_gpu(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Scope-selected variants: world == 1 needs only GPU scope (no NVLink peers);
// system-scope fences are microseconds and are paid only when peers exist.
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v, bool sys) {
  if (sys) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p, bool sys) {
  uint32_t v;
  if (sys) asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_scope(bool sys) {
  if (sys) __threadfence_system();
  else __threadfence();
}
__device__ __forceinline__ void wait_flag_ge_s(const uint32_t *flag, uint32_t epoch, bool sys, int *err, int code) {
  if (static_cast<int32_t>(ld_acquire(flag, sys) - epoch) >= 0) return;
  uint64_t t0 = globaltimer_ns();
  while (static_cast<int32_t>(ld_acquire(flag, sys) - epoch) < 0) {
    if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, code);
  }
}

// Wait on a PEER's flag with failure detection: false if it did not reach epoch
// within timeout_ns (the peer is taken as failed; no trap).
__device__ __forceinline__ bool wait_flag_or_fail(const uint32_t *flag, uint32_t epoch, bool sys, long long timeout_ns) {
  if (static_cast<int32_t>(ld_acquire(flag, sys) - epoch) >= 0) return true;
  uint64_t t0 = globaltimer_ns();
  while (static_cast<int32_t>(ld_acquire(flag, sys) - epoch) < 0) {
    if ((long long)(globaltimer_ns() - t0) > timeout_ns) return false;
  }
  return true;
}

// Wait until the counter reaches target; false after timeout_ns (a peer that should add to it
// failed; no trap).  Scope-selected acquire (peers add with system-scope atomics over NVLink).
__device__ __forceinline__ bool wait_ctr_or_fail(const int *ctr, int target, bool sys, long long timeout_ns) {
  auto ld = [&]() {
    int v;
    if (sys) asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    else asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    return v;
  };
  if (ld() >= target) return true;
  const uint64_t t0 = globaltimer_ns();
  while (ld() < target)
    if ((long long)(globaltimer_ns() - t0) > timeout_ns) return false;
  return true;
}

// Spin until *flag >= epoch (wrap-safe), bounded.
__device__ __forceinline__ void wait_flag_ge(const uint32_t *flag, uint32_t epoch, int *err, int code) {
  if (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) >= 0) return;
  uint64_t t0 = globaltimer_ns();
  while (static_cast<int32_t>(ld_acquire_sys(flag) - epoch) < 0) {
    if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, code);
  }
}
__device__ __forceinline__ void wait_ctr_ge(const int *ctr, int target, int *err, int code) {
  if (ld_acquire_gpu(ctr) >= target) return;
  uint64_t t0 = globaltimer_ns();
  while (ld_acquire_gpu(ctr) < target) {
    if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, code);
  }
}

// Grid-wide barrier for a cooperative launch (all CTAs co-resident).  `count`
// is a 64-bit counter that is never reset: barrier i of call `epoch` (1-based)
// completes when count reaches ((epoch-1)*nbar + i+1) * nct (nct = CTAs of the rank's grid).
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned long long *count, uint32_t epoch, int nbar, int i, int *err,
                                             unsigned nct) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target =
        ((unsigned long long)(epoch - 1) * nbar + (unsigned long long)(i + 1)) * nct;
    __threadfence();
    atomicAdd(count, 1ull);
    if (ld_acquire_gpu_u64(count) < target) {
      uint64_t t0 = globaltimer_ns();
      while (ld_acquire_gpu_u64(count) < target)
        if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, 0x3001);
    }
    __threadfence();
  }
  __syncthreads();
}

// Grid barrier on a counter that starts at 0 for this call (barrier i completes
// at (i + 1) * nct arrivals): the number of barriers may vary per call.
__device__ __forceinline__ void grid_barrier_z(unsigned long long *count, int i, int *err, unsigned nct) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long target = (unsigned long long)(i + 1) * nct;
    __threadfence();
    atomicAdd(count, 1ull);
    if (ld_acquire_gpu_u64(count) < target) {
      uint64_t t0 = globaltimer_ns();
      while (ld_acquire_gpu_u64(count) < target)
        if (globaltimer_ns() - t0 > kWaitTimeoutNs) device_fail(err, 0x3002);
    }
    __threadfence();
  }
  __syncthreads();
}

// Programmatic dependent launch: wait until the previous grid in the stream has completed and its
// memory is visible (a no-op without the launch attribute).
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace tg
