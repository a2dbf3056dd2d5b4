// Tensor memory (TMEM) as plain storage, inline PTX for sm_100a.
//
// The stencil kernels use TMEM for what it is outside MMA: 128 lanes x 512
// 32-bit columns per SM that a warp reads with tcgen05.ld at several times
// shared memory's bandwidth (tools/tmem_probe.cu: ~390 B/SM-cycle at 16
// warps vs 128 for LDS).  Warp w of a CTA reaches lanes 32 (w % 4) .. +31
// only; with the 32x32b shapes thread t of the warp reads / writes its own
// lane, N consecutive columns.
#pragma once

#include <cstdint>

namespace sdmp {

// One warp allocates `cols` (power of two >= 32) columns and writes the base
// address to *dst (shared).  Caller: fence / CTA barrier / fence, then read.
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
  static_assert(COLS >= 32 && COLS <= 512 && (COLS & (COLS - 1)) == 0, "TMEM columns");
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "n"(COLS)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t base) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS)
               : "memory");
}
__device__ __forceinline__ void tmem_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tmem_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 8 consecutive columns of this thread's lane <-> two float4
__device__ __forceinline__ void tmem_ld8(uint32_t a, float4& p, float4& q) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(p.x), "=f"(p.y), "=f"(p.z), "=f"(p.w), "=f"(q.x), "=f"(q.y), "=f"(q.z),
                 "=f"(q.w)
               : "r"(a));
}
__device__ __forceinline__ void tmem_st8(uint32_t a, const float4& p, const float4& q) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a),
               "f"(p.x), "f"(p.y), "f"(p.z), "f"(p.w), "f"(q.x), "f"(q.y), "f"(q.z), "f"(q.w)
               : "memory");
}
// loads complete (registers valid) / stores complete (columns readable)
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
// After tmem_wait_ld: re-define the loaded registers through an (empty)
// volatile asm so no use of them can be scheduled above the wait.
__device__ __forceinline__ void tmem_pin(float4& p) {
  asm volatile("" : "+f"(p.x), "+f"(p.y), "+f"(p.z), "+f"(p.w));
}

}  // namespace sdmp
