// sxen_tc.cuh -- tcgen05 / TMEM building blocks (sm_100a inline PTX) for the tensor-core MLP head.
//
// Shared-memory operand tiles use the no-swizzle "core matrix" (interleaved) layout, CM(rows, cols) of 32-bit elements:
//     byte_offset(r, c) = (r/8) * row_group_stride + (c/4) * 128 + (r%8) * 16 + (c%4) * 4,   row_group_stride = (cols/4)*128
// i.e. 8x(16 B) core matrices stored contiguously (128 B), core matrices of one 8-row group side by side.
// The layout is self-dual: the same tile is
//   * a K-major operand   [MN = rows, K = cols]  with LBO = 128 B (next 16-byte K chunk), SBO = row_group_stride
//   * an MN-major operand [MN = cols, K = rows]  with SBO = 128 B (next 16-byte MN chunk), LBO = row_group_stride
// which is what lets one activation tile feed the forward GEMM (samples x features), the input-gradient GEMM and the
// weight-gradient GEMM (features x samples) without a transpose.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sxen_tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__host__ __device__ constexpr uint32_t cm_row_group_stride(int cols) { return static_cast<uint32_t>(cols / 4) * 128u; }
__host__ __device__ constexpr uint32_t cm_bytes(int rows, int cols) { return static_cast<uint32_t>(rows / 8) * cm_row_group_stride(cols); }
__host__ __device__ constexpr uint32_t cm_offset(int r, int c, int cols) {
  return static_cast<uint32_t>(r / 8) * cm_row_group_stride(cols) + static_cast<uint32_t>(c / 4) * 128u +
         static_cast<uint32_t>(r % 8) * 16u + static_cast<uint32_t>(c % 4) * 4u;
}

// round-to-nearest fp32 -> tf32 (the tensor core ignores the 13 low mantissa bits; rounding first removes the bias)
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

// 64-bit shared-memory matrix descriptor (sm_100 format: version 1 at bits 46-47, layout type 0 = no swizzle).
__device__ __forceinline__ uint64_t make_desc(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  return d;
}
// K-major view of a CM tile (MN = rows): the two 16-byte K chunks of one UMMA_K=8 step are `128 B` apart.
__device__ __forceinline__ uint64_t desc_k_major(uint32_t tile_addr, int cols, int k_step) {
  return make_desc(tile_addr + static_cast<uint32_t>(k_step) * 256u, 128u, cm_row_group_stride(cols));
}
// MN-major view of a CM tile (K = rows): one UMMA_K=8 step is one 8-row group.
__device__ __forceinline__ uint64_t desc_mn_major(uint32_t tile_addr, int cols, int k_step, int mn_offset = 0) {
  return make_desc(tile_addr + static_cast<uint32_t>(k_step) * cm_row_group_stride(cols) + static_cast<uint32_t>(mn_offset / 4) * 128u,
                   cm_row_group_stride(cols), 128u);
}

// ---- 128-byte-swizzled tiles, SW(rows, cols): cols in blocks of 32 elements (128 B), each block a contiguous
// [rows][32] sub-tile; inside a block 8-row groups of 1 KB, 16-byte chunks XOR-swizzled with (row % 8).  Self-dual like CM:
//   K-major  [MN = rows, K = cols]: SBO = 1024 B, K step of 8 elements = +32 B inside a block, next block = +rows*128 B
//   MN-major [MN = cols, K = rows]: LBO = rows*128 B (next 32-col block), SBO = 1024 B, K step of 8 rows = +1024 B
__host__ __device__ constexpr uint32_t sw_bytes(int rows, int cols) { return static_cast<uint32_t>(rows) * static_cast<uint32_t>(cols) * 4u; }
__host__ __device__ constexpr uint32_t sw_offset(int r, int c, int rows) {
  return static_cast<uint32_t>(c / 32) * static_cast<uint32_t>(rows) * 128u + static_cast<uint32_t>(r / 8) * 1024u +
         static_cast<uint32_t>(r % 8) * 128u + ((static_cast<uint32_t>((c % 32) / 4) ^ static_cast<uint32_t>(r % 8)) * 16u) +
         static_cast<uint32_t>(c % 4) * 4u;
}
__device__ __forceinline__ uint64_t make_desc_sw128(uint32_t smem_addr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ uint64_t sw_desc_k_major(uint32_t tile_addr, int rows, int k_step) {
  return make_desc_sw128(tile_addr + static_cast<uint32_t>(k_step / 4) * static_cast<uint32_t>(rows) * 128u +
                             static_cast<uint32_t>(k_step % 4) * 32u, 16u, 1024u);
}
__device__ __forceinline__ uint64_t sw_desc_mn_major(uint32_t tile_addr, int rows, int k_step) {
  return make_desc_sw128(tile_addr + static_cast<uint32_t>(k_step) * 1024u, static_cast<uint32_t>(rows) * 128u, 1024u);
}

// Instruction descriptor for kind::tf32, fp32 accumulate (bit layout: cute/arch/mma_sm100_desc.hpp InstrDescriptor).
__host__ __device__ constexpr uint32_t make_idesc_tf32(int m, int n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
         (static_cast<uint32_t>(b_mn_major) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate))
      : "memory");
}

// ---- 16-bit operands (bf16, kind::f16, UMMA_K = 16).  CM16(rows, cols): 8x(16 B = 8 elements) core matrices,
//     byte_offset(r, c) = (r/8) * (cols/8)*128 + (c/8)*128 + (r%8)*16 + (c%8)*2
// Self-dual exactly like the 32-bit CM tile; one UMMA_K = 16 step is two 16-byte K chunks (K-major) or two 8-row
// groups (MN-major, the pair sits LBO apart).
__host__ __device__ constexpr uint32_t cm16_row_group_stride(int cols) { return static_cast<uint32_t>(cols / 8) * 128u; }
__host__ __device__ constexpr uint32_t cm16_bytes(int rows, int cols) { return static_cast<uint32_t>(rows / 8) * cm16_row_group_stride(cols); }
__host__ __device__ constexpr uint32_t cm16_offset(int r, int c, int cols) {
  return static_cast<uint32_t>(r / 8) * cm16_row_group_stride(cols) + static_cast<uint32_t>(c / 8) * 128u +
         static_cast<uint32_t>(r % 8) * 16u + static_cast<uint32_t>(c % 8) * 2u;
}
__device__ __forceinline__ uint64_t desc16_k_major(uint32_t tile_addr, int cols, int k_step) {
  return make_desc(tile_addr + static_cast<uint32_t>(k_step) * 256u, 128u, cm16_row_group_stride(cols));
}
__device__ __forceinline__ uint64_t desc16_mn_major(uint32_t tile_addr, int cols, int k_step, int mn_offset = 0) {
  return make_desc(tile_addr + static_cast<uint32_t>(k_step) * 2u * cm16_row_group_stride(cols) + static_cast<uint32_t>(mn_offset / 8) * 128u,
                   cm16_row_group_stride(cols), 128u);
}
__host__ __device__ constexpr uint32_t make_idesc_bf16(int m, int n, bool a_mn_major, bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn_major) << 15) |
         (static_cast<uint32_t>(b_mn_major) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, bool accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate))
      : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t cols) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(smem_dst)), "r"(cols) : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t cols) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// tcgen05.commit: the mbarrier receives one arrival when every MMA issued so far by this thread has completed.
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Waits for the phase of `bar` with the given parity to complete.  A hand-off bug between warp roles shows up as a wait that
// never ends; a hung kernel takes the GPU with it, so the wait carries a watchdog: after ~2 s (4e9 cycles) it traps -- the
// host sees a CUDA error instead of a hang -- after noting which wait gave up in `dbg` (host-mapped words, may be null):
// dbg[0] = id, dbg[1] = blockIdx.x.
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.b32 %0, 1, 0, p;\n\t}\n"
      : "=r"(done)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return done != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity, uint32_t id = 0, volatile unsigned int* dbg = nullptr) {
  if (mbar_try_wait(bar, parity)) return;
  const long long t0 = clock64();
  uint32_t spins = 0;
  while (!mbar_try_wait(bar, parity)) {
    if ((++spins & 0x3ffu) == 0u && clock64() - t0 > 4000000000ll) {
      if (dbg != nullptr) {
        dbg[0] = id;
        dbg[1] = blockIdx.x;
        __threadfence_system();
      }
      __trap();
    }
  }
}

// TMEM -> registers: this warp's 32 lanes x 16 consecutive columns (thread = lane = accumulator row).
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace sxen_tc
