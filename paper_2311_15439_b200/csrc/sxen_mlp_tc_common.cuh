// sxen_mlp_tc_common.cuh -- pieces shared by the two tcgen05 MLP kernels (sxen_mlp_tc.cu: fused forward + loss + backward;
// sxen_mlp_tc_fwd.cu: forward only): the argument block, the split-bf16 tile stores, TMEM loads, the split GEMM issue loop.
#pragma once

#include <cuda_bf16.h>

#include "sxen_common.hpp"
#include "sxen_tc.cuh"

namespace sxen_mlp_tc {

using namespace sxen_tc;

constexpr int kTile = 128;
constexpr int kInMax = 32, HID = 64, OUTP = 16;  // the kernels are instantiated for input widths 16 and 32 (template IN)
constexpr int kX0CMax = kInMax + 8, HC = HID + 8;  // tile widths including the ones-column block

struct TcArgs {
  const float* params;      // W0[64x32] b0[64] W1[64x64] b1[64] W2[ow x 64] b2[ow]  (src/mlp.cpp:19-32)
  const float* features;    // N x 32
  const void* targets;      // N x ow, f32 or f64
  float* pred;              // N x ow or nullptr
  float* input_grad;        // N x 32 (training)
  double* mlp_grad;         // parameter layout, accumulated into
  double* loss_sum;         // accumulated into
  long long* grad_fixed;    // reproducible mode: parameter layout in units of 2^-52, then one double per CTA for the loss (nullptr = off)
  double* partials;         // sxen_mlp_tc2.cu: one row of `partial_stride` doubles per CTA (parameter layout); the CTA adds its
  unsigned long long partial_stride;  // gradients there and a reduction kernel folds the rows into mlp_grad (nullptr = atomics on mlp_grad)
  unsigned long long n;
  int out_w;
  int target_f32;
  int precise;              // 0: single bf16 product, 1: bf16x3, 2: bf16x4 (gemm_split)
  double upstream_scale;    // 2 / (global_batch * out_w)
  unsigned long long* timing;       // tuning aid (nullptr = off): {epilogue thread 0: cycles in the tile loop, of those waiting on the
                                    // chain, waiting on the weight-gradient MMAs; chain warp: loop cycles, waiting on the epilogue}
  volatile unsigned int* progress;  // debugging aid (nullptr = off): host-mapped words the mbar_wait watchdog writes (id, CTA)
};

// x = hi + lo with hi = bf16(x), lo = bf16(x - hi); two values per F2FP pack instruction.
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __nv_bfloat162 hp = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hp);  // low half = element 0
    const float h0 = __uint_as_float(hb << 16), h1 = __uint_as_float(hb & 0xffff0000u);
    const __nv_bfloat162 lp = __floats2bfloat162_rn(v[2 * q] - h0, v[2 * q + 1] - h1);
    h[q] = hb;
    l[q] = *reinterpret_cast<const uint32_t*>(&lp);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Row `row` of a CM16(., cols) hi/lo tile pair: columns [8*chunk, 8*chunk+8) <- v[0..8)
__device__ __forceinline__ void store_chunk(unsigned char* tile_hi, unsigned char* tile_lo, int row, int chunk, int cols,
                                            const float* v) {
  uint4 hi, lo;
  split8(v, hi, lo);
  const uint32_t off = cm16_offset(row, 8 * chunk, cols);
  *reinterpret_cast<uint4*>(tile_hi + off) = hi;
  *reinterpret_cast<uint4*>(tile_lo + off) = lo;
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// D += A*B over `ksteps` UMMA_K=16 steps with split operands.  a0/b0 are the descriptors of the hi tiles at k step 0;
// the lo tile sits `a_lo`/`b_lo` bytes further and one k step adds `a_step`/`b_step` bytes (address field = bytes >> 4).
// precise: 0 = one bf16 product; 1 = split operands, three products (hi*hi + hi*lo + lo*hi); 2 = the fourth product too
// (lo*lo, <= 2^-18 of a term: SXEN_MLP_TENSOR_BF16X4 -- predictions and input gradients within 1e-5 of the largest magnitude at
// +15 % kernel time, tools/tc_accuracy.py, profiles/r2s4_tc_lolo.log).
// The product count is dispatched ONCE per GEMM (PRODUCTS is a template argument of the issue loop): a per-k-step test of a
// run-time `precise` for the fourth product cost the default mode 5 % (0.303 -> 0.318 ms per 2^20 samples).
template <int PRODUCTS>
__device__ __forceinline__ void gemm_split_p(uint32_t d, uint32_t idesc, int ksteps, bool accumulate, uint64_t a0, uint32_t a_lo,
                                             uint32_t a_step, uint64_t b0, uint32_t b_lo, uint32_t b_step) {
  for (int ks = 0; ks < ksteps; ++ks) {
    const uint64_t ah = a0 + ((static_cast<uint64_t>(ks) * a_step) >> 4), bh = b0 + ((static_cast<uint64_t>(ks) * b_step) >> 4);
    mma_bf16(d, ah, bh, idesc, accumulate || ks > 0);
    if constexpr (PRODUCTS >= 3) {
      mma_bf16(d, ah, bh + (b_lo >> 4), idesc, true);
      mma_bf16(d, ah + (a_lo >> 4), bh, idesc, true);
    }
    if constexpr (PRODUCTS >= 4) mma_bf16(d, ah + (a_lo >> 4), bh + (b_lo >> 4), idesc, true);
  }
}
__device__ __forceinline__ void gemm_split(uint32_t d, uint32_t idesc, int ksteps, bool accumulate, int precise, uint64_t a0,
                                           uint32_t a_lo, uint32_t a_step, uint64_t b0, uint32_t b_lo, uint32_t b_step) {
  if (precise == 1) gemm_split_p<3>(d, idesc, ksteps, accumulate, a0, a_lo, a_step, b0, b_lo, b_step);
  else if (precise == 0) gemm_split_p<1>(d, idesc, ksteps, accumulate, a0, a_lo, a_step, b0, b_lo, b_step);
  else gemm_split_p<4>(d, idesc, ksteps, accumulate, a0, a_lo, a_step, b0, b_lo, b_step);
}

// The same GEMM issued from warp-uniform code: the whole warp walks the loop with warp-uniform operands (descriptors built from
// __shfl_sync'ed values live in uniform registers) and only the MMA instruction itself is predicated on `leader`.  Issued from
// inside an `if (lane == 0)` branch the compiler must assume per-thread descriptors and wraps every tcgen05.mma in a
// serialising loop (ELECT + 3 x R2UR.BROADCAST + branch): ~35 cycles per MMA against ~10 here.
__device__ __forceinline__ void mma_bf16_elect(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, bool accumulate,
                                               bool leader) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, %4, 0;\n\tsetp.ne.b32 q, %5, 0;\n\t"
      "@q tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(static_cast<uint32_t>(accumulate)), "r"(static_cast<uint32_t>(leader))
      : "memory");
}
template <int PRODUCTS>
__device__ __forceinline__ void gemm_split_uniform_p(uint32_t d, uint32_t idesc, int ksteps, bool accumulate, uint64_t a0,
                                                     uint32_t a_lo, uint32_t a_step, uint64_t b0, uint32_t b_lo, uint32_t b_step,
                                                     bool leader) {
#pragma unroll
  for (int ks = 0; ks < ksteps; ++ks) {
    const uint64_t ah = a0 + ((static_cast<uint64_t>(ks) * a_step) >> 4), bh = b0 + ((static_cast<uint64_t>(ks) * b_step) >> 4);
    mma_bf16_elect(d, ah, bh, idesc, accumulate || ks > 0, leader);
    if constexpr (PRODUCTS >= 3) {
      mma_bf16_elect(d, ah, bh + (b_lo >> 4), idesc, true, leader);
      mma_bf16_elect(d, ah + (a_lo >> 4), bh, idesc, true, leader);
    }
    if constexpr (PRODUCTS >= 4) mma_bf16_elect(d, ah + (a_lo >> 4), bh + (b_lo >> 4), idesc, true, leader);
  }
}
__device__ __forceinline__ void gemm_split_uniform(uint32_t d, uint32_t idesc, int ksteps, bool accumulate, int precise, uint64_t a0,
                                                   uint32_t a_lo, uint32_t a_step, uint64_t b0, uint32_t b_lo, uint32_t b_step,
                                                   bool leader) {
  if (precise == 1) gemm_split_uniform_p<3>(d, idesc, ksteps, accumulate, a0, a_lo, a_step, b0, b_lo, b_step, leader);
  else if (precise == 0) gemm_split_uniform_p<1>(d, idesc, ksteps, accumulate, a0, a_lo, a_step, b0, b_lo, b_step, leader);
  else gemm_split_uniform_p<4>(d, idesc, ksteps, accumulate, a0, a_lo, a_step, b0, b_lo, b_step, leader);
}

// One CTA's partial sum into the batch total: an fp64 atomic, or -- reproducible mode -- an integer atomic on the fixed-point
// shadow of the same element (order-free; sxen_mlp.cu folds the shadow into the fp64 buffer after the kernel).
// Explicit `red`: atomicAdd with its result unused compiles to ATOMG with a discarded destination for 64-bit operands, and a
// warp then issues one such instruction per L2 round trip (a 64-instruction read-out took 49 k cycles).
__device__ __forceinline__ void add_total(double* base, long long* fixed, size_t index, double v) {
  if (fixed != nullptr)
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(fixed + index), "l"(__double2ll_rn(__dmul_rn(v, 0x1p52))) : "memory");
  else
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(base + index), "d"(v) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

#ifndef SXEN_TC_SPLIT
#define SXEN_TC_SPLIT 2
#endif
constexpr int kSplit = SXEN_TC_SPLIT;           // epilogue threads per sample row: each handles HID/kSplit columns
constexpr int CPT = HID / kSplit;               // columns per thread in a hidden-layer epilogue (multiple of 16)
constexpr int kEpiThreads = kTile * kSplit;     // 8 epilogue warps (-DSXEN_TC_SPLIT=4, 16 warps at 96 registers: 0.418 vs 0.394 ms)
constexpr int kThreadsAll = kEpiThreads + 64;   // + the chain-MMA warp + the weight-gradient-MMA warp

}  // namespace sxen_mlp_tc
