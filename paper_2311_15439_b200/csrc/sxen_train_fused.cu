// sxen_train_fused.cu -- run_chunk as ONE persistent kernel (BASELINE configs[3]: simplex encode + 64-wide MLP, fused).
//
// Reference: run_chunk, /root/reference/proj/src/trainer.cpp:20-49 -- per sample: HashEncoder::encode -> Mlp::forward -> MSE
// and upstream -> Mlp::backward -> HashEncoder::encode_backward, the encoding and its gradient never leaving the core's cache.
// The unfused device path runs three kernels back to back (encode 0.22 ms + tcgen05 head 0.41 ms + encode_backward 0.30 ms per
// 2^20 samples) with the features and their gradient making a round trip through HBM (2 x 128 MB).  The encode side is bound by
// L2 requests with the tensor pipe idle, the head by the latency of its epilogue <-> MMA hand-offs with the LSU idle: they
// overlap.  One CTA per SM, 24 warps in six warpgroups with their own register budgets (setmaxnreg):
//
//   gather warps (4)    walk the simplex for the NEXT tile's 128 samples x 16 levels (sxen_device.cuh: simplex_lookup, fp64,
//                       exact blend: the same feature bits as encode_kernel), split them into bf16 hi / lo and store them
//                       straight into the double-buffered X0 operand tile in shared memory
//   chain-MMA warp      X0*W0^T | H1*W1^T | dH2*W1 | dH1*W0 on tcgen05 with TMEM accumulators; layer 1 of tile k+1 is issued
//                       as soon as its X0 tile is full -- before tile k's last backward GEMM -- so a tile costs three
//                       epilogue <-> MMA round trips instead of the unfused kernel's five
//   wgrad-MMA warp      the three weight-gradient GEMMs, accumulating in TMEM across all tiles of the CTA
//   epilogue warps (8)  bias / ReLU / output layer / loss / upstream / ReLU masks between the GEMMs (as sxen_mlp_tc.cu)
//   scatter warps (8)   read d loss / d encoding of the PREVIOUS tile out of TMEM (tcgen05.ld: a warp owns the 32 samples of
//                       its lane quadrant), repeat the lattice walk and issue the pair-merged red.global.add.v2/v4.f32 into
//                       the gradient accumulator (coarse levels into the replicas, folded by coarse_fold_kernel afterwards)
//
// Numerics are those of the unfused tensor-core step: identical feature bits in, split-bf16 GEMMs, fp32 atomics out.
#include <cuda_bf16.h>

#include <algorithm>

#include "sxen_common.hpp"
#include "sxen_encode.cuh"
#include "sxen_tc.cuh"

using namespace sxen_host;
using namespace sxen_tc;
using sxen_dev::EncodeArgs;

namespace {

constexpr int kTile = 128;
constexpr int IN = 32, HID = 64, OUTP = 16;   // L = 16 levels x F = 2 features -> 64 -> 64 -> (<= 3)
constexpr int kLevels = IN / 2;
constexpr int X0C = IN + 8, HC = HID + 8;     // tile widths including the ones-column block

// shared-memory map (bytes); every operand tile is a bf16 CM16 hi / lo pair (sxen_tc.cuh)
constexpr uint32_t kW0 = 0;
constexpr uint32_t kW1 = kW0 + 2 * cm16_bytes(HID, IN);
constexpr uint32_t kX0 = kW1 + 2 * cm16_bytes(HID, HID);          // two buffers, tile parity
constexpr uint32_t kX0Bytes = 2 * cm16_bytes(kTile, X0C);
constexpr uint32_t kH1 = kX0 + 2 * kX0Bytes;
constexpr uint32_t kH2 = kH1 + 2 * cm16_bytes(kTile, HC);
constexpr uint32_t kDY = kH2 + 2 * cm16_bytes(kTile, HC);
constexpr uint32_t kDH2 = kDY + 2 * cm16_bytes(kTile, OUTP);
constexpr uint32_t kDH1 = kDH2 + 2 * cm16_bytes(kTile, HID);
constexpr uint32_t kBias = kDH1 + 2 * cm16_bytes(kTile, HID);
constexpr uint32_t kW2f = kBias + (HID + HID + 4) * 4;
constexpr uint32_t kPP = kW2f + 3 * HID * 4;
constexpr uint32_t kSmemBytes = kPP + 2 * kTile * 4 * 4;
static_assert(kSmemBytes <= 225 * 1024, "operand tiles exceed the CTA's shared memory");

// TMEM columns (fp32)
constexpr uint32_t tS0 = 0;     // [128 x 64] layer-1 pre-activation
constexpr uint32_t tS1 = 64;    // [128 x 64] layer-2 pre-activation, later dH1
constexpr uint32_t tG0 = 128;   // [64 x 40]  dW0 | db0      (M = 64 accumulators, persistent over the CTA's tiles)
constexpr uint32_t tG1 = 168;   // [64 x 72]  dW1 | db1
constexpr uint32_t tG2 = 240;   // [64 x 16]  dW2^T
constexpr uint32_t tDX = 256;   // 2 x [128 x 32] d loss / d encoding, tile parity (drained by the scatter warps)
constexpr uint32_t kTmemCols = 512;

// warp roles: warpgroup-aligned so that setmaxnreg can give each role its own register budget
constexpr int kEpiWarps = 8, kEpiThreads = kEpiWarps * 32;     // warps 0..7   (warpgroups 0, 1)
constexpr int kChainWarp = 8, kWgradWarp = 9;                  // warps 8, 9   (warpgroup 2; warps 10, 11 idle)
constexpr int kGatherWarp0 = 12, kGatherWarps = 4;             // warps 12..15 (warpgroup 3)
constexpr int kScatterWarp0 = 16, kScatterWarps = 8;           // warps 16..23 (warpgroups 4, 5)
constexpr int kThreadsAll = (kScatterWarp0 + kScatterWarps) * 32;
constexpr int kGatherThreads = kGatherWarps * 32, kScatterThreads = kScatterWarps * 32;
// The CTA is launched with 768 threads x 80 registers = 61440; setmaxnreg only moves registers WITHIN that allocation
// (an increase blocks until other warpgroups of the CTA have released enough): 256 x 128 + 128 x 32 + 384 x 64 = 61440.
constexpr int kRegsLaunch = 80, kRegsEpi = 128, kRegsMma = 32, kRegsWalk = 64;
static_assert(2 * 128 * kRegsEpi + 128 * kRegsMma + 3 * 128 * kRegsWalk <= 6 * 128 * kRegsLaunch, "register budgets exceed the launch allocation");

struct FusedArgs {
  const float* params;      // W0[64x32] b0[64] W1[64x64] b1[64] W2[ow x 64] b2[ow]  (src/mlp.cpp:19-32)
  const void* targets;      // N x ow, f32 or f64
  double* mlp_grad;         // parameter layout, accumulated into
  double* loss_sum;         // accumulated into
  long long* grad_fixed;    // reproducible MLP gradient: parameter layout in units of 2^-52, then one double per CTA (nullptr = off)
  int out_w;
  int target_f32;
  int precise;              // 0: single bf16 product, otherwise bf16x3
  double upstream_scale;    // 2 / (global_batch * out_w)
  unsigned long long* timing;  // nullptr, or 16 counters: per role {cycles in the tile loop, cycles of those spent waiting} (a tuning aid)
};

__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const __nv_bfloat162 hp = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hp);
    const float h0 = __uint_as_float(hb << 16), h1 = __uint_as_float(hb & 0xffff0000u);
    const __nv_bfloat162 lp = __floats2bfloat162_rn(v[2 * q] - h0, v[2 * q + 1] - h1);
    h[q] = hb;
    l[q] = *reinterpret_cast<const uint32_t*>(&lp);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

__device__ __forceinline__ void store_chunk(unsigned char* tile_hi, unsigned char* tile_lo, int row, int chunk, int cols,
                                            const float* v) {
  uint4 hi, lo;
  split8(v, hi, lo);
  const uint32_t off = cm16_offset(row, 8 * chunk, cols);
  *reinterpret_cast<uint4*>(tile_hi + off) = hi;
  *reinterpret_cast<uint4*>(tile_lo + off) = lo;
}

// Row `row`, columns [4*hc, 4*hc + 4) of a CM16(., cols) hi/lo tile pair <- v[0..4): 8 bytes of the row's 16-byte chunk
__device__ __forceinline__ void store_half_chunk(unsigned char* tile_hi, unsigned char* tile_lo, int row, int hc, int cols,
                                                 const float* v) {
  uint32_t h[2], l[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const __nv_bfloat162 hp = __floats2bfloat162_rn(v[2 * q], v[2 * q + 1]);
    const uint32_t hb = *reinterpret_cast<const uint32_t*>(&hp);
    const float h0 = __uint_as_float(hb << 16), h1 = __uint_as_float(hb & 0xffff0000u);
    const __nv_bfloat162 lp = __floats2bfloat162_rn(v[2 * q] - h0, v[2 * q + 1] - h1);
    h[q] = hb;
    l[q] = *reinterpret_cast<const uint32_t*>(&lp);
  }
  const uint32_t off = cm16_offset(row, 4 * hc, cols);
  *reinterpret_cast<uint2*>(tile_hi + off) = make_uint2(h[0], h[1]);
  *reinterpret_cast<uint2*>(tile_lo + off) = make_uint2(l[0], l[1]);
}

__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void gemm_split(uint32_t d, uint32_t idesc, int ksteps, bool accumulate, int precise, uint64_t a0,
                                           uint32_t a_lo, uint32_t a_step, uint64_t b0, uint32_t b_lo, uint32_t b_step) {
  for (int ks = 0; ks < ksteps; ++ks) {
    const uint64_t ah = a0 + ((static_cast<uint64_t>(ks) * a_step) >> 4), bh = b0 + ((static_cast<uint64_t>(ks) * b_step) >> 4);
    mma_bf16(d, ah, bh, idesc, accumulate || ks > 0);
    if (precise) {
      mma_bf16(d, ah, bh + (b_lo >> 4), idesc, true);
      mma_bf16(d, ah + (a_lo >> 4), bh, idesc, true);
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void add_total(double* base, long long* fixed, size_t index, double v) {
  // explicit reds: see sxen_mlp_tc_common.cuh (atomicAdd on 64-bit operands becomes ATOMG, one L2 round trip per instruction)
  if (fixed != nullptr)
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(fixed + index), "l"(__double2ll_rn(__dmul_rn(v, 0x1p52))) : "memory");
  else
    asm volatile("red.global.add.f64 [%0], %1;" ::"l"(base + index), "d"(v) : "memory");
}

// mbar_wait that charges its cycles to `waited` when the role is being timed
__device__ __forceinline__ void mbar_wait_t(uint64_t* bar, uint32_t parity, bool timed, unsigned long long& waited) {
  if (timed) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    waited += static_cast<unsigned long long>(clock64() - t0);
  } else {
    mbar_wait(bar, parity);
  }
}

template <int N>
__device__ __forceinline__ void set_regs_inc() { asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N)); }
template <int N>
__device__ __forceinline__ void set_regs_dec() { asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N)); }

constexpr int kSplit = 2, CPT = HID / kSplit;

template <int ND>
__global__ void __launch_bounds__(kThreadsAll, 1)
train_fused_kernel(const __grid_constant__ EncodeArgs e, const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_ready;     // 256 arrivals: the epilogue has written the next GEMM's tiles and drained the TMEM scratch
  __shared__ uint64_t bar;           // the chain warp's GEMMs up to here have completed (layer 2, dH2*W1)
  __shared__ uint64_t bar_l1;        // ... layer 1 (its own barrier: it is issued a tile ahead, between two commits on `bar`)
  __shared__ uint64_t bar_g;         // every weight-gradient MMA of the tile has completed
  __shared__ uint64_t bar_w;         // chain warp -> wgrad warp: the operands of backward phase 2 / 3 are in place
  __shared__ uint64_t x0_full[2];    // gather warps -> chain warp: X0[buf] holds the tile's features
  __shared__ uint64_t x0_empty[2];   // wgrad warp's commit: nothing reads X0[buf] any more
  __shared__ uint64_t dx_full[2];    // chain warp's commit: tDX[buf] holds the tile's d loss / d encoding
  __shared__ uint64_t dx_empty[2];   // scatter warps: tDX[buf] has been read out
  __shared__ uint32_t tmem_base_slot;
  __shared__ double red_buf[kEpiWarps][4];
  __shared__ double s_scale[sxen_dev::kMaxLaunchLevels];
  __shared__ int s_res[sxen_dev::kMaxLaunchLevels];
  __shared__ int s_cshift[sxen_dev::kMaxLaunchLevels];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const bool is_epi = warp < kEpiWarps;
  float* bias = reinterpret_cast<float*>(smem + kBias);
  float* w2f = reinterpret_cast<float*>(smem + kW2f);
  float* pp = reinterpret_cast<float*>(smem + kPP);
  constexpr uint32_t loW0 = cm16_bytes(HID, IN), loW1 = cm16_bytes(HID, HID);
  constexpr uint32_t loX0 = cm16_bytes(kTile, X0C), loH = cm16_bytes(kTile, HC), loDY = cm16_bytes(kTile, OUTP),
                     loDH = cm16_bytes(kTile, HID);

  // ---- one-time setup (all warps still at the launch register budget)
  if (tid < sxen_dev::kMaxLaunchLevels) {
    s_scale[tid] = e.geom.scale[tid];
    s_res[tid] = e.geom.res[tid];
    s_cshift[tid] = e.coarse != nullptr ? e.cg.shift[tid] : -1;
  }
  if (is_epi) {
    const float* W0 = a.params;
    const float* b0 = W0 + HID * IN;
    const float* W1 = b0 + HID;
    const float* b1 = W1 + HID * HID;
    const float* W2 = b1 + HID;
    const float* b2 = W2 + a.out_w * HID;
    for (int q = tid; q < HID * IN / 8; q += kEpiThreads) {
      const int o = q / (IN / 8), ch = q % (IN / 8);
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = W0[o * IN + ch * 8 + i];
      store_chunk(smem + kW0, smem + kW0 + loW0, o, ch, IN, v);
    }
    for (int q = tid; q < HID * HID / 8; q += kEpiThreads) {
      const int o = q / (HID / 8), ch = q % (HID / 8);
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = W1[o * HID + ch * 8 + i];
      store_chunk(smem + kW1, smem + kW1 + loW1, o, ch, HID, v);
    }
    for (int q = tid; q < 3 * HID; q += kEpiThreads) w2f[q] = (q / HID) < a.out_w ? W2[q] : 0.0f;
    if (tid < HID) {
      bias[tid] = b0[tid];
      bias[HID + tid] = b1[tid];
    }
    if (tid < 4) bias[2 * HID + tid] = tid < a.out_w ? b2[tid] : 0.0f;
    if (tid < kTile) {
      float ones[8] = {1.0f, 0, 0, 0, 0, 0, 0, 0};
      store_chunk(smem + kX0, smem + kX0 + loX0, tid, IN / 8, X0C, ones);
      store_chunk(smem + kX0 + kX0Bytes, smem + kX0 + kX0Bytes + loX0, tid, IN / 8, X0C, ones);
      store_chunk(smem + kH1, smem + kH1 + loH, tid, HID / 8, HC, ones);
      store_chunk(smem + kH2, smem + kH2 + loH, tid, HID / 8, HC, ones);
      float zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      store_chunk(smem + kDY, smem + kDY + loDY, tid, 1, OUTP, zero);
    }
  }
  if (tid == 0) {
    mbar_init(&bar_ready, kEpiThreads);
    mbar_init(&bar, 1);
    mbar_init(&bar_l1, 1);
    mbar_init(&bar_g, 1);
    mbar_init(&bar_w, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&x0_full[b], kGatherThreads);
      mbar_init(&x0_empty[b], 1);
      mbar_init(&dx_full[b], 1);
      mbar_init(&dx_empty[b], kScatterThreads);
    }
  }
  if (warp == 0) tmem_alloc(&tmem_base_slot, kTmemCols);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base_slot;
  const int precise = a.precise != 0;  // this kernel issues three products in either split mode (BF16X4 = BF16X3 here)
  const unsigned long long n = e.n_samples;
  const unsigned long long n_tiles = (n + kTile - 1) / kTile;
  // tiles of this CTA: blockIdx.x, blockIdx.x + gridDim.x, ...; `k` counts them (buffer = k & 1)

  if (warp >= kGatherWarp0 && warp < kGatherWarp0 + kGatherWarps) {
    // ================================ gather warps: encode forward into X0[buf] ================================
    set_regs_dec<kRegsWalk>();
    const int row = tid - kGatherWarp0 * 32;  // the sample's row in the tile
    const bool timed = a.timing != nullptr && row == 0;
    unsigned long long w0 = 0;
    const long long t_begin = clock64();
    unsigned long long k = 0;
    for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
      const int buf = static_cast<int>(k & 1);
      if (k >= 2) mbar_wait_t(&x0_empty[buf], static_cast<uint32_t>(((k >> 1) - 1) & 1), timed, w0);
      unsigned char* xhi = smem + kX0 + buf * kX0Bytes;
      unsigned char* xlo = xhi + loX0;
      const unsigned long long s = tile * kTile + row;
      double x[ND];
      bool ok = false;
      if (s < n) {
        ok = sxen_dev::load_coords<ND>(e, s, x);
        if (!ok) atomicMin(e.status, s);  // check_input, src/encoding.cpp:183-194: zero features, reported at the next check
      }
#pragma unroll 1
      for (int hc = 0; hc < IN / 4; ++hc) {  // 2 levels = 4 features = half of a 16-byte bf16 chunk of the row
        float v[4] = {0.0f, 0.0f, 0.0f, 0.0f};
        if (ok) {
          uint32_t idx[2][ND + 1];
          double w[2][ND + 1];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int l = 2 * hc + j;
            if (sxen_dev::simplex_lookup<ND>(x, s_scale[l], e.skew, s_res[l], e.mask, idx[j], w[j])) atomicAdd(e.status + 1, 1ULL);
          }
          float t[2][ND + 1][2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float* __restrict__ tab = e.tables + static_cast<size_t>(2 * hc + j) * e.level_stride;
#pragma unroll
            for (int q = 0; q <= ND; ++q) sxen_dev::load_row<2>(tab + static_cast<size_t>(idx[j][q]) * 2, t[j][q]);
          }
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            // src/encoding.cpp:305-313: acc += w_i * entry in chain order, in double, then the cast to float
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int q = 0; q <= ND; ++q) {
              a0 = __dadd_rn(a0, __dmul_rn(w[j][q], static_cast<double>(t[j][q][0])));
              a1 = __dadd_rn(a1, __dmul_rn(w[j][q], static_cast<double>(t[j][q][1])));
            }
            v[2 * j] = static_cast<float>(a0);
            v[2 * j + 1] = static_cast<float>(a1);
          }
        }
        store_half_chunk(xhi, xlo, row, hc, X0C, v);
      }
      fence_proxy_async();   // the generic-proxy stores above must be visible to the tensor core's async-proxy reads
      mbar_arrive(&x0_full[buf]);
    }
    if (timed) {
      atomicAdd(a.timing + 0, static_cast<unsigned long long>(clock64() - t_begin));
      atomicAdd(a.timing + 1, w0);
    }
  } else if (warp >= kScatterWarp0) {
    // ================================ scatter warps: tDX[buf] -> encode_backward ================================
    set_regs_dec<kRegsWalk>();
    const int sw = warp - kScatterWarp0;
    const int quad = sw & 3;             // (warp % 4 == quad: the TMEM lanes this warp may read)
    const int half = sw >> 2;            // levels [8 * half, 8 * half + 8)
    const int row = 32 * quad + lane;
    const int red_kind = (e.cache_hints >> 2) & 3;
    const uint64_t red_pol = sxen_dev::l2_policy(red_kind);
    const bool timed = a.timing != nullptr && sw == 0 && lane == 0;
    unsigned long long w0 = 0;
    const long long t_begin = clock64();
    unsigned long long k = 0;
    for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
      const int buf = static_cast<int>(k & 1);
      mbar_wait_t(&dx_full[buf], static_cast<uint32_t>((k >> 1) & 1), timed, w0);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16_nowait(tb + (static_cast<uint32_t>(32 * quad) << 16) + tDX + 32 * buf + 16 * half, r);
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&dx_empty[buf]);
      const unsigned long long s = tile * kTile + row;
      if (s >= n) continue;
      double x[ND];
      if (!sxen_dev::load_coords<ND>(e, s, x)) continue;  // a rejected sample adds no gradient
#pragma unroll
      for (int j = 0; j < kLevels / 2; ++j) {
        const int l = (kLevels / 2) * half + j;
        uint32_t idx[ND + 1], dense[ND + 1];
        double w[ND + 1];
        if (sxen_dev::simplex_lookup<ND, true>(x, s_scale[l], e.skew, s_res[l], e.mask, idx, w, dense)) atomicAdd(e.status + 1, 1ULL);
        const float u0 = __uint_as_float(r[2 * j]), u1 = __uint_as_float(r[2 * j + 1]);
        // EncoderGradient::add, src/encoding.cpp:110-120: dst[f] += scale * upstream[f]
        float v[ND + 1][2];
#pragma unroll
        for (int q = 0; q <= ND; ++q) {
          const float wq = static_cast<float>(w[q]);
          v[q][0] = sxen_dev::canon(__fmul_rn(wq, u0));
          v[q][1] = sxen_dev::canon(__fmul_rn(wq, u1));
        }
        float* gl = e.grads + static_cast<size_t>(l) * e.level_stride;
        const int cshift = s_cshift[l];
        if (cshift >= 0) {  // coarse level: one of 2^cshift dense replicas, picked by the sample index (sxen_encode.cuh)
          const uint32_t rep = static_cast<uint32_t>(s) & ((1u << cshift) - 1u);
          gl = e.coarse + e.cg.offset[l] + static_cast<size_t>(rep) * e.cg.verts[l] * 2;
#pragma unroll
          for (int q = 0; q <= ND; ++q) idx[q] = dense[q];
        }
        bool skip = false;
#pragma unroll
        for (int q = 0; q <= ND; ++q) {
          if (skip) {
            skip = false;
            continue;
          }
          // rows idx and idx^1 share one 16-byte slot: one red.v4 for an axis-0 pair (sxen_encode.cuh)
          if (q + 1 <= ND && e.merge_pairs && (idx[q] ^ idx[q + 1 <= ND ? q + 1 : q]) == 1u) {
            const int qn = q + 1 <= ND ? q + 1 : q;
            const bool low = (idx[q] & 1u) == 0u;
            float* p = gl + static_cast<size_t>(idx[q] & ~1u) * 2;
            if (red_kind)
              sxen_dev::red_add4_policy(p, low ? v[q][0] : v[qn][0], low ? v[q][1] : v[qn][1], low ? v[qn][0] : v[q][0],
                                        low ? v[qn][1] : v[q][1], red_pol);
            else
              sxen_dev::red_add4(p, low ? v[q][0] : v[qn][0], low ? v[q][1] : v[qn][1], low ? v[qn][0] : v[q][0],
                                 low ? v[qn][1] : v[q][1]);
            skip = true;
            continue;
          }
          if (red_kind) sxen_dev::red_add2_policy(gl + static_cast<size_t>(idx[q]) * 2, v[q][0], v[q][1], red_pol);
          else sxen_dev::red_add2(gl + static_cast<size_t>(idx[q]) * 2, v[q][0], v[q][1]);
        }
      }
    }
    if (timed) {
      atomicAdd(a.timing + 4, static_cast<unsigned long long>(clock64() - t_begin));
      atomicAdd(a.timing + 5, w0);
    }
  } else if (warp == kChainWarp) {
    // ================================ chain-MMA warp ================================
    set_regs_dec<kRegsMma>();
    if (lane == 0) {
      const uint32_t sW0 = smem_u32(smem + kW0), sW1 = smem_u32(smem + kW1);
      const uint32_t sH1 = smem_u32(smem + kH1), sDH2 = smem_u32(smem + kDH2), sDH1 = smem_u32(smem + kDH1);
      const uint64_t kW0d = desc16_k_major(sW0, IN, 0), kW1d = desc16_k_major(sW1, HID, 0);
      const uint64_t kH1d = desc16_k_major(sH1, HC, 0);
      const uint64_t kDH2d = desc16_k_major(sDH2, HID, 0), kDH1d = desc16_k_major(sDH1, HID, 0);
      const uint64_t mW0d = desc16_mn_major(sW0, IN, 0), mW1d = desc16_mn_major(sW1, HID, 0);
      constexpr uint32_t kStep = 256;
      const bool timed = a.timing != nullptr;
      unsigned long long w0 = 0, w1 = 0, w2 = 0;
      const long long t_begin = clock64();
      auto layer1 = [&](unsigned long long kk) {  // S0 = X0[buf] * W0^T as soon as the gather warps have filled the tile
        const int b = static_cast<int>(kk & 1);
        mbar_wait_t(&x0_full[b], static_cast<uint32_t>((kk >> 1) & 1), timed, w0);
        tc_fence_after();
        const uint64_t kX0d = desc16_k_major(smem_u32(smem + kX0 + b * kX0Bytes), X0C, 0);
        gemm_split(tb + tS0, make_idesc_bf16(128, HID, false, false), IN / 16, false, precise, kX0d, loX0, kStep, kW0d, loW0, kStep);
        tc_commit(&bar_l1);
      };
      uint32_t ph = 0;
      unsigned long long k = 0;
      if (blockIdx.x < n_tiles) layer1(0);
      for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int buf = static_cast<int>(k & 1);
        // layer 2: S1 = H1 * W1^T
        mbar_wait_t(&bar_ready, ph, timed, w1);
        ph ^= 1;
        tc_fence_after();
        gemm_split(tb + tS1, make_idesc_bf16(128, HID, false, false), HID / 16, false, precise, kH1d, loH, kStep, kW1d, loW1, kStep);
        tc_commit(&bar);
        // backward of layer 2: S1 = dH2 * W1
        mbar_wait_t(&bar_ready, ph, timed, w1);
        ph ^= 1;
        tc_fence_after();
        mbar_arrive(&bar_w);
        gemm_split(tb + tS1, make_idesc_bf16(128, HID, false, true), HID / 16, false, precise, kDH2d, loDH, kStep, mW1d, loW1,
                   2 * cm16_row_group_stride(HID));
        tc_commit(&bar);
        // layer 1 of the NEXT tile runs in the shadow of this tile's last epilogue (S0 is free: its reader finished before
        // layer 2 was issued)
        if (tile + gridDim.x < n_tiles) layer1(k + 1);
        // backward of layer 1: tDX[buf] = dH1 * W0, once the scatter warps have drained the tile before last
        mbar_wait_t(&bar_ready, ph, timed, w1);
        ph ^= 1;
        tc_fence_after();
        mbar_arrive(&bar_w);
        if (k >= 2) {
          mbar_wait_t(&dx_empty[buf], static_cast<uint32_t>(((k >> 1) - 1) & 1), timed, w2);
          tc_fence_after();
        }
        gemm_split(tb + tDX + 32 * buf, make_idesc_bf16(128, IN, false, true), HID / 16, false, precise, kDH1d, loDH, kStep, mW0d,
                   loW0, 2 * cm16_row_group_stride(IN));
        tc_commit(&dx_full[buf]);
      }
      if (timed) {
        atomicAdd(a.timing + 8, static_cast<unsigned long long>(clock64() - t_begin));
        atomicAdd(a.timing + 9, w0);
        atomicAdd(a.timing + 10, w1);
        atomicAdd(a.timing + 11, w2);
      }
    }
  } else if (warp == kWgradWarp) {
    // ================================ wgrad-MMA warp ================================
    set_regs_dec<kRegsMma>();
    if (lane == 0) {
      const uint32_t sH1 = smem_u32(smem + kH1), sH2 = smem_u32(smem + kH2);
      const uint32_t sDY = smem_u32(smem + kDY), sDH2 = smem_u32(smem + kDH2), sDH1 = smem_u32(smem + kDH1);
      const uint64_t mH1d = desc16_mn_major(sH1, HC, 0), mH2d = desc16_mn_major(sH2, HC, 0);
      const uint64_t mDYd = desc16_mn_major(sDY, OUTP, 0), mDH2d = desc16_mn_major(sDH2, HID, 0), mDH1d = desc16_mn_major(sDH1, HID, 0);
      uint32_t phw = 0;
      bool started = false;
      unsigned long long k = 0;
      for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int buf = static_cast<int>(k & 1);
        mbar_wait(&bar_w, phw);  // G2 += H2^T * dY (dW2^T);  G1 += dH2^T * [H1 | 1]
        phw ^= 1;
        tc_fence_after();
        gemm_split(tb + tG2, make_idesc_bf16(64, OUTP, true, true), kTile / 16, started, precise, mH2d, loH,
                   2 * cm16_row_group_stride(HC), mDYd, loDY, 2 * cm16_row_group_stride(OUTP));
        gemm_split(tb + tG1, make_idesc_bf16(64, HC, true, true), kTile / 16, started, precise, mDH2d, loDH,
                   2 * cm16_row_group_stride(HID), mH1d, loH, 2 * cm16_row_group_stride(HC));
        mbar_wait(&bar_w, phw);  // G0 += dH1^T * [X0 | 1]
        phw ^= 1;
        tc_fence_after();
        const uint64_t mX0d = desc16_mn_major(smem_u32(smem + kX0 + buf * kX0Bytes), X0C, 0);
        gemm_split(tb + tG0, make_idesc_bf16(64, X0C, true, true), kTile / 16, started, precise, mDH1d, loDH,
                   2 * cm16_row_group_stride(HID), mX0d, loX0, 2 * cm16_row_group_stride(X0C));
        tc_commit(&bar_g);           // G2, G1 and G0 of this tile
        tc_commit(&x0_empty[buf]);   // ... after which nothing reads X0[buf]
        started = true;
      }
    }
  } else if (warp > kWgradWarp && warp < kGatherWarp0) {
    set_regs_dec<kRegsMma>();  // the two spare warps of the MMA warpgroup
  } else {
    // ================================ epilogue warps ================================
    set_regs_inc<kRegsEpi>();
    const int t = tid & (kTile - 1);
    const int half = (tid >> 7) & (kSplit - 1);
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t phase = 0, phase_g = 0, phase_l1 = 0;
    bool g_started = false;
    double loss_acc = 0.0;
    double db2_acc[3] = {0.0, 0.0, 0.0};
    auto ready = [&]() {
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bar_ready);
    };
    const bool timed = a.timing != nullptr && tid == 0;
    unsigned long long w0 = 0, w1 = 0, w2 = 0;
    const long long t_begin = clock64();
    auto wait_chain = [&]() {
      mbar_wait_t(&bar, phase, timed, w0);
      phase ^= 1;
      tc_fence_after();
    };
    for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const unsigned long long smp = tile * kTile + t;
      const bool valid = smp < n;
      double tgt[3] = {0.0, 0.0, 0.0};
      if (valid) {
#pragma unroll
        for (int o = 0; o < 3; ++o)
          if (o < a.out_w)
            tgt[o] = a.target_f32 ? static_cast<double>(static_cast<const float*>(a.targets)[smp * a.out_w + o])
                                  : static_cast<const double*>(a.targets)[smp * a.out_w + o];
      }
      // ---- layer 1 epilogue: S0 -> H1 (the previous tile's weight-gradient MMAs still read H1 .. dH1: wait for them first)
      uint32_t m1 = 0, m2 = 0;
      mbar_wait_t(&bar_l1, phase_l1, timed, w1);
      phase_l1 ^= 1;
      tc_fence_after();
      if (g_started) {
        mbar_wait_t(&bar_g, phase_g, timed, w2);
        phase_g ^= 1;
      }
      {
        uint32_t r[CPT / 16][16];
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(tb + lane_base + tS0 + CPT * half + 16 * q, r[q]);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float xv = __uint_as_float(r[q][i]) + bias[CPT * half + 16 * q + i];
            xv = xv > 0.0f ? xv : 0.0f;
            if (xv > 0.0f) m1 |= 1u << (16 * q + i);
            v[i] = xv;
          }
          store_chunk(smem + kH1, smem + kH1 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
          store_chunk(smem + kH1, smem + kH1 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
        }
      }
      ready();
      // ---- layer 2 epilogue: S1 -> H2, output layer, loss, dY, dH2 (CUDA cores, as sxen_mlp_tc.cu)
      wait_chain();
      {
        uint32_t r[CPT / 16][16];
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(tb + lane_base + tS1 + CPT * half + 16 * q, r[q]);
        tmem_ld_wait();
        float p0 = 0.0f, p1 = 0.0f, p2 = 0.0f;
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = CPT * half + 16 * q + i;
            float xv = __uint_as_float(r[q][i]) + bias[HID + c];
            xv = xv > 0.0f ? xv : 0.0f;
            if (xv > 0.0f) m2 |= 1u << (16 * q + i);
            v[i] = xv;
            p0 = __fmaf_rn(w2f[c], xv, p0);
            p1 = __fmaf_rn(w2f[HID + c], xv, p1);
            p2 = __fmaf_rn(w2f[2 * HID + c], xv, p2);
          }
          store_chunk(smem + kH2, smem + kH2 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
          store_chunk(smem + kH2, smem + kH2 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
        }
        *reinterpret_cast<float4*>(pp + (half * kTile + t) * 4) = make_float4(p0, p1, p2, 0.0f);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      float u[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      {
        float pr[3] = {bias[2 * HID], bias[2 * HID + 1], bias[2 * HID + 2]};
#pragma unroll
        for (int kk = 0; kk < kSplit; ++kk) {
          const float4 pk = *reinterpret_cast<const float4*>(pp + (kk * kTile + t) * 4);
          pr[0] += pk.x;
          pr[1] += pk.y;
          pr[2] += pk.z;
        }
#pragma unroll
        for (int o = 0; o < 3; ++o) {
          if (o < a.out_w && valid) {
            // src/trainer.cpp:38-44: e = pred - target, loss += e*e, upstream = 2e/(B*out_w), all in double
            const double err = static_cast<double>(pr[o]) - tgt[o];
            const double up = a.upstream_scale * err;
            u[o] = static_cast<float>(up);
            if (half == 0) {
              loss_acc += err * err;
              db2_acc[o] += up;
            }
          }
        }
      }
      if (half == 0) store_chunk(smem + kDY, smem + kDY + loDY, t, 0, OUTP, u);
      {
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = CPT * half + 16 * q + i;
            const float g = __fmaf_rn(u[2], w2f[2 * HID + c], __fmaf_rn(u[1], w2f[HID + c], __fmul_rn(u[0], w2f[c])));
            v[i] = ((m2 >> (16 * q + i)) & 1u) ? g : 0.0f;
          }
          store_chunk(smem + kDH2, smem + kDH2 + loDH, t, (CPT / 8) * half + 2 * q, HID, v);
          store_chunk(smem + kDH2, smem + kDH2 + loDH, t, (CPT / 8) * half + 2 * q + 1, HID, v + 8);
        }
      }
      ready();
      // ---- backward epilogue of layer 2: S1 -> dH1 (masked by layer 1's ReLU)
      wait_chain();
      {
        uint32_t r[CPT / 16][16];
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(tb + lane_base + tS1 + CPT * half + 16 * q, r[q]);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = ((m1 >> (16 * q + i)) & 1u) ? __uint_as_float(r[q][i]) : 0.0f;
          store_chunk(smem + kDH1, smem + kDH1 + loDH, t, (CPT / 8) * half + 2 * q, HID, v);
          store_chunk(smem + kDH1, smem + kDH1 + loDH, t, (CPT / 8) * half + 2 * q + 1, HID, v + 8);
        }
      }
      ready();
      g_started = true;
    }
    if (timed) {
      atomicAdd(a.timing + 12, static_cast<unsigned long long>(clock64() - t_begin));
      atomicAdd(a.timing + 13, w0);
      atomicAdd(a.timing + 14, w1);
      atomicAdd(a.timing + 15, w2);
    }
    // ---- weight gradients out of TMEM (M = 64 accumulators: row i in lane (i/16)*32 + i%16)
    if (g_started) mbar_wait(&bar_g, phase_g);
    tc_fence_after();
    const int row = 16 * (warp & 3) + lane;
    constexpr size_t gW0 = 0, gb0 = gW0 + HID * IN, gW1 = gb0 + HID, gb1 = gW1 + HID * HID, gW2 = gb1 + HID;
    double* const G = a.mlp_grad;
    long long* const FX = a.grad_fixed;
    if (g_started) {
      for (int c0 = 8 * half; c0 < X0C; c0 += 8 * kSplit) {
        uint32_t r[16];
        tmem_ld16_nowait(tb + lane_base + tG0 + (c0 < IN ? c0 : IN - 8), r);
        tmem_ld_wait();
        if (lane < 16) {
          if (c0 < IN) {
            for (int i = 0; i < 8; ++i) add_total(G, FX, gW0 + row * IN + c0 + i, static_cast<double>(__uint_as_float(r[i])));
          } else {
            add_total(G, FX, gb0 + row, static_cast<double>(__uint_as_float(r[8])));
          }
        }
      }
      for (int c0 = 8 * half; c0 < HC; c0 += 8 * kSplit) {
        uint32_t r[16];
        tmem_ld16_nowait(tb + lane_base + tG1 + (c0 < 64 ? c0 : 56), r);
        tmem_ld_wait();
        if (lane < 16) {
          if (c0 < 64) {
            for (int i = 0; i < 8; ++i) add_total(G, FX, gW1 + row * HID + c0 + i, static_cast<double>(__uint_as_float(r[i])));
          } else {
            add_total(G, FX, gb1 + row, static_cast<double>(__uint_as_float(r[8])));
          }
        }
      }
      if (half == 1) {
        uint32_t r[16];
        tmem_ld16_nowait(tb + lane_base + tG2, r);
        tmem_ld_wait();
        if (lane < 16)
          for (int o = 0; o < a.out_w; ++o) add_total(G, FX, gW2 + o * HID + row, static_cast<double>(__uint_as_float(r[o])));
      }
    }
    double part[4] = {loss_acc, db2_acc[0], db2_acc[1], db2_acc[2]};
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      for (int o = 16; o > 0; o >>= 1) part[kk] += __shfl_down_sync(0xffffffffu, part[kk], o);
    if (lane == 0)
      for (int kk = 0; kk < 4; ++kk) red_buf[warp][kk] = part[kk];
  }

  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    double tot[4] = {0, 0, 0, 0};
    for (int w = 0; w < kEpiWarps; ++w)
      for (int kk = 0; kk < 4; ++kk) tot[kk] += red_buf[w][kk];
    const size_t gb2 = HID * IN + HID + HID * HID + HID + a.out_w * HID;
    const size_t n_params = gb2 + a.out_w;
    if (a.grad_fixed != nullptr) reinterpret_cast<double*>(a.grad_fixed + n_params)[blockIdx.x] = tot[0];
    else atomicAdd(a.loss_sum, tot[0]);
    for (int o = 0; o < a.out_w && o < 3; ++o) add_total(a.mlp_grad, a.grad_fixed, gb2 + o, tot[1 + o]);
  }
  if (warp == 0) tmem_dealloc(tb, kTmemCols);
}

}  // namespace

// Tuning aid: 16 device counters the kernel's roles add their loop / wait cycles to (nullptr = off, the default).
static unsigned long long* g_fused_timing = nullptr;
extern "C" SXEN_API sxen_status sxen_debug_fused_timing(unsigned long long* counters_dev) {
  g_fused_timing = counters_dev;
  return SXEN_OK;
}

// Internal entry point (declared in sxen_common.hpp), used by sxen_trainer.cu.  `e` describes the whole encoder launch
// (sxen_abi.cu: sxen_encoder_fused_args); the caller launches the coarse fold afterwards.
bool sxen_train_fused_supported(const sxen_encoder_config& ec, const sxen_mlp_config& mc) {
  return ec.backend == SXEN_BACKEND_SIMPLEX && ec.features == 2 && ec.levels == kLevels && (ec.dim == 2 || ec.dim == 3) &&
         mc.input_width == IN && mc.hidden_width == HID && mc.hidden_layers == 2 && mc.output_width >= 1 && mc.output_width <= 3;
}

sxen_status sxen_train_fused_run(const EncodeArgs& e, int dim, const float* params, const void* targets, int target_f32,
                                 double* mlp_grad, double* loss_sum, long long* grad_fixed, int out_w, size_t global_batch,
                                 int precise, cudaStream_t stream, int* used_ctas) {
  if (e.n_samples == 0) return SXEN_OK;
  FusedArgs a{};
  a.params = params;
  a.targets = targets;
  a.mlp_grad = mlp_grad;
  a.loss_sum = loss_sum;
  a.grad_fixed = grad_fixed;
  a.out_w = out_w;
  a.target_f32 = target_f32;
  a.precise = precise;
  a.upstream_scale = 2.0 / static_cast<double>(global_batch * static_cast<size_t>(out_w));  // src/trainer.cpp:26-27
  a.timing = g_fused_timing;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long tiles = (e.n_samples + kTile - 1) / kTile;
  const unsigned grid = static_cast<unsigned>(std::min<unsigned long long>(tiles, static_cast<unsigned long long>(sms)));
  if (dim == 3) {
    SXEN_CUDA(cudaFuncSetAttribute(train_fused_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    train_fused_kernel<3><<<grid, kThreadsAll, kSmemBytes, stream>>>(e, a);
  } else if (dim == 2) {
    SXEN_CUDA(cudaFuncSetAttribute(train_fused_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    train_fused_kernel<2><<<grid, kThreadsAll, kSmemBytes, stream>>>(e, a);
  } else {
    return fail(SXEN_INVALID_ARGUMENT, "fused training kernel: dim %d not instantiated", dim);
  }
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (used_ctas) *used_ctas = static_cast<int>(grid);
  return SXEN_OK;
}
