// sxen_mlp_tc.cu -- the {16|32} -> 64 -> 64 -> {<=3} MLP head on 5th-generation tensor cores (tcgen05 + TMEM), fully fused:
// forward, MSE loss + upstream, input gradients and weight gradients of one 128-sample tile never leave the SM.
//
// Reference semantics: Mlp::forward / Mlp::backward and run_chunk's loss (/root/reference/proj/src/mlp.cpp:137-202,
// src/trainer.cpp:26-48).  The reference accumulates in fp64; here every GEMM runs as split-bf16 ("bf16x3"):
// x = hi + lo with hi = bf16(x), lo = bf16(x - hi), D += A_hi*B_hi + A_hi*B_lo + A_lo*B_hi in fp32 TMEM accumulators,
// i.e. ~16 mantissa bits per operand, relative error ~1e-5 per product (tests state the tolerance).
// kind::tf32 was not usable: on sm_100a MN-major tf32 operands produce zeros (tools/tc_probe.py), and the weight-gradient
// GEMMs need the sample dimension as K, i.e. MN-major views of the activation tiles.
//
// Layout: all operand tiles are bf16 CM16 tiles (sxen_tc.cuh), self-dual, so ONE activation tile [128 samples][features]
// is the K-major A operand of the next layer, the K-major A operand of the input-gradient GEMM and the MN-major operand of
// the weight-gradient GEMM.  Each tile carries one extra 8-column block whose first column is 1.0: used as the B operand of
// a weight-gradient GEMM it makes the bias gradient fall out as column `in` of the same accumulator.
// The 64 -> out_w (<= 3) output layer and its input gradient are three dot products per unit: they run on the CUDA cores in
// fp32 inside the layer-2 epilogue (partial sums of the two column halves meet through shared memory), which removes two
// tensor-core round trips from the per-tile dependency chain: X0*W0^T | H1*W1^T | dH2*W1 | dH1*W0.
// One CTA = 128 samples = 128 TMEM lanes, 256 threads: threads t and t+128 share sample t of the tile and split every
// epilogue's columns in halves (warps w and w+4 read the same TMEM lane quadrant).  The weight-gradient MMAs of a phase are
// queued behind the phase's dependent-chain MMAs and are only waited for when the tiles they read are about to be rewritten,
// so they run under the following epilogues.
#include <algorithm>

#include "sxen_mlp_tc_common.cuh"

using namespace sxen_host;
using namespace sxen_tc;
using namespace sxen_mlp_tc;

namespace {

// shared-memory map (bytes)
constexpr uint32_t kW0 = 0;                                     // CM16(64, 32) hi, lo
constexpr uint32_t kW1 = kW0 + 2 * cm16_bytes(HID, kInMax);     // CM16(64, 64) hi, lo   (regions sized for IN = 32)
constexpr uint32_t kX0 = kW1 + 2 * cm16_bytes(HID, HID);        // CM16(128, 40) hi, lo
constexpr uint32_t kH1 = kX0 + 2 * cm16_bytes(kTile, kX0CMax);  // CM16(128, 72) hi, lo
constexpr uint32_t kH2 = kH1 + 2 * cm16_bytes(kTile, HC);
constexpr uint32_t kDY = kH2 + 2 * cm16_bytes(kTile, HC);       // CM16(128, 16) hi, lo
constexpr uint32_t kDH2 = kDY + 2 * cm16_bytes(kTile, OUTP);    // CM16(128, 64) hi, lo
constexpr uint32_t kDH1 = kDH2 + 2 * cm16_bytes(kTile, HID);
constexpr uint32_t kBias = kDH1 + 2 * cm16_bytes(kTile, HID);   // b0[64], b1[64], b2[4] floats
constexpr uint32_t kW2f = kBias + (HID + HID + 4) * 4;          // output layer in fp32: W2f[3][64] (rows >= out_w zero)
constexpr uint32_t kPP = kW2f + 3 * HID * 4;                    // partial predictions pp[2][128][4]
constexpr uint32_t kSmemBytes = kPP + 4 * kTile * 4 * 4;  // pp[kSplit <= 4][128][4]

// TMEM columns (fp32): scratch accumulators (128 lanes) and the persistent weight-gradient accumulators (M = 64)
constexpr uint32_t tS0 = 0;     // [128 x 64] layer-1 pre-activation, later d(input) (32 cols)
constexpr uint32_t tS1 = 64;    // [128 x 64] layer-2 pre-activation, later dH1
constexpr uint32_t tG0 = 128;   // [64 x 40]  dW0 | db0
constexpr uint32_t tG1 = 168;   // [64 x 72]  dW1 | db1
constexpr uint32_t tG2 = 240;   // [64 x 16]  dW2^T
constexpr uint32_t kTmemCols = 256;

template <bool TRAIN, int IN>
__global__ void __launch_bounds__(kThreadsAll, 1) mlp_tc_kernel(const __grid_constant__ TcArgs a) {
  static_assert(IN == 16 || IN == 32, "input widths 16 (L=8, F=2: the reference's default encoder) and 32 (L=16, F=2)");
  constexpr int X0C = IN + 8;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_ready;  // 256 arrivals: the tiles of the next phase are written and the TMEM scratch is drained
  __shared__ uint64_t bar;        // dependent-chain MMAs of the current phase have completed
  __shared__ uint64_t bar_g;      // every weight-gradient MMA of the tile has completed
  __shared__ uint64_t bar_w;      // chain warp -> weight-gradient warp: the operands of backward phase 2 / 3 are in place
  __shared__ uint32_t tmem_base_slot;
  __shared__ double red_buf[kEpiThreads / 32][4];
  const int tid = threadIdx.x;
  const int t = tid & (kTile - 1);   // sample row inside the tile
  const int half = (tid >> 7) & (kSplit - 1);  // which slice of an epilogue's columns this thread handles
  const int warp = tid >> 5;
  const bool is_mma_warp = warp == kEpiThreads / 32;        // issues the four dependent-chain GEMMs of every tile
  const bool is_wgrad_warp = warp == kEpiThreads / 32 + 1;  // issues the three weight-gradient GEMMs (TRAIN)
  const bool is_epi = tid < kEpiThreads;
  float* bias = reinterpret_cast<float*>(smem + kBias);
  const float* W0 = a.params;
  const float* b0 = W0 + HID * IN;
  const float* W1 = b0 + HID;
  const float* b1 = W1 + HID * HID;
  const float* W2 = b1 + HID;
  const float* b2 = W2 + a.out_w * HID;

  constexpr uint32_t loW0 = cm16_bytes(HID, IN), loW1 = cm16_bytes(HID, HID);
  float* w2f = reinterpret_cast<float*>(smem + kW2f);
  float* pp = reinterpret_cast<float*>(smem + kPP);
  constexpr uint32_t loX0 = cm16_bytes(kTile, X0C), loH = cm16_bytes(kTile, HC), loDY = cm16_bytes(kTile, OUTP),
                     loDH = cm16_bytes(kTile, HID);

  // ---- one-time setup: weights (hi/lo CM16 tiles, rows = output unit, cols = input unit), biases, ones columns
  if (is_epi) {
    for (int e = tid; e < HID * IN / 8; e += kEpiThreads) {
      const int o = e / (IN / 8), ch = e % (IN / 8);
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = W0[o * IN + ch * 8 + q];
      store_chunk(smem + kW0, smem + kW0 + loW0, o, ch, IN, v);
    }
    for (int e = tid; e < HID * HID / 8; e += kEpiThreads) {
      const int o = e / (HID / 8), ch = e % (HID / 8);
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = W1[o * HID + ch * 8 + q];
      store_chunk(smem + kW1, smem + kW1 + loW1, o, ch, HID, v);
    }
    for (int e = tid; e < 3 * HID; e += kEpiThreads) w2f[e] = (e / HID) < a.out_w ? W2[e] : 0.0f;
    if (tid < HID) {
      bias[tid] = b0[tid];
      bias[HID + tid] = b1[tid];
    }
    if (tid < 4) bias[2 * HID + tid] = tid < a.out_w ? b2[tid] : 0.0f;
    if (half == 0) {
      float ones[8] = {1.0f, 0, 0, 0, 0, 0, 0, 0};
      store_chunk(smem + kX0, smem + kX0 + loX0, t, IN / 8, X0C, ones);
      store_chunk(smem + kH1, smem + kH1 + loH, t, HID / 8, HC, ones);
      store_chunk(smem + kH2, smem + kH2 + loH, t, HID / 8, HC, ones);
      float zero[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      store_chunk(smem + kDY, smem + kDY + loDY, t, 1, OUTP, zero);  // columns 8..15 of dY stay zero
    }
  }
  if (tid == 0) {
    mbar_init(&bar_ready, kEpiThreads);
    mbar_init(&bar, 1);
    mbar_init(&bar_g, 1);
    mbar_init(&bar_w, 1);
  }
  if (warp == 0) tmem_alloc(&tmem_base_slot, kTmemCols);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base_slot;
  const int precise = a.precise;
  const unsigned long long n_tiles = (a.n + kTile - 1) / kTile;
  constexpr int kPhases = TRAIN ? 4 : 2;
  bool g_started = false;

  if (is_mma_warp) {
    // =========================== MMA warp: one lane issues every tcgen05.mma of the CTA ===========================
    if ((tid & 31) == 0) {
      const uint32_t sW0 = smem_u32(smem + kW0), sW1 = smem_u32(smem + kW1);
      const uint32_t sX0 = smem_u32(smem + kX0), sH1 = smem_u32(smem + kH1), sH2 = smem_u32(smem + kH2);
      const uint32_t sDY = smem_u32(smem + kDY), sDH2 = smem_u32(smem + kDH2), sDH1 = smem_u32(smem + kDH1);
      // K-major views step 256 B per UMMA_K = 16; MN-major views step two 8-row groups
      const uint64_t kX0d = desc16_k_major(sX0, X0C, 0), kH1d = desc16_k_major(sH1, HC, 0);
      const uint64_t kW0d = desc16_k_major(sW0, IN, 0), kW1d = desc16_k_major(sW1, HID, 0);
      const uint64_t kDH2d = desc16_k_major(sDH2, HID, 0), kDH1d = desc16_k_major(sDH1, HID, 0);
      const uint64_t mW0d = desc16_mn_major(sW0, IN, 0), mW1d = desc16_mn_major(sW1, HID, 0);
      const uint64_t mX0d = desc16_mn_major(sX0, X0C, 0), mH1d = desc16_mn_major(sH1, HC, 0), mH2d = desc16_mn_major(sH2, HC, 0);
      const uint64_t mDYd = desc16_mn_major(sDY, OUTP, 0), mDH2d = desc16_mn_major(sDH2, HID, 0), mDH1d = desc16_mn_major(sDH1, HID, 0);
      constexpr uint32_t kStep = 256;
      uint32_t ph = 0;
      const bool timed = a.timing != nullptr;
      unsigned long long t_ready = 0;
      const long long t_begin = clock64();
      for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
        for (int p = 0; p < kPhases; ++p) {
          const long long t0 = timed ? clock64() : 0;
          mbar_wait(&bar_ready, ph, 0x100u + static_cast<uint32_t>(p), a.progress);
          if (timed) t_ready += static_cast<unsigned long long>(clock64() - t0);
          ph ^= 1;
          tc_fence_after();
          if (p >= 2) mbar_arrive(&bar_w);  // hand the phase to the weight-gradient warp (its private two-phase barrier)
          switch (p) {
            case 0:  // layer 1: S0 = X0 * W0^T
              gemm_split(tb + tS0, make_idesc_bf16(128, HID, false, false), IN / 16, false, precise, kX0d, loX0, kStep, kW0d, loW0, kStep);
              tc_commit(&bar);
              break;
            case 1:  // layer 2: S1 = H1 * W1^T
              gemm_split(tb + tS1, make_idesc_bf16(128, HID, false, false), HID / 16, false, precise, kH1d, loH, kStep, kW1d, loW1, kStep);
              tc_commit(&bar);
              break;
            case 2:  // S1 = dH2 * W1
              gemm_split(tb + tS1, make_idesc_bf16(128, HID, false, true), HID / 16, false, precise, kDH2d, loDH, kStep, mW1d, loW1,
                         2 * cm16_row_group_stride(HID));
              tc_commit(&bar);
              break;
            default:  // S0[:, 0:32] = dH1 * W0 (d loss / d encoding)
              gemm_split(tb + tS0, make_idesc_bf16(128, IN, false, true), HID / 16, false, precise, kDH1d, loDH, kStep, mW0d, loW0,
                         2 * cm16_row_group_stride(IN));
              tc_commit(&bar);
              break;
          }
        }
      }
      if (timed) {
        atomicAdd(a.timing + 4, static_cast<unsigned long long>(clock64() - t_begin));
        atomicAdd(a.timing + 5, t_ready);
      }
    }
  } else if (is_wgrad_warp) {
    // ============ weight-gradient warp: its own lane issues G2, G1 (phase 2) and G0 (phase 3) of every tile ============
    // A single issuing thread spends ~35 cycles per tcgen05.mma; the 72 weight-gradient MMAs of a tile would otherwise
    // sit in front of the next phase's chain MMAs in that thread's program order.  Issued from here they reach the tensor
    // pipe whenever this lane gets to them, and tcgen05.commit on bar_g tracks exactly this thread's MMAs.
    if constexpr (TRAIN) {
      if ((tid & 31) == 0) {
        const uint32_t sX0 = smem_u32(smem + kX0), sH1 = smem_u32(smem + kH1), sH2 = smem_u32(smem + kH2);
        const uint32_t sDY = smem_u32(smem + kDY), sDH2 = smem_u32(smem + kDH2), sDH1 = smem_u32(smem + kDH1);
        const uint64_t mX0d = desc16_mn_major(sX0, X0C, 0), mH1d = desc16_mn_major(sH1, HC, 0), mH2d = desc16_mn_major(sH2, HC, 0);
        const uint64_t mDYd = desc16_mn_major(sDY, OUTP, 0), mDH2d = desc16_mn_major(sDH2, HID, 0), mDH1d = desc16_mn_major(sDH1, HID, 0);
        uint32_t phw = 0;
        for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
          for (int p = 2; p < kPhases; ++p) {
            mbar_wait(&bar_w, phw, 0x200u + static_cast<uint32_t>(p), a.progress);  // the chain warp has seen this phase's operands
            phw ^= 1;
            tc_fence_after();
            if (p == 2) {  // G2 += H2^T * dY (dW2^T);  G1 += dH2^T * [H1 | 1]
              gemm_split(tb + tG2, make_idesc_bf16(64, OUTP, true, true), kTile / 16, g_started, precise, mH2d, loH,
                         2 * cm16_row_group_stride(HC), mDYd, loDY, 2 * cm16_row_group_stride(OUTP));
              gemm_split(tb + tG1, make_idesc_bf16(64, HC, true, true), kTile / 16, g_started, precise, mDH2d, loDH,
                         2 * cm16_row_group_stride(HID), mH1d, loH, 2 * cm16_row_group_stride(HC));
            } else {       // G0 += dH1^T * [X0 | 1]
              gemm_split(tb + tG0, make_idesc_bf16(64, X0C, true, true), kTile / 16, g_started, precise, mDH1d, loDH,
                         2 * cm16_row_group_stride(HID), mX0d, loX0, 2 * cm16_row_group_stride(X0C));
              tc_commit(&bar_g);  // covers G2, G1 and G0 of this tile
              g_started = true;
            }
          }
        }
      }
    }
  } else {
    // =========================== epilogue warps ===========================
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t phase = 0, phase_g = 0;
    double loss_acc = 0.0;
    double db2_acc[3] = {0.0, 0.0, 0.0};

    // hidden-layer epilogue: 32 columns of this thread's row out of a TMEM accumulator -> (bias, ReLU | mask) -> hi/lo tile
    auto ready = [&]() {
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bar_ready);
    };
    const bool timed = a.timing != nullptr && tid == 0;
    unsigned long long t_chain = 0, t_wgrad = 0;
    const long long t_begin = clock64();
    auto wait_chain = [&]() {
      const long long t0 = timed ? clock64() : 0;
      mbar_wait(&bar, phase, 0x300u, a.progress);
      if (timed) t_chain += static_cast<unsigned long long>(clock64() - t0);
      phase ^= 1;
      tc_fence_after();
    };

    // Software pipeline over tiles: the features of tile i+1 are requested right after tile i's have been written to
    // shared memory, and a tile's targets at its top, so neither global-load latency sits on the per-tile dependency chain
    // (ncu stall sampling had 9 % of the samples waiting on the feature loads and 5 % on the target loads).
    constexpr int kXCh = IN / 8;                             // 8-float chunks per feature row
    constexpr int kXThreads = kEpiThreads < kTile * kXCh ? kEpiThreads : kTile * kXCh;  // threads that stage (all, or one per chunk)
    constexpr int kXIt = (kTile * kXCh) / kXThreads;         // chunks per staging thread
    constexpr int kXRows = kXThreads / 8 / kXCh;             // 8-row groups one pass of the staging threads covers
    const bool stages = tid < kXThreads;
    float xin[kXIt][8];
    const int xch = (tid >> 3) & (kXCh - 1);
    const int xrow = (tid & 7) + 8 * ((tid >> 3) / kXCh);
    auto load_features = [&](unsigned long long tile_index) {
#pragma unroll
      for (int it = 0; it < kXIt; ++it) {
        const int row = xrow + 8 * kXRows * it;
        const unsigned long long gs = tile_index * kTile + row;
        if (stages && tile_index < n_tiles && gs < a.n) {
          const float4* p = reinterpret_cast<const float4*>(a.features + gs * IN + xch * 8);
          const float4 x0 = __ldg(p), x1 = __ldg(p + 1);
          xin[it][0] = x0.x; xin[it][1] = x0.y; xin[it][2] = x0.z; xin[it][3] = x0.w;
          xin[it][4] = x1.x; xin[it][5] = x1.y; xin[it][6] = x1.z; xin[it][7] = x1.w;
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) xin[it][q] = 0.0f;
        }
      }
    };
    load_features(blockIdx.x);

    for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
      const unsigned long long s0 = tile * kTile;
      const unsigned long long smp = s0 + t;
      const bool valid = smp < a.n;

      // ---- stage 0: features -> X0 tiles.  Lane mapping: 8 rows x 4 chunks per warp instruction keeps both the global
      // reads (64 contiguous bytes per row) and the shared stores (8 rows = 8 distinct 16-byte bank groups) efficient.
      // The previous tile's weight-gradient MMAs still read X0: wait for them before overwriting it.
      double tgt[3] = {0.0, 0.0, 0.0};
      if constexpr (TRAIN) {
        if (valid) {
#pragma unroll
          for (int o = 0; o < 3; ++o)
            if (o < a.out_w)
              tgt[o] = a.target_f32 ? static_cast<double>(static_cast<const float*>(a.targets)[smp * a.out_w + o])
                                    : static_cast<const double*>(a.targets)[smp * a.out_w + o];
        }
        if (g_started) {
          const long long t0 = timed ? clock64() : 0;
          mbar_wait(&bar_g, phase_g, 0x400u, a.progress);
          if (timed) t_wgrad += static_cast<unsigned long long>(clock64() - t0);
          phase_g ^= 1;
        }
      }
#pragma unroll
      for (int it = 0; it < kXIt; ++it)
        if (stages) store_chunk(smem + kX0, smem + kX0 + loX0, xrow + 8 * kXRows * it, xch, X0C, xin[it]);
      ready();
      if constexpr (!TRAIN) load_features(tile + gridDim.x);  // in flight under this tile's two phases

      // ---- layer 1 epilogue: S0 -> H1
      uint32_t m1 = 0, m2 = 0;  // ReLU masks of this thread's 32 units (bit i = unit 32*half + i active)
      wait_chain();
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
            float x = __uint_as_float(r[q][i]) + bias[CPT * half + 16 * q + i];
            x = x > 0.0f ? x : 0.0f;
            if (x > 0.0f) m1 |= 1u << (16 * q + i);
            v[i] = x;
          }
          store_chunk(smem + kH1, smem + kH1 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
          store_chunk(smem + kH1, smem + kH1 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
        }
      }
      ready();

      // ---- layer 2 epilogue: S1 -> H2, then the output layer, the loss and its way back to dH2 on the CUDA cores
      wait_chain();
      {
        uint32_t r[CPT / 16][16];
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(tb + lane_base + tS1 + CPT * half + 16 * q, r[q]);
        tmem_ld_wait();
        float p0 = 0.0f, p1 = 0.0f, p2 = 0.0f;  // partial predictions over this thread's 32 hidden units
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int c = CPT * half + 16 * q + i;
            float x = __uint_as_float(r[q][i]) + bias[HID + c];
            x = x > 0.0f ? x : 0.0f;
            if (x > 0.0f) m2 |= 1u << (16 * q + i);
            v[i] = x;
            p0 = __fmaf_rn(w2f[c], x, p0);
            p1 = __fmaf_rn(w2f[HID + c], x, p1);
            p2 = __fmaf_rn(w2f[2 * HID + c], x, p2);
          }
          store_chunk(smem + kH2, smem + kH2 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
          store_chunk(smem + kH2, smem + kH2 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
        }
        *reinterpret_cast<float4*>(pp + (half * kTile + t) * 4) = make_float4(p0, p1, p2, 0.0f);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");  // the two halves of every row have posted their partials
      float u[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      {
        float pr[3] = {bias[2 * HID], bias[2 * HID + 1], bias[2 * HID + 2]};
#pragma unroll
        for (int k = 0; k < kSplit; ++k) {
          const float4 pk = *reinterpret_cast<const float4*>(pp + (k * kTile + t) * 4);
          pr[0] += pk.x;
          pr[1] += pk.y;
          pr[2] += pk.z;
        }
#pragma unroll
        for (int o = 0; o < 3; ++o) {
          if (o < a.out_w) {
            if (half == 0 && valid && a.pred) a.pred[smp * a.out_w + o] = pr[o];
            if constexpr (TRAIN) {
              if (valid) {
                // src/trainer.cpp:38-44: e = pred - target, loss += e*e, upstream = 2e/(B*out_w), all in double
                const double e = static_cast<double>(pr[o]) - tgt[o];
                const double up = a.upstream_scale * e;
                u[o] = static_cast<float>(up);
                if (half == 0) {
                  loss_acc += e * e;
                  db2_acc[o] += up;
                }
              }
            }
          }
        }
      }
      if constexpr (!TRAIN) continue;  // the tiles and S1 are only rewritten after the next bar_ready rounds
      if (half == 0) store_chunk(smem + kDY, smem + kDY + loDY, t, 0, OUTP, u);  // B operand of G2 = H2^T * dY
      {
        // dH2[c] = sum_o u[o] * W2[o][c], zero where layer 2's ReLU clamped (src/mlp.cpp:189-199)
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

      // ---- backward epilogue of layer 1: S0[:, 0:32] -> d loss / d encoding, straight to global memory
      load_features(tile + gridDim.x);  // in flight under the last phase (earlier, the loads only hold scoreboards)
      wait_chain();
      if (half < IN / 16) {
        uint32_t r[16];
        tmem_ld16_nowait(tb + lane_base + tS0 + 16 * half, r);
        tmem_ld_wait();
        if (valid) {
          float4* dst = reinterpret_cast<float4*>(a.input_grad + smp * IN + 16 * half);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            __stcs(dst + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                                        __uint_as_float(r[4 * q + 3])));
        }
      }
      tc_fence_before();
      g_started = true;
    }

    if (timed) {
      atomicAdd(a.timing + 0, static_cast<unsigned long long>(clock64() - t_begin));
      atomicAdd(a.timing + 1, t_chain);
      atomicAdd(a.timing + 2, t_wgrad);
    }
    if constexpr (TRAIN) {
      // ---- weight gradients out of TMEM.  An M = 64 accumulator keeps row i in lane (i/16)*32 + i%16 (tools/tc_probe.py),
      // so lanes 0..15 of each warp hold rows 16*(warp%4) .. +15; warps w and w+4 split the columns.
      if (g_started) mbar_wait(&bar_g, phase_g, 0x401u, a.progress);
      tc_fence_after();
      const int lane = tid & 31;
      const int row = 16 * (warp & 3) + lane;  // output unit o (G0, G1) or hidden unit i (G2)
      constexpr size_t gW0 = 0, gb0 = gW0 + HID * IN, gW1 = gb0 + HID, gb1 = gW1 + HID * HID, gW2 = gb1 + HID;  // offsets
      double* const G = a.mlp_grad;
      long long* const FX = a.grad_fixed;
      if (g_started) {
        for (int c0 = 8 * half; c0 < X0C; c0 += 8 * kSplit) {  // G0: IN + 8 columns = dW0[row][0..IN), db0[row] at column IN
          uint32_t r[16];
          tmem_ld16_nowait(tb + lane_base + tG0 + (c0 < IN ? c0 : IN - 8), r);  // the last read re-covers cols IN-8..IN+7
          tmem_ld_wait();
          if (lane < 16) {
            if (c0 < IN) {
              for (int i = 0; i < 8; ++i) add_total(G, FX, gW0 + row * IN + c0 + i, static_cast<double>(__uint_as_float(r[i])));
            } else {
              add_total(G, FX, gb0 + row, static_cast<double>(__uint_as_float(r[8])));
            }
          }
        }
        for (int c0 = 8 * half; c0 < HC; c0 += 8 * kSplit) {  // G1: 72 columns = dW1[row][0..63], db1[row] at column 64
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
        if (half == 1) {  // G2: dW2^T[i = row][o]
          uint32_t r[16];
          tmem_ld16_nowait(tb + lane_base + tG2, r);
          tmem_ld_wait();
          if (lane < 16)
            for (int o = 0; o < a.out_w; ++o) add_total(G, FX, gW2 + o * HID + row, static_cast<double>(__uint_as_float(r[o])));
        }
      }
      // loss and output-bias gradient: per-thread fp64 partials -> warp shuffle -> one atomic per CTA (below)
      double part[4] = {loss_acc, db2_acc[0], db2_acc[1], db2_acc[2]};
#pragma unroll
      for (int k = 0; k < 4; ++k)
        for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_down_sync(0xffffffffu, part[k], o);
      if (lane == 0)
        for (int k = 0; k < 4; ++k) red_buf[warp][k] = part[k];
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (TRAIN) {
    if (tid == 0) {
      double tot[4] = {0, 0, 0, 0};
      for (int w = 0; w < kEpiThreads / 32; ++w)
        for (int k = 0; k < 4; ++k) tot[k] += red_buf[w][k];
      const size_t gb2 = HID * IN + HID + HID * HID + HID + a.out_w * HID;
      const size_t n_params = gb2 + a.out_w;
      // reproducible mode: the CTAs' loss partials (not bounded like a gradient, so not fixed point) go to one slot per CTA
      // behind the parameter words; the host side adds them to *loss_sum in CTA order
      if (a.grad_fixed != nullptr) reinterpret_cast<double*>(a.grad_fixed + n_params)[blockIdx.x] = tot[0];
      else atomicAdd(a.loss_sum, tot[0]);
      for (int o = 0; o < a.out_w && o < 3; ++o) add_total(a.mlp_grad, a.grad_fixed, gb2 + o, tot[1 + o]);
    }
  }
  if (warp == 0) tmem_dealloc(tb, kTmemCols);
}

}  // namespace

// Diagnostics: host-mapped words the kernels' mbarrier watchdog writes before it traps (wait id, CTA); nullptr = off.
static volatile unsigned int* g_tc_progress = nullptr;
extern "C" SXEN_API sxen_status sxen_debug_tc_progress(unsigned int* mapped_host_words) {
  g_tc_progress = mapped_host_words;
  return SXEN_OK;
}
static unsigned long long* g_tc_timing = nullptr;
extern "C" SXEN_API sxen_status sxen_debug_tc_timing(unsigned long long* counters_dev) {
  g_tc_timing = counters_dev;
  return SXEN_OK;
}
sxen_status sxen_mlp_tc_forward_launch(const sxen_mlp_tc::TcArgs& a, int in_w, cudaStream_t stream, int* used_ctas);  // sxen_mlp_tc_fwd.cu
sxen_status sxen_mlp_tc2_train_launch(const sxen_mlp_tc::TcArgs& a, int in_w, cudaStream_t stream, int* used_ctas);  // sxen_mlp_tc2.cu
// Which training kernel runs: 2 = two tiles in flight per SM (sxen_mlp_tc2.cu), 1 = one tile in flight (this file).
static int g_tc_variant = 2;
extern "C" SXEN_API sxen_status sxen_debug_tc_variant(int variant) {
  if (variant != 1 && variant != 2) return fail(SXEN_INVALID_ARGUMENT, "tc variant %d: 1 (one tile in flight) or 2 (two)", variant);
  g_tc_variant = variant;
  return SXEN_OK;
}

// Internal entry points used by sxen_mlp.cu / sxen_trainer.cu (declared there).
bool sxen_mlp_tc_supported(const sxen_mlp_config& c) {
  return (c.input_width == 16 || c.input_width == 32) && c.hidden_width == HID && c.hidden_layers == 2 && c.output_width >= 1 && c.output_width <= 3;
}

sxen_status sxen_mlp_tc_run(bool train, const float* params, const float* features, const void* targets, int target_f32,
                            float* pred, float* input_grad, double* mlp_grad, double* loss_sum, size_t n, int in_w, int out_w,
                            size_t global_batch, int precise, cudaStream_t stream, long long* grad_fixed, int* used_ctas,
                            double* partials, size_t partial_stride) {
  if (n == 0) return SXEN_OK;
  if (in_w != 16 && in_w != 32) return fail(SXEN_INVALID_ARGUMENT, "mlp (tensor cores): input width %d not instantiated", in_w);
  TcArgs a{};
  a.params = params;
  a.features = features;
  a.targets = targets;
  a.pred = pred;
  a.input_grad = input_grad;
  a.mlp_grad = mlp_grad;
  a.loss_sum = loss_sum;
  a.grad_fixed = train ? grad_fixed : nullptr;
  a.n = n;
  a.out_w = out_w;
  a.target_f32 = target_f32;
  a.precise = precise;
  a.upstream_scale = 2.0 / static_cast<double>(global_batch * static_cast<size_t>(out_w));  // src/trainer.cpp:26-27
  a.progress = g_tc_progress;
  a.timing = g_tc_timing;
  if (!train) return sxen_mlp_tc_forward_launch(a, in_w, stream, used_ctas);  // its own kernel: one hand-off per tile
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long tiles = (n + kTile - 1) / kTile;
  // two tiles in flight pay off from the second tile of a CTA on; a launch of at most one tile per SM (the reference's default
  // batch of 2048 is 16 tiles) only pays that kernel's fixed costs -- gradient rows to clear, a reduction kernel behind it
  if (g_tc_variant == 2 && tiles > static_cast<unsigned long long>(sms)) {
    if (a.grad_fixed == nullptr) {  // per-CTA gradient rows + a fixed-order reduction instead of contended atomics
      a.partials = partials;
      a.partial_stride = partial_stride;
    }
    return sxen_mlp_tc2_train_launch(a, in_w, stream, used_ctas);
  }
  const unsigned grid = static_cast<unsigned>(std::min<unsigned long long>(tiles, static_cast<unsigned long long>(sms)));
  auto launch = [&](auto kernel) -> sxen_status {
    SXEN_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    kernel<<<grid, kThreadsAll, kSmemBytes, stream>>>(a);
    return SXEN_OK;
  };
  sxen_status st;
  st = in_w == 32 ? launch(mlp_tc_kernel<true, 32>) : launch(mlp_tc_kernel<true, 16>);
  if (st != SXEN_OK) return st;
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (used_ctas) *used_ctas = static_cast<int>(grid);
  return SXEN_OK;
}
