// sxen_mlp_tc_fwd.cu -- Mlp::forward on the tensor cores (inference: render_image, hold-out evaluation), one epilogue <-> MMA
// hand-off per 128-sample tile.  Reference semantics: /root/reference/proj/src/mlp.cpp:137-162; numerics as sxen_mlp_tc.cu
// (split-bf16 GEMMs, fp32 accumulation in TMEM).
//
// Schedule.  X0 is double-buffered and the layer-1 GEMM of tile k+1 is issued right behind the layer-2 GEMM of tile k, so at
// the top of a tile ONE wait covers "layer 2 of the previous tile" and "layer 1 of this tile": the epilogue warps turn S1 into
// the previous tile's predictions, stage the next tile's features, turn S0 into this tile's H1 and hand over -- against two
// hand-offs per tile in the fused training kernel's forward half (0.145 -> 0.117 ms per 2^20 samples).  The kernel body also
// carries the matching three-hand-off TRAINING schedule (layer 1 of the next tile issued together with the last backward
// GEMM, the input gradient leaving through its own TMEM columns); measured, that one loses to sxen_mlp_tc.cu's schedule
// (0.423 vs 0.391 ms: the wait for the previous tile's weight-gradient MMAs lands on the critical path), so only the forward
// instantiation is built.
#include <algorithm>

#include "sxen_mlp_tc_common.cuh"

using namespace sxen_host;
using namespace sxen_tc;
using namespace sxen_mlp_tc;

namespace {

// shared-memory map (bytes)
constexpr uint32_t kW0 = 0;                                     // CM16(64, 32) hi, lo
constexpr uint32_t kW1 = kW0 + 2 * cm16_bytes(HID, kInMax);     // CM16(64, 64) hi, lo   (regions sized for IN = 32)
constexpr uint32_t kX0 = kW1 + 2 * cm16_bytes(HID, HID);        // CM16(128, 40) hi, lo -- TWO buffers, tile parity
constexpr uint32_t kX0Bytes = 2 * cm16_bytes(kTile, kX0CMax);
constexpr uint32_t kH1 = kX0 + 2 * kX0Bytes;                    // CM16(128, 72) hi, lo
constexpr uint32_t kH2 = kH1 + 2 * cm16_bytes(kTile, HC);
constexpr uint32_t kDY = kH2 + 2 * cm16_bytes(kTile, HC);       // CM16(128, 16) hi, lo
constexpr uint32_t kDH2 = kDY + 2 * cm16_bytes(kTile, OUTP);    // CM16(128, 64) hi, lo
constexpr uint32_t kDH1 = kDH2 + 2 * cm16_bytes(kTile, HID);
constexpr uint32_t kBias = kDH1 + 2 * cm16_bytes(kTile, HID);   // b0[64], b1[64], b2[4] floats
constexpr uint32_t kW2f = kBias + (HID + HID + 4) * 4;          // output layer in fp32: W2f[3][64] (rows >= out_w zero)
constexpr uint32_t kPP = kW2f + 3 * HID * 4;                    // partial predictions pp[2][128][4]
constexpr uint32_t kSmemBytes = kPP + 4 * kTile * 4 * 4;  // pp[kSplit <= 4][128][4]

// TMEM columns (fp32): scratch accumulators (128 lanes) and the persistent weight-gradient accumulators (M = 64)
constexpr uint32_t tS0 = 0;     // [128 x 64] layer-1 pre-activation
constexpr uint32_t tS1 = 64;    // [128 x 64] layer-2 pre-activation, later dH1
constexpr uint32_t tG0 = 128;   // [64 x 40]  dW0 | db0
constexpr uint32_t tG1 = 168;   // [64 x 72]  dW1 | db1
constexpr uint32_t tG2 = 240;   // [64 x 16]  dW2^T
constexpr uint32_t tDX = 256;   // [128 x 32] d(input): its own columns, so that the next tile's layer 1 can overwrite S0 at once
constexpr uint32_t kTmemCols = 512;

template <bool TRAIN, int IN>
__global__ void __launch_bounds__(kThreadsAll, 1) mlp_tc_kernel(const __grid_constant__ TcArgs a) {
  static_assert(IN == 16 || IN == 32, "input widths 16 (L=8, F=2: the reference's default encoder) and 32 (L=16, F=2)");
  constexpr int X0C = IN + 8;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_ready;  // 256 arrivals: the tiles of the next GEMM group are written and the TMEM scratch is drained
  __shared__ uint64_t bar;        // the chain warp's GEMMs up to here have completed
  __shared__ uint64_t bar_g;      // every weight-gradient MMA of the tile has completed
  __shared__ uint64_t bar_w;      // chain warp -> weight-gradient warp: the operands of backward phase 2 / 3 are in place
  __shared__ uint32_t tmem_base_slot;
  __shared__ double red_buf[kEpiThreads / 32][4];
  const int tid = threadIdx.x;
  const int t = tid & (kTile - 1);   // sample row inside the tile
  const int half = (tid >> 7) & (kSplit - 1);  // which slice of an epilogue's columns this thread handles
  const int warp = tid >> 5;
  const bool is_mma_warp = warp == kEpiThreads / 32;        // issues the dependent-chain GEMMs of every tile
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
      store_chunk(smem + kX0 + kX0Bytes, smem + kX0 + kX0Bytes + loX0, t, IN / 8, X0C, ones);
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
  bool g_started = false;

  // Schedule (round 2).  The layer-1 GEMM of tile k+1 is issued TOGETHER with the last GEMM of tile k (its X0 tile sits in the
  // second buffer, its accumulator S0 has been free since tile k's first epilogue), and the input gradient leaves through
  // its own TMEM columns (tDX) at the top of the next tile.  A tile therefore costs THREE epilogue <-> MMA round trips
  //     [S0 -> H1] -> H1*W1^T | [S1 -> H2, output layer, loss, dH2] -> dH2*W1 | [S1 -> dH1] -> dH1*W0 + X0'*W0^T
  // where the round-1 kernel paid five (0.41 ms per 2^20 samples, 53 % of its warp-stall samples in the hand-offs);
  // forward only: one round trip per tile instead of two.
  if (is_mma_warp) {
    // =========================== MMA warp: one lane issues every chain tcgen05.mma of the CTA ===========================
    if ((tid & 31) == 0) {
      const uint32_t sW0 = smem_u32(smem + kW0), sW1 = smem_u32(smem + kW1);
      const uint32_t sH1 = smem_u32(smem + kH1), sDH2 = smem_u32(smem + kDH2), sDH1 = smem_u32(smem + kDH1);
      // K-major views step 256 B per UMMA_K = 16; MN-major views step two 8-row groups
      const uint64_t kH1d = desc16_k_major(sH1, HC, 0);
      const uint64_t kW0d = desc16_k_major(sW0, IN, 0), kW1d = desc16_k_major(sW1, HID, 0);
      const uint64_t kDH2d = desc16_k_major(sDH2, HID, 0), kDH1d = desc16_k_major(sDH1, HID, 0);
      const uint64_t mW0d = desc16_mn_major(sW0, IN, 0), mW1d = desc16_mn_major(sW1, HID, 0);
      constexpr uint32_t kStep = 256;
      // (called with a CONSTANT parity only: with a run-time b and four products nvcc 12.9 loads the fourth MMA's B descriptor
      // under a predicate that is not set on this path, the instruction repeats product three and the second tile of a CTA
      // comes out 2^-9 off -- DESIGN.md 3.4)
      auto layer1 = [&](int b) {  // S0 = X0[b] * W0^T
        const uint64_t kX0d = desc16_k_major(smem_u32(smem + kX0 + b * kX0Bytes), X0C, 0);
        gemm_split(tb + tS0, make_idesc_bf16(128, HID, false, false), IN / 16, false, precise, kX0d, loX0, kStep, kW0d, loW0, kStep);
      };
      uint32_t ph = 0;
      auto wait_ready = [&]() {
        mbar_wait(&bar_ready, ph, 0x100u + static_cast<uint32_t>(ph), a.progress);
        ph ^= 1;
        tc_fence_after();
      };
      if (blockIdx.x < n_tiles) {
        wait_ready();  // the first tile's X0
        layer1(0);
        tc_commit(&bar);
      }
      int k = 0;
      for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const bool has_next = tile + gridDim.x < n_tiles;
        wait_ready();  // layer 2: S1 = H1 * W1^T
        gemm_split(tb + tS1, make_idesc_bf16(128, HID, false, false), HID / 16, false, precise, kH1d, loH, kStep, kW1d, loW1, kStep);
        if constexpr (!TRAIN) {
          if (has_next) { if ((k + 1) & 1) layer1(1); else layer1(0); }  // constant parities: see layer1
          tc_commit(&bar);
        } else {
          tc_commit(&bar);
          wait_ready();  // S1 = dH2 * W1
          mbar_arrive(&bar_w);
          gemm_split(tb + tS1, make_idesc_bf16(128, HID, false, true), HID / 16, false, precise, kDH2d, loDH, kStep, mW1d, loW1,
                     2 * cm16_row_group_stride(HID));
          tc_commit(&bar);
          wait_ready();  // tDX = dH1 * W0 (d loss / d encoding), and the next tile's layer 1 right behind it
          mbar_arrive(&bar_w);
          gemm_split(tb + tDX, make_idesc_bf16(128, IN, false, true), HID / 16, false, precise, kDH1d, loDH, kStep, mW0d, loW0,
                     2 * cm16_row_group_stride(IN));
          if (has_next) { if ((k + 1) & 1) layer1(1); else layer1(0); }  // constant parities: see layer1
          tc_commit(&bar);
        }
      }
    }
  } else if (is_wgrad_warp) {
    // ============ weight-gradient warp: its own lane issues G2, G1 (phase 2) and G0 (phase 3) of every tile ============
    if constexpr (TRAIN) {
      if ((tid & 31) == 0) {
        const uint32_t sH1 = smem_u32(smem + kH1), sH2 = smem_u32(smem + kH2);
        const uint32_t sDY = smem_u32(smem + kDY), sDH2 = smem_u32(smem + kDH2), sDH1 = smem_u32(smem + kDH1);
        const uint64_t mH1d = desc16_mn_major(sH1, HC, 0), mH2d = desc16_mn_major(sH2, HC, 0);
        const uint64_t mDYd = desc16_mn_major(sDY, OUTP, 0), mDH2d = desc16_mn_major(sDH2, HID, 0), mDH1d = desc16_mn_major(sDH1, HID, 0);
        uint32_t phw = 0;
        int k = 0;
        for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
          mbar_wait(&bar_w, phw, 0x200u, a.progress);  // G2 += H2^T * dY (dW2^T);  G1 += dH2^T * [H1 | 1]
          phw ^= 1;
          tc_fence_after();
          gemm_split(tb + tG2, make_idesc_bf16(64, OUTP, true, true), kTile / 16, g_started, precise, mH2d, loH,
                     2 * cm16_row_group_stride(HC), mDYd, loDY, 2 * cm16_row_group_stride(OUTP));
          gemm_split(tb + tG1, make_idesc_bf16(64, HC, true, true), kTile / 16, g_started, precise, mDH2d, loDH,
                     2 * cm16_row_group_stride(HID), mH1d, loH, 2 * cm16_row_group_stride(HC));
          mbar_wait(&bar_w, phw, 0x201u, a.progress);  // G0 += dH1^T * [X0 | 1]
          phw ^= 1;
          tc_fence_after();
          const uint64_t mX0d = desc16_mn_major(smem_u32(smem + kX0 + (k & 1) * kX0Bytes), X0C, 0);
          gemm_split(tb + tG0, make_idesc_bf16(64, X0C, true, true), kTile / 16, g_started, precise, mDH1d, loDH,
                     2 * cm16_row_group_stride(HID), mX0d, loX0, 2 * cm16_row_group_stride(X0C));
          tc_commit(&bar_g);  // covers G2, G1 and G0 of this tile
          g_started = true;
        }
      }
    }
  } else {
    // =========================== epilogue warps ===========================
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t phase = 0, phase_g = 0;
    double loss_acc = 0.0;
    double db2_acc[3] = {0.0, 0.0, 0.0};

    auto ready = [&]() {
      fence_proxy_async();
      tc_fence_before();
      mbar_arrive(&bar_ready);
    };
    auto wait_chain = [&]() {
      mbar_wait(&bar, phase, 0x300u + static_cast<uint32_t>(phase), a.progress);
      phase ^= 1;
      tc_fence_after();
    };

    // Software pipeline over tiles: a tile's features are requested a tile ahead (registers) and written into the X0
    // buffer of its parity while the previous tile's backward GEMMs run.
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
    // Lane mapping of the staging: 8 rows x 4 chunks per warp instruction keeps both the global reads (64 contiguous bytes
    // per row) and the shared stores (8 rows = 8 distinct 16-byte bank groups) efficient.
    auto stage_features = [&](int b) {
#pragma unroll
      for (int it = 0; it < kXIt; ++it)
        if (stages) store_chunk(smem + kX0 + b * kX0Bytes, smem + kX0 + b * kX0Bytes + loX0, xrow + 8 * kXRows * it, xch, X0C, xin[it]);
    };
    // d loss / d encoding of one tile: tDX -> global memory
    auto store_input_grad = [&](unsigned long long tile_index) {
      if (half < IN / 16) {
        uint32_t r[16];
        tmem_ld16_nowait(tb + lane_base + tDX + 16 * half, r);
        tmem_ld_wait();
        const unsigned long long smp = tile_index * kTile + t;
        if (smp < a.n) {
          float4* dst = reinterpret_cast<float4*>(a.input_grad + smp * IN + 16 * half);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            __stcs(dst + q, make_float4(__uint_as_float(r[4 * q]), __uint_as_float(r[4 * q + 1]), __uint_as_float(r[4 * q + 2]),
                                        __uint_as_float(r[4 * q + 3])));
        }
      }
    };
    // layer-2 epilogue of one tile, forward only: S1 -> ReLU -> output layer -> predictions
    auto forward_out = [&](unsigned long long tile_index) {
      uint32_t r[CPT / 16][16];
#pragma unroll
      for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(tb + lane_base + tS1 + CPT * half + 16 * q, r[q]);
      tmem_ld_wait();
      float p0 = 0.0f, p1 = 0.0f, p2 = 0.0f;
#pragma unroll
      for (int q = 0; q < CPT / 16; ++q) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = CPT * half + 16 * q + i;
          float x = __uint_as_float(r[q][i]) + bias[HID + c];
          x = x > 0.0f ? x : 0.0f;
          p0 = __fmaf_rn(w2f[c], x, p0);
          p1 = __fmaf_rn(w2f[HID + c], x, p1);
          p2 = __fmaf_rn(w2f[2 * HID + c], x, p2);
        }
      }
      *reinterpret_cast<float4*>(pp + (half * kTile + t) * 4) = make_float4(p0, p1, p2, 0.0f);
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");
      if (half == 0) {
        float pr[3] = {bias[2 * HID], bias[2 * HID + 1], bias[2 * HID + 2]};
#pragma unroll
        for (int k = 0; k < kSplit; ++k) {
          const float4 pk = *reinterpret_cast<const float4*>(pp + (k * kTile + t) * 4);
          pr[0] += pk.x;
          pr[1] += pk.y;
          pr[2] += pk.z;
        }
        const unsigned long long smp = tile_index * kTile + t;
        if (smp < a.n && a.pred)
          for (int o = 0; o < a.out_w && o < 3; ++o) a.pred[smp * a.out_w + o] = pr[o];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiThreads) : "memory");  // pp is rewritten by the next tile
    };

    load_features(blockIdx.x);
    if (blockIdx.x < n_tiles) {
      stage_features(0);
      ready();
    }
    load_features(static_cast<unsigned long long>(blockIdx.x) + gridDim.x);

    int k = 0;
    unsigned long long prev_tile = 0;
    for (unsigned long long tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
      const unsigned long long smp = tile * kTile + t;
      const bool valid = smp < a.n;
      const bool has_next = tile + gridDim.x < n_tiles;
      double tgt[3] = {0.0, 0.0, 0.0};
      if constexpr (TRAIN) {
        if (valid) {
#pragma unroll
          for (int o = 0; o < 3; ++o)
            if (o < a.out_w)
              tgt[o] = a.target_f32 ? static_cast<double>(static_cast<const float*>(a.targets)[smp * a.out_w + o])
                                    : static_cast<const double*>(a.targets)[smp * a.out_w + o];
        }
      }
      // ---- top of the tile: this tile's layer 1 (and the previous tile's last GEMM) have completed
      wait_chain();
      if constexpr (TRAIN) {
        if (k > 0) store_input_grad(prev_tile);
        if (g_started) {  // the previous tile's weight-gradient MMAs read H1 .. dH1 and its X0 buffer: all free after this
          mbar_wait(&bar_g, phase_g, 0x400u, a.progress);
          phase_g ^= 1;
        }
      } else {
        if (k > 0) forward_out(prev_tile);
        if (has_next) {  // the buffer of the other parity was last read by the previous tile's layer 1: complete
          stage_features((k + 1) & 1);
          load_features(tile + 2ull * gridDim.x);
        }
      }
      // ---- layer 1 epilogue: S0 -> H1
      uint32_t m1 = 0, m2 = 0;  // ReLU masks of this thread's 32 units (bit i = unit 32*half + i active)
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
      prev_tile = tile;
      if constexpr (!TRAIN) continue;  // forward only: the layer-2 epilogue runs at the top of the next tile

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
        for (int kk = 0; kk < kSplit; ++kk) {
          const float4 pk = *reinterpret_cast<const float4*>(pp + (kk * kTile + t) * 4);
          pr[0] += pk.x;
          pr[1] += pk.y;
          pr[2] += pk.z;
        }
#pragma unroll
        for (int o = 0; o < 3; ++o) {
          if (o < a.out_w) {
            if (half == 0 && valid && a.pred) a.pred[smp * a.out_w + o] = pr[o];
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
      // ---- in the shadow of dH2*W1: the NEXT tile's features into the X0 buffer of its parity (last read by the layer 1 and
      // the weight-gradient GEMM of the tile before this one: both complete, see the waits at the top), and the request for
      // the tile after that
      if (has_next) {
        stage_features((k + 1) & 1);
        load_features(tile + 2ull * gridDim.x);
      }
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
      ready();  // -> dH1*W0 into tDX, G0, and the next tile's layer 1
      g_started = true;
    }
    // ---- the last tile's results
    if (k > 0) {
      wait_chain();
      if constexpr (TRAIN) store_input_grad(prev_tile);
      else forward_out(prev_tile);
    }
    tc_fence_before();

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
      for (int kk = 0; kk < 4; ++kk)
        for (int o = 16; o > 0; o >>= 1) part[kk] += __shfl_down_sync(0xffffffffu, part[kk], o);
      if (lane == 0)
        for (int kk = 0; kk < 4; ++kk) red_buf[warp][kk] = part[kk];
    }
  }

  tc_fence_before();
  __syncthreads();
  if constexpr (TRAIN) {
    if (tid == 0) {
      double tot[4] = {0, 0, 0, 0};
      for (int w = 0; w < kEpiThreads / 32; ++w)
        for (int kk = 0; kk < 4; ++kk) tot[kk] += red_buf[w][kk];
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

sxen_status sxen_mlp_tc_forward_launch(const TcArgs& a, int in_w, cudaStream_t stream, int* used_ctas) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long tiles = (a.n + kTile - 1) / kTile;
  const unsigned grid = static_cast<unsigned>(std::min<unsigned long long>(tiles, static_cast<unsigned long long>(sms)));
  auto launch = [&](auto kernel) -> sxen_status {
    SXEN_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    kernel<<<grid, kThreadsAll, kSmemBytes, stream>>>(a);
    return SXEN_OK;
  };
  if (sxen_status st = in_w == 32 ? launch(mlp_tc_kernel<false, 32>) : launch(mlp_tc_kernel<false, 16>)) return st;
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (used_ctas) *used_ctas = static_cast<int>(grid);
  return SXEN_OK;
}
