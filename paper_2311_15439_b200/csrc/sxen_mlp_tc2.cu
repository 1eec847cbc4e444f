// sxen_mlp_tc2.cu -- the fused training kernel of the tensor-core MLP head (forward + loss + backward, as sxen_mlp_tc.cu)
// with TWO 128-sample tiles in flight per SM.
//
// Why.  sxen_mlp_tc.cu walks one tile through five epilogue <-> MMA hand-offs; its epilogue warps work 7.3k of the 12.0k
// cycles a tile takes and the tensor pipe is busy for a fifth of them (profiles/r2_mlp_tc_timing.txt): the tile is a serial
// chain.  Here two groups of eight warps each own a tile, so one group's conversions run under the other group's GEMMs.
// There are no dedicated MMA warps: 16 warps leave each thread 128 registers (18 would leave 96 -- the register file is
// allocated in units of four warps -- and the 222 KB of operand tiles leave no L1 to catch spills: a version that spilled
// 300 bytes ran its epilogues 2.4x slower).  A group hands a phase over with one named barrier, after which three elected
// lanes issue its GEMMs: the dependent-chain GEMM (warp 0 of the group), dW2 / dW0 (warp 5) and dW1 (warp 6), each
// committing to its own mbarrier.
//
// Shared memory is what limits the number of tiles in flight: a tile's operand set (X0, H1, H2, dY, dH2, dH1, each a hi/lo
// pair of bf16 CM16 tiles) is 164 KB.  The set is not live all at once, though.  With tiles numbered j = 0, 1, 2 ... in the
// order the CTA starts them (group = j % 2):
//     H1_j   lives from its epilogue to the end of the tile's phase-2 GEMMs (layer 2, dW1),
//     H2_j   only feeds dW2 (phase 2); dH1_j is written after that and dies with phase 3,
//     dH2_j  (+ dY_j in its spare column block) lives for phase 2 only.
// Three [128 x 72] buffers in a ring carry H1 / H2 / dH1 of both tiles -- H1_j = ring[j % 3], H2_j = dH1_j = ring[(j+2) % 3],
// which is the buffer H1_(j-1) leaves when tile j-1's phase-2 GEMMs complete -- and ONE buffer carries dH2 | dY of whichever
// tile is in phase 2.  208 KB with the weights and the two X0 tiles.  The ring fixes the order: tile j's second epilogue
// waits for tile j-1's phase-2 GEMMs (its own group's previous tile is two tiles back and long done).
//
// Numerics, layouts and the CUDA-core output layer are those of sxen_mlp_tc.cu; each group accumulates its weight gradients in
// its own TMEM columns (all 512 are in use) and the two sets meet when the CTA adds them to the batch total.  Reference semantics: Mlp::forward / Mlp::backward and
// run_chunk's loss (/root/reference/proj/src/mlp.cpp:137-202, src/trainer.cpp:26-48).
#include <algorithm>
#include <type_traits>

#include "sxen_mlp_tc_common.cuh"

using namespace sxen_host;
using namespace sxen_tc;
using namespace sxen_mlp_tc;

namespace {

constexpr int kGroups = 2;
constexpr int kGroupThreads = kTile * kSplit;   // epilogue threads of one group (one tile)
constexpr int kEpi2 = kGroups * kGroupThreads;
constexpr int kThreads2 = kEpi2;                // every warp is an epilogue warp; three lanes per group also issue its GEMMs

// shared-memory map (bytes)
constexpr uint32_t kHBytes = 2 * cm16_bytes(kTile, HC);          // one ring buffer: CM16(128, 72) hi, lo
constexpr uint32_t kX0Bytes = 2 * cm16_bytes(kTile, kX0CMax);    // CM16(128, 40) hi, lo
constexpr uint32_t kW0 = 0;                                      // CM16(64, 32) hi, lo
constexpr uint32_t kW1 = kW0 + 2 * cm16_bytes(HID, kInMax);      // CM16(64, 64) hi, lo
constexpr uint32_t kX0 = kW1 + 2 * cm16_bytes(HID, HID);         // one per group
constexpr uint32_t kRing = kX0 + kGroups * kX0Bytes;             // three buffers
constexpr uint32_t kDH2 = kRing + 3 * kHBytes;                   // CM16(128, 72): columns 0..63 dH2, 64..71 dY
constexpr uint32_t kBias = kDH2 + kHBytes;                       // b0[64], b1[64], b2[4] floats
constexpr uint32_t kW2f = kBias + (HID + HID + 4) * 4;           // output layer in fp32: W2f[3][64] (rows >= out_w zero)
constexpr uint32_t kPP = kW2f + 3 * HID * 4;                     // partial predictions pp[group][kSplit][128][4]
constexpr uint32_t kSmemBytes = kPP + kGroups * kSplit * kTile * 4 * 4;
static_assert(kSmemBytes <= 227 * 1024, "operand tiles of two tiles in flight must fit one SM");

// TMEM columns (fp32), + 256 * group: scratch accumulators (128 lanes) and the group's weight-gradient accumulators (M = 64)
constexpr uint32_t tS0 = 0;      // [128 x 64] layer-1 pre-activation, later d(input) (IN cols)
constexpr uint32_t tS1 = 64;     // [128 x 64] layer-2 pre-activation, later dH1
constexpr uint32_t tG0 = 128;    // [64 x 40]  dW0 | db0
constexpr uint32_t tG1 = 168;    // [64 x 72]  dW1 | db1
constexpr uint32_t tG2 = 240;    // [64 x 8]   dW2^T (read as 16 columns)
constexpr uint32_t kTmemGroup = 256;
constexpr uint32_t kTmemCols = 512;

template <int IN, bool TIMED>
__global__ void __launch_bounds__(kThreads2, 1) mlp_tc2_kernel(const __grid_constant__ TcArgs a) {
  static_assert(IN == 16 || IN == 32, "input widths 16 (L=8, F=2: the reference's default encoder) and 32 (L=16, F=2)");
  constexpr int X0C = IN + 8;
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar_chain[kGroups];  // the group's dependent-chain GEMM of the current phase has completed
  __shared__ uint64_t bar_p2[kGroups];     // ... the phase-2 chain GEMM (reads the shared dH2 buffer), once per tile
  __shared__ uint64_t bar_g2[kGroups];     // dW2 GEMM of the group's tile complete (its H2 buffer may become dH1)
  __shared__ uint64_t bar_g1[kGroups];     // dW1 GEMM complete (H1 and dH2 | dY of the tile are dead)
  __shared__ uint64_t bar_g0[kGroups];     // dW0 GEMM complete (X0 and dH1 of the tile are dead)
  __shared__ uint32_t tmem_base_slot;
  __shared__ double red_buf[kEpi2 / 32][4];
  __shared__ double acc_buf[4][kGroups * kTile];  // running {loss, db2[0..2]} per tile row and group (component-major: no bank conflicts)
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int g = tid / kGroupThreads;                     // group = which of the two tiles in flight
  const int lt = tid - g * kGroupThreads;                // thread index inside the group
  const int t = lt & (kTile - 1);                        // sample row inside the tile
  const int half = (lt >> 7) & (kSplit - 1);             // which slice of an epilogue's columns this thread handles
  const int lw = (lt >> 5);                              // warp index inside the group
  float* bias = reinterpret_cast<float*>(smem + kBias);
  const float* W0 = a.params;
  const float* b0 = W0 + HID * IN;
  const float* W1 = b0 + HID;
  const float* b1 = W1 + HID * HID;
  const float* W2 = b1 + HID;
  const float* b2 = W2 + a.out_w * HID;

  constexpr uint32_t loW0 = cm16_bytes(HID, IN), loW1 = cm16_bytes(HID, HID);
  constexpr uint32_t loX0 = cm16_bytes(kTile, X0C), loH = cm16_bytes(kTile, HC);
  float* w2f = reinterpret_cast<float*>(smem + kW2f);

  // ---- one-time setup: weights (hi/lo CM16 tiles, rows = output unit, cols = input unit), biases, ones columns
  {
    for (int e = tid; e < HID * IN / 8; e += kEpi2) {
      const int o = e / (IN / 8), ch = e % (IN / 8);
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = W0[o * IN + ch * 8 + q];
      store_chunk(smem + kW0, smem + kW0 + loW0, o, ch, IN, v);
    }
    for (int e = tid; e < HID * HID / 8; e += kEpi2) {
      const int o = e / (HID / 8), ch = e % (HID / 8);
      float v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = W1[o * HID + ch * 8 + q];
      store_chunk(smem + kW1, smem + kW1 + loW1, o, ch, HID, v);
    }
    for (int e = tid; e < 3 * HID; e += kEpi2) w2f[e] = (e / HID) < a.out_w ? W2[e] : 0.0f;
    if (tid < HID) {
      bias[tid] = b0[tid];
      bias[HID + tid] = b1[tid];
    }
    if (tid < 4) bias[2 * HID + tid] = tid < a.out_w ? b2[tid] : 0.0f;
    float ones[8] = {1.0f, 0, 0, 0, 0, 0, 0, 0};
    if (half == 0) store_chunk(smem + kX0 + g * kX0Bytes, smem + kX0 + g * kX0Bytes + loX0, t, IN / 8, X0C, ones);
    for (int b = g * kSplit + half; b < 3; b += kGroups * kSplit)  // the ring buffers keep a ones block whatever they hold
      store_chunk(smem + kRing + b * kHBytes, smem + kRing + b * kHBytes + loH, t, HID / 8, HC, ones);
  }
  if (tid == 0) {
    for (int k = 0; k < kGroups; ++k) {
      mbar_init(&bar_chain[k], 1);
      mbar_init(&bar_p2[k], 1);
      mbar_init(&bar_g2[k], 2);  // the weight-gradient GEMMs have two issuing lanes each
      mbar_init(&bar_g1[k], 2);
      mbar_init(&bar_g0[k], 2);
    }
  }
  if (warp == 0) tmem_alloc(&tmem_base_slot, kTmemCols);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base_slot;
  {
    // the weight-gradient accumulators start at zero (their GEMMs only ever accumulate): warp (quadrant, slice) of a group
    // clears its 32 lanes of a slice of the group's 128 accumulator columns
    const uint32_t base = tb + kTmemGroup * g + tG0 + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    for (int c = (128 / kSplit) * half; c < (128 / kSplit) * (half + 1); c += 16)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(base + c), "r"(0)
          : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }
  const int precise = a.precise;
  // Where the CTA's parameter gradients go.  148 CTAs adding to the same 6467 words serialise in L2 (the read-out at the end of
  // a 2^20-sample launch cost 4 % of the kernel, a mid-kernel flush 16 us): with `partials` every CTA owns a row, clears it here
  // and a reduction kernel adds the rows in a fixed order afterwards.
  double* const grad_out = a.partials != nullptr ? a.partials + blockIdx.x * a.partial_stride : a.mlp_grad;
  if (a.partials != nullptr)
    for (unsigned long long e = tid; e < a.partial_stride; e += kThreads2) grad_out[e] = 0.0;
  __syncthreads();
  const unsigned long long n_tiles = (a.n + kTile - 1) / kTile;
  const unsigned long long my_tiles = n_tiles > blockIdx.x ? (n_tiles - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const unsigned long long group_tiles[kGroups] = {(my_tiles + 1) / 2, my_tiles / 2};  // tile j of the CTA belongs to group j % 2
  constexpr uint32_t kStep = 256;                                  // K-major views: one UMMA_K = 16 step
  constexpr uint32_t kStepH = 2 * cm16_row_group_stride(HC);        // MN-major views: two 8-row groups
  const uint32_t sW0 = smem_u32(smem + kW0), sW1 = smem_u32(smem + kW1), sD = smem_u32(smem + kDH2);
  const uint32_t sX0b = smem_u32(smem + kX0), sRing = smem_u32(smem + kRing);

  {
    // =========================== epilogue warps: group g walks tiles g, g + 2, ... of the CTA ===========================
    // Register budget (128, no spills): the epilogues work on 16 accumulator columns at a time, keep the running loss /
    // output-bias sums in shared memory and count tiles in 32 bits.
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t tg = tb + kTmemGroup * g;  // this group's TMEM columns
    const uint32_t S0 = tg + lane_base + tS0, S1 = tg + lane_base + tS1;
    unsigned char* const X0 = smem + kX0 + g * kX0Bytes;
    unsigned char* const D = smem + kDH2;
    float* const pp = reinterpret_cast<float*>(smem + kPP) + g * kSplit * kTile * 4;
    double* const acc = &acc_buf[0][g * kTile + t];  // {loss, db2[0..2]} of this row's samples, stride kAcc (slice 0 threads only)
    constexpr int kAcc = kGroups * kTile;
    uint32_t phase = 0, phase_g0 = 0, phase_g2 = 0, phase_x = 0;
    int r1 = g;  // ring index of this tile's H1 buffer
    if (half == 0) acc[0] = acc[kAcc] = acc[2 * kAcc] = acc[3 * kAcc] = 0.0;

    // Hand-over of phase P: the group's threads have written the operand tiles and drained the TMEM scratch; one named
    // barrier later three elected lanes issue the phase's GEMMs.  K-major views step 256 B per UMMA_K = 16, MN-major views
    // two 8-row groups.  The first weight-gradient GEMMs of the group overwrite its accumulators.
    auto hand_over = [&](auto phase_tag, uint32_t sH1, uint32_t sH2) {
      constexpr int P = decltype(phase_tag)::value;
      fence_proxy_async();
      tc_fence_before();
      asm volatile("bar.sync %0, %1;" ::"r"(2 + 2 * g), "n"(kGroupThreads) : "memory");
      // GEMM issue from warp-uniform code (gemm_split_uniform): everything the descriptors are built from goes through
      // __shfl_sync so that the compiler keeps it in uniform registers; one lane's instructions reach the tensor core.
      const int lw_u = __shfl_sync(0xffffffffu, lw, 0);
      if (lw_u == 0 || (P >= 2 && lw_u >= 4)) {
        const bool leader = (lt & 31) == 0;
        const uint32_t g_u = static_cast<uint32_t>(__shfl_sync(0xffffffffu, g, 0));
        const uint32_t tg_u = __shfl_sync(0xffffffffu, tg, 0);
        const uint32_t sH1_u = __shfl_sync(0xffffffffu, sH1, 0), sH2_u = __shfl_sync(0xffffffffu, sH2, 0);
        const uint32_t sX0 = sX0b + g_u * kX0Bytes;
        tc_fence_after();
        if (lw_u == 0) {
          if constexpr (P == 0)  // layer 1: S0 = X0 * W0^T
            gemm_split_uniform(tg_u + tS0, make_idesc_bf16(128, HID, false, false), IN / 16, false, precise, desc16_k_major(sX0, X0C, 0),
                               loX0, kStep, desc16_k_major(sW0, IN, 0), loW0, kStep, leader);
          else if constexpr (P == 1)  // layer 2: S1 = H1 * W1^T
            gemm_split_uniform(tg_u + tS1, make_idesc_bf16(128, HID, false, false), HID / 16, false, precise,
                               desc16_k_major(sH1_u, HC, 0), loH, kStep, desc16_k_major(sW1, HID, 0), loW1, kStep, leader);
          else if constexpr (P == 2)  // S1 = dH2 * W1
            gemm_split_uniform(tg_u + tS1, make_idesc_bf16(128, HID, false, true), HID / 16, false, precise, desc16_k_major(sD, HC, 0),
                               loH, kStep, desc16_mn_major(sW1, HID, 0), loW1, 2 * cm16_row_group_stride(HID), leader);
          else  // S0[:, 0:IN] = dH1 * W0 (d loss / d encoding); dH1 sits in the tile's H2 buffer
            gemm_split_uniform(tg_u + tS0, make_idesc_bf16(128, IN, false, true), HID / 16, false, precise,
                               desc16_k_major(sH2_u, HC, 0), loH, kStep, desc16_mn_major(sW0, IN, 0), loW0,
                               2 * cm16_row_group_stride(IN), leader);
          if (leader) {
            if constexpr (P == 2) tc_commit(&bar_p2[g_u]);
            tc_commit(&bar_chain[g_u]);
          }
        } else {
          // Weight-gradient GEMMs, always accumulating (the accumulators start at zero).  K = the tile's 128 samples = eight
          // UMMA_K steps; each GEMM is issued four steps each by two warps so that no warp is held up much longer than the
          // chain GEMM takes anyway (the next hand-over waits for the group's slowest warp).
          // Reproducible mode: two lanes' MMAs into one accumulator reach the tensor core in an order that can change from
          // run to run, and fp32 sums depend on it -- there the first lane issues all eight steps and the second only commits.
          const bool one_issuer = a.grad_fixed != nullptr;
          const uint32_t second = static_cast<uint32_t>(lw_u & 1);  // which four K steps
          const int kHalfK = one_issuer ? (second ? 0 : kTile / 16) : kTile / 32;
          const uint32_t kofs = second * (kTile / 32) * kStepH;
          if constexpr (P == 2) {
            if (lw_u < 6) {  // G2 += H2^T * dY (dW2^T): on its own barrier, the tile's third epilogue overwrites H2 with dH1
              gemm_split_uniform(tg_u + tG2, make_idesc_bf16(64, 8, true, true), kHalfK, true, precise,
                                 desc16_mn_major(sH2_u + kofs, HC, 0), loH, kStepH, desc16_mn_major(sD + kofs, HC, 0, HID), loH, kStepH,
                                 leader);
              if (leader) tc_commit(&bar_g2[g_u]);
            } else {  // G1 += dH2^T * [H1 | 1]
              gemm_split_uniform(tg_u + tG1, make_idesc_bf16(64, HC, true, true), kHalfK, true, precise,
                                 desc16_mn_major(sD + kofs, HC, 0), loH, kStepH, desc16_mn_major(sH1_u + kofs, HC, 0), loH, kStepH, leader);
              if (leader) tc_commit(&bar_g1[g_u]);
            }
          } else if constexpr (P == 3) {
            if (lw_u >= 6) {  // G0 += dH1^T * [X0 | 1]
              const uint32_t xofs = second * (kTile / 32) * 2 * cm16_row_group_stride(X0C);
              gemm_split_uniform(tg_u + tG0, make_idesc_bf16(64, X0C, true, true), kHalfK, true, precise,
                                 desc16_mn_major(sH2_u + kofs, HC, 0), loH, kStepH, desc16_mn_major(sX0 + xofs, X0C, 0), loX0,
                                 2 * cm16_row_group_stride(X0C), leader);
              if (leader) tc_commit(&bar_g0[g_u]);
            }
          }
        }
      }
      __syncwarp();
    };
    const bool timed = TIMED && lt == 0;
    unsigned long long t_chain = 0, t_wgrad = 0, t_cross = 0;
    const long long t_begin = TIMED ? clock64() : 0;
    auto timed_wait = [&](uint64_t* bar_ptr, uint32_t parity, uint32_t id, unsigned long long& bucket) {
      if constexpr (TIMED) {
        const long long t0 = clock64();
        mbar_wait(bar_ptr, parity, id, a.progress);
        if (timed) bucket += static_cast<unsigned long long>(clock64() - t0);
      } else {
        mbar_wait(bar_ptr, parity, id, a.progress);
      }
    };
    auto wait_chain = [&]() {
      timed_wait(&bar_chain[g], phase, 0x300u + static_cast<uint32_t>(g), t_chain);
      phase ^= 1;
      tc_fence_after();
    };

    // feature staging: the group's threads cover the tile's 8-float chunks, 8 rows x IN/8 chunks per warp instruction
    constexpr int kXCh = IN / 8;
    constexpr int kXThreads = kGroupThreads < kTile * kXCh ? kGroupThreads : kTile * kXCh;
    constexpr int kXIt = (kTile * kXCh) / kXThreads;
    constexpr int kXRows = kXThreads / 8 / kXCh;
    const bool stages = lt < kXThreads;
    float xin[kXIt][8];
    const int xch = (lt >> 3) & (kXCh - 1);
    const int xrow = (lt & 7) + 8 * ((lt >> 3) / kXCh);
    const uint32_t tiles32 = static_cast<uint32_t>(n_tiles);  // the launcher keeps n below 2^38 samples
    const uint32_t tile_stride = static_cast<uint32_t>(kGroups) * gridDim.x;
    auto load_features = [&](uint32_t tile_index) {
#pragma unroll
      for (int it = 0; it < kXIt; ++it) {
        const int row = xrow + 8 * kXRows * it;
        const unsigned long long gs = static_cast<unsigned long long>(tile_index) * kTile + row;
        if (stages && tile_index < tiles32 && gs < a.n) {
          // read once: keep the features out of the little L1 this kernel leaves (28 KB; the targets are prefetched into it)
          const float4* p = reinterpret_cast<const float4*>(a.features + gs * IN + xch * 8);
          float4 x0, x1;
          asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x0.x), "=f"(x0.y), "=f"(x0.z), "=f"(x0.w) : "l"(p));
          asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x1.x), "=f"(x1.y), "=f"(x1.z), "=f"(x1.w) : "l"(p + 1));
          xin[it][0] = x0.x; xin[it][1] = x0.y; xin[it][2] = x0.z; xin[it][3] = x0.w;
          xin[it][4] = x1.x; xin[it][5] = x1.y; xin[it][6] = x1.z; xin[it][7] = x1.w;
        } else {
#pragma unroll
          for (int q = 0; q < 8; ++q) xin[it][q] = 0.0f;
        }
      }
    };
    // ---- the group's weight-gradient accumulators -> batch total (fp64 atomics or fixed point), then back to zero.
    // An M = 64 accumulator keeps row i in lane (i/16)*32 + i%16 (tools/tc_probe.py): lanes 0..15 of a warp hold rows
    // 16*(warp%4) .. +15.  Warp (quadrant, slice) owns its lanes of the slice's half of the 128 accumulator columns, reads
    // and clears exactly those, so no warp waits for another.  Run every kFlushTiles tiles of the group, and once more for both
    // groups together when the CTA is done: the accumulators are fp32 and a sum over T tiles is off by ~T * 2^-24 of its size
    // -- left to the end of a 2^24-sample launch (443 tiles per group) the parameter gradients were 2.5e-4 off the fp64
    // reference, against 1e-5 at 2^20 samples.  A flush is 6467 reds, one wavefront each on a data pipe that is busy already
    // (~22 k cycles, two tiles' worth), hence not more often.
    constexpr uint32_t kFlushTiles = 64;
    // `final_pass`: the CTA is done -- both groups' accumulators are summed, sixteen warps share the columns, nothing is cleared.
    auto flush_gradients = [&](bool final_pass) {
      constexpr size_t gW0 = 0, gb0 = gW0 + HID * IN, gW1 = gb0 + HID, gb1 = gW1 + HID * HID, gW2 = gb1 + HID;  // parameter layout
      constexpr int kG1 = tG1 - tG0, kG2 = tG2 - tG0;  // accumulator columns relative to tG0: dW0|db0, dW1|db1, dW2^T
      const int lane = lt & 31;
      const size_t row = 16 * (warp & 3) + lane;  // output unit (dW0, dW1) or hidden unit (dW2^T)
      // eight blocks of 16 columns: a group's warp takes four, in the final pass two -- which two rotates with the CTA so that
      // the CTAs, all finishing together, do not walk the same addresses in the same order
      const int first_blk = final_pass ? 2 * ((2 * g + half + static_cast<int>(blockIdx.x)) & 3) : 4 * half;
      const int n_blk = final_pass ? 2 : 4;
      for (int blk = first_blk; blk < first_blk + n_blk; ++blk) {
        const int c_base = 16 * blk;
        float v[16];
        {
          uint32_t r[16];
          tmem_ld16_nowait((final_pass ? tb : tg) + lane_base + tG0 + c_base, r);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) v[k] = __uint_as_float(r[k]);
          if (final_pass && group_tiles[1] > 0) {
            tmem_ld16_nowait(tb + kTmemGroup + lane_base + tG0 + c_base, r);
            tmem_ld_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) v[k] += __uint_as_float(r[k]);
          }
        }
        if (lane < 16) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = c_base + k;
            const double d = static_cast<double>(v[k]);
            if (c < kG1) {
              if (c < IN) add_total(grad_out, a.grad_fixed, gW0 + row * IN + c, d);
              else if (c == IN) add_total(grad_out, a.grad_fixed, gb0 + row, d);
            } else if (c < kG2) {
              if (c - kG1 < HID) add_total(grad_out, a.grad_fixed, gW1 + row * HID + (c - kG1), d);
              else if (c - kG1 == HID) add_total(grad_out, a.grad_fixed, gb1 + row, d);
            } else if (c - kG2 < a.out_w) {
              add_total(grad_out, a.grad_fixed, gW2 + static_cast<size_t>(c - kG2) * HID + row, d);
            }
          }
        }
        if (!final_pass)
          asm volatile(
              "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(tg + lane_base + tG0 + c_base),
              "r"(0)
              : "memory");
      }
      if (!final_pass) {
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();  // ordered before the next weight-gradient GEMMs by the hand-over barrier
      }
    };
    static_assert(kSplit == 2, "flush_gradients splits the accumulator columns in two halves");
    uint32_t tiles_done = 0;
    uint32_t next_flush = kFlushTiles / 2 + blockIdx.x % (kFlushTiles / 2);  // differs from CTA to CTA: the flushes do not coincide
    const uint32_t first_tile = blockIdx.x + static_cast<uint32_t>(g) * gridDim.x;
    load_features(first_tile);

    for (uint32_t tile = first_tile; tile < tiles32; tile += tile_stride) {
      const int r2 = r1 == 0 ? 2 : r1 - 1;  // (r1 + 2) % 3
      unsigned char* const H1 = smem + kRing + r1 * kHBytes;
      unsigned char* const H2 = smem + kRing + r2 * kHBytes;  // later dH1

      // ---- stage 0: features -> X0.  The group's previous tile's dW0 GEMM still reads X0 (and the ring buffer that is about
      // to become H1): wait for it first.
      if (tile != first_tile) {
        timed_wait(&bar_g0[g], phase_g0, 0x400u + static_cast<uint32_t>(g), t_wgrad);
        phase_g0 ^= 1;
        // every kFlushTiles tiles.  Every GEMM into the accumulators is done here: dW2 was waited for in the tile's third
        // epilogue, dW0 just above.
        if (tiles_done == next_flush) {
          next_flush += kFlushTiles;
          timed_wait(&bar_g1[g], (tiles_done - 1) & 1, 0x410u + static_cast<uint32_t>(g), t_wgrad);
          tc_fence_after();
          const long long tf0 = TIMED ? clock64() : 0;
          flush_gradients(false);
          if (timed) atomicAdd(a.timing + 6, static_cast<unsigned long long>(clock64() - tf0));
        }
      }
#pragma unroll
      for (int it = 0; it < kXIt; ++it)
        if (stages) store_chunk(X0, X0 + loX0, xrow + 8 * kXRows * it, xch, X0C, xin[it]);
      hand_over(std::integral_constant<int, 0>{}, smem_u32(H1), smem_u32(H2));

      // ---- layer 1 epilogue: S0 -> H1
      uint32_t m1 = 0, m2 = 0;  // ReLU masks of this thread's units (bit i = unit CPT*half + i active)
      wait_chain();
      uint32_t ra[CPT / 16][16];
#pragma unroll
      for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(S0 + CPT * half + 16 * q, ra[q]);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < CPT / 16; ++q) {
        const uint32_t(&r)[16] = ra[q];
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          float x = __uint_as_float(r[k]) + bias[CPT * half + 16 * q + k];
          x = x > 0.0f ? x : 0.0f;
          if (x > 0.0f) m1 |= 1u << (16 * q + k);
          v[k] = x;
        }
        store_chunk(H1, H1 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
        store_chunk(H1, H1 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
      }
      hand_over(std::integral_constant<int, 1>{}, smem_u32(H1), smem_u32(H2));

      // ---- layer 2 epilogue: S1 -> H2, then the output layer, the loss and its way back to dH2 on the CUDA cores
      const unsigned long long smp = static_cast<unsigned long long>(tile) * kTile + t;
      const bool valid = smp < a.n;
      // the row's targets are needed after the layer-2 conversion: loaded there, the L2 round trip cost 8 % of the kernel's
      // stall samples; held in registers across the conversion, they spill.  So: pull the line into L1 now, load later.
      if (valid) {
        const char* tp = static_cast<const char*>(a.targets) + smp * a.out_w * (a.target_f32 ? 4 : 8);
        asm volatile("prefetch.global.L1 [%0];" ::"l"(tp));
      }
      wait_chain();
      if (tile != first_tile || g > 0) {
        // H2 goes where the other group's tile keeps H1, dH2 | dY where it keeps its own: both are dead once that tile's
        // phase-2 GEMMs (chain: dH2 * W1, weight gradients: dW2, dW1) have completed
        // (three barriers: the three GEMMs come from different lanes, and a commit only covers its own lane's MMAs)
        timed_wait(&bar_g1[g ^ 1], phase_x, 0x500u + static_cast<uint32_t>(g), t_cross);
        timed_wait(&bar_g2[g ^ 1], phase_x, 0x520u + static_cast<uint32_t>(g), t_cross);
        timed_wait(&bar_p2[g ^ 1], phase_x, 0x510u + static_cast<uint32_t>(g), t_cross);
        phase_x ^= 1;
      }
      {
        float p0 = 0.0f, p1 = 0.0f, p2 = 0.0f;  // partial predictions over this thread's hidden units
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          uint32_t r[16];
          tmem_ld16_nowait(S1 + CPT * half + 16 * q, r);
          tmem_ld_wait();
          float v[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = CPT * half + 16 * q + k;
            float x = __uint_as_float(r[k]) + bias[HID + c];
            x = x > 0.0f ? x : 0.0f;
            if (x > 0.0f) m2 |= 1u << (16 * q + k);
            v[k] = x;
            p0 = __fmaf_rn(w2f[c], x, p0);
            p1 = __fmaf_rn(w2f[HID + c], x, p1);
            p2 = __fmaf_rn(w2f[2 * HID + c], x, p2);
          }
          store_chunk(H2, H2 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
          store_chunk(H2, H2 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
        }
        *reinterpret_cast<float4*>(pp + (half * kTile + t) * 4) = make_float4(p0, p1, p2, 0.0f);
      }
      double tgt[3] = {0.0, 0.0, 0.0};
      if (valid) {
#pragma unroll
        for (int o = 0; o < 3; ++o)
          if (o < a.out_w)
            tgt[o] = a.target_f32 ? static_cast<double>(static_cast<const float*>(a.targets)[smp * a.out_w + o])
                                  : static_cast<const double*>(a.targets)[smp * a.out_w + o];
      }
      // the slices of every row have posted their partials (one named barrier per group)
      asm volatile("bar.sync %0, %1;" ::"r"(1 + 2 * g), "n"(kGroupThreads) : "memory");
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
            if (valid) {
              // src/trainer.cpp:38-44: e = pred - target, loss += e*e, upstream = 2e/(B*out_w), all in double
              const double e = static_cast<double>(pr[o]) - tgt[o];
              const double up = a.upstream_scale * e;
              u[o] = static_cast<float>(up);
              if (half == 0) {
                acc[0] += e * e;
                acc[(1 + o) * kAcc] += up;
              }
            }
          }
        }
      }
      if (half == 0) store_chunk(D, D + loH, t, HID / 8, HC, u);  // dY: B operand of G2 = H2^T * dY
      {
        // dH2[c] = sum_o u[o] * W2[o][c], zero where layer 2's ReLU clamped (src/mlp.cpp:189-199)
#pragma unroll
        for (int q = 0; q < CPT / 16; ++q) {
          float v[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int c = CPT * half + 16 * q + k;
            const float gr = __fmaf_rn(u[2], w2f[2 * HID + c], __fmaf_rn(u[1], w2f[HID + c], __fmul_rn(u[0], w2f[c])));
            v[k] = ((m2 >> (16 * q + k)) & 1u) ? gr : 0.0f;
          }
          store_chunk(D, D + loH, t, (CPT / 8) * half + 2 * q, HC, v);
          store_chunk(D, D + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
        }
      }
      hand_over(std::integral_constant<int, 2>{}, smem_u32(H1), smem_u32(H2));

      // ---- backward epilogue of layer 2: S1 -> dH1 (masked by layer 1's ReLU), into the buffer H2 leaves
      wait_chain();
      timed_wait(&bar_g2[g], phase_g2, 0x600u + static_cast<uint32_t>(g), t_wgrad);  // dW2 has consumed H2
      phase_g2 ^= 1;
      uint32_t rb[CPT / 16][16];
#pragma unroll
      for (int q = 0; q < CPT / 16; ++q) tmem_ld16_nowait(S1 + CPT * half + 16 * q, rb[q]);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < CPT / 16; ++q) {
        const uint32_t(&r)[16] = rb[q];
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = ((m1 >> (16 * q + k)) & 1u) ? __uint_as_float(r[k]) : 0.0f;
        store_chunk(H2, H2 + loH, t, (CPT / 8) * half + 2 * q, HC, v);
        store_chunk(H2, H2 + loH, t, (CPT / 8) * half + 2 * q + 1, HC, v + 8);
      }
      hand_over(std::integral_constant<int, 3>{}, smem_u32(H1), smem_u32(H2));

      // ---- backward epilogue of layer 1: S0[:, 0:IN] -> d loss / d encoding, straight to global memory
      load_features(tile + tile_stride);  // in flight under the last phase
      wait_chain();
      if (half < IN / 16) {
        // The thread holds 16 consecutive floats (four 16-byte chunks) of its row; written as they are, one store instruction
        // would touch 32 rows = 32 cache lines.  A 4x4 transpose of chunks inside each quad of lanes (two butterfly rounds)
        // makes lane p of a quad hold chunk p of the quad's four rows, so one instruction writes 64 contiguous bytes of 8 rows.
        uint32_t r[16];
        tmem_ld16_nowait(S0 + 16 * half, r);
        tmem_ld_wait();
        const int lane = lt & 31, p = lane & 3;
#pragma unroll
        for (int c = 0; c < 2; ++c) {  // round 1, partner lane ^ 2: chunks {c, c + 2} -- keep the one whose bit 1 equals p's
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t lo = r[4 * c + k], hi = r[4 * (c + 2) + k];
            const uint32_t send = (p & 2) ? lo : hi;
            const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 2);
            r[4 * c + k] = (p & 2) ? got : lo;
            r[4 * (c + 2) + k] = (p & 2) ? hi : got;
          }
        }
#pragma unroll
        for (int c = 0; c < 4; c += 2) {  // round 2, partner lane ^ 1: chunks {c, c + 1}
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t lo = r[4 * c + k], hi = r[4 * (c + 1) + k];
            const uint32_t send = (p & 1) ? lo : hi;
            const uint32_t got = __shfl_xor_sync(0xffffffffu, send, 1);
            r[4 * c + k] = (p & 1) ? got : lo;
            r[4 * (c + 1) + k] = (p & 1) ? hi : got;
          }
        }
        // now r[4j .. 4j+3] = chunk p of row (t - p + j)
        const unsigned long long row0 = static_cast<unsigned long long>(tile) * kTile + (t - p);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (row0 + j < a.n)
            __stcs(reinterpret_cast<float4*>(a.input_grad + (row0 + j) * IN + 16 * half + 4 * p),
                   make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                               __uint_as_float(r[4 * j + 3])));
        }
      }
      tc_fence_before();
      r1 = r2;
      ++tiles_done;
    }

    if (timed && g == 0) {
      atomicAdd(a.timing + 0, static_cast<unsigned long long>(clock64() - t_begin));
      atomicAdd(a.timing + 1, t_chain);
      atomicAdd(a.timing + 2, t_wgrad);
      atomicAdd(a.timing + 3, t_cross);
    }
    // ---- the last tiles' weight gradients
    if (group_tiles[g] > 0) {  // the group's last tile: dW1 (its barrier's phases were the other group's to follow) and dW0
      mbar_wait(&bar_g1[g], static_cast<uint32_t>((group_tiles[g] - 1) & 1), 0x700u + static_cast<uint32_t>(g), a.progress);
      mbar_wait(&bar_g0[g], phase_g0, 0x710u + static_cast<uint32_t>(g), a.progress);
    }
    tc_fence_before();
    __syncthreads();  // both groups' accumulators are final (a group without tiles still holds the zeros it started with)
    tc_fence_after();
    {
      const long long tf0 = TIMED ? clock64() : 0;
      if (my_tiles > 0) flush_gradients(true);
      if (timed && g == 0) atomicAdd(a.timing + 7, static_cast<unsigned long long>(clock64() - tf0));
    }
    const int lane = tid & 31;
    // loss and output-bias gradient: per-thread fp64 partials -> warp shuffle -> one atomic per CTA (below)
    double part[4] = {0.0, 0.0, 0.0, 0.0};
    if (half == 0)
      for (int k = 0; k < 4; ++k) part[k] = acc[k * kAcc];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      for (int o = 16; o > 0; o >>= 1) part[k] += __shfl_down_sync(0xffffffffu, part[k], o);
    if (lane == 0)
      for (int k = 0; k < 4; ++k) red_buf[warp][k] = part[k];
  }

  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    double tot[4] = {0, 0, 0, 0};
    for (int w = 0; w < kEpi2 / 32; ++w)
      for (int k = 0; k < 4; ++k) tot[k] += red_buf[w][k];
    const size_t gb2 = HID * IN + HID + HID * HID + HID + a.out_w * HID;
    const size_t n_params = gb2 + a.out_w;
    // reproducible mode: the CTAs' loss partials (not bounded like a gradient, so not fixed point) go to one slot per CTA
    // behind the parameter words; the host side adds them to *loss_sum in CTA order
    if (a.grad_fixed != nullptr) reinterpret_cast<double*>(a.grad_fixed + n_params)[blockIdx.x] = tot[0];
    else atomicAdd(a.loss_sum, tot[0]);
    for (int o = 0; o < a.out_w && o < 3; ++o) add_total(grad_out, a.grad_fixed, gb2 + o, tot[1 + o]);
  }
  if (warp == 0) tmem_dealloc(tb, kTmemCols);
}

// mlp_grad[p] += sum over the CTAs' rows, in a fixed order: 32 strided partial sums per parameter (at most five loads per thread,
// all in flight at once -- with eight the kernel was a chain of 19 dependent L2 round trips, 12 us), then those in sequence.
__global__ void __launch_bounds__(1024) reduce_partials_kernel(double* __restrict__ mlp_grad, const double* __restrict__ partials,
                                                               unsigned rows, unsigned long long stride, unsigned n_params) {
  __shared__ double part[32][33];
  const unsigned px = threadIdx.x & 31, sy = threadIdx.x >> 5;
  const unsigned p = blockIdx.x * 32 + px;
  double v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const unsigned r = sy + 32 * k;
    v[k] = (p < n_params && r < rows) ? partials[r * stride + p] : 0.0;
  }
  double sum = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) sum += v[k];
  for (unsigned r = sy + 256; r < rows; r += 32)  // more than 256 CTAs: not on any current part
    if (p < n_params) sum += partials[r * stride + p];
  part[sy][px] = sum;
  __syncthreads();
  if (sy == 0 && p < n_params) {
    double total = part[0][px];
#pragma unroll
    for (int k = 1; k < 32; ++k) total += part[k][px];
    mlp_grad[p] += total;
  }
}

}  // namespace

// Launch (sxen_mlp_tc.cu: sxen_mlp_tc_run picks between this kernel and the one-tile-in-flight kernel).
sxen_status sxen_mlp_tc2_train_launch(const sxen_mlp_tc::TcArgs& a, int in_w, cudaStream_t stream, int* used_ctas) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned long long tiles = (a.n + kTile - 1) / kTile;
  if (tiles >> 32) return fail(SXEN_INVALID_ARGUMENT, "mlp (tensor cores): %llu samples in one launch (limit 2^39)", a.n);
  const unsigned grid = static_cast<unsigned>(std::min<unsigned long long>(tiles, static_cast<unsigned long long>(sms)));
  auto launch = [&](auto kernel) -> sxen_status {
    SXEN_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kSmemBytes)));
    kernel<<<grid, kThreads2, kSmemBytes, stream>>>(a);
    return SXEN_OK;
  };
  const bool timed = a.timing != nullptr;
  const sxen_status st = in_w == 32 ? (timed ? launch(mlp_tc2_kernel<32, true>) : launch(mlp_tc2_kernel<32, false>))
                                    : (timed ? launch(mlp_tc2_kernel<16, true>) : launch(mlp_tc2_kernel<16, false>));
  if (st != SXEN_OK) return st;
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (a.partials != nullptr) {
    const unsigned n_params = static_cast<unsigned>(HID * in_w + HID + HID * HID + HID + a.out_w * HID + a.out_w);
    reduce_partials_kernel<<<(n_params + 31) / 32, 1024, 0, stream>>>(a.mlp_grad, a.partials, grid, a.partial_stride, n_params);
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  if (used_ctas) *used_ctas = static_cast<int>(grid);
  return SXEN_OK;
}
