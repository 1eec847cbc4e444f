// sxen_encode.cuh -- the encode / encode_backward kernels (sm_100a).
//
// One thread owns one sample and LPT consecutive levels.  For each (sample, level) it walks the simplex once
// (sxen_device.cuh: simplex_lookup; grid_lookup for the grid backend's 2^ND corners) and then
//   forward  : gathers the vertex rows (read-only path, one vector load per row) and blends them,
//   backward : scatter-adds weight * upstream into the gradient rows with one vector `red.global.add` per row -- one
//              red.v4 for the two rows of an axis-0 pair; coarse levels go to replicated dense accumulators that
//              coarse_fold_kernel adds into the hashed rows before the call returns,
//   both     : does the two off the same lattice walk (the fused fwd+bwd kernel).
// Memory-system-bound integer/gather work (L2 tag lookups): no tensor cores here by design.
// Reference semantics: HashEncoder::encode / encode_backward, /root/reference/proj/src/encoding.cpp:295-335.
#pragma once

#include "sxen_adam.cuh"
#include "sxen_device.cuh"

namespace sxen_dev {

enum : int { kModeFwd = 1, kModeBwd = 2, kModeBoth = 3 };

struct EncodeArgs {
  const void* x;                 // N x ND coordinates, f64 or f32
  const float* upstream;         // N x row_width (backward / both)
  float* out;                    // N x row_width (forward / both)
  const float* tables;           // encoder level 0; level l at + l*level_stride
  float* grads;                  // accumulator level 0, same layout
  unsigned long long* status;    // [0] first rejected sample (atomicMin), [1] clamped cells (LookupCounters::out_of_bounds)
  unsigned long long n_samples;
  unsigned long long level_stride;  // T*F floats
  uint32_t mask;                 // T-1
  int32_t level0;                // first encoder level of this launch
  int32_t n_levels;              // levels in this launch (<= kMaxLaunchLevels)
  int32_t row_width;             // L*F
  int32_t features;              // F (used by the dynamic-F kernels)
  int32_t groups;                // ceil(n_levels / LPT)
  int32_t groups_shift;          // log2(groups) when a power of two, else -1
  int32_t coord_f32;             // coordinate element type
  int32_t level_major;           // 1: blockIdx.y = level group
  int32_t span_groups;           // sample-major: level groups one blockIdx.y slice covers (a power of two when groups_shift
                                 // >= 0, then groups_shift = log2(span_groups)); == groups unless the launch is chunked
  int32_t vec;                   // proven float alignment of every thread's out/upstream chunk: 4, 2 or 1
  uint32_t agg_mask;             // bit l: warp-aggregate the backward atomics of local level l
  int32_t merge_pairs;           // F == 2: one red.v4 for two chain vertices in the same 16-byte slot
  int32_t cache_hints;           // F == 2: gather L2 policy + 4 * red L2 policy (0 none, 1 evict_last, 2 evict_first, 3 evict_unchanged)
  double skew;                   // F_n
  long long* fixed;              // reproducible mode: 64-bit fixed-point accumulator, same layout as grads (nullptr = off)
  const double* upstream64;      // reproducible mode: upstream as the reference's doubles (nullptr: widen `upstream`)
  float* coarse;                 // replicated dense accumulators of the coarse levels (nullptr = none)
  LevelGeom geom;
  CoarseGeom cg;                 // geometry of `coarse`
};

// Sum v[] over the lanes of `m` that hold the same key, leaving the total in the group's lowest lane.
// Returns true on the lane that must issue the atomic.
template <int F>
__device__ __forceinline__ bool warp_merge_rows(unsigned m, unsigned long long key, float (&v)[F]) {
  const unsigned peers = __match_any_sync(m, key);
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(peers) - 1;
  unsigned todo = (lane == leader) ? (peers & ~(1u << lane)) : 0u;
  while (__any_sync(m, todo != 0u)) {
    const int src = todo ? (__ffs(todo) - 1) : lane;
#pragma unroll
    for (int f = 0; f < F; ++f) {
      const float t = __shfl_sync(m, v[f], src);
      if (todo) v[f] += t;
    }
    todo &= todo - 1u;
  }
  return lane == leader;
}

template <int ND>
__device__ __forceinline__ bool load_coords(const EncodeArgs& a, unsigned long long s, double (&x)[ND]) {
  if (a.coord_f32) {
    const float* xp = static_cast<const float*>(a.x) + s * ND;
#pragma unroll
    for (int i = 0; i < ND; ++i) x[i] = static_cast<double>(__ldg(xp + i));
  } else {
    const double* xp = static_cast<const double*>(a.x) + s * ND;
#pragma unroll
    for (int i = 0; i < ND; ++i) x[i] = __ldg(xp + i);
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    ok = ok && (x[i] >= 0.0 && x[i] <= 1.0);           // check_input, src/encoding.cpp:189 (NaN fails both)
    x[i] = (kOneBelow < x[i]) ? kOneBelow : x[i];      // std::min(x, one_below), src/encoding.cpp:204
  }
  return ok;
}

// REPRO (backward / both): besides the fp32 atomics every contribution is ALSO added as 64-bit fixed point (units of
// 2^-52) with red.global.add.u64 -- integer addition is associative, so the sums do not depend on the order the atomics
// land in and a training run is bit-reproducible, like the reference's fixed worker-order merge (src/trainer.cpp:125-128,
// tests/test_neural.cpp:370-408).  The product w * upstream is taken in fp64 as the reference does (src/encoding.cpp:116);
// the fp32 accumulator keeps carrying the touched marker, the NaN / range check and an approximate value.
constexpr double kFixedScale = 0x1p52, kFixedUnit = 0x1p-52;
__device__ __forceinline__ void red_add_fixed(long long* p, double v) {
  const long long q = __double2ll_rn(__dmul_rn(v, kFixedScale));
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(q) : "memory");
}

template <int ND, int F, int LPT, int MODE, bool EXACT, bool GRID = false, bool REPRO = false>
__global__ void __launch_bounds__((LPT >= 4 || GRID) ? 256 : 512)
encode_kernel(const __grid_constant__ EncodeArgs a) {
  constexpr int V = GRID ? (1 << ND) : (ND + 1);  // vertices per (sample, level): gather_grid / gather_simplex
  constexpr bool kFwd = (MODE & kModeFwd) != 0;
  constexpr bool kBwd = (MODE & kModeBwd) != 0;
  constexpr int K = LPT * F;

  __shared__ double s_scale[kMaxLaunchLevels];
  __shared__ int s_res[kMaxLaunchLevels];
  __shared__ int s_cshift[kMaxLaunchLevels];
  if (threadIdx.x < kMaxLaunchLevels) {
    s_scale[threadIdx.x] = a.geom.scale[threadIdx.x];
    s_res[threadIdx.x] = a.geom.res[threadIdx.x];
    s_cshift[threadIdx.x] = (kBwd && a.coarse != nullptr) ? a.cg.shift[threadIdx.x] : -1;
  }
  __syncthreads();

  unsigned long long s;
  int g;
  if (a.level_major) {
    g = blockIdx.y;
    s = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  } else {
    const unsigned long long gid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (a.groups_shift >= 0) {
      // chunked launch: blockIdx.y walks contiguous ranges of span_groups level groups, sample-major inside a range, so the
      // rows of one range of levels (tables + accumulator) are what L2 holds while that range is in flight
      s = gid >> a.groups_shift;
      g = static_cast<int>(gid & static_cast<unsigned long long>(a.span_groups - 1)) + static_cast<int>(blockIdx.y) * a.span_groups;
    } else {
      s = gid / static_cast<unsigned long long>(a.groups);
      g = static_cast<int>(gid - s * static_cast<unsigned long long>(a.groups));
    }
  }
  const bool in_range = s < a.n_samples && g < a.groups;

  double x[ND];
  bool ok = false;
  if (in_range) ok = load_coords<ND>(a, s, x);
  const unsigned live = __ballot_sync(0xffffffffu, ok);
  if (!in_range) return;

  const int l_begin = g * LPT;
  const bool full = l_begin + LPT <= a.n_levels;
  const size_t chunk = static_cast<size_t>(s) * a.row_width + static_cast<size_t>(a.level0 + l_begin) * F;

  if (!ok) {
    // The reference throws std::invalid_argument before touching anything (src/encoding.cpp:183-194).  Here the
    // sample is reported through the status word, its features are written as zeros, and it adds no gradient.
    atomicMin(a.status, s);
    if constexpr (kFwd) {
      for (int j = 0; j < LPT; ++j)
        if (l_begin + j < a.n_levels)
          for (int f = 0; f < F; ++f) a.out[chunk + j * F + f] = 0.0f;
    }
    return;
  }

  float upv[K];
  float outv[K];
  double upd[REPRO ? K : 1];
  const int gather_kind = a.cache_hints & 3, red_kind = (a.cache_hints >> 2) & 3;
  const uint64_t gather_pol = l2_policy(gather_kind), red_pol = l2_policy(red_kind);
  if constexpr (kBwd) {
    if (full) {
      load_stream<K>(a.upstream + chunk, upv, a.vec);
    } else {
#pragma unroll
      for (int q = 0; q < K; ++q) upv[q] = (l_begin + q / F < a.n_levels) ? __ldcs(a.upstream + chunk + q) : 0.0f;
    }
    if constexpr (REPRO) {
#pragma unroll
      for (int q = 0; q < K; ++q)
        upd[q] = (a.upstream64 != nullptr && l_begin + q / F < a.n_levels) ? __ldcs(a.upstream64 + chunk + q)
                                                                           : static_cast<double>(upv[q]);
    }
  }

#pragma unroll
  for (int j = 0; j < LPT; ++j) {
    const int l = l_begin + j;
    const bool has = l < a.n_levels;
    unsigned aggm = 0u;
    if constexpr (kBwd) {
      if (a.agg_mask != 0u) aggm = __ballot_sync(live, has && ((a.agg_mask >> l) & 1u));
    }
    if (has) {
      uint32_t idx[V];
      uint32_t dense[V];
      double w[V];
      bool oob;
      if constexpr (GRID) oob = grid_lookup<ND, kBwd>(x, s_scale[l], s_res[l], a.mask, idx, w, dense);
      else oob = simplex_lookup<ND, kBwd>(x, s_scale[l], a.skew, s_res[l], a.mask, idx, w, dense);
      // LookupCounters::out_of_bounds: the reference bumps it in encode AND in encode_backward (src/encoding.cpp:222,241),
      // so the fused walk counts for both
      if (oob) atomicAdd(a.status + 1, (kFwd && kBwd) ? 2ULL : 1ULL);
      const size_t level_off = static_cast<size_t>(a.level0 + l) * a.level_stride;

      if constexpr (kFwd) {
        const float* __restrict__ tab = a.tables + level_off;
        float e[V][F];
        if constexpr (F == 2) {
          // (a 128-bit load for the two rows of an axis-0 pair, or a dense L1-resident shadow of the coarse levels, buys
          // nothing here: the gathers are bound by sector requests on the L1 miss path, and the pair's second row
          // already hits the sector its first row fetched -- profiles/r1_coarse_shadow_tables_negative.log)
          if (gather_kind) {
#pragma unroll
            for (int k = 0; k < V; ++k) load_row2_policy(tab + static_cast<size_t>(idx[k]) * F, e[k], gather_pol);
          } else {
#pragma unroll
            for (int k = 0; k < V; ++k) load_row<F>(tab + static_cast<size_t>(idx[k]) * F, e[k]);
          }
        } else {
#pragma unroll
          for (int k = 0; k < V; ++k) load_row<F>(tab + static_cast<size_t>(idx[k]) * F, e[k]);
        }
        if constexpr (EXACT) {
          // src/encoding.cpp:305-313: acc starts at 0.0, acc += w_i * entry in chain order, all in double.
          double acc[F];
#pragma unroll
          for (int f = 0; f < F; ++f) acc[f] = 0.0;
#pragma unroll
          for (int k = 0; k < V; ++k) {
#pragma unroll
            for (int f = 0; f < F; ++f) acc[f] = __dadd_rn(acc[f], __dmul_rn(w[k], static_cast<double>(e[k][f])));
          }
#pragma unroll
          for (int f = 0; f < F; ++f) outv[j * F + f] = static_cast<float>(acc[f]);
        } else {
          float acc[F];
#pragma unroll
          for (int f = 0; f < F; ++f) acc[f] = 0.0f;
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const float wk = static_cast<float>(w[k]);
#pragma unroll
            for (int f = 0; f < F; ++f) acc[f] = __fmaf_rn(wk, e[k][f], acc[f]);
          }
#pragma unroll
          for (int f = 0; f < F; ++f) outv[j * F + f] = acc[f];
        }
      }

      if constexpr (kBwd) {
        float* gl = a.grads + level_off;
        const bool agg = (aggm >> (threadIdx.x & 31)) & 1u;
        // EncoderGradient::add, src/encoding.cpp:110-120: dst[f] += scale * upstream[f]
        float v[V][F];
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const float wk = static_cast<float>(w[k]);
#pragma unroll
          for (int f = 0; f < F; ++f) v[k][f] = canon(__fmul_rn(wk, upv[j * F + f]));
        }
        // Coarse level: a few thousand hot rows take every sample's atomics and the L2 atomic unit serialises per
        // address (profiles/r1_per_level_n*.log: level 0 costs 4-12x a fine level).  Such levels accumulate into one of
        // 2^shift dense replicas picked by the sample index (rows = dense lattice positions instead of hashed rows);
        // coarse_fold_kernel adds the replicas into the hashed rows right after this launch.
        if constexpr (REPRO) {
          // exact sums next to the fp32 ones, straight into the hashed rows (before idx[] is redirected to a replica)
          long long* fl = a.fixed + level_off;
#pragma unroll
          for (int k = 0; k < V; ++k) {
#pragma unroll
            for (int f = 0; f < F; ++f) red_add_fixed(fl + static_cast<size_t>(idx[k]) * F + f, __dmul_rn(w[k], upd[j * F + f]));
          }
        }
        const int cshift = s_cshift[l];
        if (cshift >= 0) {
          const uint32_t rep = static_cast<uint32_t>(s) & ((1u << cshift) - 1u);
          gl = a.coarse + a.cg.offset[l] + static_cast<size_t>(rep) * a.cg.verts[l] * F;
#pragma unroll
          for (int k = 0; k < V; ++k) idx[k] = dense[k];  // (a step along axis 0 is +1 here too: the pair merge applies)
        }
        bool skip = false;
#pragma unroll
        for (int k = 0; k < V; ++k) {
          if (skip) {
            skip = false;
            continue;
          }
          if constexpr (F == 2) {
            // The hash multiplies axis 0 by 1 (include/sxen/hashing.hpp:16), so the chain step along axis 0 from an even
            // coordinate lands on the neighbouring row: rows idx and idx^1 share one 16-byte slot and take ONE
            // red.v4 instead of two red.v2 (half the L2 atomic requests for that pair).  Grid backend: corners m and
            // m+1 (m even) differ along axis 0 only, the same pair.
            if (k + 1 < V && a.merge_pairs && !agg) {
              if ((idx[k] ^ idx[k + 1 < V ? k + 1 : k]) == 1u) {
                const int kn = k + 1 < V ? k + 1 : k;
                const bool low = (idx[k] & 1u) == 0u;
                float* p = gl + static_cast<size_t>(idx[k] & ~1u) * 2;
                if (red_kind)
                  red_add4_policy(p, low ? v[k][0] : v[kn][0], low ? v[k][1] : v[kn][1], low ? v[kn][0] : v[k][0],
                                  low ? v[kn][1] : v[k][1], red_pol);
                else
                  red_add4(p, low ? v[k][0] : v[kn][0], low ? v[k][1] : v[kn][1], low ? v[kn][0] : v[k][0],
                           low ? v[kn][1] : v[k][1]);
                skip = true;
                continue;
              }
            }
          }
          bool issue = true;
          if (agg) {
            const unsigned long long key = (static_cast<unsigned long long>(l) << 32) | idx[k];
            issue = warp_merge_rows<F>(aggm, key, v[k]);
          }
          if constexpr (F == 2) {
            if (issue && red_kind) {
              red_add2_policy(gl + static_cast<size_t>(idx[k]) * F, v[k][0], v[k][1], red_pol);
              issue = false;
            }
          }
          if (issue) red_row<F>(gl + static_cast<size_t>(idx[k]) * F, v[k]);
        }
      }
    }
  }

  if constexpr (kFwd) {
    if (full) {
      store_stream<K>(a.out + chunk, outv, a.vec);
    } else {
#pragma unroll
      for (int q = 0; q < K; ++q)
        if (l_begin + q / F < a.n_levels) __stcs(a.out + chunk + q, outv[q]);
    }
  }
}

// Any F in [1, 64] and both backends: one thread per (sample, level), features walked one at a time.
// Always the exact fp64 chain-order blend.  The slow-but-general path.
template <int ND, int MODE, bool GRID>
__global__ void __launch_bounds__(256) encode_generic_kernel(const __grid_constant__ EncodeArgs a) {
  constexpr bool kFwd = (MODE & kModeFwd) != 0;
  constexpr bool kBwd = (MODE & kModeBwd) != 0;
  const unsigned long long gid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned long long s = gid / static_cast<unsigned long long>(a.n_levels);
  const int l = static_cast<int>(gid - s * static_cast<unsigned long long>(a.n_levels));
  if (s >= a.n_samples) return;
  double x[ND];
  const bool ok = load_coords<ND>(a, s, x);
  const int F = a.features;
  const size_t chunk = static_cast<size_t>(s) * a.row_width + static_cast<size_t>(a.level0 + l) * F;
  if (!ok) {
    atomicMin(a.status, s);
    if constexpr (kFwd)
      for (int f = 0; f < F; ++f) a.out[chunk + f] = 0.0f;
    return;
  }
  const size_t level_off = static_cast<size_t>(a.level0 + l) * a.level_stride;
  const float* __restrict__ tab = a.tables + level_off;
  float* __restrict__ gl = a.grads + level_off;

  if constexpr (GRID) {
    GridCell<ND> cell;
    if (grid_prepare<ND>(x, a.geom.scale[l], a.geom.res[l], cell)) atomicAdd(a.status + 1, 1ULL);
    for (int f = 0; f < F; ++f) {
      double acc = 0.0;
      float up = 0.0f;
      double upd = 0.0;
      if constexpr (kBwd) {
        up = __ldg(a.upstream + chunk + f);
        upd = a.upstream64 != nullptr ? __ldg(a.upstream64 + chunk + f) : static_cast<double>(up);
      }
#pragma unroll 1
      for (int m = 0; m < (1 << ND); ++m) {
        uint32_t idx;
        double w;
        grid_corner<ND>(cell, m, a.mask, idx, w);
        if constexpr (kFwd)
          acc = __dadd_rn(acc, __dmul_rn(w, static_cast<double>(__ldg(tab + static_cast<size_t>(idx) * F + f))));
        if constexpr (kBwd) {
          red_add(gl + static_cast<size_t>(idx) * F + f, canon(__fmul_rn(static_cast<float>(w), up)));
          if (a.fixed != nullptr) red_add_fixed(a.fixed + level_off + static_cast<size_t>(idx) * F + f, __dmul_rn(w, upd));
        }
      }
      if constexpr (kFwd) a.out[chunk + f] = static_cast<float>(acc);
    }
  } else {
    uint32_t idx[ND + 1];
    double w[ND + 1];
    if (simplex_lookup<ND>(x, a.geom.scale[l], a.skew, a.geom.res[l], a.mask, idx, w)) atomicAdd(a.status + 1, 1ULL);
    for (int f = 0; f < F; ++f) {
      if constexpr (kFwd) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k <= ND; ++k)
          acc = __dadd_rn(acc, __dmul_rn(w[k], static_cast<double>(__ldg(tab + static_cast<size_t>(idx[k]) * F + f))));
        a.out[chunk + f] = static_cast<float>(acc);
      }
      if constexpr (kBwd) {
        const float up = __ldg(a.upstream + chunk + f);
#pragma unroll
        for (int k = 0; k <= ND; ++k)
          red_add(gl + static_cast<size_t>(idx[k]) * F + f, canon(__fmul_rn(static_cast<float>(w[k]), up)));
        if (a.fixed != nullptr) {
          const double upd = a.upstream64 != nullptr ? __ldg(a.upstream64 + chunk + f) : static_cast<double>(up);
#pragma unroll
          for (int k = 0; k <= ND; ++k)
            red_add_fixed(a.fixed + level_off + static_cast<size_t>(idx[k]) * F + f, __dmul_rn(w[k], upd));
        }
      }
    }
  }
}

// Parity probe: the vertex chain itself.  idx: N x total_levels x V, w likewise (doubles).
template <int ND, bool GRID>
__global__ void __launch_bounds__(256)
encode_debug_kernel(const __grid_constant__ EncodeArgs a, uint32_t* __restrict__ idx_out, double* __restrict__ w_out,
                    int total_levels) {
  constexpr int V = GRID ? (1 << ND) : (ND + 1);
  const unsigned long long gid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned long long s = gid / static_cast<unsigned long long>(a.n_levels);
  const int l = static_cast<int>(gid - s * static_cast<unsigned long long>(a.n_levels));
  if (s >= a.n_samples) return;
  double x[ND];
  const bool ok = load_coords<ND>(a, s, x);
  const size_t o = (static_cast<size_t>(s) * total_levels + (a.level0 + l)) * V;
  if (!ok) {
    atomicMin(a.status, s);
    for (int k = 0; k < V; ++k) {
      idx_out[o + k] = 0u;
      w_out[o + k] = 0.0;
    }
    return;
  }
  if constexpr (GRID) {
    GridCell<ND> cell;
    grid_prepare<ND>(x, a.geom.scale[l], a.geom.res[l], cell);
#pragma unroll 1
    for (int m = 0; m < V; ++m) {
      uint32_t idx;
      double w;
      grid_corner<ND>(cell, m, a.mask, idx, w);
      idx_out[o + m] = idx;
      w_out[o + m] = w;
    }
  } else {
    uint32_t idx[V];
    double w[V];
    simplex_lookup<ND>(x, a.geom.scale[l], a.skew, a.geom.res[l], a.mask, idx, w);
#pragma unroll
    for (int k = 0; k < V; ++k) {
      idx_out[o + k] = idx[k];
      w_out[o + k] = w[k];
    }
  }
}

// SparseAdamState::step (src/optimizer.cpp:54-84) driven by the BATCH instead of by a scan of the accumulator: one thread
// per (sample, level) repeats the lattice walk of the backward that filled the accumulator and claims each of its rows
// with a 64-bit atomic exchange against the untouched pattern; the first claimant gets the row's gradient and applies
// the update, later ones see -0.0f and move on.  Visits exactly the touched rows, each once, in O(batch * L * V) work --
// the scan reads all L*T rows, 36 of a 2048-sample training step's 93 us (profiles/r1s3_small_batch_launches.csv).
// Only valid when every touched row comes from THIS batch (the single-GPU trainer's step), F == 2.
template <int ND, bool GRID>
__global__ void __launch_bounds__(256)
sparse_adam_walk_kernel(const __grid_constant__ EncodeArgs a, const __grid_constant__ AdamWalkArgs o) {
  constexpr int V = GRID ? (1 << ND) : (ND + 1);
  if (o.gate != nullptr && *o.gate != kAdamNoBad) return;
  const unsigned long long gid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned long long s = gid / static_cast<unsigned long long>(a.n_levels);
  const int l = static_cast<int>(gid - s * static_cast<unsigned long long>(a.n_levels));
  if (s >= a.n_samples) return;
  double x[ND];
  if (!load_coords<ND>(a, s, x)) return;  // a rejected sample added no gradient (encode_kernel)
  const size_t level_row0 = static_cast<size_t>(a.level0 + l) * (static_cast<size_t>(a.mask) + 1u);
  constexpr unsigned long long kUntouchedRow = (static_cast<unsigned long long>(kUntouchedBits) << 32) | kUntouchedBits;
  auto claim_and_update = [&](uint32_t row) {
    const size_t r = level_row0 + row;
    const unsigned long long got = atomicExch(reinterpret_cast<unsigned long long*>(o.grads + r), kUntouchedRow);
    const uint32_t gx_bits = static_cast<uint32_t>(got), gy_bits = static_cast<uint32_t>(got >> 32);
    if (gx_bits == kUntouchedBits) return;  // untouched, or already claimed by another thread
    double gx = static_cast<double>(__uint_as_float(gx_bits)), gy = static_cast<double>(__uint_as_float(gy_bits));
    const bool repro = o.fixed != nullptr;
    const bool okx = isfinite(gx) && (!repro || fabs(gx) < 1024.0), oky = isfinite(gy) && (!repro || fabs(gy) < 1024.0);
    if (repro) {  // the row is this thread's now: take the order-free sums and re-arm them
      const longlong2 q = o.fixed[r];
      o.fixed[r] = make_longlong2(0, 0);
      gx = __dmul_rn(static_cast<double>(q.x), kFixedUnit);
      gy = __dmul_rn(static_cast<double>(q.y), kFixedUnit);
    }
    if (!okx || !oky) {
      atomicMin(o.status, static_cast<unsigned long long>(2 * r + (okx ? 1 : 0)));  // src/optimizer.cpp:73-76
      return;
    }
    double2 mm = o.m[r], vv = o.v[r];
    float2 t = o.tables[r];
    const double dx = adam_delta(gx, mm.x, vv.x, o.c);
    const double dy = adam_delta(gy, mm.y, vv.y, o.c);
    o.m[r] = mm;
    o.v[r] = vv;
    t.x = static_cast<float>(__dadd_rn(static_cast<double>(t.x), dx));
    t.y = static_cast<float>(__dadd_rn(static_cast<double>(t.y), dy));
    o.tables[r] = t;
  };
  if constexpr (GRID) {
    GridCell<ND> cell;
    grid_prepare<ND>(x, a.geom.scale[l], a.geom.res[l], cell);
#pragma unroll 1
    for (int m = 0; m < V; ++m) {
      uint32_t idx;
      double w;
      grid_corner<ND>(cell, m, a.mask, idx, w);
      claim_and_update(idx);
    }
  } else {
    uint32_t idx[V];
    double w[V];
    simplex_lookup<ND>(x, a.geom.scale[l], a.skew, a.geom.res[l], a.mask, idx, w);
#pragma unroll 1
    for (int k = 0; k < V; ++k) claim_and_update(idx[k]);
  }
}

// Adds the dense replicas of one launch's coarse levels into the hashed gradient rows and re-arms them with -0.0f.
// One thread per (vertex, feature) of a level (blockIdx.y = local level).  Each replica slot is claimed with an atomic
// exchange, so a backward kernel of another stream that is still adding loses nothing: whatever lands after the exchange
// is carried by that stream's own fold.  A slot still holding -0.0f was not touched; the sum of touched slots can be
// +0.0f but never -0.0f, and -0.0f + (+0.0f) = +0.0f marks the hashed row touched exactly as a direct add would.
template <int ND>
__global__ void __launch_bounds__(256) coarse_fold_kernel(const __grid_constant__ EncodeArgs a) {
  const int l = blockIdx.y;
  const int cshift = a.cg.shift[l];
  if (l >= a.n_levels || cshift < 0) return;
  const int F = a.features;
  const uint32_t verts = a.cg.verts[l];
  const unsigned long long e = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= static_cast<unsigned long long>(verts) * F) return;
  const uint32_t v = static_cast<uint32_t>(e / F);
  const int f = static_cast<int>(e - static_cast<unsigned long long>(v) * F);
  float* cb = a.coarse + a.cg.offset[l] + static_cast<size_t>(v) * F + f;
  const size_t rstride = static_cast<size_t>(verts) * F;
  const uint32_t reps = 1u << cshift;
  float sum = 0.0f;
  bool any = false;
  // replicas in batches: all loads of a batch, then all exchanges, are independent and in flight together
  constexpr uint32_t kBatch = 8;
  for (uint32_t r0 = 0; r0 < reps; r0 += kBatch) {
    uint32_t seen[kBatch];
#pragma unroll
    for (uint32_t i = 0; i < kBatch; ++i)
      seen[i] = (r0 + i < reps) ? __float_as_uint(__ldcg(cb + (r0 + i) * rstride)) : 0x80000000u;
#pragma unroll
    for (uint32_t i = 0; i < kBatch; ++i)
      if (seen[i] != 0x80000000u) seen[i] = atomicExch(reinterpret_cast<unsigned int*>(cb + (r0 + i) * rstride), 0x80000000u);
#pragma unroll
    for (uint32_t i = 0; i < kBatch; ++i) {
      if (seen[i] != 0x80000000u) {
        sum += __uint_as_float(seen[i]);
        any = true;
      }
    }
  }
  if (!any) return;
  const uint32_t side = static_cast<uint32_t>(a.geom.res[l]) + 1u;
  uint32_t rest = v, h = 0;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    const uint32_t c = rest % side;
    rest /= side;
    h ^= c * prime_of(i);
  }
  const size_t level_off = static_cast<size_t>(a.level0 + l) * a.level_stride;
  red_add(a.grads + level_off + static_cast<size_t>(h & a.mask) * F + f, sum);
}

// ---- host-side launch plumbing, one translation unit per ND (sxen_encode_nd.cu) -----------------------------

struct EncodeLaunch {
  int repro;            // reproducible mode (EncodeArgs::fixed != nullptr): the REPRO instantiation, F == 2, LPT <= 2
  int chunk_levels;     // sample-major launches: levels per blockIdx.y slice (0 = one slice); used when it is LPT * 2^k
  int features;         // F, any
  int lpt;              // requested levels per thread
  int mode;             // kModeFwd / kModeBwd / kModeBoth
  int exact;            // fp64 blend
  int grid_backend;     // 0 simplex, 1 grid
  int block_threads;
};

// Each returns cudaSuccess/err; *used_lpt reports the levels-per-thread actually instantiated.
cudaError_t launch_encode_nd1(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd2(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd3(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd4(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd5(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd6(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd7(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);
cudaError_t launch_encode_nd8(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int* used_lpt);

// coarse_fold_kernel over the levels of the launch `a` describes (no-op when none is replicated)
cudaError_t launch_fold_nd1(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd2(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd3(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd4(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd5(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd6(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd7(const EncodeArgs&, cudaStream_t);
cudaError_t launch_fold_nd8(const EncodeArgs&, cudaStream_t);

// sparse_adam_walk_kernel over the levels of the launch `a` describes
cudaError_t launch_adam_walk_nd1(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd2(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd3(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd4(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd5(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd6(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd7(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);
cudaError_t launch_adam_walk_nd8(const EncodeArgs&, const AdamWalkArgs&, int grid_backend, cudaStream_t);

cudaError_t launch_debug_nd1(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd2(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd3(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd4(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd5(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd6(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd7(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);
cudaError_t launch_debug_nd8(EncodeArgs&, int grid_backend, uint32_t*, double*, int total_levels, cudaStream_t);

}  // namespace sxen_dev
