// sxen_device.cuh -- device-side building blocks shared by every kernel of libsxen_b200.
//
// All lattice arithmetic is fp64 with explicit round-to-nearest intrinsics (__dmul_rn/__dadd_rn/
// __dsub_rn): nvcc never contracts those into FMAs, which is what makes vertex selection and hash
// indices bit-identical to the reference's x86-64 build (no -march => no FMA;
// /root/reference/proj/src/CMakeLists.txt:15-17).  Citations: file:line under /root/reference/proj/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sxen_dev {

constexpr int kMaxLaunchLevels = 32;  // levels one kernel launch can carry in its argument block
constexpr double kOneBelow = 0x1.fffffffffffffp-1;  // std::nextafter(1.0, 0.0), src/encoding.cpp:201

// include/sxen/hashing.hpp:16-18 (kHashPrimes)
__host__ __device__ constexpr uint32_t prime_of(int i) {
  return i == 0 ? 1u : i == 1 ? 2654435761u : i == 2 ? 805459861u : i == 3 ? 3674653429u
       : i == 4 ? 2097192037u : i == 5 ? 1434869437u : i == 6 ? 2165219737u : 4294967291u;
}

// include/sxen/rng.hpp:9-14
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// include/sxen/rng.hpp:16-18
__host__ __device__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
  return mix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

// draw `counter` (1-based) of a CounterRng with this key as next_double(lo, hi): include/sxen/rng.hpp:31-37
__device__ __forceinline__ double rng_double(uint64_t key, uint64_t counter, double lo, double span) {
  const uint64_t u = mix64(key + 0x9e3779b97f4a7c15ULL * counter);
  const double d = __dmul_rn(static_cast<double>(u >> 11), 0x1.0p-53);  // exact: 53-bit integer times 2^-53
  return __dadd_rn(lo, __dmul_rn(span, d));
}

// Per-launch level geometry, passed by value in the kernel argument block.
struct LevelGeom {
  double scale[kMaxLaunchLevels];  // simplex: res_l / S_n (src/encoding.cpp:200); grid: (double)res_l (:255)
  int32_t res[kMaxLaunchLevels];   // res_l (src/encoding.cpp:198)
};

// Replicated accumulators of the coarse levels of one launch (backward only; sxen_encode.cuh).
struct CoarseGeom {
  uint32_t offset[kMaxLaunchLevels];  // float offset of the level's first replica inside the coarse buffer
  uint32_t verts[kMaxLaunchLevels];   // (res_l + 1)^dim lattice vertices
  int32_t shift[kMaxLaunchLevels];    // log2(replicas), -1 = the level accumulates straight into its hashed rows
};

// One (sample, level) simplex lookup: gather_simplex, src/encoding.cpp:196-242.
//   x        coordinates already clamped with min(x, nextafter(1,0))   (:201-204)
//   returns  idx[k], w[k] for the vertex chain k = 0..ND, and whether the cell was clamped (:211-218)
//   dense    (DENSE only) vertex k's position in the level's dense lattice, sum_i c_i * (res+1)^i: the address of the
//            replicated coarse-level accumulators (sxen_encode.cuh); not part of the reference
template <int ND, bool DENSE = false>
__device__ __forceinline__ bool simplex_lookup(const double (&x)[ND], double scale, double skew, int res,
                                               uint32_t mask, uint32_t (&idx)[ND + 1], double (&w)[ND + 1],
                                               uint32_t* dense = nullptr) {
  double y[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) y[i] = __dmul_rn(x[i], scale);
  // skew_in_place, src/lattice.cpp:40-45: sum starts at 0.0 and 0.0 + y0 == y0 for y0 >= +0.
  double sum = y[0];
#pragma unroll
  for (int i = 1; i < ND; ++i) sum = __dadd_rn(sum, y[i]);
  const double shift = __dmul_rn(skew, sum);

  bool oob = false;
  double fr[ND];
  uint32_t term[ND];   // axis_term(i, base_i)        src/encoding.cpp:17-20
  uint32_t delta[ND];  // term(base_i) ^ term(base_i+1): the XOR applied when the chain steps along axis i (:231-238)
  uint32_t h = 0;
  uint32_t d0 = 0, stride = 1;
  uint32_t dstep[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    const double yi = __dadd_rn(y[i], shift);
    int b = __double2int_rd(yi);  // floor + cast; |yi| < 2^27 so int32 holds what the reference keeps in int64
    if (b < 0 || b + 1 > res) {
      oob = true;
      b = min(max(b, 0), res - 1);
    }
    double f = __dsub_rn(yi, static_cast<double>(b));
    f = (f < 0.0) ? 0.0 : ((kOneBelow < f) ? kOneBelow : f);  // std::clamp(.., 0.0, one_below), :219-220
    fr[i] = f;
    const uint32_t p = prime_of(i);
    term[i] = static_cast<uint32_t>(b) * p;
    delta[i] = term[i] ^ (static_cast<uint32_t>(b + 1) * p);
    h ^= term[i];
    if constexpr (DENSE) {
      d0 += static_cast<uint32_t>(b) * stride;
      dstep[i] = stride;
      stride *= static_cast<uint32_t>(res + 1);
    }
  }

  // subdivide, src/lattice.cpp:72-103: stable descending insertion sort.  rank[i] = position of axis i in that
  // order = #{j : f_j > f_i} + #{j < i : f_j == f_i}; computed branch-free, no register-array indexing.
  int rank[ND];
#pragma unroll
  for (int i = 0; i < ND; ++i) rank[i] = 0;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
#pragma unroll
    for (int j = i + 1; j < ND; ++j) {
      const bool j_first = fr[j] > fr[i];  // strict: ties keep ascending axis order (include/sxen/lattice.hpp:90-93)
      rank[i] += j_first ? 1 : 0;
      rank[j] += j_first ? 0 : 1;
    }
  }

  // barycentric_weights (src/lattice.cpp:139-147) over sorted[k] = fr[axis with rank k], and the chain walk
  // (src/encoding.cpp:229-240): vertex k = base + sum of unit steps along the axes with rank < k.
  double prev = 0.0;
  idx[0] = h & mask;
  if constexpr (DENSE) dense[0] = d0;
#pragma unroll
  for (int k = 0; k < ND; ++k) {
    double sk = 0.0;
    uint32_t dk = 0, ds = 0;
#pragma unroll
    for (int i = 0; i < ND; ++i) {
      const bool hit = rank[i] == k;
      sk = hit ? fr[i] : sk;
      dk = hit ? delta[i] : dk;
      if constexpr (DENSE) ds = hit ? dstep[i] : ds;
    }
    w[k] = (k == 0) ? __dsub_rn(1.0, sk) : __dsub_rn(prev, sk);
    prev = sk;
    h ^= dk;
    idx[k + 1] = h & mask;
    if constexpr (DENSE) {
      d0 += ds;
      dense[k + 1] = d0;
    }
  }
  w[ND] = prev;
  return oob;
}

// One (sample, level) grid lookup: gather_grid, src/encoding.cpp:244-285, split in two so the 2^ND corners never
// have to live in registers at once.  grid_prepare does the per-axis work (:254-268); grid_corner produces corner m
// (bit d of m set = axis d at base+1), weight = running product in axis order starting from 1.0 (:273-283).
template <int ND>
struct GridCell {
  double w0[ND], w1[ND];
  uint32_t t0[ND], t1[ND];
};

template <int ND>
__device__ __forceinline__ bool grid_prepare(const double (&x)[ND], double scale, int res, GridCell<ND>& c) {
  bool oob = false;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
    const double yi = __dmul_rn(x[i], scale);
    int b = __double2int_rd(yi);
    if (b < 0 || b + 1 > res) {
      oob = true;
      b = min(max(b, 0), res - 1);
    }
    double f = __dsub_rn(yi, static_cast<double>(b));
    f = (f < 0.0) ? 0.0 : ((kOneBelow < f) ? kOneBelow : f);
    c.w1[i] = f;
    c.w0[i] = __dsub_rn(1.0, f);
    const uint32_t p = prime_of(i);
    c.t0[i] = static_cast<uint32_t>(b) * p;
    c.t1[i] = static_cast<uint32_t>(b + 1) * p;
  }
  return oob;
}

template <int ND>
__device__ __forceinline__ void grid_corner(const GridCell<ND>& c, int m, uint32_t mask, uint32_t& idx, double& w) {
  double weight = 1.0;
  uint32_t h = 0;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    const bool bit = (m >> d) & 1;
    weight = __dmul_rn(weight, bit ? c.w1[d] : c.w0[d]);
    h ^= bit ? c.t1[d] : c.t0[d];
  }
  idx = h & mask;
  w = weight;
}

// All 2^ND corners of one (sample, level) grid cell at once, in gather_grid's order (src/encoding.cpp:273-283: corner m,
// bit d of m = axis d at base+1, weight = running product over the axes starting from 1.0).  For the tuned kernel at
// ND <= 3, where the 2^ND (index, weight) pairs fit in registers.  `dense` as in simplex_lookup.
template <int ND, bool DENSE = false>
__device__ __forceinline__ bool grid_lookup(const double (&x)[ND], double scale, int res, uint32_t mask,
                                            uint32_t (&idx)[1 << ND], double (&w)[1 << ND], uint32_t* dense = nullptr) {
  GridCell<ND> c;
  const bool oob = grid_prepare<ND>(x, scale, res, c);
  uint32_t base[ND], stride[ND];
  if constexpr (DENSE) {
    uint32_t st = 1;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      // t0 = base * prime(d); the base coordinate itself: recompute from the weights' cell (b = t0 / prime is not exact
      // in u32 arithmetic), so redo the floor the way grid_prepare did
      const double yi = __dmul_rn(x[d], scale);
      int b = __double2int_rd(yi);
      b = min(max(b, 0), res - 1);
      base[d] = static_cast<uint32_t>(b);
      stride[d] = st;
      st *= static_cast<uint32_t>(res + 1);
    }
  }
#pragma unroll
  for (int m = 0; m < (1 << ND); ++m) {
    grid_corner<ND>(c, m, mask, idx[m], w[m]);
    if constexpr (DENSE) {
      uint32_t dv = 0;
#pragma unroll
      for (int d = 0; d < ND; ++d) dv += (base[d] + ((m >> d) & 1)) * stride[d];
      dense[m] = dv;
    }
  }
  return oob;
}

// ---- memory helpers -------------------------------------------------------------------------

// Gradient contributions below 2^-100 are added as +0.0f.  This keeps every partial sum on the 2^-123 grid, so the
// fp32 atomic (which flushes subnormals to sign-preserving zero) can never produce -0.0f, the "untouched" marker.
__device__ __forceinline__ float canon(float v) { return (fabsf(v) < 0x1p-100f) ? 0.0f : v; }

__device__ __forceinline__ void red_add(float* p, float a) {
  asm volatile("red.global.add.f32 [%0], %1;" ::"l"(p), "f"(a) : "memory");
}
__device__ __forceinline__ void red_add2(float* p, float a, float b) {
  asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(a), "f"(b) : "memory");
}
__device__ __forceinline__ void red_add4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// L2 cache-policy words for the table gathers / gradient reds (sxen_tuning.cache_hints, F == 2 kernels):
//   kind 0 none, 1 evict_last, 2 evict_first, 3 evict_unchanged.
__device__ __forceinline__ uint64_t l2_policy(int kind) {
  uint64_t pol = 0;
  if (kind == 1) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  if (kind == 2) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (kind == 3) asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void load_row2_policy(const float* p, float (&e)[2], uint64_t pol) {
  asm volatile("ld.global.nc.L2::cache_hint.v2.f32 {%0, %1}, [%2], %3;" : "=f"(e[0]), "=f"(e[1]) : "l"(p), "l"(pol));
}
__device__ __forceinline__ void red_add2_policy(float* p, float a, float b, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(p), "f"(a), "f"(b), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add4_policy(float* p, float a, float b, float c, float d, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d), "l"(pol) : "memory");
}

// F contiguous floats of a table row through the read-only path (vectorised when F allows).
template <int F>
__device__ __forceinline__ void load_row(const float* __restrict__ p, float (&e)[F]) {
  if constexpr (F % 4 == 0) {
#pragma unroll
    for (int q = 0; q < F / 4; ++q) {
      const float4 v = __ldg(reinterpret_cast<const float4*>(p) + q);
      e[4 * q + 0] = v.x; e[4 * q + 1] = v.y; e[4 * q + 2] = v.z; e[4 * q + 3] = v.w;
    }
  } else if constexpr (F % 2 == 0) {
#pragma unroll
    for (int q = 0; q < F / 2; ++q) {
      const float2 v = __ldg(reinterpret_cast<const float2*>(p) + q);
      e[2 * q + 0] = v.x; e[2 * q + 1] = v.y;
    }
  } else {
#pragma unroll
    for (int q = 0; q < F; ++q) e[q] = __ldg(p + q);
  }
}

template <int F>
__device__ __forceinline__ void red_row(float* p, const float (&v)[F]) {
  if constexpr (F % 4 == 0) {
#pragma unroll
    for (int q = 0; q < F / 4; ++q) red_add4(p + 4 * q, v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
  } else if constexpr (F % 2 == 0) {
#pragma unroll
    for (int q = 0; q < F / 2; ++q) red_add2(p + 2 * q, v[2 * q], v[2 * q + 1]);
  } else {
#pragma unroll
    for (int q = 0; q < F; ++q) red_add(p + q, v[q]);
  }
}

// K contiguous floats of a streamed (read-once / write-once) array.  `vec` (4, 2 or 1) is the float alignment the host
// proved for every thread's chunk address (row width, chunk width and base pointer all multiples of it).
template <int K>
__device__ __forceinline__ void load_stream(const float* __restrict__ p, float (&v)[K], int vec) {
  if constexpr (K % 4 == 0) {
    if (vec == 4) {
#pragma unroll
      for (int q = 0; q < K / 4; ++q) {
        const float4 t = __ldcs(reinterpret_cast<const float4*>(p) + q);
        v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
      }
      return;
    }
  }
  if constexpr (K % 2 == 0) {
    if (vec >= 2) {
#pragma unroll
      for (int q = 0; q < K / 2; ++q) {
        const float2 t = __ldcs(reinterpret_cast<const float2*>(p) + q);
        v[2 * q] = t.x; v[2 * q + 1] = t.y;
      }
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < K; ++q) v[q] = __ldcs(p + q);
}

template <int K>
__device__ __forceinline__ void store_stream(float* __restrict__ p, const float (&v)[K], int vec) {
  if constexpr (K % 4 == 0) {
    if (vec == 4) {
#pragma unroll
      for (int q = 0; q < K / 4; ++q)
        __stcs(reinterpret_cast<float4*>(p) + q, make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
      return;
    }
  }
  if constexpr (K % 2 == 0) {
    if (vec >= 2) {
#pragma unroll
      for (int q = 0; q < K / 2; ++q) __stcs(reinterpret_cast<float2*>(p) + q, make_float2(v[2 * q], v[2 * q + 1]));
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < K; ++q) __stcs(p + q, v[q]);
}

}  // namespace sxen_dev
