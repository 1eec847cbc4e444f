// tools/ubench/atom_v4.cu -- does ONE vector atomic-with-return on an interleaved [t0,t1,g0,g1] row beat a gather plus a
// red on separate arrays?  Random rows, 16 level tables of 2^19 rows, 2^20 samples x 16 levels x 4 vertices.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atom_v4 atom_v4.cu && ./atom_v4
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}

constexpr int L = 16, V = 4, LPT = 2;
#ifndef TLOG
#define TLOG 19
#endif
#ifndef NFINE
#define NFINE 16
#endif
constexpr uint32_t T = 1u << TLOG;

template <int MODE>
__global__ void __launch_bounds__(256) k(const float* __restrict__ tab, float* __restrict__ grd, float* __restrict__ tg,
                                         const float* __restrict__ up, float* __restrict__ out, uint32_t n) {
  uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t s = gid / (L / LPT), g = gid % (L / LPT);
  if (s >= n) return;
  float4 u = __ldcs(reinterpret_cast<const float4*>(up + (size_t)s * 32 + g * 4));
  float o[4];
#pragma unroll
  for (int j = 0; j < LPT; ++j) {
    int l = g * LPT + j;
    float ux = j ? u.z : u.x, uy = j ? u.w : u.y;
    float a0 = 0.f, a1 = 0.f;
    uint32_t idx[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { uint32_t h = mix(s * 64u + l * 4u + v); idx[v] = (l < 16 - NFINE) ? (mix((h & ((4096u << l) - 1)) + 77u * l) & (T - 1)) : (h & (T - 1)); }
    if (MODE == 0) {  // gather + red.v2 on separate arrays
      float2 e[V];
#pragma unroll
      for (int v = 0; v < V; ++v) e[v] = __ldg(reinterpret_cast<const float2*>(tab + ((size_t)l * T + idx[v]) * 2));
#pragma unroll
      for (int v = 0; v < V; ++v) { a0 += 0.25f * e[v].x; a1 += 0.25f * e[v].y; }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float* p = grd + ((size_t)l * T + idx[v]) * 2;
        asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(0.25f * ux), "f"(0.25f * uy) : "memory");
      }
    } else if (MODE == 1) {  // one atom.v4 with return on the interleaved row
      float4 e[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float* p = tg + ((size_t)l * T + idx[v]) * 4;
        asm volatile("atom.global.add.v4.f32 {%0,%1,%2,%3}, [%4], {%5,%6,%7,%8};"
                     : "=f"(e[v].x), "=f"(e[v].y), "=f"(e[v].z), "=f"(e[v].w)
                     : "l"(p), "f"(-0.0f), "f"(-0.0f), "f"(0.25f * ux), "f"(0.25f * uy) : "memory");
      }
#pragma unroll
      for (int v = 0; v < V; ++v) { a0 += 0.25f * e[v].x; a1 += 0.25f * e[v].y; }
    } else if (MODE == 2) {  // red.v4 without return on the interleaved row (cost of the return path)
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float* p = tg + ((size_t)l * T + idx[v]) * 4;
        asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(-0.0f), "f"(-0.0f), "f"(0.25f * ux), "f"(0.25f * uy) : "memory");
      }
    } else if (MODE == 3) {  // gather only
      float2 e[V];
#pragma unroll
      for (int v = 0; v < V; ++v) e[v] = __ldg(reinterpret_cast<const float2*>(tab + ((size_t)l * T + idx[v]) * 2));
#pragma unroll
      for (int v = 0; v < V; ++v) { a0 += 0.25f * e[v].x; a1 += 0.25f * e[v].y; }
    } else if (MODE == 4) {  // red.v2 only
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float* p = grd + ((size_t)l * T + idx[v]) * 2;
        asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(0.25f * ux), "f"(0.25f * uy) : "memory");
      }
    } else if (MODE == 6) {  // interleaved [t0 t1 g0 g1] rows: 8-byte gather of the table half + red.v2 on the gradient half
      float2 e[V];
#pragma unroll
      for (int v = 0; v < V; ++v) e[v] = __ldg(reinterpret_cast<const float2*>(tg + ((size_t)l * T + idx[v]) * 4));
#pragma unroll
      for (int v = 0; v < V; ++v) { a0 += 0.25f * e[v].x; a1 += 0.25f * e[v].y; }
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float* p = tg + ((size_t)l * T + idx[v]) * 4 + 2;
        asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(0.25f * ux), "f"(0.25f * uy) : "memory");
      }
    } else if (MODE == 5) {  // atom.v2 with return on grads only (return-path cost at 8 bytes)
      float2 e[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float* p = grd + ((size_t)l * T + idx[v]) * 2;
        asm volatile("atom.global.add.v2.f32 {%0,%1}, [%2], {%3,%4};" : "=f"(e[v].x), "=f"(e[v].y) : "l"(p), "f"(0.25f * ux), "f"(0.25f * uy) : "memory");
      }
#pragma unroll
      for (int v = 0; v < V; ++v) { a0 += 0.25f * e[v].x; a1 += 0.25f * e[v].y; }
    }
    o[j * 2] = a0; o[j * 2 + 1] = a1;
  }
  __stcs(reinterpret_cast<float4*>(out + (size_t)s * 32 + g * 4), make_float4(o[0], o[1], o[2], o[3]));
}

int main() {
  const uint32_t n = 1u << 20;
  float *tab, *grd, *tg, *up[4], *out[4];
  cudaMalloc(&tab, (size_t)L * T * 2 * 4); cudaMalloc(&grd, (size_t)L * T * 2 * 4); cudaMalloc(&tg, (size_t)L * T * 4 * 4);
  cudaMemset(tab, 0, (size_t)L * T * 8); cudaMemset(grd, 0, (size_t)L * T * 8); cudaMemset(tg, 0, (size_t)L * T * 16);
  for (int i = 0; i < 4; ++i) { cudaMalloc(&up[i], (size_t)n * 128); cudaMalloc(&out[i], (size_t)n * 128); cudaMemset(up[i], 0, (size_t)n * 128); }
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[] = {"gather + red.v2 (separate arrays)", "atom.v4 with return (interleaved)", "red.v4 no return (interleaved)",
                         "gather only", "red.v2 only", "atom.v2 with return (grads only)", "gather + red.v2, interleaved [t|g] rows"};
  dim3 grid(n * (L / LPT) / 256), block(256);
  for (int m = 0; m < 7; ++m) {
    for (int rep = 0; rep < 15; ++rep) {
      if (rep == 3) cudaEventRecord(a);
      int i = rep % 4;
      switch (m) {
        case 0: k<0><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
        case 1: k<1><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
        case 2: k<2><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
        case 3: k<3><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
        case 4: k<4><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
        case 5: k<5><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
        case 6: k<6><<<grid, block>>>(tab, grd, tg, up[i], out[i], n); break;
      }
    }
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %8.1f us/launch  (%s)\n", names[m], ms / 12 * 1e3, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
