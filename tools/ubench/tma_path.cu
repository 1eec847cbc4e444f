// tools/ubench/tma_path.cu -- is the bulk-copy (TMA) engine a second request path next to the LSU's L1-miss path?
// The forward encode is bound by the SM's L1-miss request port (l1tex2xbar 90 % busy, L2 tags 68 %).
// Three kernels over the same 64 MiB of 8-byte rows (16 tables of 2^19 rows, L2-resident, random rows):
//   lsu   : every lane gathers one random 8-byte row per iteration (ld.global.nc.v2.f32), as the encode kernels do
//   bulk  : lane 0 of every warp issues 32 cp.async.bulk copies of 16 bytes (a row pair) into the warp's shared-memory
//           slots, one mbarrier per warp counts the bytes, every lane then reads its slot
//   mixed : both in the same iteration (64 rows per warp-iteration)
// Output: rows per second of each.  If mixed ~ lsu + bulk, the two paths add up; if mixed ~ max, they share a limit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_path tma_path.cu && ./tma_path
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16; return x;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

constexpr uint32_t kRows = 16u << 19;  // 8-byte rows
constexpr int kWarps = 8;              // per CTA

template <int MODE>  // 0 lsu, 1 bulk, 2 mixed
__global__ void __launch_bounds__(kWarps * 32) k(const float2* __restrict__ tab, float* __restrict__ out, int iters,
                                                 unsigned long long* __restrict__ stuck) {
  __shared__ __align__(16) float4 slots[kWarps][32];
  __shared__ __align__(8) uint64_t bars[kWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t gwarp = blockIdx.x * kWarps + warp;
  if (MODE != 0 && lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[warp])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  float acc = 0.f;
  uint32_t parity = 0;
  for (int it = 0; it < iters; ++it) {
    const uint32_t base = (gwarp * 8191u + static_cast<uint32_t>(it)) * 64u;
    if (MODE != 0) {
      if (lane == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[warp])), "r"(32 * 16) : "memory");
#pragma unroll 8
        for (int j = 0; j < 32; ++j) {
          const uint32_t pair = mix(base + 32u + j) & (kRows / 2 - 1);
          asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                           smem_u32(&slots[warp][j])),
                       "l"(reinterpret_cast<const char*>(tab) + static_cast<size_t>(pair) * 16), "r"(smem_u32(&bars[warp]))
                       : "memory");
        }
      }
    }
    if (MODE != 1) {
      const float2 e = __ldg(tab + (mix(base + lane) & (kRows - 1)));
      acc += e.x + e.y;
    }
    if (MODE != 0) {
      uint32_t done = 0;
      for (int spin = 0; spin < (1 << 22) && !done; ++spin) {
        asm volatile(
            "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(smem_u32(&bars[warp])), "r"(parity)
            : "memory");
      }
      if (!done) {  // never expected; keeps a mistake from hanging the box
        if (lane == 0) atomicAdd(stuck, 1ULL);
        break;
      }
      parity ^= 1;
      const float4 v = slots[warp][lane];
      acc += v.x + v.w;
      __syncwarp();  // every lane has read its slot before lane 0 overwrites them
    }
  }
  if (acc == 123.456f) out[0] = acc;
}

template <int MODE>
double run(const float2* tab, float* out, unsigned long long* stuck, int iters, const char* name, int rows_per_warp_iter) {
  const int grid = 148 * 4;  // 32 warps per SM
  k<MODE><<<grid, kWarps * 32>>>(tab, out, 8, stuck);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<MODE><<<grid, kWarps * 32>>>(tab, out, iters, stuck);
  cudaEventRecord(e1);
  cudaError_t err = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double rows = static_cast<double>(grid) * kWarps * iters * rows_per_warp_iter;
  std::printf("%-6s %8.3f ms  %7.2f G rows/s  (%s)\n", name, ms, rows / (ms * 1e-3) / 1e9, cudaGetErrorString(err));
  return rows / (ms * 1e-3);
}

int main() {
  float2* tab;
  float* out;
  unsigned long long* stuck;
  cudaMalloc(&tab, static_cast<size_t>(kRows) * sizeof(float2));
  cudaMalloc(&out, 4);
  cudaMalloc(&stuck, 8);
  cudaMemset(tab, 0, static_cast<size_t>(kRows) * sizeof(float2));
  cudaMemset(stuck, 0, 8);
  const int iters = 2000;
  const double a = run<0>(tab, out, stuck, iters, "lsu", 32);
  const double b = run<1>(tab, out, stuck, iters, "bulk", 32);
  const double c = run<2>(tab, out, stuck, iters, "mixed", 64);
  unsigned long long h = 0;
  cudaMemcpy(&h, stuck, 8, cudaMemcpyDeviceToHost);
  std::printf("mixed / (lsu + bulk) = %.2f, mixed / max = %.2f, stuck warps = %llu\n", c / (a + b), c / (a > b ? a : b), h);
  return 0;
}
