// sxen_tc_probe.cu -- one tcgen05.mma on caller-supplied operands, raw TMEM dumped to global memory.
// Test infrastructure for the tensor-core path (tests/test_gpu_tc.py), built into its own library
// (tests/cuda/_build/libsxen_tc_probe.so, `make -C paper_2311_15439_b200/csrc probe`), NOT into libsxen_b200.so: pins the shared-memory descriptor conventions of
// sxen_tc.cuh (K-major and MN-major views of a core-matrix tile) and the TMEM lane mapping of M=128 and M=64
// accumulators on real hardware before the MLP kernels rely on them.
#include <cuda_bf16.h>

#include <cuda_runtime.h>

#include <cstdint>

#include "../../paper_2311_15439_b200/csrc/sxen_tc.cuh"

using namespace sxen_tc;

// 0 = ok, 1 = unsupported arguments, 2 = CUDA error (cudaGetErrorString(cudaGetLastError()) has the text).
#define PROBE_API extern "C" __attribute__((visibility("default")))
#define PROBE_CUDA(call) do { if ((call) != cudaSuccess) return 2; } while (0)
#define PROBE_REQUIRE(cond, what) do { if (!(cond)) return 1; } while (0)

namespace {

// A: logical [M][K], B: logical [N][K] (row-major floats). raw: [128][N] = TMEM lanes x columns.
__global__ void __launch_bounds__(128) tc_probe_kernel(const float* __restrict__ A, const float* __restrict__ B, int M, int N,
                                                       int K, int a_mn, int b_mn, int swz, float* __restrict__ raw) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  unsigned char* a_tile = smem;
  const int a_rows = a_mn ? K : M, a_cols = a_mn ? M : K;
  const int b_rows = b_mn ? K : N, b_cols = b_mn ? N : K;
  (void)b_cols;
  unsigned char* b_tile = smem + ((a_rows * a_cols * 4 + 1023) / 1024) * 1024;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e - m * K;
    const int r = a_mn ? k : m, c = a_mn ? m : k;
    *reinterpret_cast<float*>(a_tile + (swz ? sw_offset(r, c, a_rows) : cm_offset(r, c, a_cols))) = A[e];
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e - n * K;
    const int r = b_mn ? k : n, c = b_mn ? n : k;
    *reinterpret_cast<float*>(b_tile + (swz ? sw_offset(r, c, b_rows) : cm_offset(r, c, b_cols))) = B[e];
  }
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) tmem_alloc(&tmem_base, 256);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_tf32(M, N, a_mn != 0, b_mn != 0);
    for (int ks = 0; ks < K / 8; ++ks) {
      uint64_t da, db;
      if (swz) {
        da = a_mn ? sw_desc_mn_major(smem_u32(a_tile), a_rows, ks) : sw_desc_k_major(smem_u32(a_tile), a_rows, ks);
        db = b_mn ? sw_desc_mn_major(smem_u32(b_tile), b_rows, ks) : sw_desc_k_major(smem_u32(b_tile), b_rows, ks);
      } else {
        da = a_mn ? desc_mn_major(smem_u32(a_tile), a_cols, ks) : desc_k_major(smem_u32(a_tile), a_cols, ks);
        db = b_mn ? desc_mn_major(smem_u32(b_tile), b_cols, ks) : desc_k_major(smem_u32(b_tile), b_cols, ks);
      }
      mma_tf32(tbase, da, db, idesc, ks > 0);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0), v);
    for (int i = 0; i < 16; ++i)
      if (c0 + i < N) raw[threadIdx.x * N + c0 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tbase, 256);
}

// Same probe with bf16 operands (kind::f16, UMMA_K = 16) in CM16 tiles.
__global__ void __launch_bounds__(128) tc_probe_bf16_kernel(const float* __restrict__ A, const float* __restrict__ B, int M,
                                                            int N, int K, int a_mn, int b_mn, float* __restrict__ raw) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tmem_base;
  unsigned char* a_tile = smem;
  const int a_rows = a_mn ? K : M, a_cols = a_mn ? M : K;
  const int b_cols = b_mn ? N : K;
  unsigned char* b_tile = smem + ((a_rows * a_cols * 2 + 1023) / 1024) * 1024;
  for (int e = threadIdx.x; e < M * K; e += blockDim.x) {
    const int m = e / K, k = e - m * K;
    const int r = a_mn ? k : m, c = a_mn ? m : k;
    *reinterpret_cast<__nv_bfloat16*>(a_tile + cm16_offset(r, c, a_cols)) = __float2bfloat16(A[e]);
  }
  for (int e = threadIdx.x; e < N * K; e += blockDim.x) {
    const int n = e / K, k = e - n * K;
    const int r = b_mn ? k : n, c = b_mn ? n : k;
    *reinterpret_cast<__nv_bfloat16*>(b_tile + cm16_offset(r, c, b_cols)) = __float2bfloat16(B[e]);
  }
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  if (threadIdx.x < 32) tmem_alloc(&tmem_base, 256);
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base;
  if (threadIdx.x == 0) {
    const uint32_t idesc = make_idesc_bf16(M, N, a_mn != 0, b_mn != 0);
    for (int ks = 0; ks < K / 16; ++ks) {
      const uint64_t da = a_mn ? desc16_mn_major(smem_u32(a_tile), a_cols, ks) : desc16_k_major(smem_u32(a_tile), a_cols, ks);
      const uint64_t db = b_mn ? desc16_mn_major(smem_u32(b_tile), b_cols, ks) : desc16_k_major(smem_u32(b_tile), b_cols, ks);
      mma_bf16(tbase, da, db, idesc, ks > 0);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const int warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < N; c0 += 16) {
    float v[16];
    tmem_ld16(tbase + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>(c0), v);
    for (int i = 0; i < 16; ++i)
      if (c0 + i < N) raw[threadIdx.x * N + c0 + i] = v[i];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tbase, 256);
}

}  // namespace

PROBE_API int sxen_tc_probe_bf16(const float* a_dev, const float* b_dev, int32_t m, int32_t n,
                                                         int32_t k, int32_t a_mn_major, int32_t b_mn_major, float* raw_dev) {
  PROBE_REQUIRE((m == 64 || m == 128) && n >= 8 && n <= 256 && n % 8 == 0 && k >= 16 && k % 16 == 0, "tc probe: unsupported shape");
  const size_t smem = ((static_cast<size_t>(m) * k * 2 + 1023) / 1024) * 1024 + static_cast<size_t>(n) * k * 2 + 1024;
  PROBE_CUDA(cudaFuncSetAttribute(tc_probe_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  PROBE_CUDA(cudaMemset(raw_dev, 0, sizeof(float) * 128 * static_cast<size_t>(n)));
  tc_probe_bf16_kernel<<<1, 128, smem>>>(a_dev, b_dev, m, n, k, a_mn_major, b_mn_major, raw_dev);
  PROBE_CUDA(cudaGetLastError());
  PROBE_CUDA(cudaDeviceSynchronize());
  return 0;
}

PROBE_API int sxen_tc_probe(const float* a_dev, const float* b_dev, int32_t m, int32_t n, int32_t k,
                                                    int32_t a_mn_major, int32_t b_mn_major, int32_t swizzle128, float* raw_dev) {
  PROBE_REQUIRE((m == 64 || m == 128) && n >= 8 && n <= 256 && n % 8 == 0 && k >= 8 && k % 8 == 0, "tc probe: unsupported shape");
  PROBE_REQUIRE(m % 8 == 0 && (m == 128 ? n % 16 == 0 : true), "tc probe: N must be a multiple of 16 for M=128");
  const size_t smem = ((static_cast<size_t>(m) * k * 4 + 1023) / 1024) * 1024 + static_cast<size_t>(n) * k * 4 + 1024;
  if (swizzle128) {
    const int a_cols = a_mn_major ? m : k, b_cols = b_mn_major ? n : k;
    PROBE_REQUIRE(a_cols % 32 == 0 && b_cols % 32 == 0, "tc probe: swizzled tiles need 32-element column blocks");
  }
  PROBE_REQUIRE(smem <= 200 * 1024, "tc probe: operands exceed shared memory");
  PROBE_CUDA(cudaFuncSetAttribute(tc_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  PROBE_CUDA(cudaMemset(raw_dev, 0, sizeof(float) * 128 * static_cast<size_t>(n)));
  tc_probe_kernel<<<1, 128, smem>>>(a_dev, b_dev, m, n, k, a_mn_major, b_mn_major, swizzle128, raw_dev);
  PROBE_CUDA(cudaGetLastError());
  PROBE_CUDA(cudaDeviceSynchronize());
  return 0;
}
