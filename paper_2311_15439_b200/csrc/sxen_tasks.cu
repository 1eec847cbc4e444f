// sxen_tasks.cu -- the device side of the image-fitting task around the hot path (/root/reference/proj/src/tasks.cpp):
// the fit_image batch sampler (:112-126), pixel-centre coordinates and clamped squared error of render_image (:51-96).
// Integer sampling and the (i + 0.5) / w coordinates are bit-identical to the reference (fp64 IEEE division).
#include "sxen_common.hpp"
#include "sxen_device.cuh"

using namespace sxen_host;

namespace {

// draw s (1-based) of CounterRng(seed, step): idx = next_below(w*h); x = ((idx % w) + 0.5) / w, y = ((idx / w) + 0.5) / h
__global__ void sample_image_kernel(uint64_t key, const double* __restrict__ image, int w, int h, unsigned long long n,
                                    double* __restrict__ coords, double* __restrict__ targets) {
  const unsigned long long pixels = static_cast<unsigned long long>(w) * static_cast<unsigned long long>(h);
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long s = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; s < n; s += stride) {
    const uint64_t u = sxen_dev::mix64(key + 0x9e3779b97f4a7c15ULL * (s + 1));
    const unsigned long long idx = u % pixels;
    const int xi = static_cast<int>(idx % static_cast<unsigned long long>(w));
    const int yi = static_cast<int>(idx / static_cast<unsigned long long>(w));
    coords[2 * s] = __ddiv_rn(__dadd_rn(static_cast<double>(xi), 0.5), static_cast<double>(w));
    coords[2 * s + 1] = __ddiv_rn(__dadd_rn(static_cast<double>(yi), 0.5), static_cast<double>(h));
    const double* px = image + 3 * idx;
    targets[3 * s] = px[0];
    targets[3 * s + 1] = px[1];
    targets[3 * s + 2] = px[2];
  }
}

__global__ void pixel_centers_kernel(int w, int h, unsigned long long first, unsigned long long count, double* __restrict__ coords) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const unsigned long long p = first + i;
    const int xi = static_cast<int>(p % static_cast<unsigned long long>(w));
    const int yi = static_cast<int>(p / static_cast<unsigned long long>(w));
    coords[2 * i] = __ddiv_rn(__dadd_rn(static_cast<double>(xi), 0.5), static_cast<double>(w));      // src/tasks.cpp:71
    coords[2 * i + 1] = __ddiv_rn(__dadd_rn(static_cast<double>(yi), 0.5), static_cast<double>(h));
  }
}

// sum over `count` pixels x 3 channels of (clamp(pred, 0, 1) - pixel)^2  (src/tasks.cpp:76-78 and image_mse :35-46)
__global__ void __launch_bounds__(256) render_error_kernel(const float* __restrict__ pred, const double* __restrict__ image,
                                                           unsigned long long first, unsigned long long count,
                                                           double* __restrict__ sum) {
  __shared__ double part[8];
  double acc = 0.0;
  const unsigned long long total = count * 3ULL;
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    double p = static_cast<double>(pred[i]);
    p = p < 0.0 ? 0.0 : (1.0 < p ? 1.0 : p);
    const double e = p - image[first * 3ULL + i];
    acc += e * e;
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += part[k];
    atomicAdd(sum, t);
  }
}

int grid_for(size_t n) {
  size_t b = (n + 255) / 256;
  if (b > 148 * 8) b = 148 * 8;
  return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

extern "C" {

sxen_status sxen_sample_image_batch(uint64_t seed, uint64_t step, const double* image_dev, int32_t width, int32_t height,
                                    size_t n_samples, double* coords_dev, double* targets_dev, void* stream) {
  SXEN_REQUIRE(width >= 1 && height >= 1, "image: width and height must be >= 1");  // src/image.cpp:17-19
  SXEN_REQUIRE(n_samples == 0 || (image_dev && coords_dev && targets_dev), "sample_image_batch: null pointer");
  if (n_samples == 0) return SXEN_OK;
  const uint64_t key = sxen_dev::hash_combine(sxen_dev::mix64(seed), step);  // CounterRng(seed, step), src/tasks.cpp:116
  sample_image_kernel<<<grid_for(n_samples), 256, 0, as_stream(stream)>>>(key, image_dev, width, height, n_samples,
                                                                          coords_dev, targets_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_pixel_centers(int32_t width, int32_t height, size_t first_pixel, size_t count, double* coords_dev,
                               void* stream) {
  SXEN_REQUIRE(width >= 1 && height >= 1, "image: width and height must be >= 1");
  SXEN_REQUIRE(first_pixel + count <= static_cast<size_t>(width) * static_cast<size_t>(height), "pixel range exceeds the image");
  SXEN_REQUIRE(count == 0 || coords_dev, "pixel_centers: null pointer");
  if (count == 0) return SXEN_OK;
  pixel_centers_kernel<<<grid_for(count), 256, 0, as_stream(stream)>>>(width, height, first_pixel, count, coords_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_render_sq_error(const float* pred_dev, const double* image_dev, size_t first_pixel, size_t count,
                                 double* sum_dev, void* stream) {
  SXEN_REQUIRE(count == 0 || (pred_dev && image_dev && sum_dev), "render_sq_error: null pointer");
  if (count == 0) return SXEN_OK;
  render_error_kernel<<<grid_for(count * 3), 256, 0, as_stream(stream)>>>(pred_dev, image_dev, first_pixel, count, sum_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

}  // extern "C"
