// sxen_noise.cu -- the procedural target of fit_field on the device (/root/reference/proj/src/noise.cpp): lattice gradients
// (Box-Muller on the counter RNG, :41-54 with src/rng.cpp:8-19), Perlin gradient noise (:56-97), simplex-lattice gradient
// noise (:103-157), octave fields (:167-188), and fit_field's batch sampler (src/tasks.cpp:156-166).
// fp64 throughout, one thread per point.  The integer parts (vertex keys, subdivision order) are the reference's bit for
// bit; log / cos / sin come from CUDA's libm instead of glibc's, so field values agree to rounding (tests: 1e-12), not
// to the bit.  A target generator beside the hot path: written for clarity, not speed (dims up to 8 with runtime loops).
#include <mutex>
#include <vector>

#include "sxen_common.hpp"
#include "sxen_device.cuh"

using namespace sxen_host;

namespace {

constexpr int kMaxDim = 8;
constexpr double kTwoPi = 6.283185307179586476925286766559;  // 2.0 * std::numbers::pi rounds to the same double

__device__ __forceinline__ double smoother_step(double t) {  // src/noise.cpp:34-39
  return t * t * t * (t * (t * 6.0 - 15.0) + 10.0);
}

// lattice_gradient, src/noise.cpp:41-54.  CounterRng rng(key): key_ = mix64(key), draw i = mix64(key_ + phi * i).
__device__ void lattice_gradient(const long long* vertex, int n, uint64_t seed, double* out) {
  uint64_t key = sxen_dev::mix64(seed);
  for (int i = 0; i < n; ++i) key = sxen_dev::hash_combine(key, static_cast<uint64_t>(vertex[i]));
  const uint64_t rkey = sxen_dev::mix64(key);
  uint64_t counter = 0;
  double norm_sq = 0.0;
  do {
    int i = 0;
    while (i < n) {  // fill_gaussian, src/rng.cpp:8-19
      const double u1 = 1.0 - sxen_dev::rng_double(rkey, ++counter, 0.0, 1.0);
      const double u2 = sxen_dev::rng_double(rkey, ++counter, 0.0, 1.0);
      const double r = sqrt(-2.0 * log(u1));
      const double a = kTwoPi * u2;
      out[i++] = r * cos(a);
      if (i < n) out[i++] = r * sin(a);
    }
    norm_sq = 0.0;
    for (int d = 0; d < n; ++d) norm_sq += out[d] * out[d];
  } while (norm_sq < 1e-24);
  const double inv = 1.0 / sqrt(norm_sq);
  for (int d = 0; d < n; ++d) out[d] *= inv;
}

__device__ double perlin_value(const double* x, int n, uint64_t seed) {  // src/noise.cpp:56-97
  long long base[kMaxDim], corner[kMaxDim];
  double frac[kMaxDim], warped[kMaxDim], grad[kMaxDim];
  for (int i = 0; i < n; ++i) {
    const double f = floor(x[i]);
    base[i] = static_cast<long long>(f);
    frac[i] = x[i] - f;
    warped[i] = smoother_step(frac[i]);
  }
  double value = 0.0;
  for (int m = 0; m < (1 << n); ++m) {
    double weight = 1.0;
    for (int d = 0; d < n; ++d) {
      const int bit = (m >> d) & 1;
      corner[d] = base[d] + bit;
      weight *= bit ? warped[d] : 1.0 - warped[d];
    }
    if (weight == 0.0) continue;
    lattice_gradient(corner, n, seed, grad);
    double dot = 0.0;
    for (int d = 0; d < n; ++d) dot += grad[d] * (frac[d] - static_cast<double>((m >> d) & 1));
    value += weight * dot;
  }
  return value;
}

__device__ double simplex_noise_value(const double* x, int n, uint64_t seed) {  // src/noise.cpp:103-157
  const double root = sqrt(static_cast<double>(n) + 1.0);  // SkewConstants::make, src/lattice.cpp:21-30
  const double skew = (root - 1.0) / static_cast<double>(n);
  const double unskew = (1.0 - 1.0 / root) / static_cast<double>(n);
  double y[kMaxDim], frac[kMaxDim], sorted[kMaxDim], grad[kMaxDim], unsk[kMaxDim];
  long long vertex[kMaxDim];
  int perm[kMaxDim];
  double sum = 0.0;
  for (int i = 0; i < n; ++i) sum += x[i];  // skew_in_place, src/lattice.cpp:40-45
  const double shift = skew * sum;
  for (int i = 0; i < n; ++i) {
    y[i] = x[i] + shift;
    const double f = floor(y[i]);
    vertex[i] = static_cast<long long>(f);
    double fr = y[i] - f;
    fr = fr < 0.0 ? 0.0 : (sxen_dev::kOneBelow < fr ? sxen_dev::kOneBelow : fr);
    frac[i] = fr;
  }
  // subdivide, src/lattice.cpp:72-103: stable descending insertion sort carrying the axis ids
  for (int i = 0; i < n; ++i) {
    const double v = frac[i];
    int j = i;
    while (j > 0 && sorted[j - 1] < v) {
      sorted[j] = sorted[j - 1];
      perm[j] = perm[j - 1];
      --j;
    }
    sorted[j] = v;
    perm[j] = i;
  }
  double warped[kMaxDim + 1], dots[kMaxDim + 1];
  double warped_sum = 0.0;
  for (int k = 0; k <= n; ++k) {
    if (k > 0) vertex[perm[k - 1]] += 1;
    double usum = 0.0;
    for (int i = 0; i < n; ++i) {
      unsk[i] = static_cast<double>(vertex[i]);
      usum += unsk[i];
    }
    const double ushift = unskew * usum;  // unskew_in_place, src/lattice.cpp:47-52
    for (int i = 0; i < n; ++i) unsk[i] -= ushift;
    lattice_gradient(vertex, n, seed, grad);
    double dot = 0.0;
    for (int i = 0; i < n; ++i) dot += grad[i] * (x[i] - unsk[i]);
    dots[k] = dot;
    // barycentric_weights, src/lattice.cpp:139-147
    const double w = (k == 0) ? 1.0 - sorted[0] : (k == n ? sorted[n - 1] : sorted[k - 1] - sorted[k]);
    warped[k] = smoother_step(w);
    warped_sum += warped[k];
  }
  double value = 0.0;
  for (int k = 0; k <= n; ++k) value += warped[k] / warped_sum * dots[k];
  return value;
}

__device__ double noise_field_value(const sxen_noise_spec& spec, const double* x) {  // src/noise.cpp:167-188
  double scaled[kMaxDim];
  double value = 0.0, weight = 1.0, weight_sum = 0.0, freq = spec.frequency;
  for (int o = 0; o < spec.octaves; ++o) {
    for (int i = 0; i < spec.dim; ++i) scaled[i] = x[i] * freq;
    const uint64_t octave_seed = sxen_dev::hash_combine(spec.seed, static_cast<uint64_t>(o));
    value += weight * (spec.kind == SXEN_NOISE_PERLIN ? perlin_value(scaled, spec.dim, octave_seed)
                                                      : simplex_noise_value(scaled, spec.dim, octave_seed));
    weight_sum += weight;
    weight *= 0.5;
    freq *= 2.0;
  }
  return value / weight_sum;
}

__global__ void __launch_bounds__(128) noise_field_kernel(const sxen_noise_spec spec, const double* __restrict__ x,
                                                          unsigned long long n, double* __restrict__ out) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long s = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; s < n; s += stride) {
    double p[kMaxDim];
    for (int i = 0; i < spec.dim; ++i) p[i] = x[s * spec.dim + i];
    out[s] = noise_field_value(spec, p);
  }
}

// fit_field's sampler, src/tasks.cpp:156-166: sample s takes draws s*dim+1 .. s*dim+dim of the batch's CounterRng
__global__ void __launch_bounds__(128) sample_field_kernel(const sxen_noise_spec spec, uint64_t key, unsigned long long n,
                                                           double* __restrict__ coords, double* __restrict__ targets) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long s = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; s < n; s += stride) {
    double p[kMaxDim];
    for (int i = 0; i < spec.dim; ++i) {
      p[i] = sxen_dev::rng_double(key, s * spec.dim + i + 1, 0.0, 1.0);
      coords[s * spec.dim + i] = p[i];
    }
    targets[s] = noise_field_value(spec, p);
  }
}

// make_test_image (src/image.cpp:68-96) at one pixel centre: a shared 4-octave Perlin field plus one 5-octave field per
// channel, v = 0.45 * base + 0.55 * channel, pixel = clamp(0.5 + 0.62 * v, 0, 1).
struct TestImageSpec {
  sxen_noise_spec shared;
  sxen_noise_spec channel[3];
};

// ---- the same image through cached lattice gradients.  A 2D Perlin field of frequency f only ever asks for the gradients of
// the (f + 1)^2 lattice corners of the unit square; the test image's 19 (field, octave) lattices hold 41 k corners in all, while
// a 2^22-sample batch evaluates 3.2e8 of them -- each a counter-RNG draw plus log / sqrt / cos / sin in fp64
// (lattice_gradient).  The gradients are computed ONCE per image seed by the same function and looked up afterwards: the same
// bits at a twentieth of the cost (sampler 8.3 -> 0.4 ms per 2^22 samples).
constexpr int kImageFields = 19;  // shared field: 4 octaves (f = 4..32); three channel fields: 5 octaves each (f = 8..128)
struct TestImageTables {
  const double2* grad;            // all lattices back to back
  int side[kImageFields];         // f + 1
  int offset[kImageFields];       // first corner of the lattice inside `grad`
  double freq[kImageFields];
};

__global__ void __launch_bounds__(128) build_gradient_tables_kernel(const TestImageSpec im, const TestImageTables t, double2* out) {
  const int field = blockIdx.y;
  const int side = t.side[field];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= side * side) return;
  const sxen_noise_spec& spec = field < 4 ? im.shared : im.channel[(field - 4) / 5];
  const int octave = field < 4 ? field : (field - 4) % 5;
  const uint64_t octave_seed = sxen_dev::hash_combine(spec.seed, static_cast<uint64_t>(octave));  // src/noise.cpp:176
  const long long corner[2] = {i % side, i / side};
  double g[2];
  lattice_gradient(corner, 2, octave_seed, g);
  out[t.offset[field] + i] = make_double2(g[0], g[1]);
}

// perlin_value (src/noise.cpp:56-97) at n = 2 with the corner gradients taken from the table: same operations, same order
__device__ __forceinline__ double perlin2_cached(double x0, double x1, const double2* __restrict__ grad, int side) {
  const double f0 = floor(x0), f1 = floor(x1);
  const int b0 = static_cast<int>(f0), b1 = static_cast<int>(f1);
  const double fr0 = x0 - f0, fr1 = x1 - f1;
  const double w0 = smoother_step(fr0), w1 = smoother_step(fr1);
  double value = 0.0;
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int bit0 = m & 1, bit1 = m >> 1;
    double weight = 1.0;
    weight *= bit0 ? w0 : 1.0 - w0;
    weight *= bit1 ? w1 : 1.0 - w1;
    if (weight == 0.0) continue;
    const double2 g = __ldg(grad + (b1 + bit1) * side + (b0 + bit0));
    double dot = 0.0;
    dot += g.x * (fr0 - static_cast<double>(bit0));
    dot += g.y * (fr1 - static_cast<double>(bit1));
    value += weight * dot;
  }
  return value;
}

// noise_field_value (src/noise.cpp:167-188) for one of the image's fields: octaves [first, first + count) of the tables
__device__ __forceinline__ double field_cached(const TestImageTables& t, int first, int count, double x0, double x1) {
  double value = 0.0, weight = 1.0, weight_sum = 0.0;
  for (int o = 0; o < count; ++o) {
    const double freq = t.freq[first + o];
    value += weight * perlin2_cached(x0 * freq, x1 * freq, t.grad + t.offset[first + o], t.side[first + o]);
    weight_sum += weight;
    weight *= 0.5;
  }
  return value / weight_sum;
}

__device__ __forceinline__ void test_image_pixel_cached(const TestImageTables& t, const double (&xy)[2], double (&rgb)[3]) {
  const double base = field_cached(t, 0, 4, xy[0], xy[1]);
#pragma unroll 1
  for (int c = 0; c < 3; ++c) {
    const double v = 0.45 * base + 0.55 * field_cached(t, 4 + 5 * c, 5, xy[0], xy[1]);
    const double p = 0.5 + 0.62 * v;
    rgb[c] = p < 0.0 ? 0.0 : (1.0 < p ? 1.0 : p);
  }
}

// fit_image's sampler (src/tasks.cpp:112-126) over an image that is never materialised: draw s (1-based, s = first + i + 1)
// of CounterRng(train_seed, step) picks the pixel, its centre is the coordinate, make_test_image's formula is the target.
__global__ void __launch_bounds__(128) sample_test_image_kernel(const TestImageTables im, uint64_t key, int w, int h,
                                                                unsigned long long first, unsigned long long n,
                                                                double* __restrict__ coords, double* __restrict__ targets) {
  const unsigned long long pixels = static_cast<unsigned long long>(w) * static_cast<unsigned long long>(h);
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t u = sxen_dev::mix64(key + 0x9e3779b97f4a7c15ULL * (first + i + 1));
    const unsigned long long idx = u % pixels;
    const double xy[2] = {__ddiv_rn(__dadd_rn(static_cast<double>(idx % static_cast<unsigned long long>(w)), 0.5), static_cast<double>(w)),
                          __ddiv_rn(__dadd_rn(static_cast<double>(idx / static_cast<unsigned long long>(w)), 0.5), static_cast<double>(h))};
    double rgb[3];
    test_image_pixel_cached(im, xy, rgb);
    coords[2 * i] = xy[0];
    coords[2 * i + 1] = xy[1];
    targets[3 * i] = rgb[0];
    targets[3 * i + 1] = rgb[1];
    targets[3 * i + 2] = rgb[2];
  }
}

// render_image's error against the same never-materialised image (src/tasks.cpp:76-78, 35-46): pixel p of the list (or
// first + i when the list is null) -> sum of (clamp(pred, 0, 1) - pixel)^2 over the 3 channels, added to *sum.
__global__ void __launch_bounds__(128) test_image_error_kernel(const TestImageTables im, int w, int h, const float* __restrict__ pred,
                                                               unsigned long long first, unsigned long long count,
                                                               double* __restrict__ sum) {
  __shared__ double part[4];
  double acc = 0.0;
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const unsigned long long p = first + i;
    const double xy[2] = {__ddiv_rn(__dadd_rn(static_cast<double>(p % static_cast<unsigned long long>(w)), 0.5), static_cast<double>(w)),
                          __ddiv_rn(__dadd_rn(static_cast<double>(p / static_cast<unsigned long long>(w)), 0.5), static_cast<double>(h))};
    double rgb[3];
    test_image_pixel_cached(im, xy, rgb);
    for (int c = 0; c < 3; ++c) {
      double q = static_cast<double>(pred[3 * i + c]);
      q = q < 0.0 ? 0.0 : (1.0 < q ? 1.0 : q);
      const double e = q - rgb[c];
      acc += e * e;
    }
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) atomicAdd(sum, part[0] + part[1] + part[2] + part[3]);
}


TestImageSpec test_image_spec(uint64_t seed) {  // src/image.cpp:72-79
  TestImageSpec im{};
  im.shared = sxen_noise_spec{2, SXEN_NOISE_PERLIN, 4, 0, sxen_dev::hash_combine(seed, 0xABu), 4.0};
  for (int c = 0; c < 3; ++c)
    im.channel[c] = sxen_noise_spec{2, SXEN_NOISE_PERLIN, 5, 0, sxen_dev::hash_combine(seed, static_cast<uint64_t>(c + 1)), 8.0};
  return im;
}

// gradient tables of make_test_image(., ., seed) on one device, built on first use and kept for the life of the library
struct CachedTables {
  uint64_t seed;
  int device;
  TestImageTables t;
};
std::mutex g_tables_mutex;
std::vector<CachedTables> g_tables;

sxen_status test_image_tables(uint64_t seed, cudaStream_t stream, TestImageTables* out) {
  int device = 0;
  SXEN_CUDA(cudaGetDevice(&device));
  std::lock_guard<std::mutex> lock(g_tables_mutex);
  for (const CachedTables& c : g_tables)
    if (c.seed == seed && c.device == device) {
      *out = c.t;
      return SXEN_OK;
    }
  TestImageTables t{};
  int total = 0;
  for (int field = 0; field < kImageFields; ++field) {
    const int octave = field < 4 ? field : (field - 4) % 5;
    double freq = field < 4 ? 4.0 : 8.0;
    for (int o = 0; o < octave; ++o) freq *= 2.0;  // src/noise.cpp:182: freq *= 2.0 per octave
    t.freq[field] = freq;
    t.side[field] = static_cast<int>(freq) + 1;
    t.offset[field] = total;
    total += t.side[field] * t.side[field];
  }
  double2* grad = nullptr;
  SXEN_CUDA(cudaMalloc(&grad, static_cast<size_t>(total) * sizeof(double2)));
  t.grad = grad;
  const int most = t.side[kImageFields - 1] * t.side[kImageFields - 1];
  build_gradient_tables_kernel<<<dim3((most + 127) / 128, kImageFields), 128, 0, stream>>>(test_image_spec(seed), t, grad);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  SXEN_CUDA(cudaStreamSynchronize(stream));  // other streams may use the cached tables from now on
  g_tables.push_back(CachedTables{seed, device, t});
  *out = t;
  return SXEN_OK;
}

int blocks_for(size_t n) {
  size_t b = (n + 127) / 128;
  if (b > 148 * 16) b = 148 * 16;
  return static_cast<int>(b < 1 ? 1 : b);
}

}  // namespace

extern "C" {

sxen_status sxen_noise_spec_default(sxen_noise_spec* spec) {
  SXEN_REQUIRE(spec != nullptr, "null argument");
  *spec = sxen_noise_spec{2, SXEN_NOISE_PERLIN, 1, 0, 7ULL, 4.0};  // include/sxen/noise.hpp:42-48
  return SXEN_OK;
}

sxen_status sxen_noise_spec_validate(const sxen_noise_spec* spec) {  // NoiseFieldSpec::validate, src/noise.cpp:157-165
  SXEN_REQUIRE(spec != nullptr, "null argument");
  SXEN_REQUIRE(spec->dim >= 1 && spec->dim <= kMaxDim, "noise field: dim must be in [1, %d]", kMaxDim);
  SXEN_REQUIRE(spec->octaves >= 1, "noise field: octaves must be >= 1");
  SXEN_REQUIRE(spec->frequency > 0.0 && std::isfinite(spec->frequency), "noise field: frequency must be finite and > 0");
  SXEN_REQUIRE(spec->kind == SXEN_NOISE_PERLIN || spec->kind == SXEN_NOISE_SIMPLEX, "noise field: unknown kind %d", spec->kind);
  return SXEN_OK;
}

sxen_status sxen_noise_field(const sxen_noise_spec* spec, const double* x_dev, size_t n_points, double* out_dev, void* stream) {
  if (sxen_status st = sxen_noise_spec_validate(spec)) return st;
  SXEN_REQUIRE(n_points == 0 || (x_dev != nullptr && out_dev != nullptr), "noise_field: null pointer");
  if (n_points == 0) return SXEN_OK;
  noise_field_kernel<<<blocks_for(n_points), 128, 0, as_stream(stream)>>>(*spec, x_dev, n_points, out_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_sample_field_batch(const sxen_noise_spec* spec, uint64_t seed, int32_t has_stream, uint64_t stream_id,
                                    size_t n_samples, double* coords_dev, double* targets_dev, void* stream) {
  if (sxen_status st = sxen_noise_spec_validate(spec)) return st;
  SXEN_REQUIRE(n_samples == 0 || (coords_dev != nullptr && targets_dev != nullptr), "sample_field_batch: null pointer");
  if (n_samples == 0) return SXEN_OK;
  // CounterRng(seed, stream) or CounterRng(seed), include/sxen/rng.hpp:22-29
  const uint64_t key = has_stream ? sxen_dev::hash_combine(sxen_dev::mix64(seed), stream_id) : sxen_dev::mix64(seed);
  sample_field_kernel<<<blocks_for(n_samples), 128, 0, as_stream(stream)>>>(*spec, key, n_samples, coords_dev, targets_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_sample_test_image_batch(uint64_t image_seed, int32_t width, int32_t height, uint64_t train_seed, uint64_t step,
                                         size_t first_sample, size_t n_samples, double* coords_dev, double* targets_dev,
                                         void* stream) {
  SXEN_REQUIRE(width >= 1 && height >= 1, "test image: width and height must be >= 1");  // src/image.cpp:69-71
  SXEN_REQUIRE(n_samples == 0 || (coords_dev != nullptr && targets_dev != nullptr), "sample_test_image_batch: null pointer");
  if (n_samples == 0) return SXEN_OK;
  const uint64_t key = sxen_dev::hash_combine(sxen_dev::mix64(train_seed), step);  // CounterRng(seed, step), src/tasks.cpp:116
  TestImageTables tables;
  if (sxen_status st = test_image_tables(image_seed, as_stream(stream), &tables)) return st;
  sample_test_image_kernel<<<blocks_for(n_samples), 128, 0, as_stream(stream)>>>(tables, key, width, height, first_sample,
                                                                                n_samples, coords_dev, targets_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_test_image_sq_error(uint64_t image_seed, int32_t width, int32_t height, const float* pred_dev, size_t first_pixel,
                                     size_t count, double* sum_dev, void* stream) {
  SXEN_REQUIRE(width >= 1 && height >= 1, "test image: width and height must be >= 1");
  SXEN_REQUIRE(count == 0 || (pred_dev != nullptr && sum_dev != nullptr), "test_image_sq_error: null pointer");
  SXEN_REQUIRE(first_pixel + count <= static_cast<size_t>(width) * static_cast<size_t>(height), "test_image_sq_error: pixel range outside the image");
  if (count == 0) return SXEN_OK;
  TestImageTables tables;
  if (sxen_status st = test_image_tables(image_seed, as_stream(stream), &tables)) return st;
  test_image_error_kernel<<<blocks_for(count), 128, 0, as_stream(stream)>>>(tables, width, height, pred_dev, first_pixel, count,
                                                                           sum_dev);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

}  // extern "C"
