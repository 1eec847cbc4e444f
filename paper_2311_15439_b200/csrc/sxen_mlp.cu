// sxen_mlp.cu -- the MLP head on the device, "exact" path: any MlpConfig, fp32 parameters, fp64 accumulation in the
// reference's own summation order and without FMA contraction, so forward activations and per-sample input gradients
// are bit-identical to Mlp::forward / Mlp::backward (/root/reference/proj/src/mlp.cpp:137-202).  Parameter gradients
// are summed over the batch in fp64 (block partial sums + fp64 atomics): same value up to fp64 reassociation.
// The tensor-core path for the headline 32->64->64->{<=16} head lives in sxen_mlp_tc.cu; this file is the general one
// and its parity anchor.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "sxen_common.hpp"
#include "sxen_device.cuh"

using namespace sxen_host;

struct sxen_mlp {
  sxen_mlp_config cfg{};
  int device = 0;
  size_t param_count = 0;
  float* params = nullptr;   // per layer: weights (out x in, row-major) then biases (src/mlp.cpp:19-32)
  double* grads = nullptr;   // MlpGradient: same layout, fp64
  // batched MlpWorkspace: activations of the last forward, [N x act_width] f32, slot 0 = input (include/sxen/mlp.hpp:29-31)
  float* acts = nullptr;
  size_t acts_capacity = 0;  // samples
  size_t forward_samples = 0;
  bool forward_done = false;
  int precision = SXEN_MLP_EXACT;  // sxen_mlp_precision
  double* loss_scratch = nullptr;  // 1 double, used when the caller does not want the loss
  // reproducible mode (sxen_mlp_set_reproducible): the blocks' partial parameter gradients meet in 64-bit fixed point
  // (units of 2^-52, integer atomics: order-free) and are folded into `grads` once per backward
  long long* grads_fixed = nullptr;
  // tensor-core head: one row of parameter-gradient partial sums per CTA (sxen_mlp_tc2.cu), allocated at the first training launch
  double* tc_partials = nullptr;
  size_t tc_partial_stride = 0;
  // host-span entry points (sxen_mlp_forward_host / _backward_host): grow-only staging, [0] = in, [1] = out
  void* host_stage[2] = {nullptr, nullptr};
  size_t host_stage_bytes[2] = {0, 0};
  int layer_count() const { return cfg.hidden_layers + 1; }
  int layer_in(int l) const { return l == 0 ? cfg.input_width : cfg.hidden_width; }
  int layer_out(int l) const { return l == layer_count() - 1 ? cfg.output_width : cfg.hidden_width; }
  size_t act_width() const {
    size_t w = static_cast<size_t>(cfg.input_width);
    for (int l = 0; l < layer_count(); ++l) w += static_cast<size_t>(layer_out(l));
    return w;
  }
};

// sxen_mlp_tc.cu
bool sxen_mlp_tc_supported(const sxen_mlp_config& c);
sxen_status sxen_mlp_tc_run(bool train, const float* params, const float* features, const void* targets, int target_f32,
                            float* pred, float* input_grad, double* mlp_grad, double* loss_sum, size_t n, int in_w, int out_w,
                            size_t global_batch, int precise, cudaStream_t stream, long long* grad_fixed = nullptr,
                            int* used_ctas = nullptr, double* partials = nullptr, size_t partial_stride = 0);

namespace {

constexpr int kMaxWidth = 1 << 14;  // src/mlp.cpp:13
constexpr int kMaxLayers = 16;      // layers one kernel argument block describes

struct MlpShape {
  int layers;
  int in_w[kMaxLayers];
  int out_w[kMaxLayers];
  unsigned long long w_off[kMaxLayers];  // into params / grads
  unsigned long long b_off[kMaxLayers];
  unsigned long long a_off[kMaxLayers + 1];  // activation slot offsets inside one sample's row
  unsigned long long act_width;
};

sxen_status validate(const sxen_mlp_config& c) {
  // MlpConfig::validate, src/mlp.cpp:35-52
  SXEN_REQUIRE(c.input_width >= 1 && c.input_width <= kMaxWidth, "mlp input_width must be in [1, %d], got %d", kMaxWidth,
               c.input_width);
  SXEN_REQUIRE(c.output_width >= 1 && c.output_width <= kMaxWidth, "mlp output_width must be in [1, %d], got %d",
               kMaxWidth, c.output_width);
  SXEN_REQUIRE(c.hidden_layers >= 0, "mlp hidden_layers must be >= 0, got %d", c.hidden_layers);
  SXEN_REQUIRE(c.hidden_layers == 0 || (c.hidden_width >= 1 && c.hidden_width <= kMaxWidth),
               "mlp hidden_width must be in [1, %d], got %d", kMaxWidth, c.hidden_width);
  return SXEN_OK;
}

MlpShape shape_of(const sxen_mlp* m) {
  MlpShape s{};
  s.layers = m->layer_count();
  unsigned long long p = 0, a = 0;
  for (int l = 0; l < s.layers; ++l) {
    s.in_w[l] = m->layer_in(l);
    s.out_w[l] = m->layer_out(l);
    s.w_off[l] = p;
    p += static_cast<unsigned long long>(s.in_w[l]) * s.out_w[l];
    s.b_off[l] = p;
    p += s.out_w[l];
    s.a_off[l] = a;
    a += s.in_w[l];
  }
  s.a_off[s.layers] = a;
  s.act_width = a + s.out_w[s.layers - 1];
  return s;
}

// Mlp::init_params, src/mlp.cpp:106-113: weights He-uniform from CounterRng(seed, layer), biases zero.
__global__ void mlp_init_kernel(float* __restrict__ params, MlpShape s, uint64_t seed_key) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (int l = 0; l < s.layers; ++l) {
    const uint64_t key = sxen_dev::hash_combine(seed_key, static_cast<uint64_t>(l));
    const double bound = sqrt(6.0 / static_cast<double>(s.in_w[l]));
    const double lo = -bound, span = bound - lo;
    const size_t nw = static_cast<size_t>(s.in_w[l]) * s.out_w[l];
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nw + s.out_w[l]; i += stride) {
      params[s.w_off[l] + i] = i < nw ? static_cast<float>(sxen_dev::rng_double(key, i + 1, lo, span)) : 0.0f;
    }
  }
}

// Mlp::forward, src/mlp.cpp:137-162, one layer; fp64 accumulate in index order i = 0..in-1 starting from the bias.
// Persistent blocks keep the layer's weights transposed in shared memory (Wt[i][o]: lanes walk o, conflict-free);
// each pass handles blockDim/ow samples, the input activation is a broadcast read.
__global__ void __launch_bounds__(256)
mlp_forward_layer_smem_kernel(const float* __restrict__ params, float* __restrict__ acts, unsigned long long n_samples,
                              MlpShape s, int layer, int relu) {
  extern __shared__ float wt[];  // [in][ow] then bias[ow]
  const int in = s.in_w[layer], ow = s.out_w[layer];
  float* bias = wt + static_cast<size_t>(in) * ow;
  for (int p = threadIdx.x; p < in * ow; p += blockDim.x) {
    const int o = p / in, i = p - o * in;
    wt[static_cast<size_t>(i) * ow + o] = params[s.w_off[layer] + p];
  }
  for (int o = threadIdx.x; o < ow; o += blockDim.x) bias[o] = params[s.b_off[layer] + o];
  __syncthreads();
  const int slots = blockDim.x / ow;  // >= 1 guaranteed by the launcher
  const int slot = threadIdx.x / ow, o = threadIdx.x - slot * ow;
  if (slot >= slots) return;
  for (unsigned long long smp = static_cast<unsigned long long>(blockIdx.x) * slots + slot; smp < n_samples;
       smp += static_cast<unsigned long long>(gridDim.x) * slots) {
    const float* __restrict__ src = acts + smp * s.act_width + s.a_off[layer];
    double acc = static_cast<double>(bias[o]);
    for (int i = 0; i < in; ++i)
      acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(wt[static_cast<size_t>(i) * ow + o]), static_cast<double>(src[i])));
    if (relu && acc < 0.0) acc = 0.0;
    acts[smp * s.act_width + s.a_off[layer + 1] + o] = static_cast<float>(acc);
  }
}

// Same arithmetic for layers whose weights do not fit shared memory or that are wider than a block.
__global__ void __launch_bounds__(256)
mlp_forward_layer_kernel(const float* __restrict__ params, float* __restrict__ acts, unsigned long long n_samples,
                         MlpShape s, int layer, int relu) {
  const int in = s.in_w[layer], ow = s.out_w[layer];
  const unsigned long long gid = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const unsigned long long smp = gid / static_cast<unsigned long long>(ow);
  const int o = static_cast<int>(gid - smp * static_cast<unsigned long long>(ow));
  if (smp >= n_samples) return;
  const float* __restrict__ w = params + s.w_off[layer] + static_cast<size_t>(o) * in;
  const float* __restrict__ src = acts + smp * s.act_width + s.a_off[layer];
  double acc = static_cast<double>(params[s.b_off[layer] + o]);
  for (int i = 0; i < in; ++i)
    acc = __dadd_rn(acc, __dmul_rn(static_cast<double>(__ldg(w + i)), static_cast<double>(src[i])));
  if (relu && acc < 0.0) acc = 0.0;
  acts[smp * s.act_width + s.a_off[layer + 1] + o] = static_cast<float>(acc);
}

__global__ void copy_rows_kernel(const float* __restrict__ src, int src_w, float* __restrict__ dst,
                                 unsigned long long dst_stride, unsigned long long dst_off, unsigned long long n_samples) {
  const unsigned long long total = n_samples * static_cast<unsigned long long>(src_w);
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const unsigned long long r = i / src_w, c = i - r * src_w;
    dst[r * dst_stride + dst_off + c] = src[i];
  }
}

__global__ void gather_cols_kernel(const float* __restrict__ src, unsigned long long src_stride, unsigned long long src_off,
                                   int w, float* __restrict__ dst, unsigned long long n_samples) {
  const unsigned long long total = n_samples * static_cast<unsigned long long>(w);
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const unsigned long long r = i / w, c = i - r * w;
    dst[i] = src[r * src_stride + src_off + c];
  }
}

// Mlp::backward, src/mlp.cpp:164-202, one layer for a tile of kTile samples per block:
//   db[o] += d_o ; dW[o][i] += d_o * src[i]          (:182-187) -> block partial sums in fp64, one fp64 atomic each
//   downstream[i] = sum_o d_o * W[o][i], zeroed where the (post-ReLU) source activation is <= 0 (:189-199)
// delta_in / delta_out: [N x width] doubles (ping-pong scratch).
constexpr int kTile = 32;

// reproducible mode: a block's partial sum as 64-bit fixed point, units of 2^-52 (a non-finite sum becomes the most negative
// value, which poisons the total visibly: fold_fixed_kernel turns |total| >= 2^62 into NaN for Adam's check)
// Explicit reds: atomicAdd on a 64-bit operand with the result unused still compiles to ATOMG (destination discarded) on
// sm_100a and a warp issues one per L2 round trip (csrc/sxen_mlp_tc_common.cuh: add_total).
__device__ __forceinline__ void red_add_f64(double* p, double v) { asm volatile("red.global.add.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }
__device__ __forceinline__ void red_add_u64(long long* p, unsigned long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long to_fixed(double v) {
  return static_cast<unsigned long long>(__double2ll_rn(__dmul_rn(v, 0x1p52)));
}
// the tensor-core head's per-CTA loss partials, added to the running sum in CTA order (one thread: <= 148 terms)
__global__ void sum_parts_kernel(double* __restrict__ acc, const double* __restrict__ parts, int n) {
  double s = *acc;
  for (int i = 0; i < n; ++i) s = __dadd_rn(s, parts[i]);
  *acc = s;
}
__global__ void fold_fixed_kernel(double* __restrict__ grads, long long* __restrict__ fixed, unsigned long long n) {
  const unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const long long q = fixed[i];
  fixed[i] = 0;
  const bool sane = q > -(1LL << 62) && q < (1LL << 62);
  grads[i] = __dadd_rn(grads[i], sane ? __dmul_rn(static_cast<double>(q), 0x1p-52) : __longlong_as_double(0x7ff8000000000000LL));
}

__global__ void __launch_bounds__(256)
mlp_backward_layer_kernel(const float* __restrict__ params, const float* __restrict__ acts, double* __restrict__ grads,
                          const double* __restrict__ delta_cur, double* __restrict__ delta_next,
                          unsigned long long n_samples, MlpShape s, int layer, long long* __restrict__ fixed, int tile) {
  extern __shared__ double smem[];
  const int in = s.in_w[layer], ow = s.out_w[layer];
  // `tile` samples per block: kTile, or fewer for layers whose tile would not fit shared memory (widths up to 2^14)
  double* d_tile = smem;                                    // [tile][ow]
  float* src_tile = reinterpret_cast<float*>(smem + static_cast<size_t>(tile) * ow);  // [tile][in]
  const unsigned long long s0 = static_cast<unsigned long long>(blockIdx.x) * tile;
  const int rows = static_cast<int>(min(static_cast<unsigned long long>(tile), n_samples - s0));
  for (int i = threadIdx.x; i < rows * ow; i += blockDim.x) d_tile[i] = delta_cur[s0 * ow + i];
  for (int i = threadIdx.x; i < rows * in; i += blockDim.x) {
    const int r = i / in, c = i - r * in;
    src_tile[i] = acts[(s0 + r) * s.act_width + s.a_off[layer] + c];
  }
  __syncthreads();
  // parameter gradients: thread per parameter, samples of the tile in order
  const float* __restrict__ w = params + s.w_off[layer];
  for (int p = threadIdx.x; p < ow * in + ow; p += blockDim.x) {
    double acc = 0.0;
    if (p < ow * in) {
      const int o = p / in, i = p - o * in;
      for (int r = 0; r < rows; ++r)
        acc = __dadd_rn(acc, __dmul_rn(d_tile[r * ow + o], static_cast<double>(src_tile[r * in + i])));
      if (fixed) red_add_u64(fixed + s.w_off[layer] + p, to_fixed(acc));
      else red_add_f64(grads + s.w_off[layer] + p, acc);
    } else {
      const int o = p - ow * in;
      for (int r = 0; r < rows; ++r) acc = __dadd_rn(acc, d_tile[r * ow + o]);
      if (fixed) red_add_u64(fixed + s.b_off[layer] + o, to_fixed(acc));
      else red_add_f64(grads + s.b_off[layer] + o, acc);
    }
  }
  // downstream deltas: thread per (sample, input unit), o in order
  for (int q = threadIdx.x; q < rows * in; q += blockDim.x) {
    const int r = q / in, i = q - r * in;
    double acc = 0.0;
    for (int o = 0; o < ow; ++o)
      acc = __dadd_rn(acc, __dmul_rn(d_tile[r * ow + o], static_cast<double>(__ldg(w + static_cast<size_t>(o) * in + i))));
    if (layer > 0 && src_tile[q] <= 0.0f) acc = 0.0;
    delta_next[(s0 + r) * in + i] = acc;
  }
}

__global__ void narrow_rows_kernel(const double* __restrict__ src, float* __restrict__ dst, unsigned long long n) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long i = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = static_cast<float>(src[i]);
}

// run_chunk's loss + upstream, src/trainer.cpp:26-44: e = pred - target; loss_s = sum e^2; upstream = 2e/(B*out_w).
template <typename TT>
__global__ void mse_kernel(const float* __restrict__ pred, unsigned long long pred_stride, unsigned long long pred_off,
                           const TT* __restrict__ targets, int out_w, unsigned long long n_samples, double upstream_scale,
                           double* __restrict__ upstream, double* __restrict__ sample_loss) {
  const unsigned long long stride = static_cast<unsigned long long>(gridDim.x) * blockDim.x;
  for (unsigned long long smp = static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x; smp < n_samples;
       smp += stride) {
    double loss = 0.0;
    for (int o = 0; o < out_w; ++o) {
      const double e = __dsub_rn(static_cast<double>(pred[smp * pred_stride + pred_off + o]),
                                 static_cast<double>(targets[smp * out_w + o]));
      loss = __dadd_rn(loss, __dmul_rn(e, e));
      upstream[smp * out_w + o] = __dmul_rn(upstream_scale, e);
    }
    sample_loss[smp] = loss;
  }
}

// Deterministic sum of the per-sample losses (src/trainer.cpp:118-119 sums them in sample order; any fixed order
// differs from that only by fp64 reassociation): one block, strided partials, then a shared-memory tree.
__global__ void __launch_bounds__(1024) sum_kernel(const double* __restrict__ v, unsigned long long n, double* __restrict__ out) {
  __shared__ double part[1024];
  double acc = 0.0;
  for (unsigned long long i = threadIdx.x; i < n; i += blockDim.x) acc += v[i];
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) part[threadIdx.x] += part[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = part[0];
}

__global__ void add_scalar_kernel(double* __restrict__ acc, const double* __restrict__ v) { *acc += *v; }

int grid_for(size_t n, int block = 256) {
  size_t b = (n + block - 1) / block;
  if (b > 148 * 16) b = 148 * 16;
  return static_cast<int>(b < 1 ? 1 : b);
}

sxen_status ensure_acts(sxen_mlp* m, size_t n) {
  if (n <= m->acts_capacity) return SXEN_OK;
  cudaFree(m->acts);
  m->acts = nullptr;
  m->acts_capacity = 0;
  SXEN_CUDA(cudaMalloc(&m->acts, n * m->act_width() * sizeof(float)));
  m->acts_capacity = n;
  return SXEN_OK;
}

}  // namespace

extern "C" {

sxen_status sxen_mlp_config_default(sxen_mlp_config* cfg) {
  SXEN_REQUIRE(cfg != nullptr, "config pointer is null");
  *cfg = sxen_mlp_config{32, 64, 2, 3};  // include/sxen/mlp.hpp:11-16
  return SXEN_OK;
}

sxen_status sxen_mlp_validate(const sxen_mlp_config* cfg) {
  SXEN_REQUIRE(cfg != nullptr, "config pointer is null");
  return validate(*cfg);
}

sxen_status sxen_mlp_create(const sxen_mlp_config* cfg, int32_t device, sxen_mlp** out) {
  SXEN_REQUIRE(cfg != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  if (sxen_status st = validate(*cfg)) return st;
  SXEN_REQUIRE(cfg->hidden_layers + 1 <= kMaxLayers, "mlp: at most %d affine layers are supported on the device", kMaxLayers);
  int ndev = 0;
  SXEN_CUDA(cudaGetDeviceCount(&ndev));
  SXEN_REQUIRE(device >= 0 && device < ndev, "device %d out of range (%d visible)", device, ndev);
  DeviceGuard guard(device);
  sxen_mlp* m = new sxen_mlp();
  m->cfg = *cfg;
  m->device = device;
  const MlpShape s = shape_of(m);
  m->param_count = static_cast<size_t>(s.b_off[s.layers - 1] + s.out_w[s.layers - 1]);
  cudaError_t err = cudaMalloc(&m->params, m->param_count * sizeof(float));
  if (err == cudaSuccess) err = cudaMemset(m->params, 0, m->param_count * sizeof(float));
  if (err == cudaSuccess) err = cudaMalloc(&m->grads, m->param_count * sizeof(double));
  if (err == cudaSuccess) err = cudaMemset(m->grads, 0, m->param_count * sizeof(double));
  if (err != cudaSuccess) {
    sxen_mlp_destroy(m);
    return cuda_fail(err, "sxen_mlp_create allocation");
  }
  *out = m;
  return SXEN_OK;
}

sxen_status sxen_mlp_destroy(sxen_mlp* mlp) {
  if (!mlp) return SXEN_OK;
  DeviceGuard guard(mlp->device);
  cudaFree(mlp->params);
  cudaFree(mlp->grads);
  cudaFree(mlp->acts);
  cudaFree(mlp->loss_scratch);
  cudaFree(mlp->grads_fixed);
  cudaFree(mlp->tc_partials);
  cudaFree(mlp->host_stage[0]);
  cudaFree(mlp->host_stage[1]);
  delete mlp;
  return SXEN_OK;
}

sxen_status sxen_mlp_get_config(const sxen_mlp* mlp, sxen_mlp_config* out) {
  SXEN_REQUIRE(mlp != nullptr && out != nullptr, "null argument");
  *out = mlp->cfg;
  return SXEN_OK;
}

sxen_status sxen_mlp_parameter_count(const sxen_mlp* mlp, uint64_t* out) {
  SXEN_REQUIRE(mlp != nullptr && out != nullptr, "null argument");
  *out = mlp->param_count;
  return SXEN_OK;
}

sxen_status sxen_mlp_init_params(sxen_mlp* mlp, uint64_t seed, void* stream) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  DeviceGuard guard(mlp->device);
  mlp_init_kernel<<<grid_for(mlp->param_count), 256, 0, as_stream(stream)>>>(mlp->params, shape_of(mlp), sxen_dev::mix64(seed));
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_mlp_upload_params(sxen_mlp* mlp, const float* src_host) {
  SXEN_REQUIRE(mlp != nullptr && src_host != nullptr, "null argument");
  DeviceGuard guard(mlp->device);
  SXEN_CUDA(cudaMemcpy(mlp->params, src_host, mlp->param_count * sizeof(float), cudaMemcpyHostToDevice));
  return SXEN_OK;
}

sxen_status sxen_mlp_download_params(const sxen_mlp* mlp, float* dst_host) {
  SXEN_REQUIRE(mlp != nullptr && dst_host != nullptr, "null argument");
  DeviceGuard guard(mlp->device);
  SXEN_CUDA(cudaMemcpy(dst_host, mlp->params, mlp->param_count * sizeof(float), cudaMemcpyDeviceToHost));
  return SXEN_OK;
}

sxen_status sxen_mlp_params_dev(sxen_mlp* mlp, float** out_dev) {
  SXEN_REQUIRE(mlp != nullptr && out_dev != nullptr, "null argument");
  *out_dev = mlp->params;
  return SXEN_OK;
}

sxen_status sxen_mlp_grads_dev(sxen_mlp* mlp, double** out_dev) {
  SXEN_REQUIRE(mlp != nullptr && out_dev != nullptr, "null argument");
  *out_dev = mlp->grads;
  return SXEN_OK;
}

sxen_status sxen_mlp_grad_clear(sxen_mlp* mlp, void* stream) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  DeviceGuard guard(mlp->device);
  SXEN_CUDA(cudaMemsetAsync(mlp->grads, 0, mlp->param_count * sizeof(double), as_stream(stream)));
  return SXEN_OK;
}

sxen_status sxen_mlp_grad_download(const sxen_mlp* mlp, double* dst_host) {
  SXEN_REQUIRE(mlp != nullptr && dst_host != nullptr, "null argument");
  DeviceGuard guard(mlp->device);
  SXEN_CUDA(cudaMemcpy(dst_host, mlp->grads, mlp->param_count * sizeof(double), cudaMemcpyDeviceToHost));
  return SXEN_OK;
}

sxen_status sxen_mlp_set_precision(sxen_mlp* mlp, int32_t precision) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  SXEN_REQUIRE(precision == SXEN_MLP_EXACT || precision == SXEN_MLP_TENSOR_BF16X3 || precision == SXEN_MLP_TENSOR_BF16 ||
                   precision == SXEN_MLP_TENSOR_BF16X4,
               "mlp: unknown precision mode %d", precision);
  SXEN_REQUIRE(precision == SXEN_MLP_EXACT || sxen_mlp_tc_supported(mlp->cfg),
               "mlp: the tensor-core path covers input 16 or 32, hidden 64 x 2 layers, output <= 3; this head is %d/%d x %d/%d",
               mlp->cfg.input_width, mlp->cfg.hidden_width, mlp->cfg.hidden_layers, mlp->cfg.output_width);
  mlp->precision = precision;
  return SXEN_OK;
}

sxen_status sxen_mlp_get_precision(const sxen_mlp* mlp, int32_t* out) {
  SXEN_REQUIRE(mlp != nullptr && out != nullptr, "null argument");
  *out = mlp->precision;
  return SXEN_OK;
}

// Forward + MSE + backward of one batch in one call (what run_chunk does per sample, src/trainer.cpp:36-46).
// Tensor-core modes run the fused tcgen05 kernel; the exact mode chains forward, sxen_mse_loss and backward.
sxen_status sxen_mlp_forward_backward(sxen_mlp* mlp, const float* input_dev, const void* targets_dev,
                                      sxen_coord_type target_type, size_t n_samples, size_t global_batch, float* pred_dev,
                                      float* input_grad_dev, double* loss_sum_dev, void* stream) {
  return sxen_mlp_forward_backward_ex(mlp, input_dev, targets_dev, target_type, n_samples, global_batch, pred_dev,
                                      input_grad_dev, nullptr, loss_sum_dev, stream);
}

// + input_grad_f64_dev (may be NULL): d(loss)/d(input) as the reference's doubles (exact head only; the tensor-core head
// leaves it untouched and returns 0 in *wrote_f64 -- internal, declared in sxen_common.hpp)
sxen_status sxen_mlp_forward_backward_ex(sxen_mlp* mlp, const float* input_dev, const void* targets_dev,
                                         sxen_coord_type target_type, size_t n_samples, size_t global_batch, float* pred_dev,
                                         float* input_grad_dev, double* input_grad_f64_dev, double* loss_sum_dev, void* stream) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  SXEN_REQUIRE(n_samples == 0 || (input_dev && targets_dev && input_grad_dev), "mlp forward_backward: null pointer");
  SXEN_REQUIRE(global_batch >= 1, "mlp forward_backward: global batch must be >= 1");
  if (n_samples == 0) return SXEN_OK;
  DeviceGuard guard(mlp->device);
  cudaStream_t st = as_stream(stream);
  if (!mlp->loss_scratch) SXEN_CUDA(cudaMalloc(&mlp->loss_scratch, sizeof(double)));
  if (mlp->precision != SXEN_MLP_EXACT) {
    double* loss = loss_sum_dev ? loss_sum_dev : mlp->loss_scratch;
    mlp->forward_done = false;  // no activations are kept: a separate backward would be a logic error
    int ctas = 0;
    if (!mlp->tc_partials) {  // persistent kernel: at most one CTA per SM
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, mlp->device);
      mlp->tc_partial_stride = (mlp->param_count + 31) / 32 * 32;
      SXEN_CUDA(cudaMalloc(&mlp->tc_partials, static_cast<size_t>(sms) * mlp->tc_partial_stride * sizeof(double)));
    }
    if (sxen_status s = sxen_mlp_tc_run(true, mlp->params, input_dev, targets_dev, target_type == SXEN_COORD_F32 ? 1 : 0, pred_dev,
                                        input_grad_dev, mlp->grads, loss, n_samples, mlp->cfg.input_width, mlp->cfg.output_width,
                                        global_batch, sxen_tc_products(mlp->precision), st, mlp->grads_fixed, &ctas,
                                        mlp->tc_partials, mlp->tc_partial_stride))
      return s;
    if (mlp->grads_fixed) {  // the CTAs' partial sums met in fixed point (order-free): fold them into the fp64 buffers
      fold_fixed_kernel<<<grid_for(mlp->param_count), 256, 0, st>>>(mlp->grads, mlp->grads_fixed, mlp->param_count);
      sum_parts_kernel<<<1, 1, 0, st>>>(loss, reinterpret_cast<const double*>(mlp->grads_fixed + mlp->param_count), ctas);
      SXEN_CUDA(cudaGetLastError());
      count_launch(2);
    }
    return SXEN_OK;
  }
  if (sxen_status s = sxen_mlp_forward(mlp, input_dev, n_samples, pred_dev, stream)) return s;
  const MlpShape sh = shape_of(mlp);
  double* scratch = nullptr;  // upstream [N x ow], sample loss [N], batch sum [1]
  const size_t ow = static_cast<size_t>(mlp->cfg.output_width);
  SXEN_CUDA(cudaMallocAsync(&scratch, (n_samples * (ow + 1) + 1) * sizeof(double), st));
  double* upstream = scratch;
  double* sample_loss = scratch + n_samples * ow;
  double* batch_sum = sample_loss + n_samples;
  sxen_status s = sxen_mse_loss(mlp->acts + sh.a_off[sh.layers], sh.act_width, targets_dev, target_type,
                                mlp->cfg.output_width, n_samples, global_batch, upstream, sample_loss, batch_sum, stream);
  if (s == SXEN_OK && loss_sum_dev) {
    add_scalar_kernel<<<1, 1, 0, st>>>(loss_sum_dev, batch_sum);
    count_launch();
  }
  if (s == SXEN_OK) s = sxen_mlp_backward(mlp, upstream, n_samples, input_grad_dev, input_grad_f64_dev, stream);
  cudaFreeAsync(scratch, st);
  return s;
}

sxen_status sxen_mlp_forward(sxen_mlp* mlp, const float* input_dev, size_t n_samples, float* out_dev, void* stream) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  SXEN_REQUIRE(n_samples == 0 || input_dev != nullptr, "mlp forward: input pointer is null");
  DeviceGuard guard(mlp->device);
  if (mlp->precision != SXEN_MLP_EXACT) {
    // inference on the tensor cores: outputs only, no workspace (Mlp::backward after this is a logic error)
    SXEN_REQUIRE(n_samples == 0 || out_dev != nullptr, "mlp forward: output pointer is null");
    mlp->forward_done = false;
    return sxen_mlp_tc_run(false, mlp->params, input_dev, nullptr, 0, out_dev, nullptr, nullptr, nullptr, n_samples,
                           mlp->cfg.input_width, mlp->cfg.output_width, 1, sxen_tc_products(mlp->precision), as_stream(stream));
  }
  mlp->forward_done = true;
  mlp->forward_samples = n_samples;
  if (n_samples == 0) return SXEN_OK;
  if (sxen_status st = ensure_acts(mlp, n_samples)) return st;
  const MlpShape s = shape_of(mlp);
  cudaStream_t st = as_stream(stream);
  copy_rows_kernel<<<grid_for(n_samples * s.in_w[0]), 256, 0, st>>>(input_dev, s.in_w[0], mlp->acts, s.act_width, 0, n_samples);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  for (int l = 0; l < s.layers; ++l) {
    const int relu = l + 1 < s.layers ? 1 : 0;
    const size_t smem = (static_cast<size_t>(s.in_w[l]) * s.out_w[l] + s.out_w[l]) * sizeof(float);
    if (s.out_w[l] <= 256 && smem <= 160 * 1024) {
      if (smem > 48 * 1024)
        SXEN_CUDA(cudaFuncSetAttribute(mlp_forward_layer_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      const int slots = 256 / s.out_w[l];
      const unsigned long long want = (n_samples + slots - 1) / slots;
      const unsigned blocks = static_cast<unsigned>(std::min<unsigned long long>(want, 148ULL * 8));
      mlp_forward_layer_smem_kernel<<<blocks, 256, smem, st>>>(mlp->params, mlp->acts, n_samples, s, l, relu);
    } else {
      const unsigned long long threads = static_cast<unsigned long long>(n_samples) * s.out_w[l];
      mlp_forward_layer_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st>>>(mlp->params, mlp->acts,
                                                                                            n_samples, s, l, relu);
    }
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  if (out_dev) {
    gather_cols_kernel<<<grid_for(n_samples * mlp->cfg.output_width), 256, 0, st>>>(
        mlp->acts, s.act_width, s.a_off[s.layers], mlp->cfg.output_width, out_dev, n_samples);
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  return SXEN_OK;
}

sxen_status sxen_mlp_backward(sxen_mlp* mlp, const double* upstream_dev, size_t n_samples, float* input_grad_dev,
                              double* input_grad_f64_dev, void* stream) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  if (!mlp->forward_done)  // src/mlp.cpp:165-167
    return fail(SXEN_LOGIC_ERROR, "mlp backward called before forward populated the workspace");
  SXEN_REQUIRE(n_samples == mlp->forward_samples, "mlp backward: batch of %zu samples does not match the forward pass (%zu)",
               n_samples, mlp->forward_samples);
  SXEN_REQUIRE(n_samples == 0 || upstream_dev != nullptr, "mlp backward: upstream pointer is null");
  if (n_samples == 0) return SXEN_OK;
  DeviceGuard guard(mlp->device);
  const MlpShape s = shape_of(mlp);
  cudaStream_t st = as_stream(stream);
  int maxw = mlp->cfg.input_width;
  for (int l = 0; l < s.layers; ++l) maxw = std::max(maxw, s.out_w[l]);
  double* scratch = nullptr;
  SXEN_CUDA(cudaMallocAsync(&scratch, 2 * n_samples * static_cast<size_t>(maxw) * sizeof(double), st));
  double* cur = scratch;
  double* nxt = scratch + n_samples * static_cast<size_t>(maxw);
  SXEN_CUDA(cudaMemcpyAsync(cur, upstream_dev, n_samples * static_cast<size_t>(mlp->cfg.output_width) * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
  for (int l = s.layers - 1; l >= 0; --l) {
    // samples per block: kTile when the tile fits, else halved until it does -- MlpConfig::validate admits widths up to 2^14
    // (src/mlp.cpp:13), and the reference trains them; a block's partial sums then cover fewer samples, nothing else changes
    int tile = kTile;
    auto smem_for = [&](int tl) {
      return static_cast<size_t>(tl) * s.out_w[l] * sizeof(double) + static_cast<size_t>(tl) * s.in_w[l] * sizeof(float);
    };
    while (tile > 1 && smem_for(tile) > 200 * 1024) tile >>= 1;
    const size_t smem = smem_for(tile);
    if (smem > 200 * 1024) {
      cudaFreeAsync(scratch, st);
      return fail(SXEN_INVALID_ARGUMENT, "mlp backward: layer %d (%d x %d) exceeds the shared-memory tile of this path", l,
                  s.out_w[l], s.in_w[l]);
    }
    if (smem > 48 * 1024)
      SXEN_CUDA(cudaFuncSetAttribute(mlp_backward_layer_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    double* dst = (l == 0 && input_grad_f64_dev) ? input_grad_f64_dev : nxt;
    mlp_backward_layer_kernel<<<static_cast<unsigned>((n_samples + tile - 1) / tile), 256, smem, st>>>(
        mlp->params, mlp->acts, mlp->grads, cur, dst, n_samples, s, l, mlp->grads_fixed, tile);
    SXEN_CUDA(cudaGetLastError());
    count_launch();
    if (l == 0 && input_grad_dev) {
      narrow_rows_kernel<<<grid_for(n_samples * s.in_w[0]), 256, 0, st>>>(dst, input_grad_dev, n_samples * static_cast<size_t>(s.in_w[0]));
      SXEN_CUDA(cudaGetLastError());
      count_launch();
    }
    std::swap(cur, nxt);
  }
  if (mlp->grads_fixed) {
    fold_fixed_kernel<<<grid_for(mlp->param_count), 256, 0, st>>>(mlp->grads, mlp->grads_fixed, mlp->param_count);
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  SXEN_CUDA(cudaFreeAsync(scratch, st));
  return SXEN_OK;
}

// ---- the reference's own call shape: host spans in, host spans out (include/sxen/mlp.hpp:94-99), n samples per call
namespace {
// grow-only device staging of the host-span calls (a per-sample caller would otherwise pay cudaMalloc + cudaFree per call)
sxen_status host_stage(sxen_mlp* mlp, int which, size_t bytes) {
  if (mlp->host_stage_bytes[which] >= bytes) return SXEN_OK;
  cudaFree(mlp->host_stage[which]);
  mlp->host_stage[which] = nullptr;
  mlp->host_stage_bytes[which] = 0;
  const size_t want = std::max<size_t>(bytes, 4096);
  SXEN_CUDA(cudaMalloc(&mlp->host_stage[which], want));
  mlp->host_stage_bytes[which] = want;
  return SXEN_OK;
}
}  // namespace

sxen_status sxen_mlp_forward_host(sxen_mlp* mlp, const float* input_host, size_t n_samples, float* out_host) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  SXEN_REQUIRE(n_samples == 0 || (input_host != nullptr && out_host != nullptr), "mlp forward: null input or output pointer");
  DeviceGuard guard(mlp->device);
  if (n_samples == 0) return sxen_mlp_forward(mlp, nullptr, 0, nullptr, nullptr);
  const size_t in_bytes = n_samples * static_cast<size_t>(mlp->cfg.input_width) * sizeof(float);
  const size_t out_bytes = n_samples * static_cast<size_t>(mlp->cfg.output_width) * sizeof(float);
  if (sxen_status st = host_stage(mlp, 0, in_bytes)) return st;
  if (sxen_status st = host_stage(mlp, 1, out_bytes)) return st;
  SXEN_CUDA(cudaMemcpy(mlp->host_stage[0], input_host, in_bytes, cudaMemcpyHostToDevice));
  if (sxen_status st = sxen_mlp_forward(mlp, static_cast<const float*>(mlp->host_stage[0]), n_samples,
                                        static_cast<float*>(mlp->host_stage[1]), nullptr))
    return st;
  SXEN_CUDA(cudaMemcpy(out_host, mlp->host_stage[1], out_bytes, cudaMemcpyDeviceToHost));  // synchronises the legacy stream
  return SXEN_OK;
}

sxen_status sxen_mlp_backward_host(sxen_mlp* mlp, const double* upstream_host, size_t n_samples, double* input_grad_host) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  if (!mlp->forward_done)  // src/mlp.cpp:165-167, before anything is copied
    return fail(SXEN_LOGIC_ERROR, "mlp backward called before forward populated the workspace");
  SXEN_REQUIRE(n_samples == mlp->forward_samples, "mlp backward: batch of %zu samples does not match the forward pass (%zu)",
               n_samples, mlp->forward_samples);
  SXEN_REQUIRE(n_samples == 0 || upstream_host != nullptr, "mlp backward: upstream pointer is null");
  if (n_samples == 0) return SXEN_OK;
  DeviceGuard guard(mlp->device);
  const size_t up_bytes = n_samples * static_cast<size_t>(mlp->cfg.output_width) * sizeof(double);
  const size_t ig_bytes = n_samples * static_cast<size_t>(mlp->cfg.input_width) * sizeof(double);
  if (sxen_status st = host_stage(mlp, 0, up_bytes)) return st;
  if (sxen_status st = host_stage(mlp, 1, ig_bytes)) return st;
  SXEN_CUDA(cudaMemcpy(mlp->host_stage[0], upstream_host, up_bytes, cudaMemcpyHostToDevice));
  if (sxen_status st = sxen_mlp_backward(mlp, static_cast<const double*>(mlp->host_stage[0]), n_samples, nullptr,
                                         static_cast<double*>(mlp->host_stage[1]), nullptr))
    return st;
  if (input_grad_host) SXEN_CUDA(cudaMemcpy(input_grad_host, mlp->host_stage[1], ig_bytes, cudaMemcpyDeviceToHost));
  else SXEN_CUDA(cudaStreamSynchronize(nullptr));
  return SXEN_OK;
}

sxen_status sxen_mlp_fused_view(sxen_mlp* mlp, float** params, double** grads, long long** grads_fixed, int32_t* precision) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  *params = mlp->params;
  *grads = mlp->grads;
  *grads_fixed = mlp->grads_fixed;
  *precision = mlp->precision;
  if (!mlp->loss_scratch) {
    DeviceGuard guard(mlp->device);
    SXEN_CUDA(cudaMalloc(&mlp->loss_scratch, sizeof(double)));
  }
  mlp->forward_done = false;  // no activations are kept: a separate Mlp::backward would be a logic error
  return SXEN_OK;
}

sxen_status sxen_mlp_fused_fold(sxen_mlp* mlp, double* loss_sum_dev, int ctas, void* stream) {
  if (!mlp->grads_fixed) return SXEN_OK;
  cudaStream_t st = as_stream(stream);
  fold_fixed_kernel<<<grid_for(mlp->param_count), 256, 0, st>>>(mlp->grads, mlp->grads_fixed, mlp->param_count);
  sum_parts_kernel<<<1, 1, 0, st>>>(loss_sum_dev, reinterpret_cast<const double*>(mlp->grads_fixed + mlp->param_count), ctas);
  SXEN_CUDA(cudaGetLastError());
  count_launch(2);
  return SXEN_OK;
}

sxen_status sxen_mlp_set_reproducible(sxen_mlp* mlp, int32_t on) {
  SXEN_REQUIRE(mlp != nullptr, "mlp handle is null");
  DeviceGuard guard(mlp->device);
  if (on && !mlp->grads_fixed) {
    // + one double per CTA of the tensor-core head for its loss partial (persistent kernel: at most one CTA per SM)
    SXEN_CUDA(cudaMalloc(&mlp->grads_fixed, (mlp->param_count + 1024) * sizeof(long long)));
    SXEN_CUDA(cudaMemset(mlp->grads_fixed, 0, (mlp->param_count + 1024) * sizeof(long long)));
  } else if (!on && mlp->grads_fixed) {
    SXEN_CUDA(cudaDeviceSynchronize());
    cudaFree(mlp->grads_fixed);
    mlp->grads_fixed = nullptr;
  }
  return SXEN_OK;
}

sxen_status sxen_mlp_activations_dev(sxen_mlp* mlp, float** out_dev, size_t* act_width, size_t* output_offset) {
  SXEN_REQUIRE(mlp != nullptr && out_dev != nullptr, "null argument");
  const MlpShape s = shape_of(mlp);
  *out_dev = mlp->acts;
  if (act_width) *act_width = s.act_width;
  if (output_offset) *output_offset = s.a_off[s.layers];
  return SXEN_OK;
}

sxen_status sxen_mse_loss(const float* pred_dev, size_t pred_stride, const void* targets_dev, sxen_coord_type target_type,
                          int32_t out_w, size_t n_samples, size_t global_batch, double* upstream_dev,
                          double* sample_loss_dev, double* loss_sum_dev, void* stream) {
  SXEN_REQUIRE(out_w >= 1, "mse: output width must be >= 1");
  SXEN_REQUIRE(n_samples == 0 || (pred_dev && targets_dev && upstream_dev && sample_loss_dev), "mse: null pointer");
  SXEN_REQUIRE(global_batch >= 1, "mse: global batch must be >= 1");
  if (n_samples == 0) return SXEN_OK;
  cudaStream_t st = as_stream(stream);
  // upstream_scale = 2 / targets.size() with targets.size() = B * out_w of the WHOLE batch (src/trainer.cpp:26-27)
  const double scale = 2.0 / static_cast<double>(global_batch * static_cast<size_t>(out_w));
  if (target_type == SXEN_COORD_F32) {
    mse_kernel<float><<<grid_for(n_samples), 256, 0, st>>>(pred_dev, pred_stride, 0, static_cast<const float*>(targets_dev),
                                                           out_w, n_samples, scale, upstream_dev, sample_loss_dev);
  } else {
    mse_kernel<double><<<grid_for(n_samples), 256, 0, st>>>(pred_dev, pred_stride, 0, static_cast<const double*>(targets_dev),
                                                            out_w, n_samples, scale, upstream_dev, sample_loss_dev);
  }
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (loss_sum_dev) {
    sum_kernel<<<1, 1024, 0, st>>>(sample_loss_dev, n_samples, loss_sum_dev);
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  return SXEN_OK;
}

}  // extern "C"
