// sxen_optim.cu -- Adam updates on the device (reference: /root/reference/proj/src/optimizer.cpp).
//
// The arithmetic is the reference's, operation for operation, in fp64 with explicit round-to-nearest intrinsics so
// nvcc cannot contract mul+add into an FMA (the reference's x86-64 build does not fuse either): given the same
// gradient values the updated parameters and moments are bit-identical to AdamState::step / SparseAdamState::step.
#include <cmath>

#include "sxen_adam.cuh"
#include "sxen_common.hpp"

using namespace sxen_host;

namespace {

using sxen_dev::AdamScalars;
using sxen_dev::adam_delta;
using sxen_dev::kUntouchedBits;
constexpr unsigned long long kNoBad = sxen_dev::kAdamNoBad;

// SparseAdamState::step, src/optimizer.cpp:54-84.  One thread per table row; a row is visited iff the accumulator
// touched it (feature 0 != -0.0f), zero gradients included; untouched rows' moments do not decay.
// `fixed` != nullptr (reproducible mode, sxen_grad_set_reproducible): the gradient is the 64-bit fixed-point sum (units of
// 2^-52, order-free); the fp32 accumulator still says which rows were touched and carries the NaN / range check -- a sum
// of 2^10 or more in magnitude does not fit the fixed-point word and is reported like a non-finite gradient.
__device__ __forceinline__ bool usable(double g_f32, bool repro) {
  return isfinite(g_f32) && (!repro || fabs(g_f32) < 1024.0);
}

__global__ void sparse_adam_kernel(float* __restrict__ tables, float* __restrict__ grads, double* __restrict__ m,
                                   double* __restrict__ v, size_t rows, int features, AdamScalars c, int clear_grad,
                                   unsigned long long* __restrict__ status, const unsigned long long* __restrict__ gate,
                                   long long* __restrict__ fixed) {
  if (gate != nullptr && *gate != kNoBad) return;  // a queued step whose loss was non-finite applies no update
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t r = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const size_t base = r * static_cast<size_t>(features);
    if (__float_as_uint(grads[base]) == kUntouchedBits) continue;
    for (int f = 0; f < features; ++f) {
      const size_t i = base + static_cast<size_t>(f);
      double g = static_cast<double>(grads[i]);
      const bool ok = usable(g, fixed != nullptr);
      if (fixed != nullptr) {
        g = __dmul_rn(static_cast<double>(fixed[i]), 0x1p-52);
        if (clear_grad) fixed[i] = 0;
      }
      if (!ok) {
        atomicMin(status, static_cast<unsigned long long>(i));  // TrainingError, src/optimizer.cpp:73-76
        // the reference aborts the run here; this ABI can be called again, so the row must not keep its NaN/Inf (the next
        // backward would add into it): with clear_grad the whole row is re-armed like every other visited row
        if (clear_grad) grads[i] = __uint_as_float(kUntouchedBits);
        continue;
      }
      double mi = m[i], vi = v[i];
      const double d = adam_delta(g, mi, vi, c);
      m[i] = mi;
      v[i] = vi;
      tables[i] = static_cast<float>(__dadd_rn(static_cast<double>(tables[i]), d));
      if (clear_grad) grads[i] = __uint_as_float(kUntouchedBits);
    }
  }
}

// F == 2 fast path: 8-byte gradient/table rows, 16-byte moment rows, one vector access each.
__global__ void sparse_adam_f2_kernel(float2* __restrict__ tables, float2* __restrict__ grads, double2* __restrict__ m,
                                      double2* __restrict__ v, size_t rows, AdamScalars c, int clear_grad,
                                      unsigned long long* __restrict__ status, const unsigned long long* __restrict__ gate,
                                      longlong2* __restrict__ fixed) {
  if (gate != nullptr && *gate != kNoBad) return;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t r = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const float2 g2 = grads[r];
    if (__float_as_uint(g2.x) == kUntouchedBits) continue;
    double gx = static_cast<double>(g2.x), gy = static_cast<double>(g2.y);
    const bool okx = usable(gx, fixed != nullptr), oky = usable(gy, fixed != nullptr);
    if (fixed != nullptr) {
      const longlong2 q = fixed[r];
      gx = __dmul_rn(static_cast<double>(q.x), 0x1p-52);
      gy = __dmul_rn(static_cast<double>(q.y), 0x1p-52);
      if (clear_grad) fixed[r] = make_longlong2(0, 0);
    }
    if (!okx || !oky) {
      atomicMin(status, static_cast<unsigned long long>(2 * r + (okx ? 1 : 0)));
      if (clear_grad) grads[r] = make_float2(__uint_as_float(kUntouchedBits), __uint_as_float(kUntouchedBits));  // (see above)
      continue;
    }
    double2 mm = m[r], vv = v[r];
    float2 t = tables[r];
    const double dx = adam_delta(gx, mm.x, vv.x, c);
    const double dy = adam_delta(gy, mm.y, vv.y, c);
    m[r] = mm;
    v[r] = vv;
    t.x = static_cast<float>(__dadd_rn(static_cast<double>(t.x), dx));
    t.y = static_cast<float>(__dadd_rn(static_cast<double>(t.y), dy));
    tables[r] = t;
    if (clear_grad) grads[r] = make_float2(__uint_as_float(kUntouchedBits), __uint_as_float(kUntouchedBits));
  }
}

// AdamState::step, src/optimizer.cpp:25-41
template <typename G>
__global__ void dense_adam_kernel(float* __restrict__ params, const G* __restrict__ grads, double* __restrict__ m,
                                  double* __restrict__ v, size_t n, AdamScalars c,
                                  unsigned long long* __restrict__ status, const unsigned long long* __restrict__ gate) {
  if (gate != nullptr && *gate != kNoBad) return;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double g = static_cast<double>(grads[i]);
    if (!isfinite(g)) {
      atomicMin(status, static_cast<unsigned long long>(i));  // TrainingError, src/optimizer.cpp:35-37
      continue;
    }
    double mi = m[i], vi = v[i];
    const double d = adam_delta(g, mi, vi, c);
    m[i] = mi;
    v[i] = vi;
    params[i] = static_cast<float>(__dadd_rn(static_cast<double>(params[i]), d));
  }
}

}  // namespace

sxen_dev::AdamScalars sxen_adam_scalars(const sxen_adam_config& cfg, int64_t t) {
  AdamScalars c;
  c.beta1 = cfg.beta1;
  c.beta2 = cfg.beta2;
  c.one_minus_beta1 = 1.0 - cfg.beta1;
  c.one_minus_beta2 = 1.0 - cfg.beta2;
  c.neg_lr = -cfg.lr;
  c.epsilon = cfg.epsilon;
  c.bc1 = 1.0 - std::pow(cfg.beta1, static_cast<double>(t));  // src/optimizer.cpp:31-32,65-66
  c.bc2 = 1.0 - std::pow(cfg.beta2, static_cast<double>(t));
  return c;
}

namespace {

AdamScalars scalars(const sxen_adam_config& cfg, int64_t t) { return sxen_adam_scalars(cfg, t); }

int grid_for(size_t n) {
  size_t b = (n + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return static_cast<int>(b < 1 ? 1 : b);
}

template <class H>
sxen_status alloc_status(H* h) {
  SXEN_CUDA(cudaMalloc(&h->status, sizeof(unsigned long long)));
  SXEN_CUDA(cudaHostAlloc(&h->status_host, sizeof(unsigned long long), cudaHostAllocDefault));
  const unsigned long long none = kNoBad;
  SXEN_CUDA(cudaMemcpy(h->status, &none, sizeof(none), cudaMemcpyHostToDevice));
  return SXEN_OK;
}

template <class H>
sxen_status check_status(H* h, cudaStream_t stream, const char* what) {
  SXEN_CUDA(cudaMemcpyAsync(h->status_host, h->status, sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
  SXEN_CUDA(cudaStreamSynchronize(stream));
  if (*h->status_host != kNoBad) {
    const unsigned long long bad = *h->status_host;
    const unsigned long long none = kNoBad;
    SXEN_CUDA(cudaMemcpyAsync(h->status, &none, sizeof(none), cudaMemcpyHostToDevice, stream));
    SXEN_CUDA(cudaStreamSynchronize(stream));
    return fail(SXEN_TRAINING_ERROR, "%s %llu", what, bad);
  }
  return SXEN_OK;
}

}  // namespace

extern "C" {

sxen_status sxen_adam_config_default(sxen_adam_config* cfg) {
  SXEN_REQUIRE(cfg != nullptr, "config pointer is null");
  *cfg = sxen_adam_config{1e-3, 0.9, 0.99, 1e-15};  // include/sxen/optimizer.hpp:13-18
  return SXEN_OK;
}

sxen_status sxen_sparse_adam_create(const sxen_encoder* enc, sxen_sparse_adam** out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  DeviceGuard guard(enc->device);
  sxen_sparse_adam* o = new sxen_sparse_adam();
  o->device = enc->device;
  o->levels = enc->cfg.levels;
  o->features = enc->cfg.features;
  o->table_size = enc->cfg.table_size;
  const size_t bytes = static_cast<size_t>(o->levels) * o->table_size * static_cast<size_t>(o->features) * sizeof(double);
  cudaError_t err = cudaMalloc(&o->m, bytes);
  if (err == cudaSuccess) err = cudaMalloc(&o->v, bytes);
  if (err == cudaSuccess) err = cudaMemset(o->m, 0, bytes);
  if (err == cudaSuccess) err = cudaMemset(o->v, 0, bytes);
  if (err != cudaSuccess) {
    sxen_sparse_adam_destroy(o);
    return cuda_fail(err, "sxen_sparse_adam_create allocation");
  }
  if (sxen_status st = alloc_status(o)) {
    sxen_sparse_adam_destroy(o);
    return st;
  }
  *out = o;
  return SXEN_OK;
}

sxen_status sxen_sparse_adam_destroy(sxen_sparse_adam* opt) {
  if (!opt) return SXEN_OK;
  DeviceGuard guard(opt->device);
  cudaFree(opt->m);
  cudaFree(opt->v);
  cudaFree(opt->status);
  cudaFreeHost(opt->status_host);
  delete opt;
  return SXEN_OK;
}

sxen_status sxen_sparse_adam_step_count(const sxen_sparse_adam* opt, int64_t* out) {
  SXEN_REQUIRE(opt != nullptr && out != nullptr, "null argument");
  *out = opt->t;
  return SXEN_OK;
}

sxen_status sxen_sparse_adam_step(sxen_sparse_adam* opt, sxen_encoder* enc, sxen_grad* grad, const sxen_adam_config* cfg,
                                  int32_t clear_grad, void* stream) {
  return sxen_sparse_adam_step_gated(opt, enc, grad, cfg, clear_grad, nullptr, stream);
}

}  // extern "C"

sxen_status sxen_sparse_adam_step_gated(sxen_sparse_adam* opt, sxen_encoder* enc, sxen_grad* grad, const sxen_adam_config* cfg,
                                        int32_t clear_grad, const unsigned long long* gate_dev, void* stream) {
  SXEN_REQUIRE(opt != nullptr && enc != nullptr && grad != nullptr && cfg != nullptr, "null argument");
  // src/optimizer.cpp:57-61
  SXEN_REQUIRE(enc->cfg.levels == opt->levels && enc->cfg.features == opt->features &&
                   enc->cfg.table_size == opt->table_size && grad->levels == opt->levels &&
                   grad->features == opt->features && grad->table_size == opt->table_size &&
                   enc->device == opt->device && grad->device == opt->device,
               "sparse adam step: encoder/gradient shape mismatch");
  DeviceGuard guard(opt->device);
  ++opt->t;  // the step counter is global: it advances even for rows that are never touched (src/optimizer.cpp:64)
  const AdamScalars c = scalars(*cfg, opt->t);
  const size_t rows = static_cast<size_t>(opt->levels) * opt->table_size;
  if (opt->features == 2) {
    sparse_adam_f2_kernel<<<grid_for(rows), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<float2*>(enc->tables), reinterpret_cast<float2*>(grad->values),
        reinterpret_cast<double2*>(opt->m), reinterpret_cast<double2*>(opt->v), rows, c, clear_grad, opt->status, gate_dev,
        reinterpret_cast<longlong2*>(grad->fixed));
  } else {
    sparse_adam_kernel<<<grid_for(rows), 256, 0, as_stream(stream)>>>(enc->tables, grad->values, opt->m, opt->v, rows,
                                                                      opt->features, c, clear_grad, opt->status, gate_dev,
                                                                      grad->fixed);
  }
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

extern "C" {

sxen_status sxen_sparse_adam_check(sxen_sparse_adam* opt, void* stream) {
  SXEN_REQUIRE(opt != nullptr, "optimizer handle is null");
  DeviceGuard guard(opt->device);
  return check_status(opt, as_stream(stream), "non-finite table gradient at flat element");
}

sxen_status sxen_sparse_adam_download(const sxen_sparse_adam* opt, int32_t level, double* m_host, double* v_host) {
  SXEN_REQUIRE(opt != nullptr && m_host != nullptr && v_host != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < opt->levels, "sparse adam: level out of range");
  DeviceGuard guard(opt->device);
  const size_t per = static_cast<size_t>(opt->table_size) * static_cast<size_t>(opt->features);
  SXEN_CUDA(cudaMemcpy(m_host, opt->m + static_cast<size_t>(level) * per, per * sizeof(double), cudaMemcpyDeviceToHost));
  SXEN_CUDA(cudaMemcpy(v_host, opt->v + static_cast<size_t>(level) * per, per * sizeof(double), cudaMemcpyDeviceToHost));
  return SXEN_OK;
}

sxen_status sxen_adam_create(size_t size, int32_t device, sxen_adam** out) {
  SXEN_REQUIRE(out != nullptr, "null argument");
  *out = nullptr;
  int ndev = 0;
  SXEN_CUDA(cudaGetDeviceCount(&ndev));
  SXEN_REQUIRE(device >= 0 && device < ndev, "device %d out of range (%d visible)", device, ndev);
  DeviceGuard guard(device);
  sxen_adam* o = new sxen_adam();
  o->device = device;
  o->size = size;
  const size_t bytes = (size ? size : 1) * sizeof(double);
  cudaError_t err = cudaMalloc(&o->m, bytes);
  if (err == cudaSuccess) err = cudaMalloc(&o->v, bytes);
  if (err == cudaSuccess) err = cudaMemset(o->m, 0, bytes);
  if (err == cudaSuccess) err = cudaMemset(o->v, 0, bytes);
  if (err != cudaSuccess) {
    sxen_adam_destroy(o);
    return cuda_fail(err, "sxen_adam_create allocation");
  }
  if (sxen_status st = alloc_status(o)) {
    sxen_adam_destroy(o);
    return st;
  }
  *out = o;
  return SXEN_OK;
}

sxen_status sxen_adam_destroy(sxen_adam* opt) {
  if (!opt) return SXEN_OK;
  DeviceGuard guard(opt->device);
  cudaFree(opt->m);
  cudaFree(opt->v);
  cudaFree(opt->status);
  cudaFreeHost(opt->status_host);
  delete opt;
  return SXEN_OK;
}

sxen_status sxen_adam_step_count(const sxen_adam* opt, int64_t* out) {
  SXEN_REQUIRE(opt != nullptr && out != nullptr, "null argument");
  *out = opt->t;
  return SXEN_OK;
}

sxen_status sxen_adam_step(sxen_adam* opt, float* params_dev, const void* grads_dev, sxen_coord_type grad_type,
                           size_t size, const sxen_adam_config* cfg, void* stream) {
  return sxen_adam_step_gated(opt, params_dev, grads_dev, grad_type, size, cfg, nullptr, stream);
}

}  // extern "C"

sxen_status sxen_adam_step_gated(sxen_adam* opt, float* params_dev, const void* grads_dev, sxen_coord_type grad_type,
                                 size_t size, const sxen_adam_config* cfg, const unsigned long long* gate_dev, void* stream) {
  SXEN_REQUIRE(opt != nullptr && cfg != nullptr, "null argument");
  // src/optimizer.cpp:27-29
  SXEN_REQUIRE(size == opt->size, "adam step: parameter/gradient size mismatch");
  SXEN_REQUIRE(size == 0 || (params_dev != nullptr && grads_dev != nullptr), "adam step: null parameter or gradient pointer");
  DeviceGuard guard(opt->device);
  ++opt->t;
  if (size == 0) return SXEN_OK;
  const AdamScalars c = scalars(*cfg, opt->t);
  if (grad_type == SXEN_COORD_F32) {
    dense_adam_kernel<float><<<grid_for(size), 256, 0, as_stream(stream)>>>(
        params_dev, static_cast<const float*>(grads_dev), opt->m, opt->v, size, c, opt->status, gate_dev);
  } else {
    dense_adam_kernel<double><<<grid_for(size), 256, 0, as_stream(stream)>>>(
        params_dev, static_cast<const double*>(grads_dev), opt->m, opt->v, size, c, opt->status, gate_dev);
  }
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

extern "C" {

sxen_status sxen_adam_check(sxen_adam* opt, void* stream) {
  SXEN_REQUIRE(opt != nullptr, "optimizer handle is null");
  DeviceGuard guard(opt->device);
  return check_status(opt, as_stream(stream), "non-finite gradient at parameter");
}

}  // extern "C"
