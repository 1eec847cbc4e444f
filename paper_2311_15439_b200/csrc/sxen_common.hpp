// sxen_common.hpp -- host-side plumbing shared by the C-ABI translation units: error strings, CUDA call checks,
// handle definitions.  Nothing here is exported; the exported surface is include/sxen_cuda.h.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/sxen_cuda.h"

namespace sxen_host {

std::string& last_error();
sxen_status fail(sxen_status st, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
sxen_status cuda_fail(cudaError_t e, const char* what);
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

#define SXEN_CUDA(call)                                                   \
  do {                                                                    \
    cudaError_t e__ = (call);                                             \
    if (e__ != cudaSuccess) return ::sxen_host::cuda_fail(e__, #call);    \
  } while (0)

#define SXEN_REQUIRE(cond, ...)                                           \
  do {                                                                    \
    if (!(cond)) return ::sxen_host::fail(SXEN_INVALID_ARGUMENT, __VA_ARGS__); \
  } while (0)

// RAII device switch: handles live on one device, callers may have another current.
struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// sxen_mlp_precision -> the tensor-core kernels' `precise` argument (products per operand pair: 0 one, 1 three, 2 four)
inline int sxen_tc_products(int precision) {
  return precision == SXEN_MLP_TENSOR_BF16X3 ? 1 : precision == SXEN_MLP_TENSOR_BF16X4 ? 2 : 0;
}

}  // namespace sxen_host

struct sxen_encoder {
  sxen_encoder_config cfg{};
  int device = 0;
  std::vector<uint32_t> res;          // per-level resolution (src/encoding.cpp:159-162)
  double skew = 0.0, scale = 1.0;     // F_n, S_n
  float* tables = nullptr;            // L x T x F
  unsigned long long* status = nullptr;       // device: [0] first bad sample, [1] oob count
  unsigned long long* status_host = nullptr;  // pinned mirror
  sxen_tuning tuning{};
  uint64_t touched = 0;               // LookupCounters::touched_vertices
  uint64_t oob_base = 0;              // oob counted before the last device reset
  // staging for the *_host entry points: a three-stage pipeline (copy-in stream | compute stream | copy-out stream) over
  // kStages rotating slots of stage_samples samples each
  static constexpr int kStages = 3;
  size_t stage_samples = 0;
  double* stage_x[kStages] = {nullptr, nullptr, nullptr};      // coordinates
  float* stage_up[kStages] = {nullptr, nullptr, nullptr};      // upstream as f32
  double* stage_up64[kStages] = {nullptr, nullptr, nullptr};   // upstream as the host's f64 (allocated on first use)
  float* stage_out[kStages] = {nullptr, nullptr, nullptr};     // features
  cudaStream_t stage_stream[3] = {nullptr, nullptr, nullptr};  // [0] copy-in, [1] compute, [2] copy-out
  cudaEvent_t stage_in[kStages] = {nullptr, nullptr, nullptr};    // slot's inputs have arrived
  cudaEvent_t stage_done[kStages] = {nullptr, nullptr, nullptr};  // slot's kernels have finished
  cudaEvent_t stage_back[kStages] = {nullptr, nullptr, nullptr};  // slot's features have left
  size_t level_floats() const { return static_cast<size_t>(cfg.table_size) * static_cast<size_t>(cfg.features); }
  int vertices() const { return cfg.backend == SXEN_BACKEND_SIMPLEX ? cfg.dim + 1 : (1 << cfg.dim); }
};

struct sxen_grad {
  int device = 0;
  int levels = 0, features = 0;
  uint32_t table_size = 0;
  float* values = nullptr;  // L x T x F, untouched rows carry -0.0f in feature 0
  long long* fixed = nullptr;  // reproducible mode (sxen_grad_set_reproducible): the same sums in 64-bit fixed point, units of 2^-52
  // Coarse simplex levels (few lattice vertices, every sample's atomics land on them) accumulate into 2^shift dense
  // replicas [replica][vertex][F] that the backward launch folds into `values` before it returns (sxen_encode.cuh).
  float* coarse = nullptr;
  size_t coarse_floats = 0;
  std::vector<uint32_t> coarse_offset, coarse_verts;  // per level
  std::vector<int32_t> coarse_shift;                  // per level, -1 = none
  int dim = 0;
  std::vector<uint32_t> res;                          // lattice the replicas were laid out for
  size_t count() const { return static_cast<size_t>(levels) * table_size * static_cast<size_t>(features); }
};

struct sxen_sparse_adam {
  int device = 0;
  int levels = 0, features = 0;
  uint32_t table_size = 0;
  double* m = nullptr;
  double* v = nullptr;
  int64_t t = 0;
  unsigned long long* status = nullptr;       // device: first non-finite gradient element
  unsigned long long* status_host = nullptr;  // pinned
};

struct sxen_adam {
  int device = 0;
  size_t size = 0;
  double* m = nullptr;
  double* v = nullptr;
  int64_t t = 0;
  unsigned long long* status = nullptr;
  unsigned long long* status_host = nullptr;
};

// Update steps of a QUEUED training step (sxen_trainer_step_enqueue): the kernels return at once when *gate_dev holds a
// slot index (that step's loss was non-finite: the reference throws before updating, src/trainer.cpp:121-123).
// gate_dev == nullptr: the public sxen_sparse_adam_step / sxen_adam_step.
sxen_status sxen_sparse_adam_step_gated(sxen_sparse_adam* opt, sxen_encoder* enc, sxen_grad* grad, const sxen_adam_config* cfg,
                                        int32_t clear_grad, const unsigned long long* gate_dev, void* stream);
sxen_status sxen_adam_step_gated(sxen_adam* opt, float* params_dev, const void* grads_dev, sxen_coord_type grad_type,
                                 size_t size, const sxen_adam_config* cfg, const unsigned long long* gate_dev, void* stream);

// The same update driven by the batch (sxen_abi.cu): O(n_samples * L * V) instead of O(L * T); valid when every touched
// row of `grad` comes from the backward of exactly these samples.  sxen_sparse_adam_walk_pays: the size rule.
bool sxen_sparse_adam_walk_pays(const sxen_encoder* enc, size_t n_samples);
sxen_status sxen_sparse_adam_step_walk(sxen_sparse_adam* opt, sxen_encoder* enc, sxen_grad* grad, const void* x_dev,
                                       sxen_coord_type type, size_t n_samples, const sxen_adam_config* cfg,
                                       const unsigned long long* gate_dev, void* stream);

// Encode / encode_backward over feature rows `row_stride` floats apart (sxen_abi.cu), for the trainer's [encoding | aux] rows.
sxen_status sxen_encoder_encode_strided(sxen_encoder* enc, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                        float* out_dev, int row_stride, void* stream);
sxen_status sxen_encoder_encode_backward_strided(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                 const float* upstream_dev, int row_stride, size_t n_samples,
                                                 sxen_grad* grad, int first_level, int level_count, void* stream);

// sxen_mlp_forward_backward with d(loss)/d(input) also as doubles (exact head; NULL = not wanted), sxen_mlp.cu
extern "C" sxen_status sxen_mlp_forward_backward_ex(sxen_mlp* mlp, const float* input_dev, const void* targets_dev,
                                         sxen_coord_type target_type, size_t n_samples, size_t global_batch, float* pred_dev,
                                         float* input_grad_dev, double* input_grad_f64_dev, double* loss_sum_dev, void* stream);
// encode_backward with the upstream ALSO as doubles (reproducible mode: the fixed-point sums take the fp64 product)
sxen_status sxen_encoder_encode_backward_strided64(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                   const float* upstream_dev, const double* upstream64_dev, int row_stride,
                                                   size_t n_samples, sxen_grad* grad, int first_level, int level_count,
                                                   void* stream);

// ---- the fused training kernel (sxen_train_fused.cu) and what it needs from the encoder (sxen_abi.cu)
namespace sxen_dev { struct EncodeArgs; }
bool sxen_train_fused_supported(const sxen_encoder_config& ec, const sxen_mlp_config& mc);
// fills the argument block of one launch over ALL levels of `enc` for a backward into `grad` (geometry, replicas, policies)
sxen_status sxen_encoder_fused_args(sxen_encoder* enc, sxen_grad* grad, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                    sxen_dev::EncodeArgs* out);
// the coarse-level fold of that launch + the encoder's touched counter (forward + backward walks)
sxen_status sxen_encoder_fused_finish(sxen_encoder* enc, const sxen_dev::EncodeArgs& args, void* stream);
sxen_status sxen_train_fused_run(const sxen_dev::EncodeArgs& e, int dim, const float* params, const void* targets, int target_f32,
                                 double* mlp_grad, double* loss_sum, long long* grad_fixed, int out_w, size_t global_batch,
                                 int precise, cudaStream_t stream, int* used_ctas);
// sxen_mlp.cu: the pieces of an Mlp handle the fused kernel works on, and the fold of its reproducible partials
extern "C" sxen_status sxen_mlp_fused_view(sxen_mlp* mlp, float** params, double** grads, long long** grads_fixed, int32_t* precision);
extern "C" sxen_status sxen_mlp_fused_fold(sxen_mlp* mlp, double* loss_sum_dev, int ctas, void* stream);
