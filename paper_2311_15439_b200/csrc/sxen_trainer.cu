// sxen_trainer.cu -- one training step of train_field on the device (/root/reference/proj/src/trainer.cpp:94-136):
//   gradient pass  = run_chunk over this rank's contiguous chunk of the batch (:20-49): encode -> Mlp::forward -> MSE and
//                    upstream = 2e/(B*out_w) with B the GLOBAL batch -> Mlp::backward -> encode_backward
//   update         = SparseAdamState::step on the tables (touched rows only) + AdamState::step on the MLP (:129-130)
// The two halves are separate entry points so a multi-GPU host can all-reduce the gradient buffers in between
// (the reference merges its workers' accumulators at exactly that point, :125-128).
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "sxen_common.hpp"
#include "sxen_encode.cuh"

using namespace sxen_host;

struct sxen_trainer {
  sxen_encoder* enc = nullptr;
  sxen_mlp* mlp = nullptr;
  int device = 0;
  sxen_grad* grad = nullptr;
  sxen_sparse_adam* table_opt = nullptr;
  sxen_adam* mlp_opt = nullptr;
  size_t capacity = 0;           // samples the workspace holds
  size_t head_samples = 0;       // samples whose input gradient the last accumulate_head left in the workspace
  float* features = nullptr;     // N x L*F
  float* input_grad = nullptr;   // N x L*F
  double* input_grad64 = nullptr; // N x L*F, reproducible mode with the exact head: the same gradient as doubles
  int fused_mode = 0;            // sxen_trainer_set_fused: 0 = three kernels (default: they are faster), 1 = the fused
                                 // kernel (error if the shapes do not allow it), -1 = fused whenever the shapes allow
  bool reproducible = false;
  bool have_grad64 = false;      // the last accumulate_head filled input_grad64
  double* upstream = nullptr;    // N x out_w
  double* sample_loss = nullptr; // N
  double* loss_sum = nullptr;    // device scalar: sum of per-sample losses accumulated since the last update
  double* loss_host = nullptr;   // pinned
  // queued steps (sxen_trainer_step_enqueue / _collect): one loss per step, read back by the collect call
  double* loss_ring = nullptr;       // device, kLossRing slots
  double* loss_ring_host = nullptr;  // pinned mirror
  unsigned long long* gate = nullptr;       // device: slot of the first queued step whose loss was non-finite, else ~0
  unsigned long long* gate_host = nullptr;  // pinned
  size_t pending = 0;                // queued steps not collected yet
  bool foreign_grads = false;        // the accumulators may hold rows of batches other than the current step's
  int32_t out_w = 0, enc_w = 0;
  int32_t aux_dims = 0, in_w = 0;    // TrainConfig::aux_dims; MLP input width = enc_w + aux_dims
  const void* aux = nullptr;         // caller-owned N x aux_dims pass-through inputs of the next batch (sxen_trainer_set_aux)
  sxen_coord_type aux_type = SXEN_COORD_F64;
  uint64_t mlp_params = 0;
  // batch-sharded steps (sxen_trainer_set_comm / _step_sharded): the exchange runs on a second stream behind events
  sxen_comm* comm = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_compute = nullptr, ev_comm = nullptr;
};

namespace {

constexpr size_t kLossRing = 4096;
constexpr unsigned long long kNoFailure = ~0ULL;

// The loss half of train_field's step (src/trainer.cpp:118-123) for a queued step: loss = sum / (B * out_w) goes to the
// step's slot, a non-finite loss closes the gate (the update kernels of this and every later queued step then return
// without touching anything, as the reference throws before its optimizer steps), and the sum is re-armed.
// The encoder's rejected-sample word closes the gate too: check_input throws before anything is computed
// (src/encoding.cpp:183-194), so a batch with a coordinate outside [0,1] must not reach the optimizers either.
__global__ void loss_record_kernel(double* __restrict__ loss_sum, double* __restrict__ ring, unsigned long long slot,
                                   double denom, unsigned long long* __restrict__ gate,
                                   const unsigned long long* __restrict__ rejected_sample) {
  const double loss = __ddiv_rn(*loss_sum, denom);
  ring[slot] = loss;
  if (!isfinite(loss) || *rejected_sample != kNoFailure) atomicMin(gate, slot);
  *loss_sum = 0.0;
}

// sharded steps: 1.0 when this rank's encoder rejected a coordinate in the batch (summed over the ranks with the loss)
__global__ void reject_flag_kernel(double* __restrict__ flag, const unsigned long long* __restrict__ rejected_sample) {
  *flag = (*rejected_sample != kNoFailure) ? 1.0 : 0.0;
}

// src/trainer.cpp:32-35: the aux inputs follow the encoding in every MLP input row, narrowed to float
template <typename T>
__global__ void aux_fill_kernel(float* __restrict__ rows, int row_stride, int first_col, const T* __restrict__ aux,
                                int aux_dims, size_t n) {
  const size_t e = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= n * static_cast<size_t>(aux_dims)) return;
  const size_t s = e / static_cast<size_t>(aux_dims);
  const int a = static_cast<int>(e - s * static_cast<size_t>(aux_dims));
  rows[s * static_cast<size_t>(row_stride) + static_cast<size_t>(first_col + a)] = static_cast<float>(aux[e]);
}

sxen_status ensure_workspace(sxen_trainer* t, size_t n) {
  if (n <= t->capacity) return SXEN_OK;
  cudaFree(t->features);
  cudaFree(t->input_grad);
  cudaFree(t->input_grad64);
  cudaFree(t->upstream);
  cudaFree(t->sample_loss);
  t->input_grad64 = nullptr;
  t->features = t->input_grad = nullptr;
  t->upstream = t->sample_loss = nullptr;
  t->capacity = 0;
  SXEN_CUDA(cudaMalloc(&t->features, n * static_cast<size_t>(t->in_w) * sizeof(float)));
  SXEN_CUDA(cudaMalloc(&t->input_grad, n * static_cast<size_t>(t->in_w) * sizeof(float)));
  if (t->reproducible) SXEN_CUDA(cudaMalloc(&t->input_grad64, n * static_cast<size_t>(t->in_w) * sizeof(double)));
  SXEN_CUDA(cudaMalloc(&t->upstream, n * static_cast<size_t>(t->out_w) * sizeof(double)));
  SXEN_CUDA(cudaMalloc(&t->sample_loss, (n + 1) * sizeof(double)));
  t->capacity = n;
  return SXEN_OK;
}

// table_opt.step then mlp_opt.step (src/trainer.cpp:129-130); the accumulators are cleared for the next step (:97-100).
// walk_coords != nullptr: the table step visits the rows of that batch only (sxen_sparse_adam_step_walk) -- the caller has
// checked that nothing else was accumulated.  gate: queued steps (nullptr otherwise).
sxen_status update_impl(sxen_trainer* t, const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam,
                        const void* walk_coords, sxen_coord_type coord_type, size_t n_samples,
                        const unsigned long long* gate, void* stream) {
  if (walk_coords != nullptr) {
    if (sxen_status st = sxen_sparse_adam_step_walk(t->table_opt, t->enc, t->grad, walk_coords, coord_type, n_samples,
                                                    table_adam, gate, stream))
      return st;
  } else if (sxen_status st = sxen_sparse_adam_step_gated(t->table_opt, t->enc, t->grad, table_adam, 1, gate, stream)) {
    return st;
  }
  double* mg = nullptr;
  float* mp = nullptr;
  sxen_mlp_grads_dev(t->mlp, &mg);
  sxen_mlp_params_dev(t->mlp, &mp);
  if (sxen_status st = sxen_adam_step_gated(t->mlp_opt, mp, mg, SXEN_COORD_F64, static_cast<size_t>(t->mlp_params), mlp_adam,
                                            gate, stream))
    return st;
  t->foreign_grads = false;
  return sxen_mlp_grad_clear(t->mlp, stream);
}

}  // namespace

extern "C" {

sxen_status sxen_trainer_create(sxen_encoder* enc, sxen_mlp* mlp, sxen_trainer** out) {
  return sxen_trainer_create_aux(enc, mlp, 0, out);
}

sxen_status sxen_trainer_create_aux(sxen_encoder* enc, sxen_mlp* mlp, int32_t aux_dims, sxen_trainer** out) {
  SXEN_REQUIRE(enc != nullptr && mlp != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  sxen_encoder_config ec;
  sxen_encoder_get_config(enc, &ec);
  sxen_mlp_config mc;
  if (sxen_status st = sxen_mlp_get_config(mlp, &mc)) return st;
  // src/trainer.cpp:59-65
  SXEN_REQUIRE(aux_dims >= 0, "train: aux_dims must be >= 0");
  SXEN_REQUIRE(mc.input_width == ec.levels * ec.features + aux_dims, "train: MLP input width %d != encoded width %d + aux %d",
               mc.input_width, ec.levels * ec.features, aux_dims);
  sxen_trainer* t = new sxen_trainer();
  t->enc = enc;
  t->mlp = mlp;
  t->device = enc->device;
  t->out_w = mc.output_width;
  t->enc_w = ec.levels * ec.features;
  t->aux_dims = aux_dims;
  t->in_w = t->enc_w + aux_dims;
  DeviceGuard guard(t->device);
  sxen_status st = sxen_grad_create(enc, &t->grad);
  if (st == SXEN_OK) st = sxen_sparse_adam_create(enc, &t->table_opt);
  if (st == SXEN_OK) st = sxen_mlp_parameter_count(mlp, &t->mlp_params);
  if (st == SXEN_OK) st = sxen_adam_create(static_cast<size_t>(t->mlp_params), t->device, &t->mlp_opt);
  // loss_sum[0] = sum of the per-sample losses; loss_sum[1] = ranks whose chunk held a rejected coordinate (sharded steps)
  if (st == SXEN_OK && cudaMalloc(&t->loss_sum, 2 * sizeof(double)) != cudaSuccess) st = fail(SXEN_CUDA_ERROR, "trainer: allocation failed");
  if (st == SXEN_OK && cudaMemset(t->loss_sum, 0, 2 * sizeof(double)) != cudaSuccess) st = fail(SXEN_CUDA_ERROR, "trainer: memset failed");
  if (st == SXEN_OK && cudaHostAlloc(&t->loss_host, 2 * sizeof(double), cudaHostAllocDefault) != cudaSuccess)
    st = fail(SXEN_CUDA_ERROR, "trainer: pinned allocation failed");
  if (st == SXEN_OK && (cudaMalloc(&t->loss_ring, kLossRing * sizeof(double)) != cudaSuccess ||
                        cudaMalloc(&t->gate, sizeof(unsigned long long)) != cudaSuccess ||
                        cudaMemset(t->gate, 0xff, sizeof(unsigned long long)) != cudaSuccess))
    st = fail(SXEN_CUDA_ERROR, "trainer: allocation failed");
  if (st == SXEN_OK && (cudaHostAlloc(&t->loss_ring_host, kLossRing * sizeof(double), cudaHostAllocDefault) != cudaSuccess ||
                        cudaHostAlloc(&t->gate_host, sizeof(unsigned long long), cudaHostAllocDefault) != cudaSuccess))
    st = fail(SXEN_CUDA_ERROR, "trainer: pinned allocation failed");
  if (st != SXEN_OK) {
    sxen_trainer_destroy(t);
    return st;
  }
  *out = t;
  return SXEN_OK;
}

sxen_status sxen_trainer_destroy(sxen_trainer* t) {
  if (!t) return SXEN_OK;
  DeviceGuard guard(t->device);
  sxen_grad_destroy(t->grad);
  sxen_sparse_adam_destroy(t->table_opt);
  sxen_adam_destroy(t->mlp_opt);
  cudaFree(t->features);
  cudaFree(t->input_grad);
  cudaFree(t->input_grad64);
  cudaFree(t->upstream);
  cudaFree(t->sample_loss);
  cudaFree(t->loss_sum);
  cudaFreeHost(t->loss_host);
  cudaFree(t->loss_ring);
  cudaFree(t->gate);
  cudaFreeHost(t->loss_ring_host);
  cudaFreeHost(t->gate_host);
  if (t->comm_stream) cudaStreamDestroy(t->comm_stream);
  if (t->ev_compute) cudaEventDestroy(t->ev_compute);
  if (t->ev_comm) cudaEventDestroy(t->ev_comm);
  delete t;
  return SXEN_OK;
}

sxen_status sxen_trainer_set_aux(sxen_trainer* t, const void* aux_dev, sxen_coord_type aux_type) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  SXEN_REQUIRE(aux_dev == nullptr || t->aux_dims > 0, "train: this trainer was created with aux_dims = 0");
  t->aux = aux_dev;
  t->aux_type = aux_type;
  return SXEN_OK;
}

sxen_status sxen_trainer_table_grad(sxen_trainer* t, sxen_grad** out) {
  SXEN_REQUIRE(t != nullptr && out != nullptr, "null argument");
  *out = t->grad;
  return SXEN_OK;
}

sxen_status sxen_trainer_loss_dev(sxen_trainer* t, double** out_dev) {
  SXEN_REQUIRE(t != nullptr && out_dev != nullptr, "null argument");
  *out_dev = t->loss_sum;
  return SXEN_OK;
}

sxen_status sxen_trainer_accumulate_head(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type,
                                         const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                         size_t global_batch, void* stream) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  SXEN_REQUIRE(global_batch >= 1 && n_samples <= global_batch, "train: local chunk (%zu) exceeds the global batch (%zu)",
               n_samples, global_batch);
  if (n_samples == 0) return SXEN_OK;
  DeviceGuard guard(t->device);
  if (sxen_status st = ensure_workspace(t, n_samples)) return st;
  if (t->aux_dims > 0 && t->aux == nullptr)
    return fail(SXEN_LOGIC_ERROR, "train: aux_dims = %d but no aux inputs were set for this batch (sxen_trainer_set_aux)",
                t->aux_dims);
  // encoder.encode (src/trainer.cpp:31) into the first enc_w columns of the MLP input rows, aux inputs behind (:32-35)
  if (sxen_status st = sxen_encoder_encode_strided(t->enc, coords_dev, coord_type, n_samples, t->features,
                                                   t->aux_dims > 0 ? t->in_w : 0, stream))
    return st;
  if (t->aux_dims > 0) {
    const size_t elems = n_samples * static_cast<size_t>(t->aux_dims);
    const unsigned blocks = static_cast<unsigned>((elems + 255) / 256);
    if (t->aux_type == SXEN_COORD_F32)
      aux_fill_kernel<float><<<blocks, 256, 0, as_stream(stream)>>>(t->features, t->in_w, t->enc_w,
                                                                   static_cast<const float*>(t->aux), t->aux_dims, n_samples);
    else
      aux_fill_kernel<double><<<blocks, 256, 0, as_stream(stream)>>>(t->features, t->in_w, t->enc_w,
                                                                    static_cast<const double*>(t->aux), t->aux_dims, n_samples);
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  // mlp.forward, loss + upstream, mlp.backward (:36-46): one fused call (tensor-core kernel or the exact chain)
  int32_t precision = SXEN_MLP_EXACT;
  sxen_mlp_get_precision(t->mlp, &precision);
  t->have_grad64 = t->reproducible && precision == SXEN_MLP_EXACT && t->input_grad64 != nullptr;
  if (sxen_status st = sxen_mlp_forward_backward_ex(t->mlp, t->features, targets_dev, target_type, n_samples, global_batch,
                                                    nullptr, t->input_grad, t->have_grad64 ? t->input_grad64 : nullptr,
                                                    t->loss_sum, stream))
    return st;
  t->head_samples = n_samples;
  t->foreign_grads = true;
  return SXEN_OK;
}

sxen_status sxen_trainer_accumulate_tables(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type,
                                           size_t n_samples, int32_t first_level, int32_t level_count, void* stream) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  if (n_samples == 0) return SXEN_OK;
  if (n_samples != t->head_samples)
    return fail(SXEN_LOGIC_ERROR, "train: accumulate_tables(%zu samples) without a matching accumulate_head (%zu)",
                n_samples, t->head_samples);
  DeviceGuard guard(t->device);
  // encoder.encode_backward on d(loss)/d(encoding) (:47), levels [first_level, first_level + level_count)
  return sxen_encoder_encode_backward_strided64(t->enc, coords_dev, coord_type, t->input_grad,
                                                t->have_grad64 ? t->input_grad64 : nullptr, t->aux_dims > 0 ? t->in_w : 0,
                                                n_samples, t->grad, first_level, level_count, stream);
}

// run_chunk as ONE kernel (sxen_train_fused.cu) when the shapes allow: simplex, F = 2, 16 levels, n in {2, 3}, the tensor-core
// head 32 -> 64 -> 64 -> <= 3, no aux inputs, default (fp32-atomic) table accumulation.  SXEN_FUSED_TRAIN=0 keeps the three
// kernels (a measuring aid).
static bool fused_step_applies(const sxen_trainer* t) {
  static const bool enabled = [] {
    const char* env = std::getenv("SXEN_FUSED_TRAIN");
    return env == nullptr || std::atoi(env) != 0;
  }();
  if (!enabled || t->fused_mode == 0 || t->aux_dims != 0 || t->grad->fixed != nullptr) return false;
  int32_t precision = SXEN_MLP_EXACT;
  sxen_mlp_get_precision(t->mlp, &precision);
  if (precision == SXEN_MLP_EXACT) return false;
  sxen_encoder_config ec;
  sxen_encoder_get_config(t->enc, &ec);
  sxen_mlp_config mc;
  sxen_mlp_get_config(t->mlp, &mc);
  return sxen_train_fused_supported(ec, mc);
}

static sxen_status accumulate_fused(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type, const void* targets_dev,
                                    sxen_coord_type target_type, size_t n_samples, size_t global_batch, void* stream) {
  SXEN_REQUIRE(global_batch >= 1 && n_samples <= global_batch, "train: local chunk (%zu) exceeds the global batch (%zu)",
               n_samples, global_batch);
  SXEN_REQUIRE(targets_dev != nullptr, "train: targets pointer is null");
  DeviceGuard guard(t->device);
  sxen_dev::EncodeArgs e;
  if (sxen_status st = sxen_encoder_fused_args(t->enc, t->grad, coords_dev, coord_type, n_samples, &e)) return st;
  float* params = nullptr;
  double* grads = nullptr;
  long long* fixed = nullptr;
  int32_t precision = 0;
  if (sxen_status st = sxen_mlp_fused_view(t->mlp, &params, &grads, &fixed, &precision)) return st;
  sxen_encoder_config ec;
  sxen_encoder_get_config(t->enc, &ec);
  int ctas = 0;
  if (sxen_status st = sxen_train_fused_run(e, ec.dim, params, targets_dev, target_type == SXEN_COORD_F32 ? 1 : 0, grads,
                                            t->loss_sum, fixed, t->out_w, global_batch,
                                            sxen_tc_products(precision), as_stream(stream), &ctas))
    return st;
  if (sxen_status st = sxen_mlp_fused_fold(t->mlp, t->loss_sum, ctas, stream)) return st;
  t->head_samples = 0;
  return sxen_encoder_fused_finish(t->enc, e, stream);
}

sxen_status sxen_trainer_accumulate(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type,
                                    const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                    size_t global_batch, void* stream) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  t->foreign_grads = true;  // (the whole-step entry points reset this around their own call)
  if (n_samples > 0 && fused_step_applies(t))
    return accumulate_fused(t, coords_dev, coord_type, targets_dev, target_type, n_samples, global_batch, stream);
  if (t->fused_mode == 1)
    return fail(SXEN_INVALID_ARGUMENT, "train: the fused kernel was required (sxen_trainer_set_fused) but does not cover this "
                                       "configuration (simplex, F=2, 16 levels, dim 2|3, tensor-core head 32-64-64-<=3, no aux, "
                                       "default accumulation)");
  if (sxen_status st = sxen_trainer_accumulate_head(t, coords_dev, coord_type, targets_dev, target_type, n_samples,
                                                    global_batch, stream))
    return st;
  if (n_samples == 0) return SXEN_OK;
  sxen_encoder_config ec;
  sxen_encoder_get_config(t->enc, &ec);
  return sxen_trainer_accumulate_tables(t, coords_dev, coord_type, n_samples, 0, ec.levels, stream);
}

sxen_status sxen_trainer_loss(sxen_trainer* t, size_t global_batch, double* loss_out, void* stream) {
  SXEN_REQUIRE(t != nullptr && loss_out != nullptr, "null argument");
  DeviceGuard guard(t->device);
  cudaStream_t s = as_stream(stream);
  SXEN_CUDA(cudaMemcpyAsync(t->loss_host, t->loss_sum, sizeof(double), cudaMemcpyDeviceToHost, s));
  SXEN_CUDA(cudaStreamSynchronize(s));
  // loss /= batch * out_w; non-finite -> TrainingError (src/trainer.cpp:120-123)
  const double loss = *t->loss_host / (static_cast<double>(global_batch) * static_cast<double>(t->out_w));
  *loss_out = loss;
  if (!std::isfinite(loss)) return fail(SXEN_TRAINING_ERROR, "loss became non-finite");
  return sxen_encoder_check(t->enc, stream);
}

sxen_status sxen_trainer_update(sxen_trainer* t, const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam,
                                void* stream) {
  SXEN_REQUIRE(t != nullptr && table_adam != nullptr && mlp_adam != nullptr, "null argument");
  DeviceGuard guard(t->device);
  if (sxen_status st = update_impl(t, table_adam, mlp_adam, nullptr, SXEN_COORD_F64, 0, nullptr, stream)) return st;
  SXEN_CUDA(cudaMemsetAsync(t->loss_sum, 0, sizeof(double), as_stream(stream)));
  return SXEN_OK;
}

sxen_status sxen_trainer_check(sxen_trainer* t, void* stream) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  if (sxen_status st = sxen_sparse_adam_check(t->table_opt, stream)) return st;
  return sxen_adam_check(t->mlp_opt, stream);
}

sxen_status sxen_trainer_step(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type, const void* targets_dev,
                              sxen_coord_type target_type, size_t n_samples, const sxen_adam_config* table_adam,
                              const sxen_adam_config* mlp_adam, double* loss_out, void* stream) {
  SXEN_REQUIRE(n_samples >= 1, "train: batch_size must be >= 1");  // src/trainer.cpp:57
  SXEN_REQUIRE(t != nullptr && table_adam != nullptr && mlp_adam != nullptr, "null argument");
  if (t->pending != 0)
    return fail(SXEN_LOGIC_ERROR, "train: %zu queued steps not collected (sxen_trainer_collect first)", t->pending);
  // One queued step, collected at once: the device-side gate keeps "throw before the update" for a non-finite loss
  // (src/trainer.cpp:121-123) and the loss, the gate and the three error words come back on ONE stream synchronisation
  // (the separate loss / check entry points cost four).
  if (sxen_status st = sxen_trainer_step_enqueue(t, coords_dev, coord_type, targets_dev, target_type, n_samples, table_adam,
                                                 mlp_adam, stream))
    return st;
  double loss = 0.0;
  size_t count = 0;
  int64_t failed = -1;
  const sxen_status st = sxen_trainer_collect(t, &loss, 1, &count, &failed, stream);
  if (loss_out) *loss_out = loss;
  return st;
}

sxen_status sxen_trainer_step_enqueue(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type,
                                      const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                      const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam, void* stream) {
  SXEN_REQUIRE(t != nullptr && table_adam != nullptr && mlp_adam != nullptr, "null argument");
  SXEN_REQUIRE(n_samples >= 1, "train: batch_size must be >= 1");  // src/trainer.cpp:57
  if (t->pending >= kLossRing)
    return fail(SXEN_LOGIC_ERROR, "train: %zu queued steps not collected (sxen_trainer_collect first)", t->pending);
  const bool own_rows_only = !t->foreign_grads;  // nothing accumulated since the last update but this step's batch
  if (sxen_status st = sxen_trainer_accumulate(t, coords_dev, coord_type, targets_dev, target_type, n_samples, n_samples, stream))
    return st;
  DeviceGuard guard(t->device);
  cudaStream_t s = as_stream(stream);
  loss_record_kernel<<<1, 1, 0, s>>>(t->loss_sum, t->loss_ring, static_cast<unsigned long long>(t->pending),
                                     static_cast<double>(n_samples) * static_cast<double>(t->out_w), t->gate, t->enc->status);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  ++t->pending;
  // table_opt.step, mlp_opt.step (src/trainer.cpp:129-130), skipped on the device when the gate is closed; a small batch
  // visits its own rows instead of scanning all L*T
  const bool walk = own_rows_only && sxen_sparse_adam_walk_pays(t->enc, n_samples);
  return update_impl(t, table_adam, mlp_adam, walk ? coords_dev : nullptr, coord_type, n_samples, t->gate, stream);
}

sxen_status sxen_trainer_set_fused(sxen_trainer* t, int32_t mode) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  SXEN_REQUIRE(mode >= -1 && mode <= 1, "train: fused mode must be -1 (auto), 0 (off) or 1 (required)");
  t->fused_mode = mode;
  return SXEN_OK;
}

sxen_status sxen_trainer_set_reproducible(sxen_trainer* t, int32_t on) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  if (t->pending != 0)
    return fail(SXEN_LOGIC_ERROR, "train: %zu queued steps not collected (sxen_trainer_collect first)", t->pending);
  DeviceGuard guard(t->device);
  if (sxen_status st = sxen_grad_set_reproducible(t->grad, on)) return st;
  if (sxen_status st = sxen_mlp_set_reproducible(t->mlp, on)) return st;
  t->reproducible = on != 0;
  t->capacity = 0;  // the workspace is re-made with (or without) the f64 gradient rows at the next step
  t->have_grad64 = false;
  return SXEN_OK;
}

// ------------------------------------------------------------------------------------------------ batch-sharded step
sxen_status sxen_trainer_set_comm(sxen_trainer* t, sxen_comm* comm) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  if (comm != nullptr) {
    int32_t device = -1;
    if (sxen_status st = sxen_comm_info(comm, nullptr, nullptr, &device, nullptr)) return st;
    SXEN_REQUIRE(device == t->device, "train: the communicator lives on device %d, the trainer on device %d", device, t->device);
    DeviceGuard guard(t->device);
    if (t->comm_stream == nullptr) {
      SXEN_CUDA(cudaStreamCreateWithFlags(&t->comm_stream, cudaStreamNonBlocking));
      SXEN_CUDA(cudaEventCreateWithFlags(&t->ev_compute, cudaEventDisableTiming));
      SXEN_CUDA(cudaEventCreateWithFlags(&t->ev_comm, cudaEventDisableTiming));
    }
  }
  t->comm = comm;
  return SXEN_OK;
}

sxen_status sxen_trainer_allreduce_head(sxen_trainer* t, void* stream) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  if (t->comm == nullptr) return SXEN_OK;
  double* mg = nullptr;
  if (sxen_status st = sxen_mlp_grads_dev(t->mlp, &mg)) return st;
  if (sxen_status st = sxen_comm_allreduce(t->comm, mg, static_cast<size_t>(t->mlp_params), SXEN_COORD_F64, stream)) return st;
  t->foreign_grads = true;
  return sxen_comm_allreduce(t->comm, t->loss_sum, 2, SXEN_COORD_F64, stream);
}

sxen_status sxen_trainer_allreduce_levels(sxen_trainer* t, int32_t first_level, int32_t level_count, void* stream) {
  SXEN_REQUIRE(t != nullptr, "trainer handle is null");
  sxen_encoder_config ec;
  sxen_encoder_get_config(t->enc, &ec);
  SXEN_REQUIRE(first_level >= 0 && level_count >= 0 && first_level + level_count <= ec.levels,
               "level range [%d, %d) outside the encoder's %d levels", first_level, first_level + level_count, ec.levels);
  if (t->comm == nullptr || level_count == 0) return SXEN_OK;
  const size_t per_level = static_cast<size_t>(ec.table_size) * static_cast<size_t>(ec.features);
  t->foreign_grads = true;  // the accumulator now holds other ranks' rows: the table update must scan, not walk this batch
  if (sxen_status st = sxen_comm_allreduce(t->comm, t->grad->values + static_cast<size_t>(first_level) * per_level,
                                           static_cast<size_t>(level_count) * per_level, SXEN_COORD_F32, stream))
    return st;
  if (t->grad->fixed == nullptr) return SXEN_OK;
  return sxen_comm_allreduce(t->comm, t->grad->fixed + static_cast<size_t>(first_level) * per_level,
                             static_cast<size_t>(level_count) * per_level, SXEN_ELEM_I64, stream);
}

sxen_status sxen_trainer_step_sharded(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type,
                                      const void* targets_dev, sxen_coord_type target_type, size_t global_batch,
                                      const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam,
                                      int32_t level_chunks, double* loss_out, void* stream) {
  SXEN_REQUIRE(t != nullptr && table_adam != nullptr && mlp_adam != nullptr, "null argument");
  SXEN_REQUIRE(global_batch >= 1, "train: batch_size must be >= 1");  // src/trainer.cpp:57
  SXEN_REQUIRE(coords_dev != nullptr && targets_dev != nullptr, "null argument");
  if (t->pending != 0)
    return fail(SXEN_LOGIC_ERROR, "train: %zu queued steps not collected (sxen_trainer_collect first)", t->pending);
  int32_t world = 1, rank = 0;
  if (t->comm != nullptr)
    if (sxen_status st = sxen_comm_info(t->comm, &world, &rank, nullptr, nullptr)) return st;
  SXEN_REQUIRE(t->aux_dims == 0 || world == 1, "train: aux_dims > 0 is single-GPU on the device path");
  sxen_encoder_config ec;
  sxen_encoder_get_config(t->enc, &ec);
  // the reference's contiguous chunks with ranks as the workers: chunk = ceil(B / W), src/trainer.cpp:93,107-108
  const size_t chunk = (global_batch + static_cast<size_t>(world) - 1) / static_cast<size_t>(world);
  const size_t begin = std::min(global_batch, static_cast<size_t>(rank) * chunk);
  const size_t n_local = std::min(global_batch, begin + chunk) - begin;
  const size_t csize = coord_type == SXEN_COORD_F32 ? sizeof(float) : sizeof(double);
  const size_t tsize = target_type == SXEN_COORD_F32 ? sizeof(float) : sizeof(double);
  const char* x = static_cast<const char*>(coords_dev) + begin * static_cast<size_t>(ec.dim) * csize;
  const char* y = static_cast<const char*>(targets_dev) + begin * static_cast<size_t>(t->out_w) * tsize;
  DeviceGuard guard(t->device);
  cudaStream_t s = as_stream(stream);
  cudaStream_t cs = t->comm != nullptr ? t->comm_stream : s;
  auto hand_to_comm = [&]() -> sxen_status {  // what the compute stream has queued so far precedes the next exchange
    if (cs == s) return SXEN_OK;
    SXEN_CUDA(cudaEventRecord(t->ev_compute, s));
    SXEN_CUDA(cudaStreamWaitEvent(cs, t->ev_compute, 0));
    return SXEN_OK;
  };
  // run_chunk's head on this rank's chunk (src/trainer.cpp:31-46), upstream scaled by the GLOBAL batch (:26-27)
  if (sxen_status st = sxen_trainer_accumulate_head(t, x, coord_type, y, target_type, n_local, global_batch, stream)) return st;
  reject_flag_kernel<<<1, 1, 0, s>>>(t->loss_sum + 1, t->enc->status);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (sxen_status st = hand_to_comm()) return st;
  if (sxen_status st = sxen_trainer_allreduce_head(t, cs)) return st;   // under the first range's backward
  const int chunks = std::max(1, std::min<int>(level_chunks <= 0 ? 4 : level_chunks, ec.levels));
  const int per = (ec.levels + chunks - 1) / chunks;
  for (int first = 0; first < ec.levels; first += per) {
    const int count = std::min(per, ec.levels - first);
    if (n_local > 0)
      if (sxen_status st = sxen_trainer_accumulate_tables(t, x, coord_type, n_local, first, count, stream)) return st;
    if (sxen_status st = hand_to_comm()) return st;
    if (sxen_status st = sxen_trainer_allreduce_levels(t, first, count, cs)) return st;
  }
  if (cs != s) {
    SXEN_CUDA(cudaEventRecord(t->ev_comm, cs));
    SXEN_CUDA(cudaStreamWaitEvent(s, t->ev_comm, 0));
  }
  // the merged loss decides, identically on every rank, whether the step is applied (src/trainer.cpp:118-123)
  SXEN_CUDA(cudaMemcpyAsync(t->loss_host, t->loss_sum, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
  SXEN_CUDA(cudaStreamSynchronize(s));
  const double loss = t->loss_host[0] / (static_cast<double>(global_batch) * static_cast<double>(t->out_w));
  if (loss_out) *loss_out = loss;
  auto drop_step = [&]() -> sxen_status {
    if (sxen_status st = sxen_grad_clear(t->grad, stream)) return st;
    if (sxen_status st = sxen_mlp_grad_clear(t->mlp, stream)) return st;
    SXEN_CUDA(cudaMemsetAsync(t->loss_sum, 0, 2 * sizeof(double), s));
    t->foreign_grads = false;
    return SXEN_OK;
  };
  if (t->loss_host[1] != 0.0) {  // some rank's chunk held a coordinate outside [0,1]: nobody updates (src/encoding.cpp:183-194)
    if (sxen_status st = drop_step()) return st;
    if (sxen_status st = sxen_encoder_check(t->enc, stream)) return st;  // this rank's own sample, named
    return fail(SXEN_INVALID_ARGUMENT, "encode: a coordinate outside [0,1] was rejected on another rank");
  }
  if (!std::isfinite(loss)) {
    if (sxen_status st = drop_step()) return st;
    return fail(SXEN_TRAINING_ERROR, "loss became non-finite");
  }
  if (sxen_status st = update_impl(t, table_adam, mlp_adam, nullptr, coord_type, 0,
                                   nullptr, stream))
    return st;
  SXEN_CUDA(cudaMemsetAsync(t->loss_sum, 0, 2 * sizeof(double), s));
  return sxen_trainer_check(t, stream);
}

sxen_status sxen_trainer_pending(const sxen_trainer* t, size_t* out) {
  SXEN_REQUIRE(t != nullptr && out != nullptr, "null argument");
  *out = t->pending;
  return SXEN_OK;
}

sxen_status sxen_trainer_collect(sxen_trainer* t, double* losses_out, size_t capacity, size_t* count_out,
                                 int64_t* failed_out, void* stream) {
  SXEN_REQUIRE(t != nullptr && count_out != nullptr, "null argument");
  SXEN_REQUIRE(capacity >= t->pending && (losses_out != nullptr || t->pending == 0),
               "train: %zu queued losses do not fit the caller's buffer (%zu)", t->pending, capacity);
  DeviceGuard guard(t->device);
  cudaStream_t s = as_stream(stream);
  const size_t n = t->pending;
  *count_out = n;
  if (failed_out) *failed_out = -1;
  if (n == 0) return SXEN_OK;
  SXEN_CUDA(cudaMemcpyAsync(t->loss_ring_host, t->loss_ring, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  SXEN_CUDA(cudaMemcpyAsync(t->gate_host, t->gate, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  // the three error words ride on the same synchronisation: the encoder's first rejected sample and the optimizers' first
  // non-finite gradient element.  All clear (the normal case) = one stream sync per collect; anything else takes the
  // checking entry points below, which re-read, reset and word the error.
  SXEN_CUDA(cudaMemcpyAsync(t->enc->status_host, t->enc->status, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SXEN_CUDA(cudaMemcpyAsync(t->table_opt->status_host, t->table_opt->status, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SXEN_CUDA(cudaMemcpyAsync(t->mlp_opt->status_host, t->mlp_opt->status, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  SXEN_CUDA(cudaStreamSynchronize(s));
  const bool words_clear = t->enc->status_host[0] == kNoFailure && *t->table_opt->status_host == kNoFailure &&
                           *t->mlp_opt->status_host == kNoFailure;
  t->pending = 0;
  for (size_t i = 0; i < n; ++i) losses_out[i] = t->loss_ring_host[i];
  if (*t->gate_host != kNoFailure) {
    const unsigned long long bad = *t->gate_host;
    SXEN_CUDA(cudaMemsetAsync(t->gate, 0xff, sizeof(unsigned long long), s));
    // the gated steps left their gradients in the accumulators (the reference's are in the same state when it throws,
    // and it drops them with the aborted run): clear them so the handle can go on from the last applied step
    if (sxen_status st = sxen_grad_clear(t->grad, stream)) return st;
    if (sxen_status st = sxen_mlp_grad_clear(t->mlp, stream)) return st;
    t->foreign_grads = false;
    SXEN_CUDA(cudaStreamSynchronize(s));
    if (failed_out) *failed_out = static_cast<int64_t>(bad);
    // the gated steps bumped both optimizers' step counters on the host without applying an update: take them back, so the
    // next applied step uses the bias correction of the number of updates actually made (src/optimizer.cpp:31-32,64-66)
    const int64_t skipped = static_cast<int64_t>(n) - static_cast<int64_t>(bad);
    t->table_opt->t -= skipped;
    t->mlp_opt->t -= skipped;
    // re-read and reset the latched error words so they cannot surface on an unrelated later collect
    const bool rejected = t->enc->status_host[0] != kNoFailure;
    const sxen_status enc_st = sxen_encoder_check(t->enc, stream);
    sxen_trainer_check(t, stream);
    if (rejected && enc_st != SXEN_OK) return enc_st;  // std::invalid_argument: thrown before the step changed anything
    return fail(SXEN_TRAINING_ERROR, "loss became non-finite (queued step %llu of %zu)", bad, n);
  }
  if (words_clear) return SXEN_OK;
  if (sxen_status st = sxen_encoder_check(t->enc, stream)) return st;
  return sxen_trainer_check(t, stream);
}

}  // extern "C"
