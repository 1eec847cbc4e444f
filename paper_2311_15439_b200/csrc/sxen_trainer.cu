// sxen_trainer.cu -- one training step of train_field on the device (/root/reference/proj/src/trainer.cpp:94-136):
//   gradient pass  = run_chunk over this rank's contiguous chunk of the batch (:20-49): encode -> Mlp::forward -> MSE and
//                    upstream = 2e/(B*out_w) with B the GLOBAL batch -> Mlp::backward -> encode_backward
//   update         = SparseAdamState::step on the tables (touched rows only) + AdamState::step on the MLP (:129-130)
// The two halves are separate entry points so a multi-GPU host can all-reduce the gradient buffers in between
// (the reference merges its workers' accumulators at exactly that point, :125-128).
#include <cmath>

#include "sxen_common.hpp"

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
  double* upstream = nullptr;    // N x out_w
  double* sample_loss = nullptr; // N
  double* loss_sum = nullptr;    // device scalar: sum of per-sample losses accumulated since the last update
  double* loss_host = nullptr;   // pinned
  int32_t out_w = 0, enc_w = 0;
  uint64_t mlp_params = 0;
};

namespace {

sxen_status ensure_workspace(sxen_trainer* t, size_t n) {
  if (n <= t->capacity) return SXEN_OK;
  cudaFree(t->features);
  cudaFree(t->input_grad);
  cudaFree(t->upstream);
  cudaFree(t->sample_loss);
  t->features = t->input_grad = nullptr;
  t->upstream = t->sample_loss = nullptr;
  t->capacity = 0;
  SXEN_CUDA(cudaMalloc(&t->features, n * static_cast<size_t>(t->enc_w) * sizeof(float)));
  SXEN_CUDA(cudaMalloc(&t->input_grad, n * static_cast<size_t>(t->enc_w) * sizeof(float)));
  SXEN_CUDA(cudaMalloc(&t->upstream, n * static_cast<size_t>(t->out_w) * sizeof(double)));
  SXEN_CUDA(cudaMalloc(&t->sample_loss, (n + 1) * sizeof(double)));
  t->capacity = n;
  return SXEN_OK;
}

}  // namespace

extern "C" {

sxen_status sxen_trainer_create(sxen_encoder* enc, sxen_mlp* mlp, sxen_trainer** out) {
  SXEN_REQUIRE(enc != nullptr && mlp != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  sxen_encoder_config ec;
  sxen_encoder_get_config(enc, &ec);
  sxen_mlp_config mc;
  if (sxen_status st = sxen_mlp_get_config(mlp, &mc)) return st;
  // src/trainer.cpp:61-65 (aux_dims = 0: this path feeds the encoding straight into the head)
  SXEN_REQUIRE(mc.input_width == ec.levels * ec.features, "train: MLP input width %d != encoded width %d + aux 0",
               mc.input_width, ec.levels * ec.features);
  sxen_trainer* t = new sxen_trainer();
  t->enc = enc;
  t->mlp = mlp;
  t->device = enc->device;
  t->out_w = mc.output_width;
  t->enc_w = ec.levels * ec.features;
  DeviceGuard guard(t->device);
  sxen_status st = sxen_grad_create(enc, &t->grad);
  if (st == SXEN_OK) st = sxen_sparse_adam_create(enc, &t->table_opt);
  if (st == SXEN_OK) st = sxen_mlp_parameter_count(mlp, &t->mlp_params);
  if (st == SXEN_OK) st = sxen_adam_create(static_cast<size_t>(t->mlp_params), t->device, &t->mlp_opt);
  if (st == SXEN_OK && cudaMalloc(&t->loss_sum, sizeof(double)) != cudaSuccess) st = fail(SXEN_CUDA_ERROR, "trainer: allocation failed");
  if (st == SXEN_OK && cudaMemset(t->loss_sum, 0, sizeof(double)) != cudaSuccess) st = fail(SXEN_CUDA_ERROR, "trainer: memset failed");
  if (st == SXEN_OK && cudaHostAlloc(&t->loss_host, sizeof(double), cudaHostAllocDefault) != cudaSuccess)
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
  cudaFree(t->upstream);
  cudaFree(t->sample_loss);
  cudaFree(t->loss_sum);
  cudaFreeHost(t->loss_host);
  delete t;
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
  // encoder.encode (src/trainer.cpp:31)
  if (sxen_status st = sxen_encoder_encode(t->enc, coords_dev, coord_type, n_samples, t->features, stream)) return st;
  // mlp.forward, loss + upstream, mlp.backward (:36-46): one fused call (tensor-core kernel or the exact chain)
  if (sxen_status st = sxen_mlp_forward_backward(t->mlp, t->features, targets_dev, target_type, n_samples, global_batch,
                                                 nullptr, t->input_grad, t->loss_sum, stream))
    return st;
  t->head_samples = n_samples;
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
  return sxen_encoder_encode_backward_levels(t->enc, coords_dev, coord_type, t->input_grad, n_samples, t->grad,
                                             first_level, level_count, stream);
}

sxen_status sxen_trainer_accumulate(sxen_trainer* t, const void* coords_dev, sxen_coord_type coord_type,
                                    const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                    size_t global_batch, void* stream) {
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
  // table_opt.step then mlp_opt.step (src/trainer.cpp:129-130); the accumulators are cleared for the next step (:97-100)
  if (sxen_status st = sxen_sparse_adam_step(t->table_opt, t->enc, t->grad, table_adam, 1, stream)) return st;
  double* mg = nullptr;
  float* mp = nullptr;
  sxen_mlp_grads_dev(t->mlp, &mg);
  sxen_mlp_params_dev(t->mlp, &mp);
  if (sxen_status st = sxen_adam_step(t->mlp_opt, mp, mg, SXEN_COORD_F64, static_cast<size_t>(t->mlp_params), mlp_adam, stream))
    return st;
  if (sxen_status st = sxen_mlp_grad_clear(t->mlp, stream)) return st;
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
  if (sxen_status st = sxen_trainer_accumulate(t, coords_dev, coord_type, targets_dev, target_type, n_samples, n_samples, stream))
    return st;
  double loss = 0.0;
  const sxen_status loss_st = sxen_trainer_loss(t, n_samples, &loss, stream);
  if (loss_out) *loss_out = loss;
  if (loss_st != SXEN_OK) return loss_st;  // the reference throws before updating (src/trainer.cpp:121-123)
  if (sxen_status st = sxen_trainer_update(t, table_adam, mlp_adam, stream)) return st;
  return sxen_trainer_check(t, stream);
}

}  // extern "C"
