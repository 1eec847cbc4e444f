// sxen_b200_train.hpp -- header-only C++ mirror of the reference's trainer and tasks over the C ABI (sxen_cuda.h):
//   TrainConfig / TrainResult / train_field     include/sxen/trainer.hpp:15-54, src/trainer.cpp:53-139
//   psnr_from_mse / render (MSE form) / fit_image / fit_field   include/sxen/tasks.hpp, src/tasks.cpp:30-194
// Same names, defaults, argument meaning and exception types as the reference (namespace sxen::b200).  What differs is
// where the data lives: a BatchSampler fills DEVICE spans (the two samplers the reference ships, fit_image's and
// fit_field's, are device kernels behind sxen_sample_image_batch / sxen_sample_field_batch, bit-identical batches), and
// the training loop queues whole steps on the stream (sxen_trainer_step_enqueue) and reads the losses back in windows
// instead of once per step -- the step's kernels, not the host round trip, set the pace at the reference's default
// batch of 2048.  No arithmetic happens in this header apart from fit_field's hold-out statistics (host doubles, the
// reference's own loop, src/tasks.cpp:176-192).  The host program needs no CUDA headers: device buffers come from
// sxen_device_alloc.
#pragma once

#include <algorithm>
#include <cmath>
#include <exception>
#include <functional>
#include <thread>

#include "sxen_b200.hpp"

namespace sxen::b200 {

// RAII device array through the C ABI.
template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  DeviceBuffer(std::size_t count, int device) : n_(count), device_(device) {
    void* p = nullptr;
    check(sxen_device_alloc(device, count * sizeof(T), &p));
    p_ = static_cast<T*>(p);
  }
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)), device_(o.device_) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      sxen_device_free(device_, p_);
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
      device_ = o.device_;
    }
    return *this;
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { sxen_device_free(device_, p_); }
  T* data() const { return p_; }
  std::size_t size() const { return n_; }
  DeviceSpan<T> span(std::size_t count) const { return {p_, count}; }
  DeviceSpan<const T> cspan(std::size_t count) const { return {p_, count}; }
  void upload(std::span<const T> src, void* stream = nullptr) {
    if (src.size() > n_) throw std::invalid_argument("DeviceBuffer::upload: source larger than the buffer");
    check(sxen_device_upload(device_, p_, src.data(), src.size() * sizeof(T), stream));
  }
  std::vector<T> download(std::size_t count, void* stream = nullptr) const {
    std::vector<T> out(count);
    check(sxen_device_download(device_, out.data(), p_, count * sizeof(T), stream));
    return out;
  }
  void zero(void* stream = nullptr) { check(sxen_device_zero(device_, p_, n_ * sizeof(T), stream)); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
  int device_ = 0;
};

// include/sxen/optimizer.hpp:24-40 (dense Adam over a caller-owned device parameter array)
class AdamState {
 public:
  AdamState(std::size_t size, int device = 0) { check(sxen_adam_create(size, device, &h_)); }
  AdamState(const AdamState&) = delete;
  AdamState& operator=(const AdamState&) = delete;
  ~AdamState() { sxen_adam_destroy(h_); }
  std::int64_t step_count() const {
    std::int64_t t = 0;
    check(sxen_adam_step_count(h_, &t));
    return t;
  }
  void step(DeviceSpan<float> params, DeviceSpan<const double> grads, const AdamConfig& cfg, void* stream = nullptr) {
    if (params.size != grads.size) throw std::invalid_argument("adam step: parameter/gradient size mismatch");
    const sxen_adam_config c = cfg.c();
    check(sxen_adam_step(h_, params.data, grads.data, SXEN_COORD_F64, params.size, &c, stream));
    check(sxen_adam_check(h_, stream));  // TrainingError on a non-finite gradient (src/optimizer.cpp:35-37)
  }

 private:
  sxen_adam* h_ = nullptr;
};

// include/sxen/trainer.hpp:15-24, same defaults.  `threads` is accepted and ignored: the batch is one launch, the
// reference's worker fan-out has no analogue on one device (ranks play that role across devices).
struct TrainConfig {
  int batch_size = 2048;
  int steps = 10000;
  int aux_dims = 0;  // extra inputs appended verbatim after the encoding
  AdamConfig table_adam{.lr = 1e-2, .beta1 = 0.9, .beta2 = 0.99, .epsilon = 1e-15};
  AdamConfig mlp_adam{.lr = 1e-3, .beta1 = 0.9, .beta2 = 0.99, .epsilon = 1e-15};
  std::uint64_t seed = 1234;
  int threads = 0;
  int record_every = 100;
  int queue_window = 256;  // steps queued between two loss read-backs (1 = the reference's per-step cadence); <= 4096
  int level_chunks = 4;    // batch-sharded runs: level ranges whose gradient exchange overlaps the next range's backward
  bool reproducible = false;  // order-free fixed-point gradient sums (sxen_trainer_set_reproducible): bit-identical runs for a fixed
                              // seed, as the reference's are for a fixed (seed, threads) (tests/test_neural.cpp:370-408)
};

// include/sxen/trainer.hpp:26-32 with device spans: coords = batch x dim, aux = batch x aux_dims pass-through inputs (empty
// when aux_dims == 0), targets = batch x output_width, all f64, filled by work queued on `stream`.  Called on the
// coordinating thread only; determinism comes from (seed, step).
using BatchSampler = std::function<void(int step, DeviceSpan<double> coords, DeviceSpan<double> aux,
                                        DeviceSpan<double> targets, void* stream)>;

// One rank's end of the gradient exchange of a batch-sharded run (sxen_comm_*, sxen_cuda.h).  The reference's analogue is
// the worker fan-out and worker-order merge inside train_field (src/trainer.cpp:101-128); ranks are the workers here.
class Comm {
 public:
  Comm() = default;
  // NCCL, one process per GPU: rank 0 calls unique_id() and hands the bytes to its peers over any side channel.
  static sxen_comm_id unique_id() {
    sxen_comm_id id{};
    check(sxen_comm_unique_id(&id));
    return id;
  }
  Comm(const sxen_comm_id& id, int world, int rank, int device) { check(sxen_comm_create(&id, world, rank, device, &h_)); }
  // LOCAL: every rank in this process, one host thread per rank (train_field_local below); devices[r] = rank r's device.
  static std::vector<Comm> local(const std::vector<int>& devices) {
    std::vector<std::int32_t> dev(devices.begin(), devices.end());
    std::vector<sxen_comm*> raw(devices.size(), nullptr);
    check(sxen_comm_create_local(static_cast<std::int32_t>(dev.size()), dev.data(), raw.data()));
    std::vector<Comm> out(devices.size());
    for (std::size_t r = 0; r < raw.size(); ++r) out[r].h_ = raw[r];
    return out;
  }
  Comm(Comm&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Comm& operator=(Comm&& o) noexcept {
    if (this != &o) {
      sxen_comm_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  ~Comm() { sxen_comm_destroy(h_); }
  sxen_comm* handle() const { return h_; }
  int world() const {
    std::int32_t w = 1;
    if (h_) check(sxen_comm_info(h_, &w, nullptr, nullptr, nullptr));
    return w;
  }
  int rank() const {
    std::int32_t r = 0;
    if (h_) check(sxen_comm_info(h_, nullptr, &r, nullptr, nullptr));
    return r;
  }

 private:
  sxen_comm* h_ = nullptr;
};

// include/sxen/trainer.hpp:34-38
struct TrainResult {
  std::vector<std::pair<int, double>> loss_curve;  // (step, batch MSE before that step's update)
  double final_loss = 0.0;
  int steps_run = 0;
};

// sxen::train_field (src/trainer.cpp:53-139).  Throws TrainingError when a loss or gradient goes non-finite -- tables,
// MLP and moments are then as they were before the offending step, as in the reference -- and std::invalid_argument
// for the reference's argument checks (:55-65).
//
// comm != nullptr: this process (or thread) is ONE RANK of a batch-sharded run.  encoder / mlp are this rank's replicas,
// initialised like every other rank's; the sampler fills the WHOLE batch on every rank (it is deterministic in (seed, step),
// as the reference's contract requires, include/sxen/trainer.hpp:29-30), the rank runs its contiguous chunk
// (src/trainer.cpp:93,107-108), gradients and the loss are summed over the ranks where the reference merges its workers
// (:125-128) and every rank applies the identical update -- sxen_trainer_step_sharded, one loss read-back per step.
inline TrainResult train_field(HashEncoder& encoder, Mlp& mlp, const BatchSampler& sampler, const TrainConfig& cfg,
                               int device = 0, void* stream = nullptr, const Comm* comm = nullptr) {
  if (cfg.batch_size < 1) throw std::invalid_argument("train: batch_size must be >= 1");
  if (cfg.steps < 0) throw std::invalid_argument("train: steps must be >= 0");
  if (cfg.aux_dims < 0) throw std::invalid_argument("train: aux_dims must be >= 0");  // src/trainer.cpp:59
  if (cfg.record_every < 1) throw std::invalid_argument("train: record_every must be >= 1");
  if (cfg.queue_window < 1 || cfg.queue_window > 4096) throw std::invalid_argument("train: queue_window must be in [1, 4096]");
  if (!sampler) throw std::invalid_argument("train: sampler must be callable");
  struct Handle {
    sxen_trainer* h = nullptr;
    ~Handle() { sxen_trainer_destroy(h); }
  } trainer;
  check(sxen_trainer_create_aux(encoder.handle(), mlp.handle(), cfg.aux_dims, &trainer.h));  // width check, :61-65
  if (cfg.reproducible) check(sxen_trainer_set_reproducible(trainer.h, 1));
  const std::size_t batch = static_cast<std::size_t>(cfg.batch_size);
  const std::size_t dim = static_cast<std::size_t>(encoder.config().dim);
  const std::size_t out_w = static_cast<std::size_t>(mlp.config().output_width);
  // one batch slot: the sampler's work and the step's kernels are ordered on `stream`, so step k+1's sampler cannot
  // overwrite what step k's queued kernels still read
  const std::size_t aux_w = static_cast<std::size_t>(cfg.aux_dims);
  DeviceBuffer<double> coords(batch * dim, device), targets(batch * out_w, device), aux(batch * aux_w, device);
  if (aux_w > 0) check(sxen_trainer_set_aux(trainer.h, aux.data(), SXEN_COORD_F64));
  const sxen_adam_config ta = cfg.table_adam.c(), ma = cfg.mlp_adam.c();
  TrainResult result;
  if (comm != nullptr && comm->handle() != nullptr) {
    if (aux_w > 0 && comm->world() > 1) throw std::invalid_argument("train: aux_dims > 0 is single-GPU on the device path");
    check(sxen_trainer_set_comm(trainer.h, comm->handle()));
    for (int step = 0; step < cfg.steps; ++step) {
      sampler(step, coords.span(batch * dim), aux.span(batch * aux_w), targets.span(batch * out_w), stream);
      double loss = 0.0;
      const sxen_status st = sxen_trainer_step_sharded(trainer.h, coords.data(), SXEN_COORD_F64, targets.data(), SXEN_COORD_F64,
                                                       batch, &ta, &ma, cfg.level_chunks, &loss, stream);
      if (st == SXEN_TRAINING_ERROR && !std::isfinite(loss))
        throw TrainingError("loss became non-finite at step " + std::to_string(step));  // src/trainer.cpp:121-123
      check(st);
      if (step % cfg.record_every == 0 || step == cfg.steps - 1) result.loss_curve.emplace_back(step, loss);
      result.final_loss = loss;
    }
    result.steps_run = cfg.steps;
    return result;
  }
  std::vector<double> losses(static_cast<std::size_t>(cfg.queue_window));
  int first = 0;
  for (int step = 0; step < cfg.steps; ++step) {
    sampler(step, coords.span(batch * dim), aux.span(batch * aux_w), targets.span(batch * out_w), stream);
    check(sxen_trainer_step_enqueue(trainer.h, coords.data(), SXEN_COORD_F64, targets.data(), SXEN_COORD_F64, batch, &ta, &ma,
                                    stream));
    if (step + 1 - first == cfg.queue_window || step == cfg.steps - 1) {
      std::size_t count = 0;
      std::int64_t failed = -1;
      const sxen_status st = sxen_trainer_collect(trainer.h, losses.data(), losses.size(), &count, &failed, stream);
      const std::size_t good = (st == SXEN_TRAINING_ERROR && failed >= 0) ? static_cast<std::size_t>(failed) : count;
      for (std::size_t k = 0; k < good; ++k) {
        const int s = first + static_cast<int>(k);
        if (s % cfg.record_every == 0 || s == cfg.steps - 1) result.loss_curve.emplace_back(s, losses[k]);
        result.final_loss = losses[k];
      }
      if (st == SXEN_TRAINING_ERROR && failed >= 0)
        throw TrainingError("loss became non-finite at step " + std::to_string(first + static_cast<int>(failed)));
      check(st);
      first = step + 1;
    }
  }
  result.steps_run = cfg.steps;
  return result;
}

// One model replica of a batch-sharded run inside ONE process (train_field_local): rank r's encoder and MLP on device r.
struct Replica {
  HashEncoder* encoder = nullptr;
  Mlp* mlp = nullptr;
  int device = 0;
  void* stream = nullptr;
};

// train_field with the reference's own layout -- one worker THREAD per chunk of the batch (src/trainer.cpp:101-116) -- where
// every worker drives a GPU: rank r trains replicas[r] through a LOCAL communicator (the library's peer-memory all-reduce;
// two replicas may share a device).  make_sampler(r) returns rank r's BatchSampler (each rank fills its own device buffers
// with the same (seed, step) stream).  Returns rank 0's result -- the loss curve is the same on every rank, and so are the
// trained replicas, bit for bit (the exchange sums in rank order on one rank per slice).  An exception on any rank
// breaks the group, every worker returns, and the first exception is rethrown here.
inline TrainResult train_field_local(const std::vector<Replica>& replicas, const std::function<BatchSampler(int rank)>& make_sampler,
                                     const TrainConfig& cfg) {
  if (replicas.empty()) throw std::invalid_argument("train: no replicas");
  std::vector<int> devices;
  for (const Replica& r : replicas) {
    if (r.encoder == nullptr || r.mlp == nullptr) throw std::invalid_argument("train: a replica lacks its encoder or MLP");
    devices.push_back(r.device);
  }
  std::vector<Comm> comms = Comm::local(devices);
  std::vector<TrainResult> results(replicas.size());
  std::vector<std::exception_ptr> errors(replicas.size());
  std::vector<std::thread> workers;
  for (std::size_t r = 0; r < replicas.size(); ++r) {
    workers.emplace_back([&, r] {
      try {
        results[r] = train_field(*replicas[r].encoder, *replicas[r].mlp, make_sampler(static_cast<int>(r)), cfg,
                                 replicas[r].device, replicas[r].stream, &comms[r]);
      } catch (...) {
        errors[r] = std::current_exception();
        sxen_comm_abort(comms[r].handle());  // peers waiting for this rank leave their collective with CommError
      }
    });
  }
  for (std::thread& w : workers) w.join();
  // the rank that failed first in rank order speaks (peers of a failed rank only report the broken group)
  std::exception_ptr first_comm;
  for (std::size_t r = 0; r < errors.size(); ++r) {
    if (!errors[r]) continue;
    try {
      std::rethrow_exception(errors[r]);
    } catch (const CommError&) {
      if (!first_comm) first_comm = errors[r];
    } catch (...) {
      std::rethrow_exception(errors[r]);
    }
  }
  if (first_comm) std::rethrow_exception(first_comm);
  return results[0];
}

// ------------------------------------------------------------------------------------------------ tasks
inline constexpr double kPsnrCap = 99.0;  // include/sxen/tasks.hpp:14

// src/tasks.cpp:30-33
inline double psnr_from_mse(double mse) {
  if (!(mse > 0.0)) return kPsnrCap;
  return std::min(kPsnrCap, 10.0 * std::log10(1.0 / mse));
}

// include/sxen/image.hpp: row-major width x height x 3 doubles in [0, 1]
struct ImageDataset {
  int width = 0, height = 0;
  std::vector<double> pixels;
  void validate() const {  // src/image.cpp:16-29
    if (width < 1 || height < 1) throw std::invalid_argument("image: width and height must be >= 1");
    if (pixels.size() != static_cast<std::size_t>(width) * static_cast<std::size_t>(height) * 3)
      throw std::invalid_argument("image: pixel buffer size != width*height*3");
    for (double v : pixels)
      if (!(v >= 0.0 && v <= 1.0)) throw std::invalid_argument("image: pixel values must lie in [0, 1]");
  }
};

// Head arithmetic of the fitted model; no reference analogue (the reference has one, fp64-accumulated path = exact).
enum class MlpPrecision {
  exact = SXEN_MLP_EXACT, tensor_bf16x3 = SXEN_MLP_TENSOR_BF16X3, tensor_bf16 = SXEN_MLP_TENSOR_BF16,
  tensor_bf16x4 = SXEN_MLP_TENSOR_BF16X4
};

// include/sxen/tasks.hpp:30-34
struct FitImageOptions {
  std::uint64_t init_seed = 42;
  int mlp_hidden_width = 64;
  int mlp_hidden_layers = 2;
  MlpPrecision mlp_precision = MlpPrecision::exact;
};

// include/sxen/tasks.hpp:36-42
struct FitImageResult {
  HashEncoder encoder;
  Mlp mlp;
  TrainResult train;
  double final_psnr = 0.0;
  std::vector<std::pair<int, double>> psnr_curve;
};

// MSE over all channels of render_image(encoder, mlp) against the image (src/tasks.cpp:51-96 + image_mse :35-46) without
// materialising the rendered image: pixel centres -> encode -> Mlp::forward -> clamp to [0,1] -> squared error, in
// chunks of `chunk` pixels on the device.
inline double render_mse(const HashEncoder& encoder, Mlp& mlp, DeviceSpan<const double> image_dev, int width, int height,
                         int device = 0, void* stream = nullptr, std::size_t chunk = std::size_t{1} << 20) {
  if (encoder.config().dim != 2) throw std::invalid_argument("render_image: encoder dim must be 2");
  if (mlp.config().input_width != encoder.config().encoded_width() || mlp.config().output_width != 3)
    throw std::invalid_argument("render_image: model widths do not form a 2D->RGB map");
  const std::size_t total = static_cast<std::size_t>(width) * static_cast<std::size_t>(height);
  if (image_dev.size != total * 3) throw std::invalid_argument("image: pixel buffer size != width*height*3");
  const std::size_t step = std::min(chunk, total);
  const std::size_t enc_w = static_cast<std::size_t>(encoder.config().encoded_width());
  DeviceBuffer<double> coords(step * 2, device), acc(1, device);
  DeviceBuffer<float> feats(step * enc_w, device), pred(step * 3, device);
  acc.zero(stream);
  for (std::size_t first = 0; first < total; first += step) {
    const std::size_t n = std::min(step, total - first);
    check(sxen_pixel_centers(width, height, first, n, coords.data(), stream));
    encoder.encode(coords.cspan(n * 2), feats.span(n * enc_w), stream);
    mlp.forward(feats.cspan(n * enc_w), pred.span(n * 3), stream);
    check(sxen_render_sq_error(pred.data(), image_dev.data, first, n, acc.data(), stream));
  }
  const double sum = acc.download(1, stream)[0];
  encoder.check_async(stream);
  return sum / (3.0 * static_cast<double>(total));
}

// sxen::render_image (src/tasks.cpp:51-96): the fitted model at every pixel centre, clamped to [0, 1].  `threads` is
// accepted and ignored (the rows are one device batch per chunk).
inline ImageDataset render_image(const HashEncoder& encoder, Mlp& mlp, int width, int height, int /*threads*/ = 0,
                                 int device = 0, void* stream = nullptr, std::size_t chunk = std::size_t{1} << 20) {
  if (encoder.config().dim != 2) throw std::invalid_argument("render_image: encoder dim must be 2");
  if (mlp.config().input_width != encoder.config().encoded_width() || mlp.config().output_width != 3)
    throw std::invalid_argument("render_image: model widths do not form a 2D->RGB map");
  if (width < 1 || height < 1) throw std::invalid_argument("image: width and height must be >= 1");
  ImageDataset out;
  out.width = width;
  out.height = height;
  const std::size_t total = static_cast<std::size_t>(width) * static_cast<std::size_t>(height);
  out.pixels.resize(3 * total);
  const std::size_t step = std::min(chunk, total);
  const std::size_t enc_w = static_cast<std::size_t>(encoder.config().encoded_width());
  DeviceBuffer<double> coords(step * 2, device);
  DeviceBuffer<float> feats(step * enc_w, device), pred(step * 3, device);
  for (std::size_t first = 0; first < total; first += step) {
    const std::size_t n = std::min(step, total - first);
    check(sxen_pixel_centers(width, height, first, n, coords.data(), stream));
    encoder.encode(coords.cspan(n * 2), feats.span(n * enc_w), stream);
    mlp.forward(feats.cspan(n * enc_w), pred.span(n * 3), stream);
    const std::vector<float> p = pred.download(n * 3, stream);
    for (std::size_t i = 0; i < n * 3; ++i) out.pixels[first * 3 + i] = std::clamp(static_cast<double>(p[i]), 0.0, 1.0);
  }
  encoder.check_async(stream);
  return out;
}

// src/tasks.cpp:35-49
inline double image_mse(const ImageDataset& a, const ImageDataset& b) {
  if (a.width != b.width || a.height != b.height || a.pixels.size() != b.pixels.size())
    throw std::invalid_argument("image_mse: shape mismatch");
  double sum = 0.0;
  for (std::size_t i = 0; i < a.pixels.size(); ++i) {
    const double e = a.pixels[i] - b.pixels[i];
    sum += e * e;
  }
  return sum / static_cast<double>(a.pixels.size());
}
inline double image_psnr(const ImageDataset& a, const ImageDataset& b) { return psnr_from_mse(image_mse(a, b)); }

// sxen::fit_image (src/tasks.cpp:98-137)
inline FitImageResult fit_image(const ImageDataset& image, const EncoderConfig& encoder_cfg, const TrainConfig& train_cfg,
                                const FitImageOptions& opt = {}, int device = 0, void* stream = nullptr) {
  image.validate();
  if (encoder_cfg.dim != 2) throw std::invalid_argument("fit_image: encoder dim must be 2");
  HashEncoder encoder(encoder_cfg, device);
  encoder.init_tables(opt.init_seed, stream);  // :104
  Mlp mlp(MlpConfig{encoder_cfg.encoded_width(), opt.mlp_hidden_width, opt.mlp_hidden_layers, 3}, device);
  mlp.init_params(sxen_hash_combine(opt.init_seed, 1), stream);  // :107
  if (opt.mlp_precision != MlpPrecision::exact) check(sxen_mlp_set_precision(mlp.handle(), static_cast<int>(opt.mlp_precision)));
  DeviceBuffer<double> image_dev(image.pixels.size(), device);
  image_dev.upload(image.pixels, stream);
  const int w = image.width, h = image.height;
  const std::uint64_t seed = train_cfg.seed;
  const double* px = image_dev.data();
  const BatchSampler sampler = [=](int step, DeviceSpan<double> coords, DeviceSpan<double> /*aux*/,
                                   DeviceSpan<double> targets, void* s) {  // :112-126
    check(sxen_sample_image_batch(seed, static_cast<std::uint64_t>(step), px, w, h, coords.size / 2, coords.data,
                                  targets.data, s));
  };
  TrainResult train = train_field(encoder, mlp, sampler, train_cfg, device, stream);
  FitImageResult result{std::move(encoder), std::move(mlp), std::move(train), 0.0, {}};
  for (const auto& [s, loss] : result.train.loss_curve) result.psnr_curve.emplace_back(s, psnr_from_mse(loss));  // :130-132
  result.final_psnr =
      psnr_from_mse(render_mse(result.encoder, result.mlp, image_dev.cspan(image.pixels.size()), w, h, device, stream));
  return result;
}

// fit_image on make_test_image(width, height, image_seed) WITHOUT the image in memory (BASELINE configs[2], the gigapixel fit:
// 32768 x 32768 would be 26 GB as doubles): the sampler (src/tasks.cpp:112-126) draws the pixel and evaluates the image's
// procedural definition (src/image.cpp:68-96) there, sxen_sample_test_image_batch.  comm != nullptr: this call is one rank of a
// batch-sharded run (train_field above).  The final PSNR is render_image's over the first psnr_pixels pixels in row-major
// order (the whole image when it has no more).
inline FitImageResult fit_test_image(int width, int height, std::uint64_t image_seed, const EncoderConfig& encoder_cfg,
                                     const TrainConfig& train_cfg, const FitImageOptions& opt = {}, int device = 0,
                                     void* stream = nullptr, const Comm* comm = nullptr, std::size_t psnr_pixels = std::size_t{1} << 24) {
  if (width < 1 || height < 1) throw std::invalid_argument("test image: width and height must be >= 1");
  if (encoder_cfg.dim != 2) throw std::invalid_argument("fit_image: encoder dim must be 2");
  HashEncoder encoder(encoder_cfg, device);
  encoder.init_tables(opt.init_seed, stream);
  Mlp mlp(MlpConfig{encoder_cfg.encoded_width(), opt.mlp_hidden_width, opt.mlp_hidden_layers, 3}, device);
  mlp.init_params(sxen_hash_combine(opt.init_seed, 1), stream);
  if (opt.mlp_precision != MlpPrecision::exact) check(sxen_mlp_set_precision(mlp.handle(), static_cast<int>(opt.mlp_precision)));
  const std::uint64_t seed = train_cfg.seed;
  const BatchSampler sampler = [=](int step, DeviceSpan<double> coords, DeviceSpan<double> /*aux*/, DeviceSpan<double> targets,
                                   void* s) {
    check(sxen_sample_test_image_batch(image_seed, width, height, seed, static_cast<std::uint64_t>(step), 0, coords.size / 2,
                                       coords.data, targets.data, s));
  };
  TrainResult train = train_field(encoder, mlp, sampler, train_cfg, device, stream, comm);
  FitImageResult result{std::move(encoder), std::move(mlp), std::move(train), 0.0, {}};
  for (const auto& [s, loss] : result.train.loss_curve) result.psnr_curve.emplace_back(s, psnr_from_mse(loss));
  const std::size_t total = std::min(psnr_pixels, static_cast<std::size_t>(width) * static_cast<std::size_t>(height));
  const std::size_t step = std::min<std::size_t>(total, std::size_t{1} << 20);
  DeviceBuffer<double> coords(step * 2, device), sum(1, device);
  DeviceBuffer<float> feats(step * static_cast<std::size_t>(encoder_cfg.encoded_width()), device), pred(step * 3, device);
  sum.zero(stream);
  for (std::size_t first = 0; first < total; first += step) {
    const std::size_t n = std::min(step, total - first);
    check(sxen_pixel_centers(width, height, first, n, coords.data(), stream));
    result.encoder.encode(coords.cspan(n * 2), feats.span(n * static_cast<std::size_t>(encoder_cfg.encoded_width())), stream);
    result.mlp.forward(feats.cspan(n * static_cast<std::size_t>(encoder_cfg.encoded_width())), pred.span(n * 3), stream);
    check(sxen_test_image_sq_error(image_seed, width, height, pred.data(), first, n, sum.data(), stream));
  }
  result.final_psnr = psnr_from_mse(sum.download(1, stream)[0] / (3.0 * static_cast<double>(total)));
  return result;
}

// include/sxen/noise.hpp:38-50, same defaults (sxen_noise_spec_default)
enum class NoiseKind { perlin = SXEN_NOISE_PERLIN, simplex = SXEN_NOISE_SIMPLEX };
struct NoiseFieldSpec {
  int dim = 2;
  std::uint64_t seed = 7;
  NoiseKind kind = NoiseKind::perlin;
  int octaves = 1;
  double frequency = 4.0;  // lattice cells per unit of input space
  sxen_noise_spec c() const {
    sxen_noise_spec s{};
    s.dim = dim;
    s.kind = static_cast<int>(kind);
    s.octaves = octaves;
    s.seed = seed;
    s.frequency = frequency;
    return s;
  }
  void validate() const {
    const sxen_noise_spec s = c();
    check(sxen_noise_spec_validate(&s));
  }
};

// include/sxen/tasks.hpp:49-54
struct FitFieldOptions {
  std::uint64_t init_seed = 42;
  int mlp_hidden_width = 64;
  int mlp_hidden_layers = 2;
  int holdout_samples = 1 << 14;
  MlpPrecision mlp_precision = MlpPrecision::exact;
};

// include/sxen/tasks.hpp:56-62
struct FitFieldResult {
  HashEncoder encoder;
  Mlp mlp;
  TrainResult train;
  double holdout_mse = 0.0;
  double field_variance = 0.0;
};

// sxen::fit_field (src/tasks.cpp:139-194)
inline FitFieldResult fit_field(const NoiseFieldSpec& spec, const EncoderConfig& encoder_cfg, const TrainConfig& train_cfg,
                                const FitFieldOptions& opt = {}, int device = 0, void* stream = nullptr) {
  spec.validate();
  if (encoder_cfg.dim != spec.dim)
    throw std::invalid_argument("fit_field: encoder dim " + std::to_string(encoder_cfg.dim) + " != field dim " +
                                std::to_string(spec.dim));
  if (opt.holdout_samples < 2) throw std::invalid_argument("fit_field: holdout_samples must be >= 2");
  HashEncoder encoder(encoder_cfg, device);
  encoder.init_tables(opt.init_seed, stream);
  Mlp mlp(MlpConfig{encoder_cfg.encoded_width(), opt.mlp_hidden_width, opt.mlp_hidden_layers, 1}, device);
  mlp.init_params(sxen_hash_combine(opt.init_seed, 1), stream);
  if (opt.mlp_precision != MlpPrecision::exact) check(sxen_mlp_set_precision(mlp.handle(), static_cast<int>(opt.mlp_precision)));
  const sxen_noise_spec cs = spec.c();
  const std::uint64_t seed = train_cfg.seed;
  const std::size_t dim = static_cast<std::size_t>(spec.dim);
  const BatchSampler sampler = [=](int step, DeviceSpan<double> coords, DeviceSpan<double> /*aux*/,
                                   DeviceSpan<double> targets, void* s) {  // :156-166
    check(sxen_sample_field_batch(&cs, seed, 1, static_cast<std::uint64_t>(step), coords.size / dim, coords.data,
                                  targets.data, s));
  };
  TrainResult train = train_field(encoder, mlp, sampler, train_cfg, device, stream);
  // hold-out: CounterRng(hash_combine(seed, 'HOLD')) without a stream id (:172-173)
  const std::size_t n = static_cast<std::size_t>(opt.holdout_samples);
  const std::size_t enc_w = static_cast<std::size_t>(encoder_cfg.encoded_width());
  DeviceBuffer<double> coords(n * dim, device), targets(n, device);
  DeviceBuffer<float> feats(n * enc_w, device), pred(n, device);
  check(sxen_sample_field_batch(&cs, sxen_hash_combine(seed, 0x484f4c44ULL), 0, 0, n, coords.data(), targets.data(), stream));
  encoder.encode(coords.cspan(n * dim), feats.span(n * enc_w), stream);
  mlp.forward(feats.cspan(n * enc_w), pred.span(n), stream);
  const std::vector<float> p = pred.download(n, stream);
  const std::vector<double> t = targets.download(n, stream);
  encoder.check_async(stream);
  double se = 0.0, sum = 0.0, sum_sq = 0.0;  // :176-192
  for (std::size_t i = 0; i < n; ++i) {
    const double e = static_cast<double>(p[i]) - t[i];
    se += e * e;
    sum += t[i];
    sum_sq += t[i] * t[i];
  }
  const double mean = sum / static_cast<double>(n);
  FitFieldResult result{std::move(encoder), std::move(mlp), std::move(train), se / static_cast<double>(n),
                        std::max(0.0, sum_sq / static_cast<double>(n) - mean * mean)};
  return result;
}

}  // namespace sxen::b200
