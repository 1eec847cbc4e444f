// sxen_b200.hpp -- header-only C++ mirror of the reference's classes over the C ABI (sxen_cuda.h).
//
// A maintainer of the reference swaps `#include "sxen/encoding.hpp"` for this header on the hot path: same class and
// method names (namespace sxen::b200), same exception types (std::invalid_argument, std::logic_error,
// sxen::b200::TrainingError / IoError mirror include/sxen/errors.hpp:8-15), batched spans instead of one sample per
// call.  Host spans take the pipelined *_host entry points; DeviceSpan arguments take the asynchronous device ones.
// Everything below is a thin call into libsxen_b200.so -- no arithmetic happens in this header.
#pragma once

#include <cstddef>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sxen_cuda.h"

namespace sxen::b200 {

struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct TrainingError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// SXEN_NCCL_ERROR: the gradient exchange between ranks failed (no reference analogue either).
struct CommError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Re-raises a C-ABI status as the exception the reference would have thrown.
inline void check(sxen_status st) {
  if (st == SXEN_OK) return;
  const std::string msg = sxen_last_error();
  switch (st) {
    case SXEN_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case SXEN_LOGIC_ERROR: throw std::logic_error(msg);
    case SXEN_TRAINING_ERROR: throw TrainingError(msg);
    case SXEN_IO_ERROR: throw IoError(msg);
    case SXEN_NCCL_ERROR: throw CommError(msg);
    default: throw CudaError(msg);
  }
}

enum class Backend { simplex = SXEN_BACKEND_SIMPLEX, grid = SXEN_BACKEND_GRID };
enum class LevelScale { raw = SXEN_SCALE_RAW, equal_memory = SXEN_SCALE_EQUAL_MEMORY };

// include/sxen/encoding.hpp:18-33
struct EncoderConfig {
  int dim = 2;
  int levels = 8;
  std::uint32_t table_size = 1u << 16;
  int features = 2;
  int base_resolution = 16;
  double growth = 2.0;
  Backend backend = Backend::simplex;
  LevelScale level_scale = LevelScale::raw;

  int encoded_width() const { return levels * features; }
  sxen_encoder_config c() const {
    return {dim, levels, table_size, features, base_resolution, growth, static_cast<int32_t>(backend),
            static_cast<int32_t>(level_scale)};
  }
  void validate() const {
    const sxen_encoder_config cc = c();
    check(sxen_encoder_validate(&cc));
  }
};

inline double equal_memory_multiplier(int n) {
  double out = 0.0;
  check(sxen_equal_memory_multiplier(n, &out));
  return out;
}

inline std::uint32_t level_resolution(const EncoderConfig& cfg, int level) {
  const sxen_encoder_config cc = cfg.c();
  std::uint32_t out = 0;
  check(sxen_level_resolution(&cc, level, &out));
  return out;
}

struct LookupCounters {
  std::uint64_t touched_vertices = 0;
  std::uint64_t out_of_bounds = 0;
};

// Caller-owned device memory (cudaMalloc'ed by the caller); never retained by the library.
template <class T>
struct DeviceSpan {
  T* data = nullptr;
  std::size_t size = 0;
};

class HashEncoder;

// include/sxen/encoding.hpp:53-86
class EncoderGradient {
 public:
  EncoderGradient() = default;
  explicit EncoderGradient(const HashEncoder& enc);
  EncoderGradient(EncoderGradient&& o) noexcept : h_(std::exchange(o.h_, nullptr)), levels_(o.levels_), features_(o.features_), table_size_(o.table_size_) {}
  EncoderGradient& operator=(EncoderGradient&& o) noexcept {
    if (this != &o) {
      sxen_grad_destroy(h_);
      h_ = std::exchange(o.h_, nullptr);
      levels_ = o.levels_;
      features_ = o.features_;
      table_size_ = o.table_size_;
    }
    return *this;
  }
  EncoderGradient(const EncoderGradient&) = delete;
  EncoderGradient& operator=(const EncoderGradient&) = delete;
  ~EncoderGradient() { sxen_grad_destroy(h_); }

  void clear(void* stream = nullptr) { check(sxen_grad_clear(h_, stream)); }
  void merge(const EncoderGradient& other, void* stream = nullptr) { check(sxen_grad_merge(h_, other.h_, stream)); }
  std::uint64_t touched_total() const {
    std::uint64_t out = 0;
    check(sxen_grad_touched_total(h_, &out));
    return out;
  }
  int levels() const { return levels_; }
  int features() const { return features_; }
  // slice() / touched() of one level, copied to the host: values T*F floats, touched T bytes.
  void download(int level, std::vector<float>& values, std::vector<std::uint8_t>& touched) const {
    values.resize(static_cast<std::size_t>(table_size_) * static_cast<std::size_t>(features_));
    touched.resize(table_size_);
    check(sxen_grad_download(h_, level, values.data(), touched.data()));
  }
  sxen_grad* handle() const { return h_; }

 private:
  sxen_grad* h_ = nullptr;
  int levels_ = 0, features_ = 0;
  std::uint32_t table_size_ = 0;
};

// include/sxen/encoding.hpp:92-148
class HashEncoder {
 public:
  explicit HashEncoder(EncoderConfig cfg, int device = 0) : cfg_(cfg) {
    const sxen_encoder_config cc = cfg.c();
    check(sxen_encoder_create(&cc, device, &h_));
  }
  HashEncoder(HashEncoder&& o) noexcept : cfg_(o.cfg_), h_(std::exchange(o.h_, nullptr)) {}
  HashEncoder& operator=(HashEncoder&& o) noexcept {
    if (this != &o) {
      sxen_encoder_destroy(h_);
      cfg_ = o.cfg_;
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  HashEncoder(const HashEncoder&) = delete;
  HashEncoder& operator=(const HashEncoder&) = delete;
  ~HashEncoder() { sxen_encoder_destroy(h_); }

  const EncoderConfig& config() const { return cfg_; }
  std::uint32_t resolution(int level) const {
    std::uint32_t out = 0;
    check(sxen_encoder_resolution(h_, level, &out));
    return out;
  }
  void init_tables(std::uint64_t seed, void* stream = nullptr) { check(sxen_encoder_init_tables(h_, seed, stream)); }
  std::vector<float> table(int level) const {
    std::vector<float> out(static_cast<std::size_t>(cfg_.table_size) * static_cast<std::size_t>(cfg_.features));
    check(sxen_encoder_download_table(h_, level, out.data()));
    return out;
  }
  void set_table(int level, std::span<const float> values) {
    if (values.size() != static_cast<std::size_t>(cfg_.table_size) * static_cast<std::size_t>(cfg_.features))
      throw std::invalid_argument("table: wrong element count");
    check(sxen_encoder_upload_table(h_, level, values.data()));
  }
  std::uint64_t parameter_count() const {
    std::uint64_t out = 0;
    check(sxen_encoder_parameter_count(h_, &out));
    return out;
  }

  // Batched encode: x holds N*dim doubles, out N*levels*features floats (host memory).
  void encode(std::span<const double> x, std::span<float> out) const {
    const std::size_t n = batch_of(x.size());
    if (out.size() != n * static_cast<std::size_t>(cfg_.encoded_width()))
      throw std::invalid_argument("encode: output span has wrong width");
    check(sxen_encoder_encode_host(h_, x.data(), n, out.data()));
  }
  void encode_backward(std::span<const double> x, std::span<const double> upstream, EncoderGradient& grad) const {
    const std::size_t n = batch_of(x.size());
    if (upstream.size() != n * static_cast<std::size_t>(cfg_.encoded_width()))
      throw std::invalid_argument("encode_backward: upstream span has wrong width");
    check(sxen_encoder_encode_backward_host(h_, x.data(), upstream.data(), n, grad.handle()));
  }
  // Device-resident forms (asynchronous on `stream`; call check_async() to surface input errors).
  void encode(DeviceSpan<const double> x, DeviceSpan<float> out, void* stream = nullptr) const {
    check(sxen_encoder_encode(h_, x.data, SXEN_COORD_F64, batch_of(x.size), out.data, stream));
  }
  void encode(DeviceSpan<const float> x, DeviceSpan<float> out, void* stream = nullptr) const {
    check(sxen_encoder_encode(h_, x.data, SXEN_COORD_F32, batch_of(x.size), out.data, stream));
  }
  void encode_backward(DeviceSpan<const float> x, DeviceSpan<const float> upstream, EncoderGradient& grad,
                       void* stream = nullptr) const {
    check(sxen_encoder_encode_backward(h_, x.data, SXEN_COORD_F32, upstream.data, batch_of(x.size), grad.handle(), stream));
  }
  // One contiguous range of levels (multi-GPU hosts all-reduce each range's slice of the accumulator while the next
  // range computes; include/sxen_cuda.h: sxen_encoder_encode_backward_levels).
  void encode_backward(DeviceSpan<const float> x, DeviceSpan<const float> upstream, EncoderGradient& grad, int first_level,
                       int level_count, void* stream = nullptr) const {
    check(sxen_encoder_encode_backward_levels(h_, x.data, SXEN_COORD_F32, upstream.data, batch_of(x.size), grad.handle(),
                                              first_level, level_count, stream));
  }
  // encode + encode_backward of one batch off a single lattice walk (the run_chunk pair, src/trainer.cpp:31,47).
  void encode_forward_backward(DeviceSpan<const float> x, DeviceSpan<const float> upstream, DeviceSpan<float> out,
                               EncoderGradient& grad, void* stream = nullptr) const {
    check(sxen_encoder_encode_forward_backward(h_, x.data, SXEN_COORD_F32, upstream.data, batch_of(x.size), out.data,
                                               grad.handle(), stream));
  }
  void check_async(void* stream = nullptr) const { check(sxen_encoder_check(h_, stream)); }

  LookupCounters counters() const {
    sxen_lookup_counters c{};
    check(sxen_encoder_counters(h_, &c));
    return {c.touched_vertices, c.out_of_bounds};
  }
  void reset_counters() const { check(sxen_encoder_reset_counters(h_)); }
  sxen_encoder* handle() const { return h_; }

 private:
  std::size_t batch_of(std::size_t coords) const {
    if (coords % static_cast<std::size_t>(cfg_.dim) != 0)
      throw std::invalid_argument("encode: expected " + std::to_string(cfg_.dim) + " coordinates per sample");
    return coords / static_cast<std::size_t>(cfg_.dim);
  }
  EncoderConfig cfg_;
  sxen_encoder* h_ = nullptr;
};

inline EncoderGradient::EncoderGradient(const HashEncoder& enc)
    : levels_(enc.config().levels), features_(enc.config().features), table_size_(enc.config().table_size) {
  check(sxen_grad_create(enc.handle(), &h_));
}

// include/sxen/optimizer.hpp:13-18
struct AdamConfig {
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.99, epsilon = 1e-15;
  sxen_adam_config c() const { return {lr, beta1, beta2, epsilon}; }
};

// include/sxen/optimizer.hpp:42-59
class SparseAdamState {
 public:
  explicit SparseAdamState(const HashEncoder& enc) { check(sxen_sparse_adam_create(enc.handle(), &h_)); }
  SparseAdamState(const SparseAdamState&) = delete;
  SparseAdamState& operator=(const SparseAdamState&) = delete;
  ~SparseAdamState() { sxen_sparse_adam_destroy(h_); }
  std::int64_t step_count() const {
    std::int64_t t = 0;
    check(sxen_sparse_adam_step_count(h_, &t));
    return t;
  }
  void step(HashEncoder& encoder, EncoderGradient& grads, const AdamConfig& cfg, void* stream = nullptr) {
    const sxen_adam_config c = cfg.c();
    check(sxen_sparse_adam_step(h_, encoder.handle(), grads.handle(), &c, 0, stream));
    check(sxen_sparse_adam_check(h_, stream));  // TrainingError on a non-finite gradient, like the reference
  }

 private:
  sxen_sparse_adam* h_ = nullptr;
};

// include/sxen/mlp.hpp:11-25
struct MlpConfig {
  int input_width = 32, hidden_width = 64, hidden_layers = 2, output_width = 3;
  int layer_count() const { return hidden_layers + 1; }
  sxen_mlp_config c() const { return {input_width, hidden_width, hidden_layers, output_width}; }
  void validate() const {
    const sxen_mlp_config cc = c();
    check(sxen_mlp_validate(&cc));
  }
};

// include/sxen/mlp.hpp:76-108 (parameters + MlpGradient + the batched MlpWorkspace live behind one handle)
class Mlp {
 public:
  explicit Mlp(MlpConfig cfg, int device = 0) : cfg_(cfg) {
    const sxen_mlp_config cc = cfg.c();
    check(sxen_mlp_create(&cc, device, &h_));
  }
  Mlp(Mlp&& o) noexcept : cfg_(o.cfg_), h_(std::exchange(o.h_, nullptr)) {}  // movable, not copyable (include/sxen/mlp.hpp)
  Mlp& operator=(Mlp&& o) noexcept {
    if (this != &o) {
      sxen_mlp_destroy(h_);
      cfg_ = o.cfg_;
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  Mlp(const Mlp&) = delete;
  Mlp& operator=(const Mlp&) = delete;
  ~Mlp() { sxen_mlp_destroy(h_); }
  const MlpConfig& config() const { return cfg_; }
  std::size_t parameter_count() const {
    std::uint64_t n = 0;
    check(sxen_mlp_parameter_count(h_, &n));
    return static_cast<std::size_t>(n);
  }
  void init_params(std::uint64_t seed, void* stream = nullptr) { check(sxen_mlp_init_params(h_, seed, stream)); }
  std::vector<float> parameters() const {
    std::vector<float> p(parameter_count());
    check(sxen_mlp_download_params(h_, p.data()));
    return p;
  }
  void set_parameters(std::span<const float> values) {
    if (values.size() != parameter_count()) throw std::invalid_argument("mlp: parameter count mismatch");
    check(sxen_mlp_upload_params(h_, values.data()));
  }
  // The reference's call shape (include/sxen/mlp.hpp:94-99) with host spans, N samples per call: `out` is
  // MlpWorkspace::output(), `input_grad` MlpWorkspace::input_grad(); the workspace and the MlpGradient live in the handle.
  void forward(std::span<const float> input, std::span<float> out) {
    const std::size_t in_w = static_cast<std::size_t>(cfg_.input_width), out_w = static_cast<std::size_t>(cfg_.output_width);
    if (input.size() % in_w != 0 || out.size() != input.size() / in_w * out_w)  // src/mlp.cpp:138-143
      throw std::invalid_argument("mlp forward: input or output span has the wrong width");
    check(sxen_mlp_forward_host(h_, input.data(), input.size() / in_w, out.data()));
  }
  void backward(std::span<const double> upstream, std::span<double> input_grad) {
    const std::size_t in_w = static_cast<std::size_t>(cfg_.input_width), out_w = static_cast<std::size_t>(cfg_.output_width);
    if (upstream.size() % out_w != 0 || (!input_grad.empty() && input_grad.size() != upstream.size() / out_w * in_w))
      throw std::invalid_argument("mlp backward: upstream span has the wrong width");  // src/mlp.cpp:168-173
    check(sxen_mlp_backward_host(h_, upstream.data(), upstream.size() / out_w, input_grad.empty() ? nullptr : input_grad.data()));
  }
  // MlpGradient::values() / clear() (include/sxen/mlp.hpp:40-74): fp64, laid out like parameters()
  std::vector<double> gradient() const {
    std::vector<double> g(parameter_count());
    check(sxen_mlp_grad_download(h_, g.data()));
    return g;
  }
  void clear_gradient(void* stream = nullptr) { check(sxen_mlp_grad_clear(h_, stream)); }
  int layer_count() const { return cfg_.hidden_layers + 1; }
  int layer_input_width(int l) const { return l == 0 ? cfg_.input_width : cfg_.hidden_width; }
  int layer_output_width(int l) const { return l == layer_count() - 1 ? cfg_.output_width : cfg_.hidden_width; }
  // offset of layer l's weights in parameters() (per layer: out*in weights, then out biases; src/mlp.cpp:19-32)
  std::size_t layer_offset(int l) const {
    std::size_t off = 0;
    for (int k = 0; k < l; ++k)
      off += static_cast<std::size_t>(layer_input_width(k)) * layer_output_width(k) + static_cast<std::size_t>(layer_output_width(k));
    return off;
  }
  void forward(DeviceSpan<const float> input, DeviceSpan<float> out, void* stream = nullptr) {
    check(sxen_mlp_forward(h_, input.data, input.size / static_cast<std::size_t>(cfg_.input_width), out.data, stream));
  }
  void backward(DeviceSpan<const double> upstream, DeviceSpan<float> input_grad, void* stream = nullptr) {
    check(sxen_mlp_backward(h_, upstream.data, upstream.size / static_cast<std::size_t>(cfg_.output_width),
                            input_grad.data, nullptr, stream));
  }
  sxen_mlp* handle() const { return h_; }

 private:
  MlpConfig cfg_;
  sxen_mlp* h_ = nullptr;
};

}  // namespace sxen::b200
