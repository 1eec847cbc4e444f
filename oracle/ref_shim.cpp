// ref_shim.cpp -- extern "C" handle API over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  This file is our own code; it #includes the reference's public
// headers from $SXEN_REF/include at build time and is linked with the reference's own sources
// (lattice, encoding, mlp, optimizer, trainer, rng .cpp) compiled where they lie.  Outputs go to
// oracle/_ref/ only (git-ignored).  It exists to (a) validate oracle/sxen_oracle.c, (b) generate
// tests/golden fixtures, (c) serve as bench.py's `--impl reference` / cpu_baseline "reference" arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "sxen/encoding.hpp"
#include "sxen/hashing.hpp"
#include "sxen/lattice.hpp"
#include "sxen/mlp.hpp"
#include "sxen/optimizer.hpp"
#include "sxen/checkpoint.hpp"
#include "sxen/image.hpp"
#include "sxen/rng.hpp"
#include "sxen/noise.hpp"
#include "sxen/tasks.hpp"
#include "sxen/trainer.hpp"

#include <png.h>

namespace {

thread_local std::string g_err;

struct Cfg {  // layout-compatible with sxo_config
  std::int32_t dim, levels;
  std::uint32_t table_size;
  std::int32_t features, base_resolution;
  double growth;
  std::int32_t backend, level_scale;
};

struct MlpCfg {
  std::int32_t input_width, hidden_width, hidden_layers, output_width;
};

struct AdamCfg {
  double lr, beta1, beta2, epsilon;
};

sxen::EncoderConfig to_ref(const Cfg& c) {
  sxen::EncoderConfig e;
  e.dim = c.dim;
  e.levels = c.levels;
  e.table_size = c.table_size;
  e.features = c.features;
  e.base_resolution = c.base_resolution;
  e.growth = c.growth;
  e.backend = c.backend == 0 ? sxen::Backend::simplex : sxen::Backend::grid;
  e.level_scale = c.level_scale == 0 ? sxen::LevelScale::raw : sxen::LevelScale::equal_memory;
  return e;
}

sxen::MlpConfig to_ref(const MlpCfg& c) {
  sxen::MlpConfig m;
  m.input_width = c.input_width;
  m.hidden_width = c.hidden_width;
  m.hidden_layers = c.hidden_layers;
  m.output_width = c.output_width;
  return m;
}

sxen::AdamConfig to_ref(const AdamCfg& c) { return {c.lr, c.beta1, c.beta2, c.epsilon}; }

// status: 0 ok, 1 invalid_argument, 2 logic_error, 3 TrainingError, 9 other
template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 2;
  } catch (const sxen::TrainingError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

}  // namespace

extern "C" {

const char* sxr_last_error() { return g_err.c_str(); }

// ---- rng / hash / lattice free functions
std::uint64_t sxr_mix64(std::uint64_t z) { return sxen::mix64(z); }
std::uint64_t sxr_hash_combine(std::uint64_t a, std::uint64_t b) { return sxen::hash_combine(a, b); }
void sxr_rng_u64(std::uint64_t seed, int has_stream, std::uint64_t stream, std::size_t n, std::uint64_t* out) {
  sxen::CounterRng rng = has_stream ? sxen::CounterRng(seed, stream) : sxen::CounterRng(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = rng.next_u64();
}
void sxr_rng_double(std::uint64_t seed, int has_stream, std::uint64_t stream, std::size_t n, double lo,
                    double hi, int ranged, double* out) {
  sxen::CounterRng rng = has_stream ? sxen::CounterRng(seed, stream) : sxen::CounterRng(seed);
  for (std::size_t i = 0; i < n; ++i) out[i] = ranged ? rng.next_double(lo, hi) : rng.next_double();
}
std::uint32_t sxr_hash_coords(int n, const std::int64_t* c) {
  return sxen::hash_coords(std::span<const std::int64_t>(c, static_cast<std::size_t>(n)));
}
int sxr_skew_constants(int n, double* out) {
  return guarded([&] {
    const auto sc = sxen::SkewConstants::make(n);
    out[0] = sc.skew;
    out[1] = sc.unskew;
    out[2] = sc.scale;
  });
}
int sxr_subdivide(int n, const double* fracs, std::uint8_t* perm, double* sorted) {
  return guarded([&] {
    const auto s = sxen::subdivide(std::span<const double>(fracs, static_cast<std::size_t>(n)));
    for (int i = 0; i < n; ++i) {
      perm[i] = s.perm[static_cast<std::size_t>(i)];
      sorted[i] = s.sorted[static_cast<std::size_t>(i)];
    }
  });
}
int sxr_barycentric(int n, const double* sorted, double* w) {
  return guarded([&] {
    const auto b = sxen::barycentric_weights(std::span<const double>(sorted, static_cast<std::size_t>(n)));
    for (int i = 0; i <= n; ++i) w[i] = b.weights[static_cast<std::size_t>(i)];
  });
}

// ---- config
int sxr_validate(const Cfg* c) {
  return guarded([&] { to_ref(*c).validate(); });
}
int sxr_level_resolution(const Cfg* c, int level, std::uint32_t* out) {
  return guarded([&] { *out = sxen::level_resolution(to_ref(*c), level); });
}
double sxr_equal_memory_multiplier(int n) { return sxen::equal_memory_multiplier(n); }

// ---- encoder handle
void* sxr_encoder_create(const Cfg* c) {
  sxen::HashEncoder* h = nullptr;
  if (guarded([&] { h = new sxen::HashEncoder(to_ref(*c)); }) != 0) return nullptr;
  return h;
}
void sxr_encoder_destroy(void* h) { delete static_cast<sxen::HashEncoder*>(h); }
void sxr_encoder_init_tables(void* h, std::uint64_t seed) { static_cast<sxen::HashEncoder*>(h)->init_tables(seed); }
float* sxr_encoder_table(void* h, int level) { return static_cast<sxen::HashEncoder*>(h)->table(level).data(); }
std::uint32_t sxr_encoder_resolution(void* h, int level) { return static_cast<sxen::HashEncoder*>(h)->resolution(level); }
void sxr_encoder_counters(void* h, std::uint64_t* out) {
  const auto c = static_cast<sxen::HashEncoder*>(h)->counters();
  out[0] = c.touched_vertices;
  out[1] = c.out_of_bounds;
}
void sxr_encoder_reset_counters(void* h) { static_cast<sxen::HashEncoder*>(h)->reset_counters(); }

// batched encode; *bad = index of the sample that threw (or -1)
int sxr_encode(void* h, const double* x, std::size_t n_samples, float* out, long* bad) {
  auto* enc = static_cast<sxen::HashEncoder*>(h);
  const auto dim = static_cast<std::size_t>(enc->config().dim);
  const auto lf = static_cast<std::size_t>(enc->config().encoded_width());
  *bad = -1;
  std::size_t s = 0;
  const int st = guarded([&] {
    for (s = 0; s < n_samples; ++s) {
      enc->encode(std::span<const double>(x + s * dim, dim), std::span<float>(out + s * lf, lf));
    }
  });
  if (st != 0) *bad = static_cast<long>(s);
  return st;
}

// ---- gradient accumulator handle
void* sxr_grad_create(int levels, std::uint32_t table_size, int features) {
  sxen::EncoderGradient* g = nullptr;
  if (guarded([&] { g = new sxen::EncoderGradient(levels, table_size, features); }) != 0) return nullptr;
  return g;
}
void sxr_grad_destroy(void* g) { delete static_cast<sxen::EncoderGradient*>(g); }
void sxr_grad_clear(void* g) { static_cast<sxen::EncoderGradient*>(g)->clear(); }
std::size_t sxr_grad_touched_count(void* g, int level) { return static_cast<sxen::EncoderGradient*>(g)->touched(level).size(); }
// touch-order index list of a level and the matching slices (count x features doubles)
void sxr_grad_read(void* g, int level, std::uint32_t* idx, double* values) {
  auto* gr = static_cast<sxen::EncoderGradient*>(g);
  const auto t = gr->touched(level);
  const auto f = static_cast<std::size_t>(gr->features());
  for (std::size_t i = 0; i < t.size(); ++i) {
    idx[i] = t[i];
    const auto sl = gr->slice(level, t[i]);
    std::memcpy(values + i * f, sl.data(), f * sizeof(double));
  }
}
int sxr_grad_merge(void* dst, void* src) {
  return guarded([&] { static_cast<sxen::EncoderGradient*>(dst)->merge(*static_cast<sxen::EncoderGradient*>(src)); });
}

int sxr_encode_backward(void* h, const double* x, const double* upstream, std::size_t n_samples, void* g,
                        long* bad) {
  auto* enc = static_cast<sxen::HashEncoder*>(h);
  auto* gr = static_cast<sxen::EncoderGradient*>(g);
  const auto dim = static_cast<std::size_t>(enc->config().dim);
  const auto lf = static_cast<std::size_t>(enc->config().encoded_width());
  *bad = -1;
  std::size_t s = 0;
  const int st = guarded([&] {
    for (s = 0; s < n_samples; ++s) {
      enc->encode_backward(std::span<const double>(x + s * dim, dim),
                           std::span<const double>(upstream + s * lf, lf), *gr);
    }
  });
  if (st != 0) *bad = static_cast<long>(s);
  return st;
}

// ---- MLP handle
void* sxr_mlp_create(const MlpCfg* c) {
  sxen::Mlp* m = nullptr;
  if (guarded([&] { m = new sxen::Mlp(to_ref(*c)); }) != 0) return nullptr;
  return m;
}
void sxr_mlp_destroy(void* m) { delete static_cast<sxen::Mlp*>(m); }
std::size_t sxr_mlp_param_count(void* m) { return static_cast<sxen::Mlp*>(m)->parameter_count(); }
float* sxr_mlp_params(void* m) { return static_cast<sxen::Mlp*>(m)->parameters().data(); }
void sxr_mlp_init(void* m, std::uint64_t seed) { static_cast<sxen::Mlp*>(m)->init_params(seed); }

// forward (+ optional backward) over a batch; grads accumulate into mlp_grad (param_count doubles)
int sxr_mlp_forward_backward(void* mh, const float* input, std::size_t n_samples, float* out,
                             const double* upstream, double* mlp_grad, double* input_grad) {
  auto* mlp = static_cast<sxen::Mlp*>(mh);
  const auto& mc = mlp->config();
  return guarded([&] {
    sxen::MlpWorkspace ws(mc);
    sxen::MlpGradient grad(mc);
    const auto iw = static_cast<std::size_t>(mc.input_width);
    const auto ow = static_cast<std::size_t>(mc.output_width);
    for (std::size_t s = 0; s < n_samples; ++s) {
      mlp->forward(std::span<const float>(input + s * iw, iw), ws);
      if (out) std::memcpy(out + s * ow, ws.output().data(), ow * sizeof(float));
      if (upstream) {
        mlp->backward(std::span<const double>(upstream + s * ow, ow), ws, grad);
        if (input_grad) std::memcpy(input_grad + s * iw, ws.input_grad().data(), iw * sizeof(double));
      }
    }
    if (upstream && mlp_grad) {
      const auto v = grad.values();
      for (std::size_t i = 0; i < v.size(); ++i) mlp_grad[i] += v[i];
    }
  });
}

// ---- optimizers (state handles)
void* sxr_adam_create(std::size_t n) { return new sxen::AdamState(n); }
void sxr_adam_destroy(void* a) { delete static_cast<sxen::AdamState*>(a); }
int sxr_adam_step(void* a, float* params, const double* grads, std::size_t n, const AdamCfg* c) {
  return guarded([&] {
    static_cast<sxen::AdamState*>(a)->step(std::span<float>(params, n), std::span<const double>(grads, n), to_ref(*c));
  });
}
void* sxr_sparse_adam_create(int levels, std::uint32_t table_size, int features) {
  return new sxen::SparseAdamState(levels, table_size, features);
}
void sxr_sparse_adam_destroy(void* a) { delete static_cast<sxen::SparseAdamState*>(a); }
int sxr_sparse_adam_step(void* a, void* enc, void* grad, const AdamCfg* c) {
  return guarded([&] {
    static_cast<sxen::SparseAdamState*>(a)->step(*static_cast<sxen::HashEncoder*>(enc),
                                                *static_cast<sxen::EncoderGradient*>(grad), to_ref(*c));
  });
}

// ---- train_field with an explicit (pre-sampled) batch stream: coords steps x B x dim, targets
// steps x B x out_w.  Runs the reference's own train_field (src/trainer.cpp:53) and returns the
// per-step loss (record_every = 1).
int sxr_train_field(void* eh, void* mh, const double* coords, const double* targets, int steps, int batch,
                    int threads, const AdamCfg* table_adam, const AdamCfg* mlp_adam, double* loss_out) {
  auto* enc = static_cast<sxen::HashEncoder*>(eh);
  auto* mlp = static_cast<sxen::Mlp*>(mh);
  return guarded([&] {
    const auto dim = static_cast<std::size_t>(enc->config().dim);
    const auto ow = static_cast<std::size_t>(mlp->config().output_width);
    sxen::TrainConfig tc;
    tc.batch_size = batch;
    tc.steps = steps;
    tc.table_adam = to_ref(*table_adam);
    tc.mlp_adam = to_ref(*mlp_adam);
    tc.threads = threads;
    tc.record_every = 1;
    sxen::BatchSampler sampler = [&](int step, std::span<double> c, std::span<double>, std::span<double> t) {
      std::memcpy(c.data(), coords + static_cast<std::size_t>(step) * c.size(), c.size() * sizeof(double));
      std::memcpy(t.data(), targets + static_cast<std::size_t>(step) * t.size(), t.size() * sizeof(double));
      (void)dim;
      (void)ow;
    };
    const sxen::TrainResult r = sxen::train_field(*enc, *mlp, sampler, tc);
    for (std::size_t i = 0; i < r.loss_curve.size(); ++i) loss_out[r.loss_curve[i].first] = r.loss_curve[i].second;
  });
}

// train_field with pass-through inputs (TrainConfig::aux_dims, src/trainer.cpp:32-35,59-65): the sampler replays
// caller-provided coords / aux / targets, one slab per step.
int sxr_train_field_aux(void* eh, void* mh, const double* coords, const double* aux, int aux_dims, const double* targets,
                        int steps, int batch, int threads, const AdamCfg* table_adam, const AdamCfg* mlp_adam,
                        double* loss_out) {
  auto* enc = static_cast<sxen::HashEncoder*>(eh);
  auto* mlp = static_cast<sxen::Mlp*>(mh);
  return guarded([&] {
    sxen::TrainConfig tc;
    tc.batch_size = batch;
    tc.steps = steps;
    tc.aux_dims = aux_dims;
    tc.table_adam = to_ref(*table_adam);
    tc.mlp_adam = to_ref(*mlp_adam);
    tc.threads = threads;
    tc.record_every = 1;
    sxen::BatchSampler sampler = [&](int step, std::span<double> c, std::span<double> a, std::span<double> t) {
      std::memcpy(c.data(), coords + static_cast<std::size_t>(step) * c.size(), c.size() * sizeof(double));
      if (!a.empty()) std::memcpy(a.data(), aux + static_cast<std::size_t>(step) * a.size(), a.size() * sizeof(double));
      std::memcpy(t.data(), targets + static_cast<std::size_t>(step) * t.size(), t.size() * sizeof(double));
    };
    const sxen::TrainResult r = sxen::train_field(*enc, *mlp, sampler, tc);
    for (std::size_t i = 0; i < r.loss_curve.size(); ++i) loss_out[r.loss_curve[i].first] = r.loss_curve[i].second;
  });
}

// ---- CPU baseline: the reference's worker pattern (src/trainer.cpp:104-116) restricted to the
// encode + encode_backward pair, steady_clock around the fan-out (src/analysis.cpp:279-290).
// Accumulators are allocated and cleared outside the timed region.  Returns seconds (<0 on error).
double sxr_bench_fwd_bwd(void* h, const double* x, const double* upstream, std::size_t n_samples, int threads) {
  auto* enc = static_cast<sxen::HashEncoder*>(h);
  const auto& cfg = enc->config();
  if (threads < 1) threads = 1;
  const auto dim = static_cast<std::size_t>(cfg.dim);
  const auto lf = static_cast<std::size_t>(cfg.encoded_width());
  double seconds = -1.0;
  const int st = guarded([&] {
    std::vector<sxen::EncoderGradient> grads(static_cast<std::size_t>(threads));
    for (auto& g : grads) g.reset(cfg.levels, cfg.table_size, cfg.features);
    const std::size_t chunk = (n_samples + static_cast<std::size_t>(threads) - 1) / static_cast<std::size_t>(threads);
    auto work = [&](int t) {
      std::vector<float> out(lf);
      const std::size_t begin = std::min(n_samples, static_cast<std::size_t>(t) * chunk);
      const std::size_t end = std::min(n_samples, begin + chunk);
      for (std::size_t s = begin; s < end; ++s) {
        const std::span<const double> xs(x + s * dim, dim);
        enc->encode(xs, out);
        enc->encode_backward(xs, std::span<const double>(upstream + s * lf, lf), grads[static_cast<std::size_t>(t)]);
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(work, t);
    work(0);
    for (auto& th : pool) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    seconds = std::chrono::duration<double>(t1 - t0).count();
  });
  return st == 0 ? seconds : -1.0;
}

int sxr_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

// ---- libpng stand-ins (see oracle/png_stub/png.h): always fail, the reference raises IoError
int png_image_begin_read_from_file(png_image* image, const char*) {
  std::strncpy(image->message, "libpng is not available in the oracle build", sizeof(image->message) - 1);
  return 0;
}
int png_image_finish_read(png_image*, const void*, void*, int, void*) { return 0; }
void png_image_free(png_image*) {}
int png_image_write_to_file(png_image* image, const char*, int, const void*, int, const void*) {
  std::strncpy(image->message, "libpng is not available in the oracle build", sizeof(image->message) - 1);
  return 0;
}

// ---- tasks: make_test_image (src/image.cpp:68-96), fit_image (src/tasks.cpp:98-137), render_image + PSNR (:30-96)
int sxr_make_test_image(int width, int height, std::uint64_t seed, double* pixels_out) {
  return guarded([&] {
    const sxen::ImageDataset img = sxen::make_test_image(width, height, seed);
    std::memcpy(pixels_out, img.pixels.data(), img.pixels.size() * sizeof(double));
  });
}

// Runs the reference's fit_image.  Outputs: final PSNR, per-step loss (record_every = 1), trained tables (L x T*F) and
// MLP parameters.
int sxr_fit_image(const double* pixels, int width, int height, const Cfg* cfg, int batch, int steps, std::uint64_t train_seed,
                  int threads, std::uint64_t init_seed, int hidden_width, int hidden_layers, const AdamCfg* table_adam,
                  const AdamCfg* mlp_adam, double* final_psnr, double* loss_out, float* tables_out, float* mlp_out) {
  return guarded([&] {
    sxen::ImageDataset img;
    img.width = width;
    img.height = height;
    img.pixels.assign(pixels, pixels + 3 * static_cast<std::size_t>(width) * static_cast<std::size_t>(height));
    sxen::TrainConfig tc;
    tc.batch_size = batch;
    tc.steps = steps;
    tc.seed = train_seed;
    tc.threads = threads;
    tc.record_every = 1;
    tc.table_adam = to_ref(*table_adam);
    tc.mlp_adam = to_ref(*mlp_adam);
    sxen::FitImageOptions opt;
    opt.init_seed = init_seed;
    opt.mlp_hidden_width = hidden_width;
    opt.mlp_hidden_layers = hidden_layers;
    const sxen::EncoderConfig ec = to_ref(*cfg);
    sxen::FitImageResult r = sxen::fit_image(img, ec, tc, opt);
    *final_psnr = r.final_psnr;
    for (const auto& [step, loss] : r.train.loss_curve) loss_out[step] = loss;
    const std::size_t per = static_cast<std::size_t>(ec.table_size) * static_cast<std::size_t>(ec.features);
    for (int l = 0; l < ec.levels; ++l) std::memcpy(tables_out + static_cast<std::size_t>(l) * per, r.encoder.table(l).data(), per * sizeof(float));
    std::memcpy(mlp_out, r.mlp.parameters().data(), r.mlp.parameter_count() * sizeof(float));
  });
}

double sxr_psnr_from_mse(double mse) { return sxen::psnr_from_mse(mse); }

// ---- noise field + fit_field (src/noise.cpp:167-188, src/tasks.cpp:139-194)
static sxen::NoiseFieldSpec noise_spec(int dim, std::uint64_t seed, int kind, int octaves, double frequency) {
  sxen::NoiseFieldSpec spec;
  spec.dim = dim;
  spec.seed = seed;
  spec.kind = kind == 0 ? sxen::NoiseKind::perlin : sxen::NoiseKind::simplex;
  spec.octaves = octaves;
  spec.frequency = frequency;
  return spec;
}

int sxr_noise_field(int dim, std::uint64_t seed, int kind, int octaves, double frequency, const double* x, std::size_t n,
                    double* out) {
  return guarded([&] {
    const sxen::NoiseFieldSpec spec = noise_spec(dim, seed, kind, octaves, frequency);
    for (std::size_t s = 0; s < n; ++s)
      out[s] = sxen::noise_field_value(spec, std::span<const double>(x + s * static_cast<std::size_t>(dim), static_cast<std::size_t>(dim)));
  });
}

// Runs the reference's fit_field.  Outputs: per-step loss (record_every = 1), hold-out MSE, field variance.
int sxr_fit_field(int dim, std::uint64_t seed, int kind, int octaves, double frequency, const Cfg* cfg, int batch, int steps,
                  std::uint64_t train_seed, int threads, std::uint64_t init_seed, int hidden_width, int hidden_layers,
                  int holdout_samples, double* loss_out, double* holdout_mse, double* field_variance) {
  return guarded([&] {
    const sxen::NoiseFieldSpec spec = noise_spec(dim, seed, kind, octaves, frequency);
    sxen::TrainConfig tc;
    tc.batch_size = batch;
    tc.steps = steps;
    tc.seed = train_seed;
    tc.threads = threads;
    tc.record_every = 1;
    sxen::FitFieldOptions opt;
    opt.init_seed = init_seed;
    opt.mlp_hidden_width = hidden_width;
    opt.mlp_hidden_layers = hidden_layers;
    opt.holdout_samples = holdout_samples;
    sxen::FitFieldResult r = sxen::fit_field(spec, to_ref(*cfg), tc, opt);
    for (const auto& [step, loss] : r.train.loss_curve) loss_out[step] = loss;
    *holdout_mse = r.holdout_mse;
    *field_variance = r.field_variance;
  });
}

// ---- checkpoint (src/checkpoint.cpp:81-175); status 9 = IoError
int sxr_save_checkpoint(const char* path, void* enc, void* mlp) {
  return guarded([&] { sxen::save_checkpoint(path, *static_cast<sxen::HashEncoder*>(enc), static_cast<sxen::Mlp*>(mlp)); });
}
// Loads with the reference and copies out: cfg, tables (L x T*F), and the MLP section if present (has_mlp, mlp cfg, params).
int sxr_load_checkpoint(const char* path, Cfg* cfg, float* tables_out, std::size_t tables_capacity, int* has_mlp, MlpCfg* mcfg,
                        float* mlp_out, std::size_t mlp_capacity) {
  return guarded([&] {
    sxen::LoadedCheckpoint ck = sxen::load_checkpoint(path);
    const sxen::EncoderConfig& ec = ck.encoder.config();
    *cfg = Cfg{ec.dim, ec.levels, ec.table_size, ec.features, ec.base_resolution, ec.growth,
               ec.backend == sxen::Backend::simplex ? 0 : 1, 0};
    const std::size_t per = static_cast<std::size_t>(ec.table_size) * static_cast<std::size_t>(ec.features);
    if (per * static_cast<std::size_t>(ec.levels) > tables_capacity) throw std::invalid_argument("table buffer too small");
    for (int l = 0; l < ec.levels; ++l) std::memcpy(tables_out + static_cast<std::size_t>(l) * per, ck.encoder.table(l).data(), per * sizeof(float));
    *has_mlp = ck.mlp.has_value() ? 1 : 0;
    if (ck.mlp) {
      const sxen::MlpConfig& mc = ck.mlp->config();
      *mcfg = MlpCfg{mc.input_width, mc.hidden_width, mc.hidden_layers, mc.output_width};
      if (ck.mlp->parameter_count() > mlp_capacity) throw std::invalid_argument("mlp buffer too small");
      std::memcpy(mlp_out, ck.mlp->parameters().data(), ck.mlp->parameter_count() * sizeof(float));
    }
  });
}

}  // extern "C"
