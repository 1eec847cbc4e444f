// Compiled and run by tests/test_gpu_cpp_trainer.py on a B200: the C++ trainer/tasks mirror (include/sxen_b200_train.hpp)
// driving the C ABI with no Python and no CUDA headers in the host program.  Prints one "key value..." line per result;
// the pytest compares them with the reference's own runs (tests/golden/task_cases.npz, field_cases.npz).
//   argv: image.f64 width height  L T F base growth  steps batch
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>

#include "sxen_b200_train.hpp"

using namespace sxen::b200;

#define EXPECT(cond)                                            \
  do {                                                          \
    if (!(cond)) {                                              \
      std::printf("FAILED line %d: %s\n", __LINE__, #cond);     \
      return 1;                                                 \
    }                                                           \
  } while (0)

static void print_curve(const char* key, const TrainResult& r) {
  std::printf("%s", key);
  for (const auto& [s, l] : r.loss_curve) std::printf(" %.17g", l);
  std::printf("\n");
}

int main(int argc, char** argv) {
  if (argc != 11) {
    std::printf("usage: image.f64 w h L T F base growth steps batch\n");
    return 2;
  }
  ImageDataset img;
  img.width = std::atoi(argv[2]);
  img.height = std::atoi(argv[3]);
  img.pixels.resize(static_cast<std::size_t>(img.width) * img.height * 3);
  {
    std::FILE* f = std::fopen(argv[1], "rb");
    EXPECT(f != nullptr);
    EXPECT(std::fread(img.pixels.data(), sizeof(double), img.pixels.size(), f) == img.pixels.size());
    std::fclose(f);
  }
  EncoderConfig cfg;
  cfg.dim = 2;
  cfg.levels = std::atoi(argv[4]);
  cfg.table_size = static_cast<std::uint32_t>(std::atoll(argv[5]));
  cfg.features = std::atoi(argv[6]);
  cfg.base_resolution = std::atoi(argv[7]);
  cfg.growth = std::atof(argv[8]);
  TrainConfig tc;
  EXPECT(tc.batch_size == 2048 && tc.steps == 10000 && tc.record_every == 100 && tc.seed == 1234);  // trainer.hpp:15-24
  EXPECT(tc.table_adam.lr == 1e-2 && tc.mlp_adam.lr == 1e-3 && tc.table_adam.epsilon == 1e-15);
  tc.steps = std::atoi(argv[9]);
  tc.batch_size = std::atoi(argv[10]);
  tc.record_every = 1;

  // fit_image, exact head, losses read back every step and in windows of 64: the same training run
  for (int window : {1, 64}) {
    tc.queue_window = window;
    FitImageResult r = fit_image(img, cfg, tc);
    EXPECT(r.train.steps_run == tc.steps && r.train.loss_curve.size() == static_cast<std::size_t>(tc.steps));
    EXPECT(r.psnr_curve.size() == r.train.loss_curve.size());
    EXPECT(r.train.final_loss == r.train.loss_curve.back().second);
    if (window == 1) {  // render_image + image_psnr == the fused error sum behind final_psnr (src/tasks.cpp:35-96)
      const ImageDataset rendered = render_image(r.encoder, r.mlp, img.width, img.height);
      EXPECT(rendered.pixels.size() == img.pixels.size());
      EXPECT(std::abs(image_psnr(rendered, img) - r.final_psnr) <= 1e-9);
    }
    print_curve(window == 1 ? "fit_image_w1_loss" : "fit_image_w64_loss", r.train);
    std::printf("%s %.17g\n", window == 1 ? "fit_image_w1_psnr" : "fit_image_w64_psnr", r.final_psnr);
  }
  {  // tensor-core head (tcgen05 split-bf16)
    tc.queue_window = 256;
    FitImageOptions opt;
    opt.mlp_precision = MlpPrecision::tensor_bf16x3;
    const FitImageResult r = fit_image(img, cfg, tc, opt);
    print_curve("fit_image_tc_loss", r.train);
    std::printf("fit_image_tc_psnr %.17g\n", r.final_psnr);
  }
  {  // record_every / final step bookkeeping (src/trainer.cpp:132-135)
    TrainConfig t2 = tc;
    t2.steps = 23;
    t2.record_every = 10;
    t2.queue_window = 7;
    const FitImageResult r = fit_image(img, cfg, t2);
    EXPECT(r.train.loss_curve.size() == 4);
    EXPECT(r.train.loss_curve[0].first == 0 && r.train.loss_curve[1].first == 10 && r.train.loss_curve[2].first == 20 &&
           r.train.loss_curve[3].first == 22);
  }

  // fit_field, both noise kinds (the golden runs: 20 steps, batch 4096, hold-out 4096)
  for (int kind : {0, 1}) {
    EncoderConfig fc;
    fc.dim = 3;
    fc.levels = 8;
    fc.table_size = 1u << 14;
    fc.features = 2;
    fc.base_resolution = 4;
    fc.growth = 1.5;
    if (const char* e = std::getenv(kind == 0 ? "SXEN_FIELD_CFG0" : "SXEN_FIELD_CFG1")) {
      int d, l, f, b;
      long long t;
      double g;
      EXPECT(std::sscanf(e, "%d %d %lld %d %d %lf", &d, &l, &t, &f, &b, &g) == 6);
      fc.dim = d; fc.levels = l; fc.table_size = static_cast<std::uint32_t>(t); fc.features = f; fc.base_resolution = b; fc.growth = g;
    }
    NoiseFieldSpec spec;
    EXPECT(spec.dim == 2 && spec.seed == 7 && spec.octaves == 1 && spec.frequency == 4.0);  // noise.hpp:42-48
    spec.dim = fc.dim;
    spec.kind = static_cast<NoiseKind>(kind);
    spec.octaves = 2;
    TrainConfig ft;
    ft.batch_size = 4096;
    ft.steps = 20;
    ft.record_every = 1;
    FitFieldOptions fo;
    fo.holdout_samples = 4096;
    const FitFieldResult r = fit_field(spec, fc, ft, fo);
    print_curve(kind == 0 ? "fit_field_k0_loss" : "fit_field_k1_loss", r.train);
    std::printf("fit_field_k%d_holdout %.17g %.17g\n", kind, r.holdout_mse, r.field_variance);
  }

  // argument checks, as the reference throws them
  auto throws_invalid = [](auto&& fn) {
    try {
      fn();
    } catch (const std::invalid_argument&) {
      return true;
    } catch (...) {
    }
    return false;
  };
  {
    EncoderConfig c3 = cfg;
    c3.dim = 3;
    EXPECT(throws_invalid([&] { fit_image(img, c3, tc); }));
    TrainConfig bad = tc;
    bad.batch_size = 0;
    EXPECT(throws_invalid([&] { fit_image(img, cfg, bad); }));
    bad = tc;
    bad.record_every = 0;
    EXPECT(throws_invalid([&] { fit_image(img, cfg, bad); }));
    NoiseFieldSpec s3;
    s3.dim = 3;
    EXPECT(throws_invalid([&] { fit_field(s3, cfg, tc); }));
    FitFieldOptions h1;
    h1.holdout_samples = 1;
    NoiseFieldSpec s2;
    EXPECT(throws_invalid([&] { fit_field(s2, cfg, tc, h1); }));
    HashEncoder enc(cfg);
    Mlp wrong(MlpConfig{cfg.encoded_width() + 1, 64, 2, 3});
    EXPECT(throws_invalid([&] { train_field(enc, wrong, [](int, DeviceSpan<double>, DeviceSpan<double>, DeviceSpan<double>, void*) {}, tc); }));
  }

  // a non-finite loss: TrainingError naming the step; the queued updates of that and the later steps were not applied
  {
    HashEncoder enc(cfg);
    enc.init_tables(42);
    Mlp mlp(MlpConfig{cfg.encoded_width(), 64, 2, 3});
    mlp.init_params(sxen_hash_combine(42, 1));
    std::vector<std::vector<float>> before;
    for (int l = 0; l < cfg.levels; ++l) before.push_back(enc.table(l));
    const std::vector<float> params_before = mlp.parameters();
    const std::size_t batch = 512;
    std::vector<double> hx(batch * 2, 0.25), ht(batch * 3, std::numeric_limits<double>::quiet_NaN());
    const BatchSampler nan_sampler = [&](int, DeviceSpan<double> coords, DeviceSpan<double>, DeviceSpan<double> targets, void* s) {
      check(sxen_device_upload(0, coords.data, hx.data(), hx.size() * sizeof(double), s));
      check(sxen_device_upload(0, targets.data, ht.data(), ht.size() * sizeof(double), s));
    };
    TrainConfig t3;
    t3.batch_size = static_cast<int>(batch);
    t3.steps = 8;
    t3.queue_window = 8;
    bool thrown = false;
    try {
      train_field(enc, mlp, nan_sampler, t3);
    } catch (const TrainingError& e) {
      thrown = std::strstr(e.what(), "step 0") != nullptr;
    }
    EXPECT(thrown);
    for (int l = 0; l < cfg.levels; ++l) {
      const std::vector<float> now = enc.table(l);
      EXPECT(std::memcmp(now.data(), before[static_cast<std::size_t>(l)].data(), now.size() * sizeof(float)) == 0);
    }
    const std::vector<float> params_now = mlp.parameters();
    EXPECT(std::memcmp(params_now.data(), params_before.data(), params_now.size() * sizeof(float)) == 0);

    // ... and at a later step: finite targets for steps 0-2, NaN from step 3 on -> "step 3", three losses usable
    std::vector<double> good(batch * 3, 0.5);
    const BatchSampler late = [&](int step, DeviceSpan<double> coords, DeviceSpan<double>, DeviceSpan<double> targets, void* s) {
      check(sxen_device_upload(0, coords.data, hx.data(), hx.size() * sizeof(double), s));
      check(sxen_device_upload(0, targets.data, (step < 3 ? good : ht).data(), ht.size() * sizeof(double), s));
    };
    thrown = false;
    try {
      train_field(enc, mlp, late, t3);
    } catch (const TrainingError& e) {
      thrown = std::strstr(e.what(), "step 3") != nullptr;
    }
    EXPECT(thrown);
    // the trainer stays usable afterwards
    const BatchSampler fine = [&](int, DeviceSpan<double> coords, DeviceSpan<double>, DeviceSpan<double> targets, void* s) {
      check(sxen_device_upload(0, coords.data, hx.data(), hx.size() * sizeof(double), s));
      check(sxen_device_upload(0, targets.data, good.data(), good.size() * sizeof(double), s));
    };
    const TrainResult ok = train_field(enc, mlp, fine, t3);
    EXPECT(ok.steps_run == 8 && std::isfinite(ok.final_loss));
    EXPECT(ok.loss_curve.front().second > ok.final_loss);
  }
  // tests/test_neural.cpp:439-462: encoder + aux widths against the head's input width
  {
    EncoderConfig ec;
    ec.dim = 2;
    ec.levels = 2;
    ec.table_size = 1u << 6;
    ec.features = 2;
    ec.base_resolution = 4;
    HashEncoder enc(ec);
    Mlp mlp(MlpConfig{ec.encoded_width() + 1, 8, 1, 1});
    TrainConfig t4;
    t4.threads = 1;
    EXPECT(throws_invalid(
        [&] { train_field(enc, mlp, [](int, DeviceSpan<double>, DeviceSpan<double>, DeviceSpan<double>, void*) {}, t4); }));
    t4.aux_dims = 1;  // now the widths line up
    t4.steps = 3;
    t4.batch_size = 4;
    std::vector<double> c(8, 0.5), a(4, 0.7), tg(4, 0.1);
    const BatchSampler ok = [&](int, DeviceSpan<double> coords, DeviceSpan<double> aux, DeviceSpan<double> targets, void* s) {
      check(sxen_device_upload(0, coords.data, c.data(), c.size() * sizeof(double), s));
      check(sxen_device_upload(0, aux.data, a.data(), a.size() * sizeof(double), s));
      check(sxen_device_upload(0, targets.data, tg.data(), tg.size() * sizeof(double), s));
    };
    const TrainResult r = train_field(enc, mlp, ok, t4);
    EXPECT(r.steps_run == 3 && std::isfinite(r.final_loss));
  }
  std::printf("launches %llu\n", static_cast<unsigned long long>(sxen_launch_count()));
  std::printf("train_tasks ok\n");
  return 0;
}
