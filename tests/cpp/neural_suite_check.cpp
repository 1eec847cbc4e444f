// Compiled and run by tests/test_gpu_cpp_suite.py on the GPU box: the MLP / optimizer cases of the reference's `neural`
// suite (/root/reference/proj/tests/test_neural.cpp:39-309) as a C++ host program over include/sxen_b200.hpp, with the
// reference's host-span call shape: Mlp::forward(span<const float>, span<float> out), Mlp::backward(span<const double>,
// span<double> input_grad), gradient() for MlpGradient::values().  Links libsxen_b200.so only.
// (The train_field cases of that suite run from C++ in tests/cpp/train_tasks_check.cpp.)
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "sxen_b200.hpp"
#include "sxen_b200_train.hpp"

using namespace sxen::b200;

static int g_failed = 0;
static const char* g_case = "";
#define EXPECT(cond)                                                      \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("FAILED %s line %d: %s\n", g_case, __LINE__, #cond);    \
      ++g_failed;                                                         \
    }                                                                     \
  } while (0)

template <class E, class Fn>
static bool throws(Fn&& fn) {
  try {
    fn();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

struct Lcg {
  std::uint64_t s;
  double next(double lo, double hi) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return lo + (hi - lo) * (static_cast<double>(s >> 11) * 0x1.0p-53);
  }
};

static MlpConfig tiny_mlp(int in, int hidden, int layers, int out) { return MlpConfig{in, hidden, layers, out}; }

static std::vector<float> random_input(int width, std::uint64_t seed) {
  Lcg rng{seed};
  std::vector<float> v(static_cast<std::size_t>(width));
  for (float& x : v) x = static_cast<float>(rng.next(-1.0, 1.0));
  return v;
}

static std::vector<float> forward_vec(Mlp& mlp, std::span<const float> input) {
  std::vector<float> out(static_cast<std::size_t>(mlp.config().output_width));
  mlp.forward(input, out);
  return out;
}

// dense fp64 forward from the parameter vector (per layer: out x in weights row-major, then out biases)
static std::vector<double> dense_forward(const Mlp& mlp, const std::vector<float>& params, std::span<const float> input) {
  std::vector<double> cur(input.begin(), input.end()), next;
  for (int l = 0; l < mlp.layer_count(); ++l) {
    const int in_w = mlp.layer_input_width(l), out_w = mlp.layer_output_width(l);
    const float* w = params.data() + mlp.layer_offset(l);
    const float* b = w + static_cast<std::size_t>(in_w) * out_w;
    next.assign(static_cast<std::size_t>(out_w), 0.0);
    for (int o = 0; o < out_w; ++o) {
      double dot = b[o];
      for (int i = 0; i < in_w; ++i) dot += static_cast<double>(w[static_cast<std::size_t>(o) * in_w + i]) * cur[i];
      next[o] = (l + 1 < mlp.layer_count()) ? std::max(dot, 0.0) : dot;
    }
    cur = next;
  }
  return cur;
}

int main() {
  g_case = "config validation";  // :39-48
  EXPECT(!throws<std::exception>([] { tiny_mlp(4, 8, 2, 3).validate(); }));
  EXPECT(!throws<std::exception>([] { tiny_mlp(4, 8, 0, 3).validate(); }));
  EXPECT(throws<std::invalid_argument>([] { tiny_mlp(0, 8, 2, 3).validate(); }));
  EXPECT(throws<std::invalid_argument>([] { tiny_mlp(4, 0, 2, 3).validate(); }));
  EXPECT(throws<std::invalid_argument>([] { tiny_mlp(4, 8, -1, 3).validate(); }));
  EXPECT(throws<std::invalid_argument>([] { tiny_mlp(4, 8, 2, 0).validate(); }));
  EXPECT(tiny_mlp(4, 8, 2, 3).layer_count() == 3 && tiny_mlp(4, 8, 0, 3).layer_count() == 1);

  g_case = "zero parameters produce zero output";  // :50-56
  {
    Mlp mlp(tiny_mlp(6, 12, 2, 4));
    for (float v : forward_vec(mlp, random_input(6, 31))) EXPECT(v == 0.0f);
  }

  g_case = "identity single layer";  // :58-66
  {
    Mlp mlp(tiny_mlp(5, 1, 0, 5));
    auto p = mlp.parameters();
    for (int o = 0; o < 5; ++o) p[static_cast<std::size_t>(o) * 5 + o] = 1.0f;
    mlp.set_parameters(p);
    const auto input = random_input(5, 32);
    EXPECT(forward_vec(mlp, input) == input);
  }

  g_case = "forward matches the dense matrix product";  // :68-81
  {
    Mlp mlp(tiny_mlp(8, 16, 2, 3));
    mlp.init_params(41);
    const auto params = mlp.parameters();
    for (int it = 0; it < 200; ++it) {
      const auto input = random_input(8, 1000 + static_cast<std::uint64_t>(it));
      const auto got = forward_vec(mlp, input);
      const auto want = dense_forward(mlp, params, input);
      for (int o = 0; o < 3; ++o) EXPECT(std::abs(static_cast<double>(got[o]) - want[o]) <= 1e-5 * std::max(1.0, std::abs(want[o])));
    }
  }

  g_case = "initialization is seed-deterministic and bias-free";  // :83-100
  {
    Mlp a(tiny_mlp(8, 16, 2, 3)), b(tiny_mlp(8, 16, 2, 3)), c(tiny_mlp(8, 16, 2, 3));
    a.init_params(7);
    b.init_params(7);
    c.init_params(8);
    const auto pa = a.parameters();
    EXPECT(pa == b.parameters() && pa != c.parameters());
    for (int l = 0; l < a.layer_count(); ++l) {
      const std::size_t bias0 = a.layer_offset(l) + static_cast<std::size_t>(a.layer_input_width(l)) * a.layer_output_width(l);
      for (int o = 0; o < a.layer_output_width(l); ++o) EXPECT(pa[bias0 + o] == 0.0f);
    }
  }

  g_case = "backward requires a cached forward pass";  // :102-109
  {
    Mlp mlp(tiny_mlp(4, 8, 1, 2));
    mlp.init_params(1);
    const std::array<double, 2> up{1.0, 1.0};
    std::vector<double> ig(4);
    EXPECT(throws<std::logic_error>([&] { mlp.backward(up, ig); }));
  }

  g_case = "zero upstream produces zero gradients";  // :111-121
  {
    Mlp mlp(tiny_mlp(4, 8, 2, 2));
    mlp.init_params(2);
    forward_vec(mlp, random_input(4, 33));
    const std::array<double, 2> up{0.0, 0.0};
    std::vector<double> ig(4, 1.0);
    mlp.backward(up, ig);
    for (double g : mlp.gradient()) EXPECT(g == 0.0);
    for (double g : ig) EXPECT(g == 0.0);
  }

  g_case = "single affine layer closed form";  // :123-151
  {
    Mlp mlp(tiny_mlp(3, 1, 0, 2));
    mlp.init_params(3);
    const auto input = random_input(3, 34);
    const auto w = mlp.parameters();
    forward_vec(mlp, input);
    const std::array<double, 2> up{0.7, -1.3};
    std::vector<double> ig(3);
    mlp.backward(up, ig);
    const auto g = mlp.gradient();
    for (int o = 0; o < 2; ++o) {
      EXPECT(std::abs(g[6 + o] - up[o]) <= 1e-12 * std::abs(up[o]));
      for (int i = 0; i < 3; ++i) {
        const double want = up[o] * static_cast<double>(input[i]);
        EXPECT(std::abs(g[static_cast<std::size_t>(o) * 3 + i] - want) <= 1e-6 * std::abs(want));
      }
    }
    for (int i = 0; i < 3; ++i) {
      double want = 0.0;
      for (int o = 0; o < 2; ++o) want += up[o] * static_cast<double>(w[static_cast<std::size_t>(o) * 3 + i]);
      EXPECT(std::abs(ig[i] - want) <= 1e-6 * std::abs(want));
    }
  }

  g_case = "backward accumulates across calls; clear";  // :153-190
  {
    Mlp once(tiny_mlp(4, 8, 1, 2)), twice(tiny_mlp(4, 8, 1, 2));
    once.init_params(4);
    twice.init_params(4);
    const auto input = random_input(4, 35);
    const std::array<double, 2> up{0.4, 0.9};
    std::vector<double> ig(4);
    forward_vec(once, input);
    once.backward(up, ig);
    for (int r = 0; r < 2; ++r) {
      forward_vec(twice, input);
      twice.backward(up, ig);
    }
    const auto a = once.gradient(), b = twice.gradient();
    bool any = false;
    for (std::size_t i = 0; i < a.size(); ++i) {
      any |= a[i] != 0.0;
      EXPECT(std::abs(b[i] - 2.0 * a[i]) <= 1e-12 * std::abs(2.0 * a[i]));
    }
    EXPECT(any);
    twice.clear_gradient();
    for (double g : twice.gradient()) EXPECT(g == 0.0);
  }

  g_case = "full-stack gradients match central finite differences";  // :192-228
  {
    Mlp mlp(tiny_mlp(4, 8, 2, 2));
    mlp.init_params(45);
    const auto input = random_input(4, 38);
    const std::array<double, 2> up{0.8, -0.6};
    std::vector<double> ig(4);
    forward_vec(mlp, input);
    mlp.backward(up, ig);
    const auto grad = mlp.gradient();
    auto params = mlp.parameters();
    auto loss = [&] {
      const auto out = forward_vec(mlp, input);
      return up[0] * static_cast<double>(out[0]) + up[1] * static_cast<double>(out[1]);
    };
    Lcg pick{39};
    const double h = 1e-3;
    for (int it = 0; it < 10; ++it) {
      const std::size_t pi = static_cast<std::size_t>(pick.next(0.0, 1.0) * static_cast<double>(params.size())) % params.size();
      const float saved = params[pi];
      params[pi] = static_cast<float>(static_cast<double>(saved) + h);
      mlp.set_parameters(params);
      const double hi = loss();
      params[pi] = static_cast<float>(static_cast<double>(saved) - h);
      mlp.set_parameters(params);
      const double lo = loss();
      params[pi] = saved;
      mlp.set_parameters(params);
      const double fd = (hi - lo) / (2.0 * h);
      EXPECT(std::abs(fd - grad[pi]) <= 1e-3 * std::max(1.0, std::abs(grad[pi])));
    }
  }

  g_case = "mlp span validation";  // src/mlp.cpp:138-143,168-173
  {
    Mlp mlp(tiny_mlp(4, 8, 1, 2));
    std::vector<float> in5(5), out2(2), out3(3), in4(4);
    EXPECT(throws<std::invalid_argument>([&] { mlp.forward(in5, out2); }));
    EXPECT(throws<std::invalid_argument>([&] { mlp.forward(in4, out3); }));
    mlp.forward(in4, out2);
    std::vector<double> up3(3), ig4(4);
    EXPECT(throws<std::invalid_argument>([&] { mlp.backward(up3, ig4); }));
  }

  g_case = "adaptive-moment steps";  // :230-274
  {
    auto adam_once = [](std::vector<float> p, const std::vector<double>& g, const AdamConfig& cfg, int steps, std::int64_t* count) {
      DeviceBuffer<float> dp(p.size(), 0);
      DeviceBuffer<double> dg(g.size(), 0);
      dp.upload(p);
      dg.upload(g);
      AdamState opt(p.size());
      for (int t = 0; t < steps; ++t) opt.step(dp.span(p.size()), dg.cspan(g.size()), cfg);
      if (count) *count = opt.step_count();
      p = dp.download(p.size());
      return p;
    };
    std::int64_t count = 0;
    auto p = adam_once({0.5f, -0.25f, 1.0f}, {0.0, 0.0, 0.0}, AdamConfig{}, 1, &count);
    EXPECT(count == 1 && p[0] == 0.5f && p[1] == -0.25f && p[2] == 1.0f);
    AdamConfig cfg;
    cfg.lr = 0.1;
    p = adam_once({1.0f, 1.0f}, {0.5, -0.02}, cfg, 1, nullptr);  // step 1 moves by -lr * g / (|g| + eps)
    EXPECT(std::abs(p[0] - 0.9) <= 1e-6 * 0.9 && std::abs(p[1] - 1.1) <= 1e-6 * 1.1);
    cfg.lr = 0.01;
    const auto p199 = adam_once({0.0f}, {0.3}, cfg, 199, nullptr), p200 = adam_once({0.0f}, {0.3}, cfg, 200, nullptr);
    const double last_delta = static_cast<double>(p200[0]) - static_cast<double>(p199[0]);
    EXPECT(std::abs(last_delta + cfg.lr) <= 0.05 * cfg.lr);
    EXPECT(throws<TrainingError>([&] { adam_once({0.0f}, {std::nan("")}, AdamConfig{}, 1, nullptr); }));
  }

  g_case = "sparse table update touches only accumulated entries";  // :276-309
  {
    EncoderConfig cfg;
    cfg.dim = 2;
    cfg.levels = 2;
    cfg.table_size = 1u << 6;
    cfg.features = 2;
    cfg.base_resolution = 4;
    HashEncoder enc(cfg);
    enc.init_tables(9);
    const auto before0 = enc.table(0), before1 = enc.table(1);
    EncoderGradient grad(enc);
    std::vector<float> v(static_cast<std::size_t>(cfg.table_size) * 2, 0.0f);
    std::vector<std::uint8_t> t(cfg.table_size, 0);
    v[10] = 0.25f;  // row 5: grad.add(0, 5, 1.0, {0.25, -0.5})
    v[11] = -0.5f;
    t[5] = 1;
    check(sxen_grad_upload(grad.handle(), 0, v.data(), t.data()));
    AdamConfig opt_cfg;
    opt_cfg.lr = 0.05;
    SparseAdamState opt(enc);
    opt.step(enc, grad, opt_cfg);
    EXPECT(opt.step_count() == 1);
    const auto after0 = enc.table(0);
    for (std::size_t i = 0; i < before0.size(); ++i) {
      if (i == 10) EXPECT(std::abs(after0[i] - (before0[i] - opt_cfg.lr)) <= 1e-5 * std::abs(before0[i] - opt_cfg.lr));
      else if (i == 11) EXPECT(std::abs(after0[i] - (before0[i] + opt_cfg.lr)) <= 1e-5 * std::abs(before0[i] + opt_cfg.lr));
      else EXPECT(after0[i] == before0[i]);
    }
    EXPECT(enc.table(1) == before1);
  }

  if (g_failed) {
    std::printf("neural suite: %d check(s) failed\n", g_failed);
    return 1;
  }
  std::printf("neural suite ok\n");
  return 0;
}
