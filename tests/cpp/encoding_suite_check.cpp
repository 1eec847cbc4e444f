// Compiled and run by tests/test_gpu_cpp_suite.py on the GPU box: a C++ host that includes include/sxen_b200.hpp where the
// reference's tests include "sxen/encoding.hpp" and makes the reference's own per-sample span calls
// (HashEncoder::encode(span<const double>, span<float>), encode_backward(x, upstream, grad)) -- the cases of
// /root/reference/proj/tests/test_encoding.cpp against the device path.  Links libsxen_b200.so only (no CUDA headers).
//
// Expected values come from a from-scratch pipeline in this file (the idea of the reference's tests/oracles.hpp, written
// independently: explicit skew matrix product, index sort, vertex walk, 64-bit hash products), not from the library.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <numeric>
#include <stdexcept>
#include <vector>

#include "sxen_b200.hpp"

using namespace sxen::b200;

static int g_failed = 0;
#define EXPECT(cond)                                                      \
  do {                                                                    \
    if (!(cond)) {                                                        \
      std::printf("FAILED %s line %d: %s\n", g_case, __LINE__, #cond);    \
      ++g_failed;                                                         \
    }                                                                     \
  } while (0)
static const char* g_case = "";

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

// ---- test-side helpers (not the library's code paths)
struct Lcg {  // points for the property cases; any stream of doubles in [0, 1) will do
  std::uint64_t s;
  double next() {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    return static_cast<double>(s >> 11) * 0x1.0p-53;
  }
};

static const std::uint64_t kPrime[8] = {1ull,          2654435761ull, 805459861ull,  3674653429ull,
                                        2097192037ull, 1434869437ull, 2165219737ull, 4294967291ull};

static std::uint32_t hash_of(const std::vector<std::int64_t>& v) {
  std::uint64_t h = 0;
  for (std::size_t i = 0; i < v.size(); ++i) h ^= ((static_cast<std::uint64_t>(v[i]) & 0xffffffffull) * kPrime[i]) & 0xffffffffull;
  return static_cast<std::uint32_t>(h);
}

// One level of the simplex encoding from first principles; `rows` = that level's table (T*F floats).
static std::vector<double> simplex_level(int n, std::uint32_t res, std::uint32_t T, int F, const std::vector<float>& rows,
                                         const double* x) {
  const double below_one = std::nextafter(1.0, 0.0);
  const double scale = static_cast<double>(res) / std::sqrt(n + 1.0);
  const double f = (std::sqrt(n + 1.0) - 1.0) / n;
  std::vector<double> v(n), y(n), fr(n);
  for (int i = 0; i < n; ++i) v[i] = std::min(x[i], below_one) * scale;
  for (int i = 0; i < n; ++i) {  // y = (I + f 1 1^T) v, row by row
    double acc = 0.0;
    for (int j = 0; j < n; ++j) acc += (i == j ? 1.0 + f : f) * v[j];
    y[i] = acc;
  }
  std::vector<std::int64_t> cell(n);
  for (int i = 0; i < n; ++i) {
    cell[i] = std::clamp<std::int64_t>(static_cast<std::int64_t>(std::floor(y[i])), 0, static_cast<std::int64_t>(res) - 1);
    fr[i] = std::clamp(y[i] - static_cast<double>(cell[i]), 0.0, below_one);
  }
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return fr[a] > fr[b]; });
  std::vector<double> out(F, 0.0);
  for (int k = 0; k <= n; ++k) {
    if (k > 0) cell[order[k - 1]] += 1;
    const double w = k == 0 ? 1.0 - fr[order[0]] : (k == n ? fr[order[n - 1]] : fr[order[k - 1]] - fr[order[k]]);
    const std::uint32_t idx = hash_of(cell) & (T - 1u);
    for (int c = 0; c < F; ++c) out[c] += w * static_cast<double>(rows[static_cast<std::size_t>(idx) * F + c]);
  }
  return out;
}

static std::vector<double> grid_level(int n, std::uint32_t res, std::uint32_t T, int F, const std::vector<float>& rows,
                                      const double* x) {
  const double below_one = std::nextafter(1.0, 0.0);
  std::vector<std::int64_t> cell(n), corner(n);
  std::vector<double> fr(n);
  for (int i = 0; i < n; ++i) {
    const double y = std::min(x[i], below_one) * static_cast<double>(res);
    cell[i] = std::clamp<std::int64_t>(static_cast<std::int64_t>(std::floor(y)), 0, static_cast<std::int64_t>(res) - 1);
    fr[i] = std::clamp(y - static_cast<double>(cell[i]), 0.0, below_one);
  }
  std::vector<double> out(F, 0.0);
  for (int m = 0; m < (1 << n); ++m) {
    double w = 1.0;
    for (int d = 0; d < n; ++d) {
      const int up = (m >> d) & 1;
      corner[d] = cell[d] + up;
      w *= up ? fr[d] : 1.0 - fr[d];
    }
    const std::uint32_t idx = hash_of(corner) & (T - 1u);
    for (int c = 0; c < F; ++c) out[c] += w * static_cast<double>(rows[static_cast<std::size_t>(idx) * F + c]);
  }
  return out;
}

static EncoderConfig small_config(Backend backend, int dim, int levels = 2) {  // test_encoding.cpp:16-27
  EncoderConfig cfg;
  cfg.dim = dim;
  cfg.levels = levels;
  cfg.table_size = 1u << 10;
  cfg.features = 2;
  cfg.base_resolution = 4;
  cfg.growth = 2.0;
  cfg.backend = backend;
  cfg.level_scale = LevelScale::raw;
  return cfg;
}

static std::vector<float> encode_vec(const HashEncoder& enc, std::span<const double> x) {
  std::vector<float> out(static_cast<std::size_t>(enc.config().encoded_width()));
  enc.encode(x, out);
  return out;
}

static void fill_table(HashEncoder& enc, int level, float value) {
  std::vector<float> t(static_cast<std::size_t>(enc.config().table_size) * enc.config().features, value);
  enc.set_table(level, t);
}

int main() {
  const Backend both[2] = {Backend::simplex, Backend::grid};
  Lcg rng{20231115};

  g_case = "zero tables encode to zero";  // :138-147
  for (Backend b : both) {
    HashEncoder enc(small_config(b, 3));
    for (int it = 0; it < 50; ++it) {
      const std::array<double, 3> x{rng.next(), rng.next(), rng.next()};
      for (float v : encode_vec(enc, x)) EXPECT(v == 0.0f);
    }
  }

  g_case = "lattice vertex reads back its entry";  // :149-174
  for (Backend b : both) {
    HashEncoder enc(small_config(b, 2, 1));
    auto t = enc.table(0);
    t[0] = 0.25f;
    t[1] = -0.75f;
    enc.set_table(0, t);
    const std::array<double, 2> origin{0.0, 0.0};
    const auto out = encode_vec(enc, origin);
    EXPECT(out[0] == 0.25f && out[1] == -0.75f);
  }
  {
    const EncoderConfig cfg = small_config(Backend::grid, 2, 1);
    HashEncoder enc(cfg);
    const std::uint32_t idx = hash_of({2, 1}) & (cfg.table_size - 1u);
    auto t = enc.table(0);
    t[idx * 2] = 1.5f;
    t[idx * 2 + 1] = 2.5f;
    enc.set_table(0, t);
    const std::array<double, 2> x{0.5, 0.25};
    const auto out = encode_vec(enc, x);
    EXPECT(out[0] == 1.5f && out[1] == 2.5f);
  }

  g_case = "grid frozen blends";  // :176-206
  {
    EncoderConfig cfg = small_config(Backend::grid, 1, 1);
    cfg.base_resolution = 1;
    cfg.features = 1;
    HashEncoder enc(cfg);
    auto t = enc.table(0);
    t[hash_of({0}) & (cfg.table_size - 1u)] = 2.0f;
    t[hash_of({1}) & (cfg.table_size - 1u)] = 6.0f;
    enc.set_table(0, t);
    for (double s : {0.0, 0.25, 0.5, 0.75}) {
      const std::array<double, 1> x{s};
      EXPECT(std::abs(encode_vec(enc, x)[0] - (2.0 + 4.0 * s)) <= 1e-6 * (2.0 + 4.0 * s));
    }
  }

  g_case = "both backends match the independent pipeline";  // :224-251
  for (Backend b : both) {
    for (int n = 1; n <= 7; ++n) {
      const EncoderConfig cfg = small_config(b, n, 3);
      HashEncoder enc(cfg);
      enc.init_tables(77);
      std::vector<std::vector<float>> tables;
      for (int l = 0; l < cfg.levels; ++l) tables.push_back(enc.table(l));
      double worst = 0.0;
      for (int it = 0; it < 200; ++it) {
        std::array<double, 8> x{};
        for (int i = 0; i < n; ++i) x[i] = rng.next();
        const auto got = encode_vec(enc, std::span<const double>(x.data(), static_cast<std::size_t>(n)));
        for (int l = 0; l < cfg.levels; ++l) {
          const auto want = b == Backend::simplex ? simplex_level(n, enc.resolution(l), cfg.table_size, 2, tables[l], x.data())
                                                  : grid_level(n, enc.resolution(l), cfg.table_size, 2, tables[l], x.data());
          for (int c = 0; c < 2; ++c) worst = std::max(worst, std::abs(static_cast<double>(got[l * 2 + c]) - want[c]));
        }
      }
      EXPECT(worst < 1e-9);
    }
  }

  g_case = "linear in the table entries";  // :253-268
  for (Backend b : both) {
    HashEncoder enc(small_config(b, 3));
    enc.init_tables(5);
    const std::array<double, 3> x{0.31, 0.77, 0.12};
    const auto once = encode_vec(enc, x);
    for (int l = 0; l < enc.config().levels; ++l) {
      auto t = enc.table(l);
      for (float& v : t) v *= 2.0f;
      enc.set_table(l, t);
    }
    const auto twice = encode_vec(enc, x);
    for (std::size_t i = 0; i < once.size(); ++i) EXPECT(std::abs(static_cast<double>(twice[i]) - 2.0 * once[i]) < 1e-9);
  }

  g_case = "constant tables encode to the constant";  // :270-288
  for (Backend b : both) {
    for (int n = 1; n <= 7; ++n) {
      HashEncoder enc(small_config(b, n));
      for (int l = 0; l < enc.config().levels; ++l) fill_table(enc, l, 0.5f);
      for (int it = 0; it < 100; ++it) {
        std::array<double, 8> x{};
        for (int i = 0; i < n; ++i) x[i] = rng.next();
        for (float v : encode_vec(enc, std::span<const double>(x.data(), static_cast<std::size_t>(n)))) EXPECT(std::abs(v - 0.5) < 1e-7);
      }
    }
  }

  g_case = "identical config and seed are bit-identical";  // :290-306
  {
    const EncoderConfig cfg = small_config(Backend::simplex, 4);
    HashEncoder a(cfg), b(cfg);
    a.init_tables(999);
    b.init_tables(999);
    for (int l = 0; l < cfg.levels; ++l) EXPECT(a.table(l) == b.table(l));
    const std::array<double, 4> x{0.1, 0.9, 0.4, 0.6};
    EXPECT(encode_vec(a, x) == encode_vec(b, x));
  }

  g_case = "touched-vertex counters are exact";  // :308-334
  for (int n = 2; n <= 5; ++n) {
    HashEncoder simplex(small_config(Backend::simplex, n)), grid(small_config(Backend::grid, n));
    const int k = 100;
    for (int it = 0; it < k; ++it) {
      std::array<double, 8> x{};
      for (int i = 0; i < n; ++i) x[i] = rng.next();
      const std::span<const double> view(x.data(), static_cast<std::size_t>(n));
      encode_vec(simplex, view);
      encode_vec(grid, view);
    }
    const std::uint64_t levels = static_cast<std::uint64_t>(simplex.config().levels);
    EXPECT(simplex.counters().touched_vertices == k * levels * static_cast<std::uint64_t>(n + 1));
    EXPECT(grid.counters().touched_vertices == k * levels * (1ull << n));
    EXPECT(simplex.counters().out_of_bounds == 0 && grid.counters().out_of_bounds == 0);
    simplex.reset_counters();
    EXPECT(simplex.counters().touched_vertices == 0);
  }

  g_case = "unit-cube boundary points are accepted";  // :336-346
  for (Backend b : both) {
    HashEncoder enc(small_config(b, 2));
    for (const auto& x : {std::array<double, 2>{0.0, 0.0}, std::array<double, 2>{1.0, 1.0}, std::array<double, 2>{1.0, 0.0},
                          std::array<double, 2>{0.999999999, 1.0}})
      EXPECT(!throws<std::exception>([&] { encode_vec(enc, x); }));
    EXPECT(enc.counters().out_of_bounds == 0);
  }

  g_case = "encode input and shape validation";  // :348-358
  {
    HashEncoder enc(small_config(Backend::simplex, 2));
    std::vector<float> out(static_cast<std::size_t>(enc.config().encoded_width()));
    EXPECT(throws<std::invalid_argument>([&] { enc.encode(std::array<double, 3>{0.5, 0.5, 0.5}, out); }));
    EXPECT(throws<std::invalid_argument>([&] { enc.encode(std::array<double, 2>{1.5, 0.5}, out); }));
    EXPECT(throws<std::invalid_argument>([&] { enc.encode(std::array<double, 2>{-0.1, 0.5}, out); }));
    EXPECT(throws<std::invalid_argument>([&] { enc.encode(std::array<double, 2>{std::nan(""), 0.5}, out); }));
    std::vector<float> bad(out.size() + 1);
    EXPECT(throws<std::invalid_argument>([&] { enc.encode(std::array<double, 2>{0.5, 0.5}, bad); }));
    EXPECT(!throws<std::exception>([&] { enc.encode(std::array<double, 2>{0.5, 0.5}, out); }));  // the handle lives on
  }

  g_case = "backward: zero upstream leaves only zero slices";  // :389-401
  {
    HashEncoder enc(small_config(Backend::simplex, 3));
    enc.init_tables(4);
    EncoderGradient grad(enc);
    const std::array<double, 3> x{0.2, 0.6, 0.9};
    const std::vector<double> up(static_cast<std::size_t>(enc.config().encoded_width()), 0.0);
    enc.encode_backward(x, up, grad);
    EXPECT(grad.touched_total() == static_cast<std::uint64_t>(enc.config().levels) * 4u);
    std::vector<float> v;
    std::vector<std::uint8_t> t;
    for (int l = 0; l < grad.levels(); ++l) {
      grad.download(l, v, t);
      for (float g : v) EXPECT(g == 0.0f);
    }
  }

  g_case = "backward: one-hot upstream recovers the weights";  // :403-435
  for (Backend b : both) {
    HashEncoder enc(small_config(b, 2));
    enc.init_tables(6);
    const EncoderConfig& cfg = enc.config();
    for (int it = 0; it < 20; ++it) {
      const std::array<double, 2> x{rng.next(), rng.next()};
      const int hot_l = it % cfg.levels, hot_f = it % cfg.features;
      std::vector<double> up(static_cast<std::size_t>(cfg.encoded_width()), 0.0);
      up[static_cast<std::size_t>(hot_l * cfg.features + hot_f)] = 1.0;
      EncoderGradient grad(enc);
      enc.encode_backward(x, up, grad);
      double sum = 0.0;
      std::vector<float> v;
      std::vector<std::uint8_t> t;
      for (int l = 0; l < cfg.levels; ++l) {
        grad.download(l, v, t);
        for (std::uint32_t r = 0; r < cfg.table_size; ++r)
          for (int c = 0; c < cfg.features; ++c) {
            const float g = v[static_cast<std::size_t>(r) * cfg.features + c];
            if (l != hot_l || c != hot_f) EXPECT(g == 0.0f);
            else {
              EXPECT(g >= 0.0f);
              sum += g;
            }
          }
      }
      EXPECT(std::abs(sum - 1.0) <= 2e-7);  // f32 accumulator rows here (the reference's are fp64: 1e-12)
    }
  }

  g_case = "backward matches finite differences";  // :437-480
  for (Backend b : both) {
    HashEncoder enc(small_config(b, 2));
    enc.init_tables(8);
    const EncoderConfig& cfg = enc.config();
    const std::array<double, 2> x{0.37, 0.58};
    std::vector<double> up(static_cast<std::size_t>(cfg.encoded_width()));
    for (double& u : up) u = 2.0 * rng.next() - 1.0;
    EncoderGradient grad(enc);
    enc.encode_backward(x, up, grad);
    auto loss = [&] {
      const auto out = encode_vec(enc, x);
      double acc = 0.0;
      for (std::size_t i = 0; i < out.size(); ++i) acc += up[i] * static_cast<double>(out[i]);
      return acc;
    };
    const float h = 1e-3f;
    int checked = 0;
    std::vector<float> v;
    std::vector<std::uint8_t> t;
    for (int l = 0; l < cfg.levels && checked < 8; ++l) {
      grad.download(l, v, t);
      for (std::uint32_t r = 0; r < cfg.table_size && checked < 8; ++r) {
        if (!t[r]) continue;
        const int c = static_cast<int>(r % static_cast<std::uint32_t>(cfg.features));
        const std::size_t at = static_cast<std::size_t>(r) * cfg.features + c;
        auto tab = enc.table(l);
        const float saved = tab[at];
        tab[at] = saved + h;
        enc.set_table(l, tab);
        const double hi = loss();
        tab[at] = saved - h;
        enc.set_table(l, tab);
        const double lo = loss();
        tab[at] = saved;
        enc.set_table(l, tab);
        const double fd = (hi - lo) / (2.0 * static_cast<double>(h));
        const double analytic = v[at];
        EXPECT(std::abs(fd - analytic) < 1e-3 * std::max(1.0, std::abs(analytic)));
        ++checked;
      }
    }
    EXPECT(checked > 0);
  }

  g_case = "backward shape validation";  // :482-491
  {
    HashEncoder enc(small_config(Backend::simplex, 2)), other(small_config(Backend::simplex, 2, 3));
    EncoderGradient good(enc), bad(other);
    const std::vector<double> up(static_cast<std::size_t>(enc.config().encoded_width()), 0.0), short_up(up.size() - 1, 0.0);
    const std::array<double, 2> x{0.5, 0.5};
    EXPECT(throws<std::invalid_argument>([&] { enc.encode_backward(x, short_up, good); }));
    EXPECT(throws<std::invalid_argument>([&] { enc.encode_backward(x, up, bad); }));
    EXPECT(throws<std::invalid_argument>([&] { good.merge(bad); }));  // :384-386
  }

  g_case = "parameter count";  // :493-497
  {
    const EncoderConfig cfg = small_config(Backend::simplex, 3, 5);
    EXPECT(HashEncoder(cfg).parameter_count() == 5ull * cfg.table_size * 2ull);
  }

  if (g_failed) {
    std::printf("encoding suite: %d check(s) failed\n", g_failed);
    return 1;
  }
  std::printf("encoding suite ok\n");
  return 0;
}
