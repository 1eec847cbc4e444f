// sxen_b200_analysis.hpp -- header-only C++ mirror of the reference's kernel-timing protocol over the C ABI:
//   KernelBenchConfig / KernelBenchReport / bench_kernel   include/sxen/analysis.hpp:20-29,56-75, src/analysis.cpp:233-313
//   write_kernel_csv / read_kernel_csv                     src/analysis.cpp:122,340-372 (same header, same column order)
// The protocol is the reference's: a single-level encoder whose resolution is the largest side with side^n <= cells,
// `samples` points from CounterRng(seed, 1), `reps` passes over them, set-up outside the timed region, steady_clock around
// the passes, vertices per sample from the exact lookup counters.  What differs: one pass over the points is ONE kernel
// launch on the device, and the clock stops after the stream has drained.  Reports of the reference CLI and of this
// library share the CSV schema, so the n = 2..6 sweep can be laid side by side.  The rest of the reference's analysis
// suite (volume ratios, Monte-Carlo utilisation, JSON emitters) is out of scope.
#pragma once

#include <chrono>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <sstream>

#include "sxen_b200_train.hpp"

namespace sxen::b200 {

// include/sxen/analysis.hpp:56-65, same defaults
struct KernelBenchConfig {
  int n = 3;
  std::uint64_t cells = std::uint64_t{1} << 21;
  int samples = 1 << 10;
  int reps = 1000;
  Backend backend = Backend::simplex;
  std::uint32_t table_size = 1u << 19;
  int features = 2;
  std::uint64_t seed = 99;
};

// include/sxen/analysis.hpp:20-29
struct KernelBenchReport {
  int n = 0;
  Backend backend = Backend::simplex;
  std::uint64_t cells = 0;
  int samples = 0;
  int reps = 0;
  double seconds = 0.0;
  double vertices_per_sample = 0.0;
};

// Largest integer side with side^n <= cells (src/analysis.cpp:243-257), in exact integer arithmetic.
inline std::uint32_t bench_side(int n, std::uint64_t cells) {
  auto pow_le = [&](std::uint64_t side) {  // side^n <= cells without overflow
    std::uint64_t p = 1;
    for (int i = 0; i < n; ++i) {
      if (side != 0 && p > cells / side) return false;
      p *= side;
    }
    return p <= cells;
  };
  std::uint64_t side = static_cast<std::uint64_t>(std::llround(std::pow(static_cast<double>(cells), 1.0 / n)));
  if (side < 1) side = 1;
  while (side > 1 && !pow_le(side)) --side;
  while (pow_le(side + 1)) ++side;
  return static_cast<std::uint32_t>(side);
}

// sxen::bench_kernel (src/analysis.cpp:233-313)
inline KernelBenchReport bench_kernel(const KernelBenchConfig& cfg, int device = 0, void* stream = nullptr) {
  if (cfg.n < 1 || cfg.n > 8) throw std::invalid_argument("bench: n must be in [1, 8]");
  if (cfg.cells < 1) throw std::invalid_argument("bench: cells must be >= 1");
  if (cfg.samples < 1 || cfg.reps < 1) throw std::invalid_argument("bench: samples and reps must be >= 1");
  const std::uint32_t side = bench_side(cfg.n, cfg.cells);
  EncoderConfig ec;
  ec.dim = cfg.n;
  ec.levels = 1;
  ec.table_size = cfg.table_size;
  ec.features = cfg.features;
  ec.base_resolution = static_cast<int>(side);
  ec.growth = 2.0;
  ec.backend = cfg.backend;
  ec.level_scale = LevelScale::raw;
  HashEncoder enc(ec, device);
  enc.init_tables(cfg.seed, stream);
  const std::size_t samples = static_cast<std::size_t>(cfg.samples), dim = static_cast<std::size_t>(cfg.n);
  const std::size_t width = static_cast<std::size_t>(ec.encoded_width());
  DeviceBuffer<double> x(samples * dim, device);
  DeviceBuffer<float> out(samples * width, device);
  check(sxen_rng_fill_dev(cfg.seed, 1, 1, 1, 0.0, 1.0, x.data(), samples * dim, SXEN_COORD_F64, stream));  // :269-271 (draws are 1-based)
  enc.encode(x.cspan(samples * dim), out.span(samples * width), stream);  // warm-up, outside the timed region
  (void)out.download(1, stream);                                          // ... and drained
  int reps = cfg.reps;
  double seconds = 0.0;
  for (;;) {
    enc.reset_counters();
    const auto t0 = std::chrono::steady_clock::now();
    for (int r = 0; r < reps; ++r) enc.encode(x.cspan(samples * dim), out.span(samples * width), stream);
    const std::vector<float> probe = out.download(1, stream);  // synchronises the stream
    seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (!std::isfinite(probe[0])) throw std::runtime_error("bench: encode produced non-finite values");
    if (seconds >= 1e-3 || reps > (1 << 28)) break;  // :296-301: raise reps until the timer resolves
    reps *= 10;
  }
  enc.check_async(stream);
  KernelBenchReport r;
  r.n = cfg.n;
  r.backend = cfg.backend;
  r.cells = 1;
  for (int i = 0; i < cfg.n; ++i) r.cells *= side;
  r.samples = cfg.samples;
  r.reps = reps;
  r.seconds = seconds;
  r.vertices_per_sample = static_cast<double>(enc.counters().touched_vertices) /
                          (static_cast<double>(reps) * static_cast<double>(cfg.samples));
  return r;
}

inline constexpr const char* kKernelHeader = "n,backend,cells,samples,reps,seconds,vertices_per_sample";  // :122

// src/analysis.cpp:340-348: stable column order, doubles printed so that they read back bit-exactly
inline void write_kernel_csv(const std::string& path, std::span<const KernelBenchReport> rows) {
  std::ofstream f(path, std::ios::trunc);
  if (!f) throw IoError("cannot open '" + path + "' for writing");
  f << kKernelHeader << "\n";
  char buf[64];
  for (const KernelBenchReport& r : rows) {
    f << r.n << "," << (r.backend == Backend::simplex ? "simplex" : "grid") << "," << r.cells << "," << r.samples << ","
      << r.reps << ",";
    std::snprintf(buf, sizeof buf, "%.17g", r.seconds);
    f << buf << ",";
    std::snprintf(buf, sizeof buf, "%.17g", r.vertices_per_sample);
    f << buf << "\n";
  }
  f.flush();
  if (!f) throw IoError("write to '" + path + "' failed");
}

// src/analysis.cpp:350-372: rejects unknown headers, wrong column counts, unknown backends and malformed numbers
inline std::vector<KernelBenchReport> read_kernel_csv(const std::string& path) {
  std::ifstream f(path);
  if (!f) throw IoError("cannot open '" + path + "'");
  std::string line;
  if (!std::getline(f, line)) throw IoError("csv '" + path + "' is empty");
  if (line != kKernelHeader)
    throw IoError("csv '" + path + "' header mismatch: expected '" + kKernelHeader + "', got '" + line + "'");
  std::vector<KernelBenchReport> out;
  while (std::getline(f, line)) {
    if (line.empty()) continue;
    std::vector<std::string> fields;
    std::stringstream ss(line);
    for (std::string cell; std::getline(ss, cell, ',');) fields.push_back(cell);
    if (!line.empty() && line.back() == ',') fields.emplace_back();
    if (fields.size() != 7) throw IoError("csv '" + path + "': expected 7 columns");
    KernelBenchReport r;
    try {
      std::size_t used = 0;
      auto whole = [&](const std::string& s, auto conv) {
        auto v = conv(s, &used);
        if (used != s.size()) throw std::invalid_argument(s);
        return v;
      };
      r.n = static_cast<int>(whole(fields[0], [](const std::string& s, std::size_t* u) { return std::stoll(s, u); }));
      if (fields[1] == "simplex") r.backend = Backend::simplex;
      else if (fields[1] == "grid") r.backend = Backend::grid;
      else throw IoError("csv: unknown backend '" + fields[1] + "'");
      r.cells = static_cast<std::uint64_t>(whole(fields[2], [](const std::string& s, std::size_t* u) { return std::stoull(s, u); }));
      r.samples = static_cast<int>(whole(fields[3], [](const std::string& s, std::size_t* u) { return std::stoll(s, u); }));
      r.reps = static_cast<int>(whole(fields[4], [](const std::string& s, std::size_t* u) { return std::stoll(s, u); }));
      r.seconds = whole(fields[5], [](const std::string& s, std::size_t* u) { return std::stod(s, u); });
      r.vertices_per_sample = whole(fields[6], [](const std::string& s, std::size_t* u) { return std::stod(s, u); });
    } catch (const IoError&) {
      throw;
    } catch (const std::exception&) {
      throw IoError("csv '" + path + "': malformed field");
    }
    out.push_back(r);
  }
  return out;
}

}  // namespace sxen::b200
