// sxen_b200_checkpoint.hpp -- header-only C++ mirror of the reference's checkpoint files over the C ABI
// (include/sxen/checkpoint.hpp:12-38, src/checkpoint.cpp:81-175): the little-endian "SXEN" / "SXML" format, so a model
// trained on the device loads into the reference (inspect, render) and a reference-written file loads onto the device.
//
//   "SXEN" | version u32 | n, L, T, F, N_base u32 | growth f64 | backend u32 | L blocks of T*F f32
//   ["SXML" | version u32 | layer_count, input, hidden, output u32 | per layer: out*in f32 weights, out f32 biases]
//
// Host-side file I/O only: tables and parameters move through HashEncoder::table / set_table and Mlp::parameters /
// set_parameters.  Same error type (IoError) and rejections as the reference; round trips are bit-exact.
#pragma once

#include <cstring>
#include <fstream>
#include <optional>

#include "sxen_b200.hpp"

namespace sxen::b200 {

// include/sxen/checkpoint.hpp:12-15
struct LoadedCheckpoint {
  HashEncoder encoder;
  std::optional<Mlp> mlp;
};

namespace checkpoint_detail {

inline constexpr char kEncoderMagic[4] = {'S', 'X', 'E', 'N'};
inline constexpr char kMlpMagic[4] = {'S', 'X', 'M', 'L'};
inline constexpr std::uint32_t kEncoderVersion = 1, kMlpVersion = 1;

// the format is little-endian; every host this library runs on (x86-64, aarch64) is too
template <class T>
void put(std::ostream& f, const T& v) {
  f.write(reinterpret_cast<const char*>(&v), sizeof(T));
}
inline void get_bytes(std::istream& f, void* dst, std::size_t n) {
  f.read(static_cast<char*>(dst), static_cast<std::streamsize>(n));
  if (static_cast<std::size_t>(f.gcount()) != n) throw IoError("checkpoint: unexpected end of file");
}
template <class T>
T get(std::istream& f) {
  T v;
  get_bytes(f, &v, sizeof(T));
  return v;
}

}  // namespace checkpoint_detail

// sxen::save_checkpoint (src/checkpoint.cpp:81-112)
inline void save_checkpoint(const std::string& path, const HashEncoder& encoder, const Mlp* mlp = nullptr) {
  using namespace checkpoint_detail;
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  if (!f) throw IoError("cannot open '" + path + "' for writing");
  const EncoderConfig& ec = encoder.config();
  f.write(kEncoderMagic, 4);
  put<std::uint32_t>(f, kEncoderVersion);
  put<std::uint32_t>(f, static_cast<std::uint32_t>(ec.dim));
  put<std::uint32_t>(f, static_cast<std::uint32_t>(ec.levels));
  put<std::uint32_t>(f, ec.table_size);
  put<std::uint32_t>(f, static_cast<std::uint32_t>(ec.features));
  put<std::uint32_t>(f, static_cast<std::uint32_t>(ec.base_resolution));
  put<double>(f, ec.growth);
  put<std::uint32_t>(f, ec.backend == Backend::simplex ? 0u : 1u);
  for (int l = 0; l < ec.levels; ++l) {
    const std::vector<float> t = encoder.table(l);
    f.write(reinterpret_cast<const char*>(t.data()), static_cast<std::streamsize>(t.size() * sizeof(float)));
  }
  if (mlp != nullptr) {
    const MlpConfig& mc = mlp->config();
    f.write(kMlpMagic, 4);
    put<std::uint32_t>(f, kMlpVersion);
    put<std::uint32_t>(f, static_cast<std::uint32_t>(mc.layer_count()));
    put<std::uint32_t>(f, static_cast<std::uint32_t>(mc.input_width));
    put<std::uint32_t>(f, static_cast<std::uint32_t>(mc.hidden_width));
    put<std::uint32_t>(f, static_cast<std::uint32_t>(mc.output_width));
    const std::vector<float> p = mlp->parameters();  // per layer: weights then biases (src/mlp.cpp:19-32)
    f.write(reinterpret_cast<const char*>(p.data()), static_cast<std::streamsize>(p.size() * sizeof(float)));
  }
  f.flush();
  if (!f) throw IoError("write to '" + path + "' failed");
}

// sxen::load_checkpoint (src/checkpoint.cpp:114-175).  The level-scale mode is not part of the file: pass the mode the
// checkpoint was trained with so the level resolutions reconstruct identically.
inline LoadedCheckpoint load_checkpoint(const std::string& path, LevelScale level_scale = LevelScale::raw, int device = 0) {
  using namespace checkpoint_detail;
  std::ifstream f(path, std::ios::binary);
  if (!f) throw IoError("cannot open '" + path + "' for reading");
  char magic[4];
  get_bytes(f, magic, 4);
  if (std::memcmp(magic, kEncoderMagic, 4) != 0) throw IoError("checkpoint: bad encoder section magic");
  const std::uint32_t version = get<std::uint32_t>(f);
  if (version != kEncoderVersion)
    throw IoError("checkpoint: unsupported encoder section version " + std::to_string(version));
  EncoderConfig ec;
  const std::uint32_t dim = get<std::uint32_t>(f), levels = get<std::uint32_t>(f), table_size = get<std::uint32_t>(f),
                      features = get<std::uint32_t>(f), base = get<std::uint32_t>(f);
  const double growth = get<double>(f);
  const std::uint32_t backend_tag = get<std::uint32_t>(f);
  if (backend_tag > 1) throw IoError("checkpoint: unknown backend tag");
  if (dim > 64 || levels > (1u << 20) || features > (1u << 20) || base > (1u << 30))
    throw IoError("checkpoint: invalid encoder config: field out of range");
  ec.dim = static_cast<int>(dim);
  ec.levels = static_cast<int>(levels);
  ec.table_size = table_size;
  ec.features = static_cast<int>(features);
  ec.base_resolution = static_cast<int>(base);
  ec.growth = growth;
  ec.backend = backend_tag == 0 ? Backend::simplex : Backend::grid;
  ec.level_scale = level_scale;
  try {
    ec.validate();
  } catch (const std::invalid_argument& e) {
    throw IoError(std::string("checkpoint: invalid encoder config: ") + e.what());
  }
  HashEncoder encoder(ec, device);
  std::vector<float> block(static_cast<std::size_t>(table_size) * features);
  for (int l = 0; l < ec.levels; ++l) {
    get_bytes(f, block.data(), block.size() * sizeof(float));
    encoder.set_table(l, block);
  }
  LoadedCheckpoint out{std::move(encoder), std::nullopt};
  f.read(magic, 4);
  if (f.gcount() == 0) return out;  // no MLP section
  if (f.gcount() != 4 || std::memcmp(magic, kMlpMagic, 4) != 0) throw IoError("checkpoint: bad mlp section magic");
  const std::uint32_t mlp_version = get<std::uint32_t>(f);
  if (mlp_version != kMlpVersion) throw IoError("checkpoint: unsupported mlp section version " + std::to_string(mlp_version));
  const std::uint32_t layer_count = get<std::uint32_t>(f), inp = get<std::uint32_t>(f), hid = get<std::uint32_t>(f),
                      outw = get<std::uint32_t>(f);
  if (layer_count < 1) throw IoError("checkpoint: mlp layer count must be >= 1");
  if (layer_count > (1u << 20) || inp > (1u << 30) || hid > (1u << 30) || outw > (1u << 30))
    throw IoError("checkpoint: invalid mlp config: field out of range");
  MlpConfig mc{static_cast<int>(inp), static_cast<int>(hid), static_cast<int>(layer_count) - 1, static_cast<int>(outw)};
  try {
    mc.validate();
  } catch (const std::invalid_argument& e) {
    throw IoError(std::string("checkpoint: invalid mlp config: ") + e.what());
  }
  Mlp mlp(mc, device);
  std::vector<float> params(mlp.parameter_count());
  get_bytes(f, params.data(), params.size() * sizeof(float));
  mlp.set_parameters(params);
  char extra;
  f.read(&extra, 1);
  if (f.gcount() != 0) throw IoError("checkpoint: trailing bytes after mlp section");
  out.mlp.emplace(std::move(mlp));
  return out;
}

}  // namespace sxen::b200
