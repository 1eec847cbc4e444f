// Compiled and run by tests/test_cpp_wrapper.py (CPU: the rejections that need no device) and by
// tests/test_gpu_cpp_trainer.py (B200: reference-written files load and re-save byte for byte) --
// include/sxen_b200_checkpoint.hpp.   argv: <scratch dir> [ref_with_mlp.sxen ref_without_mlp.sxen]
#include <cstdio>
#include <fstream>
#include <iterator>
#include <string>
#include <vector>

#include "sxen_b200_checkpoint.hpp"

using namespace sxen::b200;

#define EXPECT(cond)                                            \
  do {                                                          \
    if (!(cond)) {                                              \
      std::printf("FAILED line %d: %s\n", __LINE__, #cond);     \
      return 1;                                                 \
    }                                                           \
  } while (0)

template <class Fn>
bool throws_io(Fn&& fn) {
  try {
    fn();
  } catch (const IoError&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static std::vector<char> slurp(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  return std::vector<char>(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}
static void spit(const std::string& path, const std::vector<char>& bytes) {
  std::ofstream f(path, std::ios::binary | std::ios::trunc);
  f.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
}

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  const std::string tmp = dir + "/c.sxen";
  // rejections that are decided before any device object exists (src/checkpoint.cpp:114-130)
  EXPECT(throws_io([&] { load_checkpoint(dir + "/does/not/exist.sxen"); }));
  spit(tmp, {'S', 'X', 'E'});
  EXPECT(throws_io([&] { load_checkpoint(tmp); }));  // truncated magic
  spit(tmp, {'N', 'O', 'P', 'E', 1, 0, 0, 0});
  EXPECT(throws_io([&] { load_checkpoint(tmp); }));  // bad magic
  spit(tmp, {'S', 'X', 'E', 'N', 9, 0, 0, 0});
  EXPECT(throws_io([&] { load_checkpoint(tmp); }));  // unsupported version
  {
    std::vector<char> b = {'S', 'X', 'E', 'N', 1, 0, 0, 0};
    const std::uint32_t fields[5] = {2, 2, 1000 /* not a power of two */, 2, 4};
    b.insert(b.end(), reinterpret_cast<const char*>(fields), reinterpret_cast<const char*>(fields) + sizeof fields);
    const double growth = 2.0;
    b.insert(b.end(), reinterpret_cast<const char*>(&growth), reinterpret_cast<const char*>(&growth) + 8);
    const std::uint32_t backend = 0;
    b.insert(b.end(), reinterpret_cast<const char*>(&backend), reinterpret_cast<const char*>(&backend) + 4);
    spit(tmp, b);
    EXPECT(throws_io([&] { load_checkpoint(tmp); }));  // invalid encoder config
    b[8 + 16 + 8 + 4] = 7;                             // backend tag 7 (and still a bad table size: tag is checked first)
    spit(tmp, b);
    EXPECT(throws_io([&] { load_checkpoint(tmp); }));
  }
  if (sxen_device_count() == 0 || argc < 4) {
    std::printf("checkpoint ok (host part)\n");
    return 0;
  }
  // reference-written files: load, re-save, compare byte for byte (round trips are bit-exact)
  for (int i = 2; i <= 3; ++i) {
    const std::string ref = argv[i];
    const std::vector<char> want = slurp(ref);
    EXPECT(!want.empty());
    LoadedCheckpoint ck = load_checkpoint(ref);
    EXPECT(ck.mlp.has_value() == (i == 2));
    save_checkpoint(tmp, ck.encoder, ck.mlp ? &*ck.mlp : nullptr);
    EXPECT(slurp(tmp) == want);
    // truncations and trailing bytes are rejected
    std::vector<char> cut(want.begin(), want.end() - 3);
    spit(tmp, cut);
    EXPECT(throws_io([&] { load_checkpoint(tmp); }));
    if (i == 2) {
      std::vector<char> more = want;
      more.push_back(0);
      spit(tmp, more);
      EXPECT(throws_io([&] { load_checkpoint(tmp); }));
    } else {
      std::vector<char> more = want;
      more.insert(more.end(), {'S', 'X', 'M', 'X'});
      spit(tmp, more);
      EXPECT(throws_io([&] { load_checkpoint(tmp); }));  // bad mlp magic
    }
  }
  // a device-trained model written here reads back identically
  {
    EncoderConfig ec;
    ec.dim = 3;
    ec.levels = 3;
    ec.table_size = 1u << 8;
    ec.features = 4;
    ec.base_resolution = 5;
    ec.growth = 1.5;
    ec.backend = Backend::grid;
    HashEncoder enc(ec);
    enc.init_tables(7);
    Mlp mlp(MlpConfig{ec.encoded_width(), 16, 1, 2});
    mlp.init_params(9);
    save_checkpoint(tmp, enc, &mlp);
    LoadedCheckpoint ck = load_checkpoint(tmp);
    EXPECT(ck.mlp.has_value() && ck.encoder.config().backend == Backend::grid && ck.encoder.config().features == 4);
    for (int l = 0; l < ec.levels; ++l) EXPECT(ck.encoder.table(l) == enc.table(l));
    EXPECT(ck.mlp->parameters() == mlp.parameters());
    EXPECT(throws_io([&] { save_checkpoint(dir + "/no/such/dir/x.sxen", enc); }));
  }
  std::printf("checkpoint ok\n");
  return 0;
}
