// Compiled and run by tests/test_cpp_wrapper.py (CPU): the C++ mirror (include/sxen_b200.hpp) builds against the C ABI
// and the host-only entry points throw the reference's exception types.  No device work.
#include <cmath>
#include <cstdio>
#include <stdexcept>

#include "sxen_b200.hpp"

using namespace sxen::b200;

#define EXPECT(cond)                                            \
  do {                                                          \
    if (!(cond)) {                                              \
      std::printf("FAILED line %d: %s\n", __LINE__, #cond);     \
      return 1;                                                 \
    }                                                           \
  } while (0)

template <class E, class Fn>
bool throws(Fn&& fn) {
  try {
    fn();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  EncoderConfig cfg;  // reference defaults, include/sxen/encoding.hpp:18-27
  EXPECT(cfg.dim == 2 && cfg.levels == 8 && cfg.table_size == (1u << 16) && cfg.features == 2);
  cfg.validate();
  EXPECT(level_resolution(cfg, 0) == 16 && level_resolution(cfg, 3) == 128);
  EXPECT(std::abs(equal_memory_multiplier(2) - std::pow(3.0, 0.25)) < 1e-12);
  EncoderConfig bad = cfg;
  bad.table_size = 1000;
  EXPECT(throws<std::invalid_argument>([&] { bad.validate(); }));
  bad = cfg;
  bad.levels = 40;
  EXPECT(throws<std::invalid_argument>([&] { bad.validate(); }));
  EXPECT(throws<std::invalid_argument>([&] { level_resolution(cfg, 8); }));
  MlpConfig mc;
  mc.validate();
  mc.output_width = 0;
  EXPECT(throws<std::invalid_argument>([&] { mc.validate(); }));
  if (sxen_device_count() == 0) {
    // no sm_100 device: constructing an encoder must fail loudly, not fall back
    EXPECT(throws<CudaError>([&] { HashEncoder enc(cfg); }));
  }
  std::printf("wrapper ok\n");
  return 0;
}
