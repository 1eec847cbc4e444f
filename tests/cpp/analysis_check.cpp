// Compiled and run by tests/test_cpp_wrapper.py (CPU: bench_side, CSV schema and error cases) and by
// tests/test_gpu_cpp_trainer.py (B200: the bench-kernel protocol itself) -- include/sxen_b200_analysis.hpp.
#include <cmath>
#include <cstdio>
#include <string>

#include "sxen_b200_analysis.hpp"

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

int main(int argc, char** argv) {
  const std::string dir = argc > 1 ? argv[1] : ".";
  // the reference's protocol sizes: 2^27 cells -> side 11585 (n=2), 512 (n=3), 107 (n=4)
  EXPECT(bench_side(2, std::uint64_t{1} << 27) == 11585);
  EXPECT(bench_side(3, std::uint64_t{1} << 27) == 512);
  EXPECT(bench_side(4, std::uint64_t{1} << 27) == 107);
  EXPECT(bench_side(1, 1000) == 1000 && bench_side(8, 1) == 1 && bench_side(3, 26) == 2 && bench_side(3, 27) == 3);
  KernelBenchConfig def;
  EXPECT(def.n == 3 && def.cells == (std::uint64_t{1} << 21) && def.samples == 1024 && def.reps == 1000 &&
         def.table_size == (1u << 19) && def.features == 2 && def.seed == 99);  // include/sxen/analysis.hpp:56-65

  // CSV: the reference's schema, doubles round-trip bit-exactly
  std::vector<KernelBenchReport> rows(2);
  rows[0] = {3, Backend::simplex, 2097152, 1024, 1000, 0.0123456789012345678, 4.0};
  rows[1] = {2, Backend::grid, 1u << 20, 7, 10, 1.0 / 3.0, 3.999999999999};
  const std::string path = dir + "/kernel.csv";
  write_kernel_csv(path, rows);
  const std::vector<KernelBenchReport> back = read_kernel_csv(path);
  EXPECT(back.size() == 2);
  for (int i = 0; i < 2; ++i) {
    EXPECT(back[i].n == rows[i].n && back[i].backend == rows[i].backend && back[i].cells == rows[i].cells &&
           back[i].samples == rows[i].samples && back[i].reps == rows[i].reps && back[i].seconds == rows[i].seconds &&
           back[i].vertices_per_sample == rows[i].vertices_per_sample);
  }
  {
    std::FILE* f = std::fopen(path.c_str(), "r");
    char line[128];
    EXPECT(f && std::fgets(line, sizeof line, f));
    std::fclose(f);
    EXPECT(std::string(line) == "n,backend,cells,samples,reps,seconds,vertices_per_sample\n");  // src/analysis.cpp:122
  }
  auto write_raw = [&](const char* text) {
    std::FILE* f = std::fopen(path.c_str(), "w");
    std::fputs(text, f);
    std::fclose(f);
  };
  write_raw("n,level,samples\n1,2,3\n");
  EXPECT(throws<IoError>([&] { read_kernel_csv(path); }));  // header mismatch
  write_raw("n,backend,cells,samples,reps,seconds,vertices_per_sample\n3,simplex,8,1,1,0.5\n");
  EXPECT(throws<IoError>([&] { read_kernel_csv(path); }));  // 6 columns
  write_raw("n,backend,cells,samples,reps,seconds,vertices_per_sample\n3,octree,8,1,1,0.5,4\n");
  EXPECT(throws<IoError>([&] { read_kernel_csv(path); }));  // unknown backend
  write_raw("n,backend,cells,samples,reps,seconds,vertices_per_sample\n3,grid,8,1,x1,0.5,4\n");
  EXPECT(throws<IoError>([&] { read_kernel_csv(path); }));  // malformed number
  write_raw("");
  EXPECT(throws<IoError>([&] { read_kernel_csv(path); }));  // empty
  EXPECT(throws<IoError>([&] { read_kernel_csv(dir + "/does/not/exist.csv"); }));
  KernelBenchConfig bad;
  bad.n = 9;
  EXPECT(throws<std::invalid_argument>([&] { bench_kernel(bad); }));
  bad = KernelBenchConfig{};
  bad.reps = 0;
  EXPECT(throws<std::invalid_argument>([&] { bench_kernel(bad); }));

  if (sxen_device_count() == 0) {
    std::printf("analysis ok (host part; no sm_100 device)\n");
    return 0;
  }
  // the protocol on the device: exact vertex counts (n+1 / 2^n), cells = side^n, a time that resolves
  for (int n = 2; n <= 4; ++n) {
    for (Backend b : {Backend::simplex, Backend::grid}) {
      KernelBenchConfig c;
      c.n = n;
      c.backend = b;
      c.samples = 1 << 12;
      c.reps = 20;
      const KernelBenchReport r = bench_kernel(c);
      const std::uint32_t side = bench_side(n, c.cells);
      std::uint64_t cells = 1;
      for (int i = 0; i < n; ++i) cells *= side;
      EXPECT(r.n == n && r.backend == b && r.cells == cells && r.samples == c.samples && r.reps >= c.reps);
      EXPECT(r.vertices_per_sample == (b == Backend::simplex ? n + 1.0 : std::pow(2.0, n)));
      EXPECT(r.seconds >= 1e-3 && r.seconds < 5.0);
      std::printf("bench_kernel n=%d %s: %.3f ns per sample\n", n, b == Backend::simplex ? "simplex" : "grid",
                  r.seconds / (static_cast<double>(r.reps) * r.samples) * 1e9);
    }
  }
  std::printf("analysis ok\n");
  return 0;
}
