// tools/ubench/die_probe.cu -- B200 is two dies with an L2 half each.  An atomic executes at the line's HOME L2 slice; from an
// SM on the other die it crosses the die-to-die fabric (ncu: lts__t_requests_srcunit_ltcfabric = half of all reds).
// This probe measures, with chained atom.add round trips timed by clock64:
//   1. which SMs sit on which die   (latency signature of each SM over a set of test lines),
//   2. the address -> home-die map and its granularity over a buffer,
//   3. red throughput from all SMs when every red goes to a near-die line, a far-die line, or a random line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o die_probe.bin die_probe.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ unsigned smid() { unsigned r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }

// One thread per CTA: CHAIN dependent atomics on each of n_lines addresses (stride bytes apart); mean cycles per atomic.
__global__ void probe(float* buf, size_t stride_floats, int n_lines, int chain, unsigned* sm_of_cta, float* lat /*[cta][line]*/,
                      int first_line, int lines_per_cta) {
  if (threadIdx.x != 0) return;
  sm_of_cta[blockIdx.x] = smid();
  const int lo = lines_per_cta ? first_line + blockIdx.x * lines_per_cta : 0;
  const int hi = lines_per_cta ? min(n_lines, lo + lines_per_cta) : n_lines;
  for (int i = lo; i < hi; ++i) {
    float* p = buf + (size_t)i * stride_floats;
    float v = atomicAdd(p, 0.0f);  // warm: bring the line into its home L2
    v = atomicAdd(p, v * 0.0f);
    long long t0 = clock64();
    for (int c = 0; c < chain; ++c) v = atomicAdd(p, v * 0.0f);  // dependent chain
    long long t1 = clock64();
    lat[(size_t)blockIdx.x * (lines_per_cta ? lines_per_cta : n_lines) + (i - lo)] = (float)(t1 - t0) / chain + v * 0.0f;
  }
}

// Throughput: every thread issues `per` reds to rows picked from `rows` (a list of row indices, 8-byte rows).
__global__ void red_rate(float* buf, const uint32_t* rows, uint32_t n_rows, int per, const unsigned char* sm_die, int want_die_xor) {
  // rows[] holds near rows for die 0 in [0, n_rows) and for die 1 in [n_rows, 2 n_rows)
  const unsigned die = sm_die[smid()] ^ want_die_xor;
  const uint32_t* r = rows + (size_t)die * n_rows;
  uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) * 2654435761u;
  for (int i = 0; i < per; ++i) {
    h = h * 1664525u + 1013904223u;
    const uint32_t row = r[(h >> 8) % n_rows];
    asm volatile("red.global.add.v2.f32 [%0], {%1, %2};" ::"l"(buf + (size_t)row * 2), "f"(1.0f), "f"(1.0f) : "memory");
  }
}

int main() {
  const size_t bytes = 64ull << 20;
  float* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
  int nsm; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  printf("SMs: %d\n", nsm);
  // ---- 1. SM signatures over 96 lines spaced 1 MiB + 4 KiB apart
  const int n_sig = 96, chain = 24;
  unsigned* d_sm; float* d_lat;
  CK(cudaMalloc(&d_sm, nsm * sizeof(unsigned))); CK(cudaMalloc(&d_lat, (size_t)nsm * 4096 * sizeof(float)));
  const size_t sig_stride = ((640u << 10) + 4096) / 4;
  probe<<<nsm, 32>>>(buf, sig_stride, n_sig, chain, d_sm, d_lat, 0, 0);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned> sm(nsm); std::vector<float> lat((size_t)nsm * n_sig);
  CK(cudaMemcpy(sm.data(), d_sm, nsm * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(lat.data(), d_lat, lat.size() * 4, cudaMemcpyDeviceToHost));
  // global latency histogram
  std::vector<float> all(lat); std::sort(all.begin(), all.end());
  printf("atomic round trip (cycles): min %.0f p10 %.0f p50 %.0f p90 %.0f max %.0f\n", all[0], all[all.size() / 10], all[all.size() / 2],
         all[all.size() * 9 / 10], all.back());
  // per line: median over SMs; an SM's signature bit = latency above the line's median
  std::vector<unsigned char> sm_die(256, 0);
  std::vector<int> votes(nsm, 0);
  std::vector<float> med(n_sig);
  for (int i = 0; i < n_sig; ++i) {
    std::vector<float> col(nsm);
    for (int c = 0; c < nsm; ++c) col[c] = lat[(size_t)c * n_sig + i];
    std::sort(col.begin(), col.end());
    med[i] = 0.5f * (col[nsm / 4] + col[nsm * 3 / 4]);  // midpoint of the two modes
  }
  // reference: CTA 0's signature; die of CTA c = majority of (sig_c[i] != sig_0[i])
  int n1 = 0;
  for (int c = 0; c < nsm; ++c) {
    int diff = 0;
    for (int i = 0; i < n_sig; ++i) diff += ((lat[(size_t)c * n_sig + i] > med[i]) != (lat[i] > med[i]));
    votes[c] = diff;
    sm_die[sm[c]] = diff > n_sig / 2;
    n1 += diff > n_sig / 2;
  }
  std::vector<int> vs(votes); std::sort(vs.begin(), vs.end());
  printf("signature distance to CTA0 over %d lines: min %d p25 %d p50 %d p75 %d max %d  -> die split %d / %d\n", n_sig, vs[0], vs[nsm / 4],
         vs[nsm / 2], vs[nsm * 3 / 4], vs.back(), nsm - n1, n1);
  // near/far latency from CTA0's view
  {
    double near = 0, far = 0; int nn = 0, nf = 0;
    for (int i = 0; i < n_sig; ++i) { if (lat[i] > med[i]) { far += lat[i]; ++nf; } else { near += lat[i]; ++nn; } }
    printf("CTA0 (sm %u): %d near lines %.1f cyc, %d far lines %.1f cyc\n", sm[0], nn, nn ? near / nn : 0, nf, nf ? far / nf : 0);
  }
  // ---- 2. address -> die map at 256-byte steps over the first 2 MiB, probed from the CTAs (die-0 CTAs only are used)
  const int step = 256, n_map = (2 << 20) / step;  // 8192 lines
  const int per_cta = (n_map + nsm - 1) / nsm;
  probe<<<nsm, 32>>>(buf, step / 4, n_map, chain, d_sm, d_lat, 0, per_cta);
  CK(cudaDeviceSynchronize());
  std::vector<float> mlat((size_t)nsm * per_cta);
  CK(cudaMemcpy(sm.data(), d_sm, nsm * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(mlat.data(), d_lat, mlat.size() * 4, cudaMemcpyDeviceToHost));
  std::vector<float> thr_src(mlat); std::sort(thr_src.begin(), thr_src.end());
  const float thr = 0.5f * (thr_src[thr_src.size() / 4] + thr_src[thr_src.size() * 3 / 4]);
  std::vector<unsigned char> home(n_map);
  for (int i = 0; i < n_map; ++i) {
    const int c = i / per_cta;
    const bool far = mlat[(size_t)c * per_cta + (i - c * per_cta)] > thr;
    home[i] = sm_die[sm[c]] ^ (far ? 1 : 0);
  }
  int runs = 1, ones = home[0];
  std::vector<int> runlen; int cur = 1;
  for (int i = 1; i < n_map; ++i) { ones += home[i]; if (home[i] != home[i - 1]) { ++runs; runlen.push_back(cur); cur = 1; } else ++cur; }
  runlen.push_back(cur);
  std::sort(runlen.begin(), runlen.end());
  printf("home-die map over 2 MiB at 256 B steps (thr %.1f cyc): %d of %d lines on die 1, %d runs, run length min %d p50 %d max %d (x256 B)\n",
         thr, ones, n_map, runs, runlen[0], runlen[runlen.size() / 2], runlen.back());
  printf("first 128 steps: ");
  for (int i = 0; i < 128; ++i) printf("%d", home[i]);
  printf("\n");
  // ---- 3. red throughput near / far / mixed, rows = 8-byte rows of the first 2 MiB mapped above
  std::vector<uint32_t> rows0, rows1;
  for (int i = 0; i < n_map; ++i)
    for (int r = 0; r < step / 8; ++r) (home[i] ? rows1 : rows0).push_back((uint32_t)(i * (step / 8) + r));
  const uint32_t n_rows = (uint32_t)std::min(rows0.size(), rows1.size());
  std::vector<uint32_t> rows(2 * (size_t)n_rows);
  std::copy(rows0.begin(), rows0.begin() + n_rows, rows.begin());
  std::copy(rows1.begin(), rows1.begin() + n_rows, rows.begin() + n_rows);
  uint32_t* d_rows; unsigned char* d_die;
  CK(cudaMalloc(&d_rows, rows.size() * 4)); CK(cudaMemcpy(d_rows, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&d_die, 256)); CK(cudaMemcpy(d_die, sm_die.data(), 256, cudaMemcpyHostToDevice));
  // mixed list: both halves interleaved, same for both dies
  std::vector<uint32_t> mixed(2 * (size_t)n_rows);
  for (uint32_t i = 0; i < n_rows; ++i) { mixed[i] = mixed[n_rows + i] = (i & 1) ? rows1[i] : rows0[i]; }
  uint32_t* d_mixed; CK(cudaMalloc(&d_mixed, mixed.size() * 4)); CK(cudaMemcpy(d_mixed, mixed.data(), mixed.size() * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int per = 64, grid = 148 * 16, block = 256;
  const char* names[3] = {"near-die rows only", "far-die rows only", "mixed rows"};
  for (int m = 0; m < 3; ++m) {
    for (int rep = 0; rep < 6; ++rep) {
      if (rep == 1) cudaEventRecord(a);
      if (m == 2) red_rate<<<grid, block>>>(buf, d_mixed, n_rows, per, d_die, 0);
      else red_rate<<<grid, block>>>(buf, d_rows, n_rows, per, d_die, m);
    }
    cudaEventRecord(b); CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double reds = 5.0 * grid * block * per;
    printf("%-20s %.1f G reds/s (%u rows per die)\n", names[m], reds / (ms * 1e-3) / 1e9, n_rows);
  }
  return 0;
}
