// sxen_abi.cu -- the C ABI of include/sxen_cuda.h: library, rng, config, encoder and gradient-accumulator entry
// points.  Host code above the kernels; every entry point cites the reference call it stands in for in the header.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <limits>

#include "sxen_common.hpp"
#include "sxen_encode.cuh"

namespace sxen_host {

std::string& last_error() {
  thread_local std::string e;
  return e;
}

sxen_status fail(sxen_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  last_error() = buf;
  return st;
}

sxen_status cuda_fail(cudaError_t e, const char* what) {
  return fail(SXEN_CUDA_ERROR, "CUDA error %d (%s) in %s", static_cast<int>(e), cudaGetErrorString(e), what);
}

std::atomic<uint64_t> g_launches{0};

}  // namespace sxen_host

using namespace sxen_host;
using sxen_dev::EncodeArgs;
using sxen_dev::EncodeLaunch;

namespace {

constexpr unsigned long long kNoBadSample = ~0ULL;
constexpr uint32_t kUntouchedBits = 0x80000000u;  // -0.0f

bool is_pow2(uint32_t v) { return v != 0 && (v & (v - 1)) == 0; }

// src/encoding.cpp:60-66
double equal_memory_multiplier(int n) {
  return std::pow(static_cast<double>(n + 1), static_cast<double>(n - 1) / (2.0 * static_cast<double>(n)));
}

// src/encoding.cpp:68-82
uint32_t level_resolution(const sxen_encoder_config& cfg, int level) {
  double r = static_cast<double>(cfg.base_resolution) * std::pow(cfg.growth, level);
  if (cfg.level_scale == SXEN_SCALE_EQUAL_MEMORY && cfg.backend == SXEN_BACKEND_SIMPLEX) {
    r *= equal_memory_multiplier(cfg.dim);
  }
  const double floored = std::floor(r);
  if (floored < 1.0) return 1;
  if (floored > static_cast<double>(SXEN_MAX_RESOLUTION)) return SXEN_MAX_RESOLUTION + 1;
  return static_cast<uint32_t>(floored);
}

// EncoderConfig::validate, src/encoding.cpp:28-58 (same order, same rejections)
sxen_status validate(const sxen_encoder_config& c) {
  SXEN_REQUIRE(c.dim >= 1 && c.dim <= SXEN_MAX_DIM, "encoder dim must be in [1, %d], got %d", SXEN_MAX_DIM, c.dim);
  SXEN_REQUIRE(c.levels >= 1, "encoder levels must be >= 1, got %d", c.levels);
  SXEN_REQUIRE(is_pow2(c.table_size), "encoder table_size must be a power of two, got %u", c.table_size);
  SXEN_REQUIRE(c.features >= 1 && c.features <= SXEN_MAX_FEATURES, "encoder features must be in [1, %d], got %d",
               SXEN_MAX_FEATURES, c.features);
  SXEN_REQUIRE(c.base_resolution >= 1, "encoder base_resolution must be >= 1, got %d", c.base_resolution);
  SXEN_REQUIRE(c.growth > 1.0 && std::isfinite(c.growth), "encoder growth must be a finite value > 1");
  SXEN_REQUIRE(c.backend == SXEN_BACKEND_SIMPLEX || c.backend == SXEN_BACKEND_GRID, "encoder backend must be 0 or 1");
  SXEN_REQUIRE(c.level_scale == SXEN_SCALE_RAW || c.level_scale == SXEN_SCALE_EQUAL_MEMORY,
               "encoder level_scale must be 0 or 1");
  const uint32_t finest = level_resolution(c, c.levels - 1);
  SXEN_REQUIRE(finest <= SXEN_MAX_RESOLUTION,
               "finest level resolution %u exceeds the supported maximum %u; lower levels, growth, or base_resolution",
               finest, SXEN_MAX_RESOLUTION);
  return SXEN_OK;
}

sxen_tuning default_tuning() {
  sxen_tuning t{};
  t.levels_per_thread = 0;  // auto
  t.block_threads = 256;
  t.level_major = -1;  // auto
  t.exact_blend = 1;
  t.warp_aggregate = 0;
  t.merge_pairs = 1;
  t.cache_hints = -1;  // auto
  t.coarse_replicas = 0;
  t.level_chunk = 0;
  return t;
}

__global__ void fill_u32_kernel(uint32_t* __restrict__ p, size_t n, uint32_t value) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = value;
}

// init_tables, src/encoding.cpp:169-176: entry i of level l = float(-1e-4 + 2e-4 * draw(i+1) of CounterRng(seed, l))
__global__ void init_tables_kernel(float* __restrict__ tables, size_t per_level, int levels, uint64_t seed_key,
                                   double lo, double span) {
  const size_t total = per_level * static_cast<size_t>(levels);
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const size_t l = i / per_level;
    const size_t e = i - l * per_level;
    const uint64_t key = sxen_dev::hash_combine(seed_key, static_cast<uint64_t>(l));  // CounterRng(seed, stream)
    tables[i] = static_cast<float>(sxen_dev::rng_double(key, static_cast<uint64_t>(e) + 1, lo, span));
  }
}

template <typename T>
__global__ void rng_fill_kernel(T* __restrict__ out, size_t n, uint64_t key, uint64_t first, double lo, double span) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = static_cast<T>(sxen_dev::rng_double(key, first + i, lo, span));
}

// EncoderGradient::merge, src/encoding.cpp:122-131, on the in-band touched encoding: a row untouched in src leaves
// dst alone; otherwise every feature is added (src's -0.0f in features > 0 cannot occur for a touched row).
__global__ void grad_merge_kernel(float* __restrict__ dst, const float* __restrict__ src, size_t rows, int features) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t r = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride) {
    const float* s = src + r * features;
    if (__float_as_uint(s[0]) == kUntouchedBits) continue;
    float* d = dst + r * features;
    for (int f = 0; f < features; ++f) d[f] = (d[f] + 0.0f) + s[f];  // +0.0f first: an untouched dst row becomes +0
  }
}

__global__ void add_i64_kernel(long long* __restrict__ dst, const long long* __restrict__ src, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] += src[i];
}

__global__ void grad_touched_kernel(const float* __restrict__ v, size_t rows, int features,
                                    unsigned long long* __restrict__ out) {
  unsigned long long local = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t r = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < rows; r += stride)
    local += (__float_as_uint(v[r * features]) != kUntouchedBits) ? 1ULL : 0ULL;
  for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(out, local);
}

int grid_for(size_t n, int block = 256) {
  size_t b = (n + block - 1) / block;
  const size_t cap = 148 * 16;  // a few waves of the 148 SMs; kernels above are grid-stride
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return static_cast<int>(b);
}

typedef cudaError_t (*encode_fn)(const EncodeLaunch&, EncodeArgs&, cudaStream_t, int*);
typedef cudaError_t (*debug_fn)(EncodeArgs&, int, uint32_t*, double*, int, cudaStream_t);

const encode_fn kEncode[8] = {sxen_dev::launch_encode_nd1, sxen_dev::launch_encode_nd2, sxen_dev::launch_encode_nd3,
                              sxen_dev::launch_encode_nd4, sxen_dev::launch_encode_nd5, sxen_dev::launch_encode_nd6,
                              sxen_dev::launch_encode_nd7, sxen_dev::launch_encode_nd8};
typedef cudaError_t (*fold_fn)(const EncodeArgs&, cudaStream_t);
typedef cudaError_t (*adam_walk_fn)(const EncodeArgs&, const sxen_dev::AdamWalkArgs&, int, cudaStream_t);
const adam_walk_fn kAdamWalk[8] = {sxen_dev::launch_adam_walk_nd1, sxen_dev::launch_adam_walk_nd2,
                                   sxen_dev::launch_adam_walk_nd3, sxen_dev::launch_adam_walk_nd4,
                                   sxen_dev::launch_adam_walk_nd5, sxen_dev::launch_adam_walk_nd6,
                                   sxen_dev::launch_adam_walk_nd7, sxen_dev::launch_adam_walk_nd8};
const fold_fn kFold[8] = {sxen_dev::launch_fold_nd1, sxen_dev::launch_fold_nd2, sxen_dev::launch_fold_nd3,
                          sxen_dev::launch_fold_nd4, sxen_dev::launch_fold_nd5, sxen_dev::launch_fold_nd6,
                          sxen_dev::launch_fold_nd7, sxen_dev::launch_fold_nd8};
const debug_fn kDebug[8] = {sxen_dev::launch_debug_nd1, sxen_dev::launch_debug_nd2, sxen_dev::launch_debug_nd3,
                            sxen_dev::launch_debug_nd4, sxen_dev::launch_debug_nd5, sxen_dev::launch_debug_nd6,
                            sxen_dev::launch_debug_nd7, sxen_dev::launch_debug_nd8};

int ptr_vec(const void* p) {
  const uintptr_t u = reinterpret_cast<uintptr_t>(p);
  return (u % 16 == 0) ? 4 : (u % 8 == 0) ? 2 : 1;
}

// Fills the launch-invariant part of the argument block.
void base_args(const sxen_encoder* enc, const void* x, sxen_coord_type type, size_t n, EncodeArgs& a) {
  std::memset(&a, 0, sizeof(a));
  a.x = x;
  a.tables = enc->tables;
  a.status = enc->status;
  a.n_samples = n;
  a.level_stride = enc->level_floats();
  a.mask = enc->cfg.table_size - 1u;
  a.row_width = enc->cfg.levels * enc->cfg.features;
  a.features = enc->cfg.features;
  a.coord_f32 = type == SXEN_COORD_F32 ? 1 : 0;
  a.skew = enc->skew;
}

// Launches below this many samples skip the coarse-level replicas (tuning.coarse_replicas == 0): a small batch puts few
// atomics on each hot row, while the fold that follows costs the same ~10 us whatever the batch
// (profiles/r1s3_small_batch_launches.csv: 14 of a 2048-sample training step's 93 us).
constexpr size_t kReplicaMinSamples = size_t{1} << 16;

void level_chunk(const sxen_encoder* enc, const sxen_grad* grad, int level0, int level_end, size_t n_samples, EncodeArgs& a) {
  a.level0 = level0;
  a.n_levels = std::min<int>(sxen_dev::kMaxLaunchLevels, level_end - level0);
  a.agg_mask = 0;
  // the replicas are laid out for the lattice of the encoder the accumulator was created from
  const bool tuned_grid = enc->cfg.backend == SXEN_BACKEND_GRID && enc->cfg.features == 2 && enc->cfg.dim >= 2 &&
                          enc->cfg.dim <= 3;
  const bool replicas = grad != nullptr && grad->coarse != nullptr &&
                        (enc->tuning.coarse_replicas > 0 || (enc->tuning.coarse_replicas == 0 && n_samples >= kReplicaMinSamples)) &&
                        (enc->cfg.backend == SXEN_BACKEND_SIMPLEX || tuned_grid) && grad->dim == enc->cfg.dim &&
                        grad->res == enc->res;
  a.coarse = replicas ? grad->coarse : nullptr;
  for (int l = 0; l < sxen_dev::kMaxLaunchLevels; ++l) {
    const bool live = l < a.n_levels;
    a.cg.shift[l] = -1;
    a.cg.offset[l] = a.cg.verts[l] = 0;
    if (live && replicas) {
      const size_t gl = static_cast<size_t>(level0 + l);
      a.cg.shift[l] = grad->coarse_shift[gl];
      a.cg.offset[l] = grad->coarse_offset[gl];
      a.cg.verts[l] = grad->coarse_verts[gl];
    }
    const uint32_t res = live ? enc->res[static_cast<size_t>(level0 + l)] : 1u;
    // simplex: s = N_l / S_n (src/encoding.cpp:200); grid: y = x * N_l (src/encoding.cpp:255)
    a.geom.scale[l] = enc->cfg.backend == SXEN_BACKEND_SIMPLEX ? static_cast<double>(res) / enc->scale
                                                               : static_cast<double>(res);
    a.geom.res[l] = static_cast<int32_t>(res);
    // a replicated level never takes the warp-merge path (its lanes leave the level body early)
    if (live && enc->tuning.warp_aggregate > 0 && a.cg.shift[l] < 0) {
      const double verts = std::pow(static_cast<double>(res) + 1.0, enc->cfg.dim);
      if (verts <= static_cast<double>(enc->tuning.warp_aggregate)) a.agg_mask |= 1u << l;
    }
  }
}

sxen_status check_batch(const sxen_encoder* enc, const void* x, sxen_coord_type type, size_t n) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  SXEN_REQUIRE(type == SXEN_COORD_F64 || type == SXEN_COORD_F32, "unknown coordinate type %d", static_cast<int>(type));
  SXEN_REQUIRE(n == 0 || x != nullptr, "coordinate pointer is null");
  SXEN_REQUIRE(n <= (1ULL << 36), "batch of %zu samples exceeds the supported launch size", n);
  return SXEN_OK;
}

// first_level / level_count select a contiguous range of encoder levels (count < 0 = all from first_level on): the
// launch reads and writes only that range's slice of every feature / upstream row and of the accumulator.
// row_stride > 0: feature / upstream rows are row_stride floats apart (>= L*F; the trainer's [encoding | aux] rows).
sxen_status run_encode(sxen_encoder* enc, const void* x, sxen_coord_type type, const float* upstream, size_t n,
                       float* out, sxen_grad* grad, int mode, cudaStream_t stream, int first_level = 0,
                       int level_count = -1, int row_stride = 0, const double* upstream64 = nullptr) {
  if (sxen_status st = check_batch(enc, x, type, n)) return st;
  SXEN_REQUIRE(row_stride == 0 || row_stride >= enc->cfg.levels * enc->cfg.features,
               "encode: row stride %d below the encoded width %d", row_stride, enc->cfg.levels * enc->cfg.features);
  if (level_count < 0) level_count = enc->cfg.levels - first_level;
  SXEN_REQUIRE(first_level >= 0 && level_count >= 0 && first_level + level_count <= enc->cfg.levels,
               "level range [%d, %d) outside the encoder's %d levels", first_level, first_level + level_count,
               enc->cfg.levels);
  if (mode & sxen_dev::kModeFwd) SXEN_REQUIRE(n == 0 || out != nullptr, "encode: output pointer is null");
  if (mode & sxen_dev::kModeBwd) {
    SXEN_REQUIRE(n == 0 || upstream != nullptr, "encode_backward: upstream pointer is null");
    SXEN_REQUIRE(grad != nullptr, "encode_backward: gradient accumulator is null");
    // src/encoding.cpp:323-325
    SXEN_REQUIRE(grad->levels == enc->cfg.levels && grad->features == enc->cfg.features &&
                     grad->table_size == enc->cfg.table_size && grad->device == enc->device,
                 "encode_backward: gradient accumulator shape mismatch");
  }
  if (n == 0 || level_count == 0) return SXEN_OK;
  DeviceGuard guard(enc->device);
  {
    // Tables + accumulator far beyond L2 (>= 192 MiB of tables) and the launch shape left to the library: the fused call
    // runs as a forward launch followed by a backward launch, each level-major -- one level group's rows of ONE array
    // stay L2-resident, where the fused kernel would need two (measured at T = 2^22, n = 3: 1.17 -> 0.84 ms).
    const size_t bytes = static_cast<size_t>(enc->cfg.levels) * enc->level_floats() * sizeof(float);
    if (mode == sxen_dev::kModeBoth && bytes >= (192ull << 20) && enc->tuning.level_major < 0) {
      if (sxen_status st = run_encode(enc, x, type, nullptr, n, out, nullptr, sxen_dev::kModeFwd, stream, first_level, level_count,
                                      row_stride))
        return st;
      return run_encode(enc, x, type, upstream, n, nullptr, grad, sxen_dev::kModeBwd, stream, first_level, level_count,
                        row_stride, upstream64);
    }
  }
  EncodeArgs a;
  base_args(enc, x, type, n, a);
  if (row_stride > 0) a.row_width = row_stride;
  a.upstream = upstream;
  a.out = out;
  a.grads = grad ? grad->values : nullptr;
  a.fixed = (grad && (mode & sxen_dev::kModeBwd)) ? grad->fixed : nullptr;
  a.upstream64 = a.fixed ? upstream64 : nullptr;
  // Launch shape left to the library (level_major < 0, levels_per_thread == 0), by table footprint B = L*T*F*4 bytes
  // (tables and accumulator are the same size; L2 is 126 MB):
  //   B <= 96 MiB   sample-major, 2 levels per thread: a warp writes whole feature rows, everything stays near L2
  //                 (fused launches at dim >= 4 take the next shape instead: n = 4, 0.93 vs 0.66 ms; separate forward /
  //                 backward launches stay sample-major, 0.69 ms the pair)
  //   B <  192 MiB  level-major, 4 levels per thread: one level group's rows at a time stay L2-resident
  //                 (T = 2^20, n = 3: fused 1.07 -> 0.54 ms)
  //   B >= 192 MiB  level-major, 2 levels per thread, and the fused call runs as forward + backward launches (above)
  const size_t table_bytes = static_cast<size_t>(enc->cfg.levels) * enc->level_floats() * sizeof(float);
  const bool big = table_bytes >= (192ull << 20);
  const bool mid = !big && (table_bytes > (96ull << 20) || (enc->cfg.dim >= 4 && mode == sxen_dev::kModeBoth));
  a.level_major = enc->tuning.level_major < 0 ? ((big || mid) ? 1 : 0) : (enc->tuning.level_major ? 1 : 0);
  a.merge_pairs = (enc->tuning.merge_pairs > 0 && enc->cfg.table_size >= 2) ? 1 : 0;
  // L2 eviction policies (profiles/r1_cache_hints.log).  Tables + gradients within reach of L2: the fused launch marks
  // its gradient lines evict_first so the table lines (cached on both dies) survive; beyond L2: gathers and reds both
  // evict_last, which keeps the hot coarse-level rows resident against the streaming fine levels.
  a.cache_hints = enc->tuning.cache_hints >= 0 ? enc->tuning.cache_hints
                  : big ? ((mode & sxen_dev::kModeFwd ? 1 : 0) | (mode & sxen_dev::kModeBwd ? 4 : 0))
                        : (mode == sxen_dev::kModeBoth ? 8 : 0);
  EncodeLaunch ln{};
  ln.features = enc->cfg.features;
  ln.lpt = enc->tuning.levels_per_thread > 0 ? enc->tuning.levels_per_thread
                                             : ((mid && enc->tuning.level_major < 0) ? 4 : 2);
  ln.mode = mode;
  // Chunked fused launch (profiles/r2_l2_window_n3.log): at dim 3, T = 2^19 the tables (64 MiB) and the accumulator (64 MiB)
  // evict each other in the 126 MB L2 when all 16 levels are live at once (gather hit rate 62 % against 93 % forward-only);
  // walking the levels as two ranges of 8 keeps a range's rows resident: 0.500 -> 0.484 ms.  Ranges must start on whole
  // 32-byte sectors of the feature rows (4 levels at F = 2) or the partial-sector stores cost more than the residency
  // gains; at dim 2 (fewer hashed levels live) one range stays faster (0.343 vs 0.357 ms).
  ln.chunk_levels = enc->tuning.level_chunk > 0 ? enc->tuning.level_chunk
                    : (enc->tuning.level_chunk == 0 && mode == sxen_dev::kModeBoth && !big && !mid && enc->cfg.dim == 3 &&
                       enc->cfg.features == 2 && table_bytes > (48ull << 20) && level_count >= 16)
                          ? 8 : 0;
  ln.exact = enc->tuning.exact_blend ? 1 : 0;
  ln.repro = a.fixed != nullptr ? 1 : 0;
  if (ln.repro) {  // the reproducible kernels exist sample-major with one or two levels per thread
    a.level_major = 0;
    ln.lpt = std::min(ln.lpt, 2);
    ln.chunk_levels = 0;
  }
  ln.grid_backend = enc->cfg.backend == SXEN_BACKEND_GRID ? 1 : 0;
  ln.block_threads = enc->tuning.block_threads;
  const int level_end = first_level + level_count;
  for (int level0 = first_level; level0 < level_end; level0 += sxen_dev::kMaxLaunchLevels) {
    level_chunk(enc, (mode & sxen_dev::kModeBwd) ? grad : nullptr, level0, level_end, n, a);
    a.vec = 4;
    if (mode & sxen_dev::kModeFwd) a.vec = std::min(a.vec, ptr_vec(out));
    if (mode & sxen_dev::kModeBwd) a.vec = std::min(a.vec, ptr_vec(upstream));
    int used = 0;
    SXEN_CUDA(kEncode[enc->cfg.dim - 1](ln, a, stream, &used));
    count_launch();
    if (a.coarse != nullptr) {
      bool any = false;
      for (int l = 0; l < a.n_levels; ++l) any = any || a.cg.shift[l] >= 0;
      if (any) {
        SXEN_CUDA(kFold[enc->cfg.dim - 1](a, stream));
        count_launch();
      }
    }
  }
  enc->touched += static_cast<uint64_t>(n) * static_cast<uint64_t>(level_count) *
                  static_cast<uint64_t>(enc->vertices()) * ((mode == sxen_dev::kModeBoth) ? 2u : 1u);
  return SXEN_OK;
}

sxen_status read_status(sxen_encoder* enc, cudaStream_t stream, bool reset_bad) {
  SXEN_CUDA(cudaMemcpyAsync(enc->status_host, enc->status, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            stream));
  SXEN_CUDA(cudaStreamSynchronize(stream));
  if (reset_bad && enc->status_host[0] != kNoBadSample) {
    const unsigned long long none = kNoBadSample;
    SXEN_CUDA(cudaMemcpyAsync(enc->status, &none, sizeof(none), cudaMemcpyHostToDevice, stream));
    SXEN_CUDA(cudaStreamSynchronize(stream));
  }
  return SXEN_OK;
}

sxen_status ensure_staging(sxen_encoder* enc, bool need_up64) {
  const size_t lf = static_cast<size_t>(enc->cfg.levels) * static_cast<size_t>(enc->cfg.features);
  if (!enc->stage_samples) {
    // samples per slot (2^17: 20 MB in, 17 MB out per pass at L*F = 32 -- large enough for the PCIe link's
    // large-transfer rate, tools/e2e_sweep.py).  SXEN_HOST_CHUNK_LOG2 (14..22) is a tuning aid.
    size_t chunk = 1u << 17;
    if (const char* env = std::getenv("SXEN_HOST_CHUNK_LOG2")) {
      const int v = std::atoi(env);
      if (v >= 14 && v <= 22) chunk = static_cast<size_t>(1) << v;
    }
    for (int i = 0; i < sxen_encoder::kStages; ++i) {
      SXEN_CUDA(cudaMalloc(&enc->stage_x[i], chunk * static_cast<size_t>(enc->cfg.dim) * sizeof(double)));
      SXEN_CUDA(cudaMalloc(&enc->stage_up[i], chunk * lf * sizeof(float)));
      SXEN_CUDA(cudaMalloc(&enc->stage_out[i], chunk * lf * sizeof(float)));
      SXEN_CUDA(cudaEventCreateWithFlags(&enc->stage_in[i], cudaEventDisableTiming));
      SXEN_CUDA(cudaEventCreateWithFlags(&enc->stage_done[i], cudaEventDisableTiming));
      SXEN_CUDA(cudaEventCreateWithFlags(&enc->stage_back[i], cudaEventDisableTiming));
    }
    for (int i = 0; i < 3; ++i) SXEN_CUDA(cudaStreamCreateWithFlags(&enc->stage_stream[i], cudaStreamNonBlocking));
    enc->stage_samples = chunk;
  }
  if (need_up64 && enc->stage_up64[0] == nullptr) {
    for (int i = 0; i < sxen_encoder::kStages; ++i)
      SXEN_CUDA(cudaMalloc(&enc->stage_up64[i], enc->stage_samples * lf * sizeof(double)));
  }
  return SXEN_OK;
}

// upstream arrives from the host as the reference's doubles (include/sxen/encoding.hpp:119); the kernels take f32.
__global__ void narrow_kernel(const double* __restrict__ src, float* __restrict__ dst, size_t n) {
  const size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = static_cast<float>(src[i]);
}

}  // namespace

// encode / encode_backward with feature rows `row_stride` floats apart (declared in sxen_common.hpp): the trainer's
// [encoding | aux] MLP input rows, src/trainer.cpp:31-35,47.
sxen_status sxen_encoder_encode_strided(sxen_encoder* enc, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                        float* out_dev, int row_stride, void* stream) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  return run_encode(enc, x_dev, type, nullptr, n_samples, out_dev, nullptr, sxen_dev::kModeFwd, as_stream(stream), 0, -1,
                    row_stride);
}

sxen_status sxen_encoder_encode_backward_strided(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                 const float* upstream_dev, int row_stride, size_t n_samples,
                                                 sxen_grad* grad, int first_level, int level_count, void* stream) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  return run_encode(enc, x_dev, type, upstream_dev, n_samples, nullptr, grad, sxen_dev::kModeBwd, as_stream(stream),
                    first_level, level_count, row_stride);
}

sxen_status sxen_encoder_encode_backward_strided64(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                   const float* upstream_dev, const double* upstream64_dev, int row_stride,
                                                   size_t n_samples, sxen_grad* grad, int first_level, int level_count,
                                                   void* stream) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  return run_encode(enc, x_dev, type, upstream_dev, n_samples, nullptr, grad, sxen_dev::kModeBwd, as_stream(stream),
                    first_level, level_count, row_stride, upstream64_dev);
}

sxen_status sxen_encoder_fused_args(sxen_encoder* enc, sxen_grad* grad, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                    EncodeArgs* out) {
  if (sxen_status st = check_batch(enc, x_dev, type, n_samples)) return st;
  SXEN_REQUIRE(grad != nullptr && out != nullptr, "null argument");
  SXEN_REQUIRE(grad->levels == enc->cfg.levels && grad->features == enc->cfg.features && grad->table_size == enc->cfg.table_size &&
                   grad->device == enc->device,
               "encode_backward: gradient accumulator shape mismatch");
  SXEN_REQUIRE(enc->cfg.levels <= sxen_dev::kMaxLaunchLevels, "fused step: more than %d levels", sxen_dev::kMaxLaunchLevels);
  EncodeArgs& a = *out;
  base_args(enc, x_dev, type, n_samples, a);
  a.grads = grad->values;
  level_chunk(enc, grad, 0, enc->cfg.levels, n_samples, a);
  a.merge_pairs = (enc->tuning.merge_pairs > 0 && enc->cfg.table_size >= 2) ? 1 : 0;
  // gathers and reds share L2 as in the fused encode launch: gradient lines evict_first (profiles/r1_cache_hints.log)
  a.cache_hints = enc->tuning.cache_hints >= 0 ? enc->tuning.cache_hints : 8;
  return SXEN_OK;
}

sxen_status sxen_encoder_fused_finish(sxen_encoder* enc, const EncodeArgs& a, void* stream) {
  if (a.coarse != nullptr) {
    bool any = false;
    for (int l = 0; l < a.n_levels; ++l) any = any || a.cg.shift[l] >= 0;
    if (any) {
      SXEN_CUDA(kFold[enc->cfg.dim - 1](a, as_stream(stream)));
      count_launch();
    }
  }
  enc->touched += static_cast<uint64_t>(a.n_samples) * static_cast<uint64_t>(enc->cfg.levels) *
                  static_cast<uint64_t>(enc->vertices()) * 2u;  // the forward walk and the backward walk (src/encoding.cpp:222,241)
  return SXEN_OK;
}

// SparseAdamState::step for the single-GPU trainer (declared in sxen_common.hpp): when the batch is small against the
// tables, the update walks the batch (sparse_adam_walk_kernel) instead of scanning all L*T accumulator rows.  The caller
// guarantees that every touched row of `grad` comes from this batch's backward.  Same arithmetic, same rows, same
// clearing as sxen_sparse_adam_step(clear_grad = 1).
bool sxen_sparse_adam_walk_pays(const sxen_encoder* enc, size_t n_samples) {
  if (enc->cfg.features != 2) return false;
  const double visits = static_cast<double>(n_samples) * enc->cfg.levels * enc->vertices();
  const double rows = static_cast<double>(enc->cfg.levels) * enc->cfg.table_size;
  return visits * 8.0 <= rows;  // a visit (lattice walk + atomic exchange) against a scanned row (one coalesced 8-byte load)
}

sxen_status sxen_sparse_adam_step_walk(sxen_sparse_adam* opt, sxen_encoder* enc, sxen_grad* grad, const void* x_dev,
                                       sxen_coord_type type, size_t n_samples, const sxen_adam_config* cfg,
                                       const unsigned long long* gate_dev, void* stream) {
  SXEN_REQUIRE(opt != nullptr && enc != nullptr && grad != nullptr && cfg != nullptr, "null argument");
  SXEN_REQUIRE(enc->cfg.features == 2 && enc->cfg.levels == opt->levels && enc->cfg.features == opt->features &&
                   enc->cfg.table_size == opt->table_size && grad->levels == opt->levels &&
                   grad->features == opt->features && grad->table_size == opt->table_size &&
                   enc->device == opt->device && grad->device == opt->device,
               "sparse adam step: encoder/gradient shape mismatch");
  DeviceGuard guard(opt->device);
  ++opt->t;  // src/optimizer.cpp:64
  if (n_samples == 0) return SXEN_OK;
  sxen_dev::AdamWalkArgs o{};
  o.tables = reinterpret_cast<float2*>(enc->tables);
  o.grads = reinterpret_cast<float2*>(grad->values);
  o.m = reinterpret_cast<double2*>(opt->m);
  o.v = reinterpret_cast<double2*>(opt->v);
  o.c = sxen_adam_scalars(*cfg, opt->t);
  o.status = opt->status;
  o.gate = gate_dev;
  o.fixed = reinterpret_cast<longlong2*>(grad->fixed);
  EncodeArgs a;
  base_args(enc, x_dev, type, n_samples, a);
  for (int level0 = 0; level0 < enc->cfg.levels; level0 += sxen_dev::kMaxLaunchLevels) {
    level_chunk(enc, nullptr, level0, enc->cfg.levels, 0, a);
    SXEN_CUDA(kAdamWalk[enc->cfg.dim - 1](a, o, enc->cfg.backend == SXEN_BACKEND_GRID ? 1 : 0, as_stream(stream)));
    count_launch();
  }
  return SXEN_OK;
}

namespace {
}  // namespace

extern "C" {

// ---------------------------------------------------------------------------------------------- library
const char* sxen_last_error(void) { return last_error().c_str(); }
const char* sxen_version(void) { return "sxen-b200 0.1 (sm_100a)"; }

int32_t sxen_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < n; ++d) {
    int major = 0;
    if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, d) == cudaSuccess && major == 10) ++ok;
  }
  return ok;
}

uint64_t sxen_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

sxen_status sxen_host_alloc(size_t bytes, void** out) {
  SXEN_REQUIRE(out != nullptr, "output pointer is null");
  SXEN_CUDA(cudaHostAlloc(out, bytes, cudaHostAllocDefault));
  return SXEN_OK;
}

sxen_status sxen_host_free(void* ptr) {
  if (ptr) SXEN_CUDA(cudaFreeHost(ptr));
  return SXEN_OK;
}

sxen_status sxen_device_alloc(int32_t device, size_t bytes, void** out_dev) {
  SXEN_REQUIRE(out_dev != nullptr, "output pointer is null");
  *out_dev = nullptr;
  int ndev = 0;
  SXEN_CUDA(cudaGetDeviceCount(&ndev));
  SXEN_REQUIRE(device >= 0 && device < ndev, "device %d out of range (%d visible)", device, ndev);
  DeviceGuard guard(device);
  SXEN_CUDA(cudaMalloc(out_dev, bytes ? bytes : 1));
  return SXEN_OK;
}

sxen_status sxen_device_free(int32_t device, void* ptr_dev) {
  if (!ptr_dev) return SXEN_OK;
  DeviceGuard guard(device);
  SXEN_CUDA(cudaFree(ptr_dev));
  return SXEN_OK;
}

sxen_status sxen_device_upload(int32_t device, void* dst_dev, const void* src_host, size_t bytes, void* stream) {
  SXEN_REQUIRE(bytes == 0 || (dst_dev != nullptr && src_host != nullptr), "null argument");
  DeviceGuard guard(device);
  SXEN_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, as_stream(stream)));
  SXEN_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return SXEN_OK;
}

sxen_status sxen_device_download(int32_t device, void* dst_host, const void* src_dev, size_t bytes, void* stream) {
  SXEN_REQUIRE(bytes == 0 || (dst_host != nullptr && src_dev != nullptr), "null argument");
  DeviceGuard guard(device);
  SXEN_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
  SXEN_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return SXEN_OK;
}

sxen_status sxen_device_zero(int32_t device, void* dst_dev, size_t bytes, void* stream) {
  SXEN_REQUIRE(bytes == 0 || dst_dev != nullptr, "null argument");
  DeviceGuard guard(device);
  SXEN_CUDA(cudaMemsetAsync(dst_dev, 0, bytes, as_stream(stream)));
  return SXEN_OK;
}

// ---------------------------------------------------------------------------------------------- rng
uint64_t sxen_mix64(uint64_t z) { return sxen_dev::mix64(z); }
uint64_t sxen_hash_combine(uint64_t a, uint64_t b) { return sxen_dev::hash_combine(a, b); }

sxen_status sxen_rng_fill_dev(uint64_t seed, int32_t has_stream, uint64_t stream_id, uint64_t first_counter, double lo,
                              double hi, void* out_dev, size_t count, sxen_coord_type type, void* stream) {
  SXEN_REQUIRE(count == 0 || out_dev != nullptr, "output pointer is null");
  SXEN_REQUIRE(first_counter >= 1, "CounterRng draws are 1-based");
  if (count == 0) return SXEN_OK;
  uint64_t key = sxen_dev::mix64(seed);                       // include/sxen/rng.hpp:26
  if (has_stream) key = sxen_dev::hash_combine(key, stream_id);  // include/sxen/rng.hpp:27
  const double span = hi - lo;
  if (type == SXEN_COORD_F32) {
    rng_fill_kernel<float><<<grid_for(count), 256, 0, as_stream(stream)>>>(static_cast<float*>(out_dev), count, key,
                                                                          first_counter, lo, span);
  } else {
    rng_fill_kernel<double><<<grid_for(count), 256, 0, as_stream(stream)>>>(static_cast<double*>(out_dev), count, key,
                                                                           first_counter, lo, span);
  }
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

// ---------------------------------------------------------------------------------------------- config
sxen_status sxen_encoder_config_default(sxen_encoder_config* cfg) {
  SXEN_REQUIRE(cfg != nullptr, "config pointer is null");
  *cfg = sxen_encoder_config{2, 8, 1u << 16, 2, 16, 2.0, SXEN_BACKEND_SIMPLEX, SXEN_SCALE_RAW};  // encoding.hpp:18-27
  return SXEN_OK;
}

sxen_status sxen_encoder_validate(const sxen_encoder_config* cfg) {
  SXEN_REQUIRE(cfg != nullptr, "config pointer is null");
  return validate(*cfg);
}

sxen_status sxen_level_resolution(const sxen_encoder_config* cfg, int32_t level, uint32_t* out) {
  SXEN_REQUIRE(cfg != nullptr && out != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < cfg->levels, "level_resolution: level out of range");  // src/encoding.cpp:69-71
  *out = level_resolution(*cfg, level);
  return SXEN_OK;
}

sxen_status sxen_equal_memory_multiplier(int32_t dim, double* out) {
  SXEN_REQUIRE(out != nullptr, "null argument");
  SXEN_REQUIRE(dim >= 1 && dim <= SXEN_MAX_DIM, "equal_memory_multiplier: dim out of range");  // src/encoding.cpp:61-63
  *out = equal_memory_multiplier(dim);
  return SXEN_OK;
}

sxen_status sxen_skew_constants(int32_t dim, double out[3]) {
  SXEN_REQUIRE(out != nullptr, "null argument");
  SXEN_REQUIRE(dim >= 1 && dim <= SXEN_MAX_DIM, "dimension must be in [1, %d], got %d", SXEN_MAX_DIM, dim);
  const double root = std::sqrt(static_cast<double>(dim) + 1.0);  // src/lattice.cpp:23
  out[0] = (root - 1.0) / static_cast<double>(dim);
  out[1] = (1.0 - 1.0 / root) / static_cast<double>(dim);
  out[2] = root;
  return SXEN_OK;
}

sxen_status sxen_hash_coords(const int64_t* coords, int32_t dim, uint32_t* out) {
  SXEN_REQUIRE(coords != nullptr && out != nullptr, "null argument");
  SXEN_REQUIRE(dim >= 1 && dim <= SXEN_MAX_DIM, "hash_index: coordinate count out of range");  // hashing.hpp:36-38
  uint32_t h = 0;
  for (int i = 0; i < dim; ++i) h ^= static_cast<uint32_t>(static_cast<uint64_t>(coords[i])) * sxen_dev::prime_of(i);
  *out = h;
  return SXEN_OK;
}

// ---------------------------------------------------------------------------------------------- encoder
sxen_status sxen_encoder_create(const sxen_encoder_config* cfg, int32_t device, sxen_encoder** out) {
  SXEN_REQUIRE(cfg != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  if (sxen_status st = validate(*cfg)) return st;
  int ndev = 0;
  SXEN_CUDA(cudaGetDeviceCount(&ndev));
  SXEN_REQUIRE(device >= 0 && device < ndev, "device %d out of range (%d visible)", device, ndev);
  int major = 0;
  SXEN_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device));
  if (major != 10) return fail(SXEN_CUDA_ERROR, "device %d is sm_%dx; this library carries sm_100a code only", device, major);
  DeviceGuard guard(device);
  sxen_encoder* e = new sxen_encoder();
  e->cfg = *cfg;
  e->device = device;
  e->tuning = default_tuning();
  e->res.resize(static_cast<size_t>(cfg->levels));
  for (int l = 0; l < cfg->levels; ++l) e->res[static_cast<size_t>(l)] = level_resolution(*cfg, l);
  double sc[3];
  sxen_skew_constants(cfg->dim, sc);
  e->skew = sc[0];
  e->scale = sc[2];
  const size_t bytes = static_cast<size_t>(cfg->levels) * e->level_floats() * sizeof(float);
  cudaError_t err = cudaMalloc(&e->tables, bytes);
  if (err == cudaSuccess) err = cudaMemset(e->tables, 0, bytes);  // tables start at zero (src/encoding.cpp:163-166)
  if (err == cudaSuccess) err = cudaMalloc(&e->status, 2 * sizeof(unsigned long long));
  if (err == cudaSuccess) err = cudaHostAlloc(&e->status_host, 2 * sizeof(unsigned long long), cudaHostAllocDefault);
  if (err == cudaSuccess) {
    const unsigned long long init[2] = {kNoBadSample, 0ULL};
    err = cudaMemcpy(e->status, init, sizeof(init), cudaMemcpyHostToDevice);
  }
  if (err != cudaSuccess) {
    sxen_encoder_destroy(e);
    return cuda_fail(err, "sxen_encoder_create allocation");
  }
  *out = e;
  return SXEN_OK;
}

sxen_status sxen_encoder_destroy(sxen_encoder* enc) {
  if (!enc) return SXEN_OK;
  DeviceGuard guard(enc->device);
  cudaFree(enc->tables);
  cudaFree(enc->status);
  cudaFreeHost(enc->status_host);
  for (int i = 0; i < sxen_encoder::kStages; ++i) {
    cudaFree(enc->stage_x[i]);
    cudaFree(enc->stage_up[i]);
    cudaFree(enc->stage_up64[i]);
    cudaFree(enc->stage_out[i]);
    if (enc->stage_in[i]) cudaEventDestroy(enc->stage_in[i]);
    if (enc->stage_done[i]) cudaEventDestroy(enc->stage_done[i]);
    if (enc->stage_back[i]) cudaEventDestroy(enc->stage_back[i]);
  }
  for (int i = 0; i < 3; ++i)
    if (enc->stage_stream[i]) cudaStreamDestroy(enc->stage_stream[i]);
  delete enc;
  return SXEN_OK;
}

sxen_status sxen_encoder_get_config(const sxen_encoder* enc, sxen_encoder_config* out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  *out = enc->cfg;
  return SXEN_OK;
}

sxen_status sxen_encoder_resolution(const sxen_encoder* enc, int32_t level, uint32_t* out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < enc->cfg.levels, "resolution: level out of range");
  *out = enc->res[static_cast<size_t>(level)];
  return SXEN_OK;
}

sxen_status sxen_encoder_parameter_count(const sxen_encoder* enc, uint64_t* out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  *out = static_cast<uint64_t>(enc->cfg.levels) * enc->cfg.table_size * static_cast<uint64_t>(enc->cfg.features);
  return SXEN_OK;
}

sxen_status sxen_encoder_set_tuning(sxen_encoder* enc, const sxen_tuning* t) {
  SXEN_REQUIRE(enc != nullptr && t != nullptr, "null argument");
  sxen_tuning d = default_tuning();
  sxen_tuning n = *t;
  if (n.levels_per_thread < 0) n.levels_per_thread = d.levels_per_thread;
  if (n.block_threads <= 0) n.block_threads = d.block_threads;
  SXEN_REQUIRE(n.block_threads % 32 == 0 && n.block_threads <= 1024, "block_threads must be a multiple of 32, <= 1024");
  SXEN_REQUIRE(n.warp_aggregate >= 0, "warp_aggregate must be >= 0");
  if (n.merge_pairs == 0) n.merge_pairs = d.merge_pairs;
  SXEN_REQUIRE(n.cache_hints >= -1 && n.cache_hints <= 15, "cache_hints must be -1 (auto) or in [0, 15]");
  enc->tuning = n;
  return SXEN_OK;
}

sxen_status sxen_encoder_get_tuning(const sxen_encoder* enc, sxen_tuning* out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  *out = enc->tuning;
  return SXEN_OK;
}

sxen_status sxen_encoder_init_tables(sxen_encoder* enc, uint64_t seed, void* stream) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  DeviceGuard guard(enc->device);
  const size_t total = static_cast<size_t>(enc->cfg.levels) * enc->level_floats();
  const double lo = -1e-4, hi = 1e-4;
  init_tables_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(enc->tables, enc->level_floats(), enc->cfg.levels,
                                                                     sxen_dev::mix64(seed), lo, hi - lo);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  return SXEN_OK;
}

sxen_status sxen_encoder_upload_table(sxen_encoder* enc, int32_t level, const float* src_host) {
  SXEN_REQUIRE(enc != nullptr && src_host != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < enc->cfg.levels, "table: level out of range");
  DeviceGuard guard(enc->device);
  SXEN_CUDA(cudaMemcpy(enc->tables + static_cast<size_t>(level) * enc->level_floats(), src_host,
                       enc->level_floats() * sizeof(float), cudaMemcpyHostToDevice));
  return SXEN_OK;
}

sxen_status sxen_encoder_download_table(const sxen_encoder* enc, int32_t level, float* dst_host) {
  SXEN_REQUIRE(enc != nullptr && dst_host != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < enc->cfg.levels, "table: level out of range");
  DeviceGuard guard(enc->device);
  SXEN_CUDA(cudaMemcpy(dst_host, enc->tables + static_cast<size_t>(level) * enc->level_floats(),
                       enc->level_floats() * sizeof(float), cudaMemcpyDeviceToHost));
  return SXEN_OK;
}

sxen_status sxen_encoder_tables_dev(sxen_encoder* enc, float** out_dev) {
  SXEN_REQUIRE(enc != nullptr && out_dev != nullptr, "null argument");
  *out_dev = enc->tables;
  return SXEN_OK;
}

sxen_status sxen_encoder_encode(sxen_encoder* enc, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                float* out_dev, void* stream) {
  return run_encode(enc, x_dev, type, nullptr, n_samples, out_dev, nullptr, sxen_dev::kModeFwd, as_stream(stream));
}

sxen_status sxen_encoder_encode_backward(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                         const float* upstream_dev, size_t n_samples, sxen_grad* grad, void* stream) {
  return run_encode(enc, x_dev, type, upstream_dev, n_samples, nullptr, grad, sxen_dev::kModeBwd, as_stream(stream));
}

sxen_status sxen_encoder_encode_forward_backward(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                 const float* upstream_dev, size_t n_samples, float* out_dev,
                                                 sxen_grad* grad, void* stream) {
  return run_encode(enc, x_dev, type, upstream_dev, n_samples, out_dev, grad, sxen_dev::kModeBoth, as_stream(stream));
}

sxen_status sxen_encoder_encode_backward_levels(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                const float* upstream_dev, size_t n_samples, sxen_grad* grad,
                                                int32_t first_level, int32_t level_count, void* stream) {
  SXEN_REQUIRE(level_count >= 0, "level_count must be >= 0");
  return run_encode(enc, x_dev, type, upstream_dev, n_samples, nullptr, grad, sxen_dev::kModeBwd, as_stream(stream),
                    first_level, level_count);
}

sxen_status sxen_encoder_encode_forward_backward_levels(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                        const float* upstream_dev, size_t n_samples, float* out_dev,
                                                        sxen_grad* grad, int32_t first_level, int32_t level_count,
                                                        void* stream) {
  SXEN_REQUIRE(level_count >= 0, "level_count must be >= 0");
  return run_encode(enc, x_dev, type, upstream_dev, n_samples, out_dev, grad, sxen_dev::kModeBoth, as_stream(stream),
                    first_level, level_count);
}

sxen_status sxen_encoder_encode_debug(sxen_encoder* enc, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                      uint32_t* idx_dev, double* w_dev, void* stream) {
  if (sxen_status st = check_batch(enc, x_dev, type, n_samples)) return st;
  SXEN_REQUIRE(n_samples == 0 || (idx_dev != nullptr && w_dev != nullptr), "encode_debug: output pointer is null");
  if (n_samples == 0) return SXEN_OK;
  DeviceGuard guard(enc->device);
  EncodeArgs a;
  base_args(enc, x_dev, type, n_samples, a);
  for (int level0 = 0; level0 < enc->cfg.levels; level0 += sxen_dev::kMaxLaunchLevels) {
    level_chunk(enc, nullptr, level0, enc->cfg.levels, 0, a);
    SXEN_CUDA(kDebug[enc->cfg.dim - 1](a, enc->cfg.backend == SXEN_BACKEND_GRID ? 1 : 0, idx_dev, w_dev,
                                       enc->cfg.levels, as_stream(stream)));
    count_launch();
  }
  return SXEN_OK;
}

sxen_status sxen_encoder_check(sxen_encoder* enc, void* stream) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  DeviceGuard guard(enc->device);
  if (sxen_status st = read_status(enc, as_stream(stream), true)) return st;
  if (enc->status_host[0] != kNoBadSample) {
    // check_input, src/encoding.cpp:189-192
    return fail(SXEN_INVALID_ARGUMENT, "encode: coordinate outside the unit cube (first offending sample %llu)",
                enc->status_host[0]);
  }
  return SXEN_OK;
}

sxen_status sxen_encoder_counters(sxen_encoder* enc, sxen_lookup_counters* out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  DeviceGuard guard(enc->device);
  SXEN_CUDA(cudaDeviceSynchronize());
  SXEN_CUDA(cudaMemcpy(enc->status_host, enc->status, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  out->touched_vertices = enc->touched;
  out->out_of_bounds = enc->status_host[1];
  return SXEN_OK;
}

sxen_status sxen_encoder_reset_counters(sxen_encoder* enc) {
  SXEN_REQUIRE(enc != nullptr, "encoder handle is null");
  DeviceGuard guard(enc->device);
  SXEN_CUDA(cudaDeviceSynchronize());
  SXEN_CUDA(cudaMemset(enc->status + 1, 0, sizeof(unsigned long long)));
  enc->touched = 0;
  return SXEN_OK;
}

// Host-buffer forms.  One pipeline serves all three: pass c copies its inputs on the copy-in stream, runs its kernels on
// the compute stream and returns its features on the copy-out stream, in slot c % kStages; a slot's inputs are
// overwritten only after its previous kernels finished, its feature buffer only after the previous copy-out finished.
// With pinned host buffers the three stages of neighbouring passes overlap and the call runs at the PCIe rate.
namespace {

sxen_status host_pipeline(sxen_encoder* enc, const double* x_host, const void* up_host, sxen_coord_type up_type,
                          size_t n_samples, float* out_host, sxen_grad* grad, int mode) {
  const bool fwd = (mode & sxen_dev::kModeFwd) != 0, bwd = (mode & sxen_dev::kModeBwd) != 0;
  const bool up64 = bwd && up_type == SXEN_COORD_F64;
  DeviceGuard guard(enc->device);
  if (sxen_status st = ensure_staging(enc, up64)) return st;
  const size_t dim = static_cast<size_t>(enc->cfg.dim);
  const size_t lf = static_cast<size_t>(enc->cfg.levels) * static_cast<size_t>(enc->cfg.features);
  cudaStream_t s_in = enc->stage_stream[0], s_k = enc->stage_stream[1], s_out = enc->stage_stream[2];
  // Pass sizes: the first pass's copy-in and the last pass's copy-out are the only transfers nothing overlaps, so the
  // passes ramp up from 2^15 samples to the slot size and back down; in between they are slot-sized, which keeps the
  // link at its large-transfer rate (tools/e2e_proto.py: 3.4 ms per 2^20 samples against 3.3 ms of raw two-way copies).
  std::vector<size_t> passes;
  {
    const size_t cap = enc->stage_samples;
    std::vector<size_t> ramp;
    size_t ramp0 = 1u << 15;
    if (const char* env = std::getenv("SXEN_HOST_RAMP_LOG2")) {  // tuning aid, like SXEN_HOST_CHUNK_LOG2
      const int v = std::atoi(env);
      if (v >= 12 && v <= 20) ramp0 = static_cast<size_t>(1) << v;
    }
    for (size_t r = ramp0; r < cap; r <<= 1) ramp.push_back(r);
    size_t ramps = 0;
    for (size_t r : ramp) ramps += 2 * r;
    if (n_samples > ramps + cap / 2) {
      for (size_t r : ramp) passes.push_back(r);
      for (size_t left = n_samples - ramps; left > 0;) {
        const size_t n = std::min(cap, left);
        passes.push_back(n);
        left -= n;
      }
      for (size_t i = ramp.size(); i-- > 0;) passes.push_back(ramp[i]);
    } else {
      const size_t per = std::min(cap, std::max<size_t>((n_samples + 7) / 8, 1u << 14));
      for (size_t left = n_samples; left > 0;) {
        const size_t n = std::min(per, left);
        passes.push_back(n);
        left -= n;
      }
    }
  }
  size_t done = 0;
  for (int c = 0; c < static_cast<int>(passes.size()); ++c) {
    const int slot = c % sxen_encoder::kStages;
    const size_t n = passes[static_cast<size_t>(c)];
    if (c >= sxen_encoder::kStages) SXEN_CUDA(cudaStreamWaitEvent(s_in, enc->stage_done[slot], 0));
    SXEN_CUDA(cudaMemcpyAsync(enc->stage_x[slot], x_host + done * dim, n * dim * sizeof(double), cudaMemcpyHostToDevice, s_in));
    if (bwd) {
      if (up64) {
        SXEN_CUDA(cudaMemcpyAsync(enc->stage_up64[slot], static_cast<const double*>(up_host) + done * lf,
                                  n * lf * sizeof(double), cudaMemcpyHostToDevice, s_in));
      } else {
        SXEN_CUDA(cudaMemcpyAsync(enc->stage_up[slot], static_cast<const float*>(up_host) + done * lf,
                                  n * lf * sizeof(float), cudaMemcpyHostToDevice, s_in));
      }
    }
    SXEN_CUDA(cudaEventRecord(enc->stage_in[slot], s_in));
    SXEN_CUDA(cudaStreamWaitEvent(s_k, enc->stage_in[slot], 0));
    if (fwd && c >= sxen_encoder::kStages) SXEN_CUDA(cudaStreamWaitEvent(s_k, enc->stage_back[slot], 0));
    if (up64) {
      narrow_kernel<<<static_cast<unsigned>((n * lf + 255) / 256), 256, 0, s_k>>>(enc->stage_up64[slot], enc->stage_up[slot], n * lf);
      SXEN_CUDA(cudaGetLastError());
      count_launch();
    }
    if (sxen_status s = run_encode(enc, enc->stage_x[slot], SXEN_COORD_F64, bwd ? enc->stage_up[slot] : nullptr, n,
                                   fwd ? enc->stage_out[slot] : nullptr, bwd ? grad : nullptr, mode, s_k))
      return s;
    SXEN_CUDA(cudaEventRecord(enc->stage_done[slot], s_k));
    if (fwd) {
      SXEN_CUDA(cudaStreamWaitEvent(s_out, enc->stage_done[slot], 0));
      SXEN_CUDA(cudaMemcpyAsync(out_host + done * lf, enc->stage_out[slot], n * lf * sizeof(float), cudaMemcpyDeviceToHost, s_out));
      SXEN_CUDA(cudaEventRecord(enc->stage_back[slot], s_out));
    }
    done += n;
  }
  SXEN_CUDA(cudaStreamSynchronize(s_k));
  if (fwd) SXEN_CUDA(cudaStreamSynchronize(s_out));
  return sxen_encoder_check(enc, s_k);
}

}  // namespace

sxen_status sxen_encoder_encode_host(sxen_encoder* enc, const double* x_host, size_t n_samples, float* out_host) {
  if (sxen_status st = check_batch(enc, x_host, SXEN_COORD_F64, n_samples)) return st;
  SXEN_REQUIRE(n_samples == 0 || out_host != nullptr, "encode: output pointer is null");
  if (n_samples == 0) return SXEN_OK;
  return host_pipeline(enc, x_host, nullptr, SXEN_COORD_F32, n_samples, out_host, nullptr, sxen_dev::kModeFwd);
}

sxen_status sxen_encoder_encode_backward_host(sxen_encoder* enc, const double* x_host, const double* upstream_host,
                                              size_t n_samples, sxen_grad* grad) {
  if (sxen_status st = check_batch(enc, x_host, SXEN_COORD_F64, n_samples)) return st;
  SXEN_REQUIRE(n_samples == 0 || upstream_host != nullptr, "encode_backward: upstream pointer is null");
  SXEN_REQUIRE(grad != nullptr, "encode_backward: gradient accumulator is null");
  if (n_samples == 0) return SXEN_OK;
  return host_pipeline(enc, x_host, upstream_host, SXEN_COORD_F64, n_samples, nullptr, grad, sxen_dev::kModeBwd);
}

sxen_status sxen_encoder_encode_forward_backward_host(sxen_encoder* enc, const double* x_host,
                                                      const void* upstream_host, sxen_coord_type upstream_type,
                                                      size_t n_samples, float* out_host, sxen_grad* grad) {
  if (sxen_status st = check_batch(enc, x_host, SXEN_COORD_F64, n_samples)) return st;
  SXEN_REQUIRE(upstream_type == SXEN_COORD_F64 || upstream_type == SXEN_COORD_F32, "unknown upstream type");
  SXEN_REQUIRE(n_samples == 0 || (upstream_host != nullptr && out_host != nullptr), "null upstream or output pointer");
  SXEN_REQUIRE(grad != nullptr, "encode_backward: gradient accumulator is null");
  if (n_samples == 0) return SXEN_OK;
  return host_pipeline(enc, x_host, upstream_host, upstream_type, n_samples, out_host, grad, sxen_dev::kModeBoth);
}

// ---------------------------------------------------------------------------------------------- gradient accumulator
sxen_status sxen_grad_create(const sxen_encoder* enc, sxen_grad** out) {
  SXEN_REQUIRE(enc != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  DeviceGuard guard(enc->device);
  sxen_grad* g = new sxen_grad();
  g->device = enc->device;
  g->levels = enc->cfg.levels;
  g->features = enc->cfg.features;
  g->table_size = enc->cfg.table_size;
  cudaError_t err = cudaMalloc(&g->values, g->count() * sizeof(float));
  if (err != cudaSuccess) {
    delete g;
    return cuda_fail(err, "sxen_grad_create allocation");
  }
  // Replicated dense accumulators for the coarse simplex levels: a level with V = (res+1)^dim lattice vertices gets
  // R = 2^floor(log2(2^17 / V)) replicas, capped at 64, when R >= 2 (at most 2^17 rows = 1 MiB per level at F = 2).
  g->dim = enc->cfg.dim;
  g->res = enc->res;
  g->coarse_offset.assign(static_cast<size_t>(g->levels), 0u);
  g->coarse_verts.assign(static_cast<size_t>(g->levels), 0u);
  g->coarse_shift.assign(static_cast<size_t>(g->levels), -1);
  {
    // (both backends address the same (res+1)^dim lattice; kernels without the replica path simply ignore the buffer)
    for (int l = 0; l < g->levels; ++l) {
      const double verts = std::pow(static_cast<double>(enc->res[static_cast<size_t>(l)]) + 1.0, enc->cfg.dim);
      if (verts > static_cast<double>(1u << 16)) continue;
      int shift = 0;
      while (shift < 6 && verts * static_cast<double>(2u << shift) <= static_cast<double>(1u << 17)) ++shift;
      if (shift < 1) continue;
      // rows per replica rounded up to even: every replica then starts on a 16-byte boundary (the F == 2 pair merge
      // issues 16-byte reds); the padding row is never touched and the fold skips it like any untouched row
      const uint32_t rows = (static_cast<uint32_t>(verts) + 1u) & ~1u;
      g->coarse_shift[static_cast<size_t>(l)] = shift;
      g->coarse_verts[static_cast<size_t>(l)] = rows;
      g->coarse_offset[static_cast<size_t>(l)] = static_cast<uint32_t>(g->coarse_floats);
      g->coarse_floats += (static_cast<size_t>(rows) << shift) * static_cast<size_t>(g->features);
    }
  }
  if (g->coarse_floats) {
    err = cudaMalloc(&g->coarse, g->coarse_floats * sizeof(float));
    if (err != cudaSuccess) {
      cudaFree(g->values);
      delete g;
      return cuda_fail(err, "sxen_grad_create allocation");
    }
    fill_u32_kernel<<<grid_for(g->coarse_floats), 256>>>(reinterpret_cast<uint32_t*>(g->coarse), g->coarse_floats,
                                                        kUntouchedBits);
    count_launch();
  }
  *out = g;
  const sxen_status st = sxen_grad_clear(g, nullptr);
  if (st == SXEN_OK) {
    if (cudaStreamSynchronize(nullptr) != cudaSuccess) return fail(SXEN_CUDA_ERROR, "sxen_grad_create sync failed");
  }
  return st;
}

sxen_status sxen_grad_destroy(sxen_grad* grad) {
  if (!grad) return SXEN_OK;
  DeviceGuard guard(grad->device);
  cudaFree(grad->values);
  cudaFree(grad->coarse);
  cudaFree(grad->fixed);
  delete grad;
  return SXEN_OK;
}

sxen_status sxen_grad_clear(sxen_grad* grad, void* stream) {
  SXEN_REQUIRE(grad != nullptr, "gradient handle is null");
  DeviceGuard guard(grad->device);
  fill_u32_kernel<<<grid_for(grad->count()), 256, 0, as_stream(stream)>>>(reinterpret_cast<uint32_t*>(grad->values),
                                                                          grad->count(), kUntouchedBits);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (grad->fixed) SXEN_CUDA(cudaMemsetAsync(grad->fixed, 0, grad->count() * sizeof(long long), as_stream(stream)));
  return SXEN_OK;
}

sxen_status sxen_grad_set_reproducible(sxen_grad* grad, int32_t on) {
  SXEN_REQUIRE(grad != nullptr, "gradient handle is null");
  DeviceGuard guard(grad->device);
  if (on && !grad->fixed) {
    SXEN_CUDA(cudaMalloc(&grad->fixed, grad->count() * sizeof(long long)));
    SXEN_CUDA(cudaDeviceSynchronize());
    return sxen_grad_clear(grad, nullptr);  // both representations start from the same (empty) state
  }
  if (!on && grad->fixed) {
    SXEN_CUDA(cudaDeviceSynchronize());
    cudaFree(grad->fixed);
    grad->fixed = nullptr;
  }
  return SXEN_OK;
}

sxen_status sxen_grad_is_reproducible(const sxen_grad* grad, int32_t* out) {
  SXEN_REQUIRE(grad != nullptr && out != nullptr, "null argument");
  *out = grad->fixed != nullptr ? 1 : 0;
  return SXEN_OK;
}

sxen_status sxen_grad_fixed_dev(sxen_grad* grad, int64_t** out_dev, size_t* count) {
  SXEN_REQUIRE(grad != nullptr && out_dev != nullptr, "null argument");
  *out_dev = reinterpret_cast<int64_t*>(grad->fixed);
  if (count) *count = grad->fixed ? grad->count() : 0;
  return SXEN_OK;
}

sxen_status sxen_grad_values_dev(sxen_grad* grad, float** out_dev, size_t* count) {
  SXEN_REQUIRE(grad != nullptr && out_dev != nullptr, "null argument");
  *out_dev = grad->values;
  if (count) *count = grad->count();
  return SXEN_OK;
}

sxen_status sxen_grad_download(const sxen_grad* grad, int32_t level, float* values_host, uint8_t* touched_host) {
  SXEN_REQUIRE(grad != nullptr && values_host != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < grad->levels, "gradient: level out of range");
  DeviceGuard guard(grad->device);
  const size_t per = static_cast<size_t>(grad->table_size) * static_cast<size_t>(grad->features);
  SXEN_CUDA(cudaMemcpy(values_host, grad->values + static_cast<size_t>(level) * per, per * sizeof(float),
                       cudaMemcpyDeviceToHost));
  for (size_t r = 0; r < grad->table_size; ++r) {
    uint32_t bits;
    std::memcpy(&bits, values_host + r * grad->features, sizeof(bits));
    const bool untouched = bits == kUntouchedBits;
    if (touched_host) touched_host[r] = untouched ? 0 : 1;
    if (untouched)
      for (int f = 0; f < grad->features; ++f) values_host[r * grad->features + f] = 0.0f;
  }
  if (grad->fixed) {  // reproducible mode: report the exact sums (rounded once to float), not the fp32-atomic ones
    std::vector<long long> q(per);
    SXEN_CUDA(cudaMemcpy(q.data(), grad->fixed + static_cast<size_t>(level) * per, per * sizeof(long long), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < per; ++i) values_host[i] = static_cast<float>(static_cast<double>(q[i]) * 0x1p-52);
  }
  return SXEN_OK;
}

sxen_status sxen_grad_download_f64(const sxen_grad* grad, int32_t level, double* values_host) {
  SXEN_REQUIRE(grad != nullptr && values_host != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < grad->levels, "gradient: level out of range");
  DeviceGuard guard(grad->device);
  const size_t per = static_cast<size_t>(grad->table_size) * static_cast<size_t>(grad->features);
  if (grad->fixed) {
    std::vector<long long> q(per);
    SXEN_CUDA(cudaMemcpy(q.data(), grad->fixed + static_cast<size_t>(level) * per, per * sizeof(long long), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < per; ++i) values_host[i] = static_cast<double>(q[i]) * 0x1p-52;  // exact: |q| < 2^53 in range
    return SXEN_OK;
  }
  std::vector<float> v(per);
  if (sxen_status st = sxen_grad_download(grad, level, v.data(), nullptr)) return st;
  for (size_t i = 0; i < per; ++i) values_host[i] = static_cast<double>(v[i]);
  return SXEN_OK;
}

sxen_status sxen_grad_upload(sxen_grad* grad, int32_t level, const float* values_host, const uint8_t* touched_host) {
  SXEN_REQUIRE(grad != nullptr && values_host != nullptr && touched_host != nullptr, "null argument");
  SXEN_REQUIRE(level >= 0 && level < grad->levels, "gradient: level out of range");
  DeviceGuard guard(grad->device);
  const size_t per = static_cast<size_t>(grad->table_size) * static_cast<size_t>(grad->features);
  std::vector<float> tmp(values_host, values_host + per);
  const float neg_zero = -0.0f;
  for (size_t r = 0; r < grad->table_size; ++r) {
    for (int f = 0; f < grad->features; ++f) {
      float& v = tmp[r * grad->features + f];
      v = touched_host[r] ? (v + 0.0f) : neg_zero;  // a touched row never carries -0.0f
    }
  }
  SXEN_CUDA(cudaMemcpy(grad->values + static_cast<size_t>(level) * per, tmp.data(), per * sizeof(float),
                       cudaMemcpyHostToDevice));
  if (grad->fixed) {
    std::vector<long long> q(per);
    for (size_t i = 0; i < per; ++i)
      q[i] = touched_host[i / grad->features] ? std::llrint(static_cast<double>(values_host[i]) * 0x1p52) : 0;
    SXEN_CUDA(cudaMemcpy(grad->fixed + static_cast<size_t>(level) * per, q.data(), per * sizeof(long long), cudaMemcpyHostToDevice));
  }
  return SXEN_OK;
}

sxen_status sxen_grad_touched_total(const sxen_grad* grad, uint64_t* out) {
  SXEN_REQUIRE(grad != nullptr && out != nullptr, "null argument");
  DeviceGuard guard(grad->device);
  unsigned long long* d = nullptr;
  SXEN_CUDA(cudaMalloc(&d, sizeof(unsigned long long)));
  cudaMemset(d, 0, sizeof(unsigned long long));
  const size_t rows = static_cast<size_t>(grad->levels) * grad->table_size;
  grad_touched_kernel<<<grid_for(rows), 256>>>(grad->values, rows, grad->features, d);
  count_launch();
  unsigned long long h = 0;
  const cudaError_t err = cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
  cudaFree(d);
  SXEN_CUDA(err);
  *out = h;
  return SXEN_OK;
}

sxen_status sxen_grad_merge(sxen_grad* dst, const sxen_grad* src, void* stream) {
  SXEN_REQUIRE(dst != nullptr && src != nullptr, "null argument");
  // src/encoding.cpp:123-125
  SXEN_REQUIRE(dst->levels == src->levels && dst->features == src->features && dst->table_size == src->table_size &&
                   dst->device == src->device,
               "EncoderGradient::merge: shape mismatch");
  DeviceGuard guard(dst->device);
  const size_t rows = static_cast<size_t>(dst->levels) * dst->table_size;
  SXEN_REQUIRE((dst->fixed != nullptr) == (src->fixed != nullptr), "EncoderGradient::merge: one accumulator is in reproducible mode, the other is not");
  grad_merge_kernel<<<grid_for(rows), 256, 0, as_stream(stream)>>>(dst->values, src->values, rows, dst->features);
  SXEN_CUDA(cudaGetLastError());
  count_launch();
  if (dst->fixed) {
    add_i64_kernel<<<grid_for(dst->count()), 256, 0, as_stream(stream)>>>(dst->fixed, src->fixed, dst->count());
    SXEN_CUDA(cudaGetLastError());
    count_launch();
  }
  return SXEN_OK;
}

}  // extern "C"
