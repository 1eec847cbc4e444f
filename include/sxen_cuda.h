/*
 * sxen_cuda.h -- C ABI of the B200-native simplex multiresolution hash encoder (libsxen_b200.so).
 *
 * This is the drop-in boundary for ONE hot path of the reference (arXiv 2311.15439 "sxen"):
 * HashEncoder::encode / encode_backward, the tiny MLP head, the Adam updates and the train step
 * that strings them together.  The reference has no FFI layer of its own; each entry point below is
 * the BATCHED form of the reference C++ call it replaces, cited as file:line under
 * /root/reference/proj/.  Plain pointers and sizes only -- no C++ or torch types.
 *
 * Conventions
 *  - Every function returns sxen_status and never throws.  On failure sxen_last_error() (thread
 *    local) holds the message.  The status values map 1:1 onto the exception types the reference
 *    throws (include/sxen/errors.hpp:8-15; std::invalid_argument / std::logic_error).
 *  - Handles are opaque and own device memory on ONE device.  Pointer arguments named *_dev are
 *    caller-owned device memory, never retained after the call's stream work completes; *_host are
 *    caller-owned host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = the legacy default stream).  Device-pointer
 *    entry points are asynchronous and stream-ordered; *_host entry points are synchronous.
 *  - Layouts are the reference's: coords N x dim row-major; features / upstream N x (L*F) with
 *    element [s*L*F + l*F + f] (src/encoding.cpp:311-313); tables L x (T*F), row-major [row][f]
 *    (include/sxen/encoding.hpp:107,145).
 *  - There is no CPU fallback: every entry point that computes requires an sm_100 device and
 *    fails with SXEN_CUDA_ERROR otherwise.
 */
#ifndef SXEN_CUDA_H
#define SXEN_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(_WIN32)
#define SXEN_API __declspec(dllexport)
#else
#define SXEN_API __attribute__((visibility("default")))
#endif

#define SXEN_MAX_DIM 8        /* include/sxen/lattice.hpp:12  kMaxDim */
#define SXEN_MAX_FEATURES 64  /* src/encoding.cpp:14           kMaxFeatures */
#define SXEN_MAX_RESOLUTION (1u << 26) /* src/encoding.cpp:15  kMaxResolution */

typedef enum sxen_status {
  SXEN_OK = 0,
  SXEN_INVALID_ARGUMENT = 1, /* std::invalid_argument (src/encoding.cpp:28-58,183-194,297-325) */
  SXEN_LOGIC_ERROR = 2,      /* std::logic_error      (src/mlp.cpp:165-167) */
  SXEN_TRAINING_ERROR = 3,   /* sxen::TrainingError   (src/trainer.cpp:121-123, src/optimizer.cpp:35-37,73-76) */
  SXEN_CUDA_ERROR = 4,       /* no reference analogue: device/runtime failure */
  SXEN_IO_ERROR = 5,         /* sxen::IoError         (include/sxen/errors.hpp:8-10) */
  SXEN_NCCL_ERROR = 6        /* no reference analogue: the gradient exchange between ranks failed (sxen_comm_*) */
} sxen_status;

typedef enum sxen_backend { SXEN_BACKEND_SIMPLEX = 0, SXEN_BACKEND_GRID = 1 } sxen_backend;           /* include/sxen/encoding.hpp:12 */
typedef enum sxen_level_scale { SXEN_SCALE_RAW = 0, SXEN_SCALE_EQUAL_MEMORY = 1 } sxen_level_scale;   /* include/sxen/encoding.hpp:13 */
typedef enum sxen_coord_type { SXEN_COORD_F64 = 0, SXEN_COORD_F32 = 1,
                               SXEN_ELEM_I64 = 2 /* sxen_comm_allreduce only: the fixed-point accumulator words */ } sxen_coord_type;

/* sxen::EncoderConfig, field for field (include/sxen/encoding.hpp:18-33). */
typedef struct sxen_encoder_config {
  int32_t dim;             /* n, input dimension, [1, 8]            default 2 */
  int32_t levels;          /* L >= 1                                default 8 */
  uint32_t table_size;     /* T entries per level, power of two     default 1<<16 */
  int32_t features;        /* F in [1, 64]                          default 2 */
  int32_t base_resolution; /* coarsest lattice resolution >= 1      default 16 */
  double growth;           /* per-level growth, finite, > 1         default 2.0 */
  int32_t backend;         /* sxen_backend                          default simplex */
  int32_t level_scale;     /* sxen_level_scale                      default raw */
} sxen_encoder_config;

/* sxen::MlpConfig (include/sxen/mlp.hpp:11-25); hidden activation is ReLU, output identity. */
typedef struct sxen_mlp_config {
  int32_t input_width;   /* default 32 */
  int32_t hidden_width;  /* default 64 */
  int32_t hidden_layers; /* default 2 */
  int32_t output_width;  /* default 3 */
} sxen_mlp_config;

/* sxen::AdamConfig (include/sxen/optimizer.hpp:13-18). */
typedef struct sxen_adam_config {
  double lr;      /* default 1e-3 */
  double beta1;   /* default 0.9 */
  double beta2;   /* default 0.99 */
  double epsilon; /* default 1e-15 */
} sxen_adam_config;

/* sxen::LookupCounters (include/sxen/encoding.hpp:44-47). */
typedef struct sxen_lookup_counters {
  uint64_t touched_vertices;
  uint64_t out_of_bounds;
} sxen_lookup_counters;

/* Launch-shape knobs of the encode kernels (no reference analogue; 0 = library default). */
typedef struct sxen_tuning {
  int32_t levels_per_thread; /* 1,2,4,16: levels one thread walks; 0 (default) = chosen with the launch shape below */
  int32_t block_threads;     /* CTA size, multiple of 32 */
  int32_t level_major;       /* 0: consecutive threads walk one sample's level groups (coalesced rows);
                                1: grid.y = level group, all samples of a group before the next (L2-resident tables);
                                -1 (default): chosen from the table footprint (level-major once tables exceed 96 MiB,
                                i.e. tables + accumulator no longer fit L2 side by side) */
  int32_t exact_blend;       /* 1: fp64 chain-order blend, features bit-identical to the reference; 0: fp32 FMA blend */
  int32_t warp_aggregate;    /* backward: merge equal rows inside a warp before the atomic on levels whose
                                lattice has at most this many vertices (0 = off) */
  int32_t merge_pairs;       /* backward, F == 2: chain vertices whose rows share a 16-byte slot (idx, idx^1) take one
                                red.v4 instead of two red.v2.  1 = on (default), -1 = off, 0 = library default */
  int32_t cache_hints;       /* F == 2 kernels: L2 eviction policy of the table gathers + 4 * policy of the gradient reds
                                (0 none, 1 evict_last, 2 evict_first, 3 evict_unchanged).  -1 = chosen from the
                                footprint; 0 = plain accesses */
  int32_t coarse_replicas;   /* backward: levels with at most 2^16 lattice vertices accumulate into replicated dense
                                arrays that the same call folds into the hashed rows (relieves the per-address
                                serialisation of the L2 atomic unit).  0 = library default: on for launches of at least
                                2^16 samples (below, the fold costs more than the contention it removes), 1 = always,
                                -1 = off */
  int32_t level_chunk;       /* sample-major launches: the grid walks the levels in contiguous ranges of this many levels
                                (blockIdx.y = range; sample-major inside a range), so only one range's table and accumulator
                                rows are live in L2 at a time.  Used when it is levels_per_thread * 2^k.  0 = library
                                default (8 for the fused launch at dim 3 when tables + accumulator only just fit L2:
                                profiles/r2_l2_window_n3.log), -1 = off */
} sxen_tuning;

typedef struct sxen_encoder sxen_encoder;   /* sxen::HashEncoder     (include/sxen/encoding.hpp:92-148) */
typedef struct sxen_grad sxen_grad;         /* sxen::EncoderGradient (include/sxen/encoding.hpp:53-86) */
typedef struct sxen_mlp sxen_mlp;           /* sxen::Mlp + MlpGradient + batched MlpWorkspace (include/sxen/mlp.hpp) */
typedef struct sxen_sparse_adam sxen_sparse_adam; /* sxen::SparseAdamState (include/sxen/optimizer.hpp:42-59) */
typedef struct sxen_adam sxen_adam;         /* sxen::AdamState       (include/sxen/optimizer.hpp:21-37) */

/* ------------------------------------------------------------------ library */
SXEN_API const char* sxen_last_error(void);
SXEN_API const char* sxen_version(void);
/* Number of visible CUDA devices with compute capability 10.x (0 when none / no driver). */
SXEN_API int32_t sxen_device_count(void);
/* Kernels launched by this library since load (all handles, all streams); bench.py's gpu_launches. */
SXEN_API uint64_t sxen_launch_count(void);

/* Pinned host memory for callers of the *_host entry points (pageable memory works too, but copies then serialise). */
SXEN_API sxen_status sxen_host_alloc(size_t bytes, void** out);
SXEN_API sxen_status sxen_host_free(void* ptr);
/* Device buffers for a host that does not link the CUDA runtime itself (the C++ trainer/tasks mirror,
 * include/sxen_b200_train.hpp): plain cudaMalloc / cudaFree / cudaMemcpyAsync + stream sync / cudaMemsetAsync. */
SXEN_API sxen_status sxen_device_alloc(int32_t device, size_t bytes, void** out_dev);
SXEN_API sxen_status sxen_device_free(int32_t device, void* ptr_dev);
SXEN_API sxen_status sxen_device_upload(int32_t device, void* dst_dev, const void* src_host, size_t bytes, void* stream);
SXEN_API sxen_status sxen_device_download(int32_t device, void* dst_host, const void* src_dev, size_t bytes, void* stream);
SXEN_API sxen_status sxen_device_zero(int32_t device, void* dst_dev, size_t bytes, void* stream);

/* ------------------------------------------------------------------ rng (include/sxen/rng.hpp:9-54), host-side */
SXEN_API uint64_t sxen_mix64(uint64_t z);
SXEN_API uint64_t sxen_hash_combine(uint64_t a, uint64_t b);
/* Fills out_dev[i] = lo + (hi-lo)*next_double() for draws first_counter+i (1-based) of
 * CounterRng(seed) (has_stream=0) or CounterRng(seed, stream_id); as f64 or f32 (rounded from the f64 value). */
SXEN_API sxen_status sxen_rng_fill_dev(uint64_t seed, int32_t has_stream, uint64_t stream_id, uint64_t first_counter,
                                       double lo, double hi, void* out_dev, size_t count, sxen_coord_type type,
                                       void* stream);

/* ------------------------------------------------------------------ config (src/encoding.cpp:28-82) */
SXEN_API sxen_status sxen_encoder_config_default(sxen_encoder_config* cfg);
SXEN_API sxen_status sxen_encoder_validate(const sxen_encoder_config* cfg);                       /* EncoderConfig::validate */
SXEN_API sxen_status sxen_level_resolution(const sxen_encoder_config* cfg, int32_t level, uint32_t* out); /* level_resolution */
SXEN_API sxen_status sxen_equal_memory_multiplier(int32_t dim, double* out);                      /* equal_memory_multiplier */
/* out[0]=F_n (skew), out[1]=G_n (unskew), out[2]=S_n (scale): SkewConstants::make (src/lattice.cpp:21-30) */
SXEN_API sxen_status sxen_skew_constants(int32_t dim, double out[3]);
/* hash_coords (include/sxen/hashing.hpp:23-29), host-side helper */
SXEN_API sxen_status sxen_hash_coords(const int64_t* coords, int32_t dim, uint32_t* out);

/* ------------------------------------------------------------------ encoder (src/encoding.cpp:157-335) */
/* HashEncoder::HashEncoder: validates, computes the per-level resolutions, allocates zeroed tables on `device`. */
SXEN_API sxen_status sxen_encoder_create(const sxen_encoder_config* cfg, int32_t device, sxen_encoder** out);
SXEN_API sxen_status sxen_encoder_destroy(sxen_encoder* enc);
SXEN_API sxen_status sxen_encoder_get_config(const sxen_encoder* enc, sxen_encoder_config* out);
SXEN_API sxen_status sxen_encoder_resolution(const sxen_encoder* enc, int32_t level, uint32_t* out); /* HashEncoder::resolution */
SXEN_API sxen_status sxen_encoder_parameter_count(const sxen_encoder* enc, uint64_t* out);           /* parameter_count */
SXEN_API sxen_status sxen_encoder_set_tuning(sxen_encoder* enc, const sxen_tuning* tuning);
SXEN_API sxen_status sxen_encoder_get_tuning(const sxen_encoder* enc, sxen_tuning* out);
/* HashEncoder::init_tables (src/encoding.cpp:169-176): counter RNG evaluated on the device, bit-identical. */
SXEN_API sxen_status sxen_encoder_init_tables(sxen_encoder* enc, uint64_t seed, void* stream);
/* HashEncoder::table(level) (include/sxen/encoding.hpp:107): T*F floats. */
SXEN_API sxen_status sxen_encoder_upload_table(sxen_encoder* enc, int32_t level, const float* src_host);
SXEN_API sxen_status sxen_encoder_download_table(const sxen_encoder* enc, int32_t level, float* dst_host);
/* Device pointer of level 0; levels are contiguous, level l starts at ptr + l*T*F. */
SXEN_API sxen_status sxen_encoder_tables_dev(sxen_encoder* enc, float** out_dev);

/* HashEncoder::encode, batched (src/encoding.cpp:295-315).  x_dev: N x dim (type), out_dev: N x L*F f32. */
SXEN_API sxen_status sxen_encoder_encode(sxen_encoder* enc, const void* x_dev, sxen_coord_type type, size_t n_samples,
                                         float* out_dev, void* stream);
/* Parity probe: the per-(sample, level) vertex chain the encode kernels use.
 * idx_dev: N x L x V u32, w_dev: N x L x V f64, V = dim+1 (simplex) or 2^dim (grid). */
SXEN_API sxen_status sxen_encoder_encode_debug(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                               size_t n_samples, uint32_t* idx_dev, double* w_dev, void* stream);
/* HashEncoder::encode_backward, batched (src/encoding.cpp:317-335).  upstream_dev: N x L*F f32. */
SXEN_API sxen_status sxen_encoder_encode_backward(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                  const float* upstream_dev, size_t n_samples, sxen_grad* grad,
                                                  void* stream);
/* encode + encode_backward of the same batch in ONE kernel (one lattice walk per (sample, level));
 * the run_chunk pair of src/trainer.cpp:31,47 when upstream does not depend on this batch's features. */
SXEN_API sxen_status sxen_encoder_encode_forward_backward(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                          const float* upstream_dev, size_t n_samples, float* out_dev,
                                                          sxen_grad* grad, void* stream);
/* The same two calls restricted to encoder levels [first_level, first_level + level_count): only that slice of every
 * upstream / feature row and of the accumulator is read and written.  A batch-sharded multi-GPU step walks the levels in
 * chunks and all-reduces each chunk's slice of the accumulator (contiguous: level l starts at values + l*T*F) on a
 * second stream while the next chunk computes. */
SXEN_API sxen_status sxen_encoder_encode_backward_levels(sxen_encoder* enc, const void* x_dev, sxen_coord_type type,
                                                         const float* upstream_dev, size_t n_samples, sxen_grad* grad,
                                                         int32_t first_level, int32_t level_count, void* stream);
SXEN_API sxen_status sxen_encoder_encode_forward_backward_levels(sxen_encoder* enc, const void* x_dev,
                                                                 sxen_coord_type type, const float* upstream_dev,
                                                                 size_t n_samples, float* out_dev, sxen_grad* grad,
                                                                 int32_t first_level, int32_t level_count, void* stream);
/* Synchronises `stream` and reports what the reference would have thrown for this encoder's launches since the
 * last check: SXEN_INVALID_ARGUMENT with the first sample whose coordinate is NaN or outside [0,1]
 * (check_input, src/encoding.cpp:183-194).  Such samples write zero features and add no gradient. */
SXEN_API sxen_status sxen_encoder_check(sxen_encoder* enc, void* stream);
/* HashEncoder::counters / reset_counters (include/sxen/encoding.hpp:122-128). Synchronises the device. */
SXEN_API sxen_status sxen_encoder_counters(sxen_encoder* enc, sxen_lookup_counters* out);
SXEN_API sxen_status sxen_encoder_reset_counters(sxen_encoder* enc);

/* Host-buffer forms: the call a user of the reference makes, batched.  x_host: N x dim doubles (the reference's
 * own coordinate type), copied to the device through pinned staging, synchronous, errors reported directly. */
SXEN_API sxen_status sxen_encoder_encode_host(sxen_encoder* enc, const double* x_host, size_t n_samples, float* out_host);
SXEN_API sxen_status sxen_encoder_encode_backward_host(sxen_encoder* enc, const double* x_host,
                                                       const double* upstream_host, size_t n_samples, sxen_grad* grad);
/* encode + encode_backward of one host batch in a single pipelined pass: chunks are copied in, run through the fused
 * kernel and copied out on rotating streams so H2D, compute and D2H overlap.  upstream_host is N x L*F of
 * `upstream_type` (f64 = the reference's type, narrowed on the device; f32 = half the bytes over PCIe). */
SXEN_API sxen_status sxen_encoder_encode_forward_backward_host(sxen_encoder* enc, const double* x_host,
                                                               const void* upstream_host, sxen_coord_type upstream_type,
                                                               size_t n_samples, float* out_host, sxen_grad* grad);

/* ------------------------------------------------------------------ gradient accumulator (src/encoding.cpp:84-137) */
/* EncoderGradient(levels, table_size, features): dense f32 device buffer L x T x F.  "Touched" is carried in-band:
 * an untouched row holds -0.0f in feature 0; any accumulated contribution (zeros are added as +0.0f) clears it. */
SXEN_API sxen_status sxen_grad_create(const sxen_encoder* enc, sxen_grad** out);
SXEN_API sxen_status sxen_grad_destroy(sxen_grad* grad);
SXEN_API sxen_status sxen_grad_clear(sxen_grad* grad, void* stream);                 /* EncoderGradient::clear */
SXEN_API sxen_status sxen_grad_values_dev(sxen_grad* grad, float** out_dev, size_t* count); /* for all-reduce */
/* EncoderGradient::slice + touched for one level: values_host T*F floats (-0.0 reported as 0), touched_host T bytes. */
SXEN_API sxen_status sxen_grad_download(const sxen_grad* grad, int32_t level, float* values_host, uint8_t* touched_host);
/* Inverse of sxen_grad_download: overwrites one level (rows with touched_host[r]==0 become untouched). */
SXEN_API sxen_status sxen_grad_upload(sxen_grad* grad, int32_t level, const float* values_host, const uint8_t* touched_host);
SXEN_API sxen_status sxen_grad_touched_total(const sxen_grad* grad, uint64_t* out); /* EncoderGradient::touched_total */
/* Reproducible accumulation (opt-in; on != 0 allocates a second L x T x F buffer of 64-bit words).  The reference's gradient
 * sums are bit-reproducible for a fixed (seed, threads): per-worker fp64 accumulators merged in worker order
 * (src/trainer.cpp:125-128, tests/test_neural.cpp:370-408).  fp32 atomics are not: the order they land in changes the low
 * bits, and Adam (epsilon 1e-15) turns low bits of near-zero gradients into lr-sized steps.  In this mode every backward
 * ALSO adds each contribution -- the fp64 product w * upstream, as src/encoding.cpp:116 -- as 64-bit fixed point in units of
 * 2^-52 with integer atomics (associative: order-free), and the optimizers, sxen_grad_download* and sxen_grad_merge use those
 * sums.  The fp32 accumulator keeps carrying "touched" and the non-finite check; a sum of magnitude >= 2^10 is outside the
 * fixed-point range and is reported by the optimizer like a non-finite gradient.  Costs two more L2 atomics per row. */
SXEN_API sxen_status sxen_grad_set_reproducible(sxen_grad* grad, int32_t on);
SXEN_API sxen_status sxen_grad_is_reproducible(const sxen_grad* grad, int32_t* out);
/* the fixed-point words (NULL / 0 when the mode is off): for an all-reduce of type SXEN_ELEM_I64 next to the values */
SXEN_API sxen_status sxen_grad_fixed_dev(sxen_grad* grad, int64_t** out_dev, size_t* count);
/* EncoderGradient::slice as the reference's doubles: the exact fixed-point sums in reproducible mode, else the f32 values. */
SXEN_API sxen_status sxen_grad_download_f64(const sxen_grad* grad, int32_t level, double* values_host);
/* EncoderGradient::merge (src/encoding.cpp:122-131): dst += src, touched = union. */
SXEN_API sxen_status sxen_grad_merge(sxen_grad* dst, const sxen_grad* src, void* stream);

/* ------------------------------------------------------------------ optimizers (src/optimizer.cpp) */
SXEN_API sxen_status sxen_adam_config_default(sxen_adam_config* cfg);
/* SparseAdamState: fp64 moments L x T x F, global step counter. */
SXEN_API sxen_status sxen_sparse_adam_create(const sxen_encoder* enc, sxen_sparse_adam** out);
SXEN_API sxen_status sxen_sparse_adam_destroy(sxen_sparse_adam* opt);
SXEN_API sxen_status sxen_sparse_adam_step_count(const sxen_sparse_adam* opt, int64_t* out);
/* SparseAdamState::step (src/optimizer.cpp:54-84): updates only touched rows, fp64 math without FMA contraction.
 * clear_grad != 0 resets the accumulator in the same pass.  Non-finite gradients set SXEN_TRAINING_ERROR, reported
 * by sxen_sparse_adam_check. */
SXEN_API sxen_status sxen_sparse_adam_step(sxen_sparse_adam* opt, sxen_encoder* enc, sxen_grad* grad,
                                           const sxen_adam_config* cfg, int32_t clear_grad, void* stream);
SXEN_API sxen_status sxen_sparse_adam_check(sxen_sparse_adam* opt, void* stream);
/* Moments of one level for inspection: m_host, v_host T*F doubles. */
SXEN_API sxen_status sxen_sparse_adam_download(const sxen_sparse_adam* opt, int32_t level, double* m_host, double* v_host);

/* AdamState over a dense f32 parameter vector (src/optimizer.cpp:25-41); gradients f64 or f32 (grad_type). */
SXEN_API sxen_status sxen_adam_create(size_t size, int32_t device, sxen_adam** out);
SXEN_API sxen_status sxen_adam_destroy(sxen_adam* opt);
SXEN_API sxen_status sxen_adam_step_count(const sxen_adam* opt, int64_t* out);
SXEN_API sxen_status sxen_adam_step(sxen_adam* opt, float* params_dev, const void* grads_dev, sxen_coord_type grad_type,
                                    size_t size, const sxen_adam_config* cfg, void* stream);
SXEN_API sxen_status sxen_adam_check(sxen_adam* opt, void* stream);

/* ------------------------------------------------------------------ MLP head (src/mlp.cpp) */
SXEN_API sxen_status sxen_mlp_config_default(sxen_mlp_config* cfg);
SXEN_API sxen_status sxen_mlp_validate(const sxen_mlp_config* cfg);                       /* MlpConfig::validate */
/* Mlp::Mlp: validates, allocates zeroed f32 parameters (per layer: weights out x in row-major, then biases --
 * src/mlp.cpp:19-32) and the fp64 MlpGradient on `device`. */
SXEN_API sxen_status sxen_mlp_create(const sxen_mlp_config* cfg, int32_t device, sxen_mlp** out);
SXEN_API sxen_status sxen_mlp_destroy(sxen_mlp* mlp);
SXEN_API sxen_status sxen_mlp_get_config(const sxen_mlp* mlp, sxen_mlp_config* out);
SXEN_API sxen_status sxen_mlp_parameter_count(const sxen_mlp* mlp, uint64_t* out);         /* Mlp::parameter_count */
SXEN_API sxen_status sxen_mlp_init_params(sxen_mlp* mlp, uint64_t seed, void* stream);     /* Mlp::init_params, bit-identical */
SXEN_API sxen_status sxen_mlp_upload_params(sxen_mlp* mlp, const float* src_host);         /* Mlp::parameters() */
SXEN_API sxen_status sxen_mlp_download_params(const sxen_mlp* mlp, float* dst_host);
SXEN_API sxen_status sxen_mlp_params_dev(sxen_mlp* mlp, float** out_dev);
SXEN_API sxen_status sxen_mlp_grads_dev(sxen_mlp* mlp, double** out_dev);                  /* MlpGradient::values(), for all-reduce */
SXEN_API sxen_status sxen_mlp_grad_clear(sxen_mlp* mlp, void* stream);                     /* MlpGradient::clear */
/* Reproducible MlpGradient (exact head): the thread blocks' partial sums meet in 64-bit fixed point (units of 2^-52,
 * integer atomics) instead of fp64 atomics, so the gradient does not depend on block scheduling -- the counterpart of the
 * reference's fixed worker-order merge (src/mlp.cpp:83-88, src/trainer.cpp:125-128). */
SXEN_API sxen_status sxen_mlp_set_reproducible(sxen_mlp* mlp, int32_t on);
SXEN_API sxen_status sxen_mlp_grad_download(const sxen_mlp* mlp, double* dst_host);
/* Mlp::forward, batched (src/mlp.cpp:137-162). input_dev: N x input_width f32; out_dev (may be NULL): N x output_width.
 * The activations stay in the handle (the batched MlpWorkspace) for the matching backward. */
SXEN_API sxen_status sxen_mlp_forward(sxen_mlp* mlp, const float* input_dev, size_t n_samples, float* out_dev, void* stream);
/* Mlp::backward, batched (src/mlp.cpp:164-202). upstream_dev: N x output_width f64; parameter gradients accumulate into
 * the handle's MlpGradient; d(loss)/d(input) is written as f32 (input_grad_dev) and/or f64 (input_grad_f64_dev), either
 * may be NULL.  SXEN_LOGIC_ERROR if no forward populated the workspace. */
SXEN_API sxen_status sxen_mlp_backward(sxen_mlp* mlp, const double* upstream_dev, size_t n_samples, float* input_grad_dev,
                                       double* input_grad_f64_dev, void* stream);
/* The same two calls with the reference's HOST spans (include/sxen/mlp.hpp:94-99; MlpWorkspace::output() and
 * ::input_grad() are the out arguments): input_host N x input_width f32 -> out_host N x output_width f32; upstream_host
 * N x output_width f64 -> input_grad_host N x input_width f64 (may be NULL).  Synchronous; same status codes. */
SXEN_API sxen_status sxen_mlp_forward_host(sxen_mlp* mlp, const float* input_host, size_t n_samples, float* out_host);
SXEN_API sxen_status sxen_mlp_backward_host(sxen_mlp* mlp, const double* upstream_host, size_t n_samples,
                                            double* input_grad_host);
/* Arithmetic of the head.  EXACT (default): fp64 accumulation in the reference's order, any shape, bit-identical outputs.
 * TENSOR_*: the fused tcgen05 kernel for the {16|32} -> 64 -> 64 -> {<=3} head; BF16X3 = split-bf16 operands (three MMAs per
 * product: predictions within 1.5e-5 of their largest magnitude, measured 6e-6 .. 1.1e-5), BF16X4 = the same with the fourth
 * (lo x lo) product: within 1e-5 (measured 4.6e-6 .. 7.3e-6) at +15 % kernel time, BF16 = single bf16 product (~4e-3). */
typedef enum sxen_mlp_precision {
  SXEN_MLP_EXACT = 0, SXEN_MLP_TENSOR_BF16X3 = 1, SXEN_MLP_TENSOR_BF16 = 2, SXEN_MLP_TENSOR_BF16X4 = 3
} sxen_mlp_precision;
SXEN_API sxen_status sxen_mlp_set_precision(sxen_mlp* mlp, int32_t precision);
SXEN_API sxen_status sxen_mlp_get_precision(const sxen_mlp* mlp, int32_t* out);
/* Mlp::forward + run_chunk's MSE/upstream + Mlp::backward of one batch (src/trainer.cpp:36-46) in one call: parameter
 * gradients accumulate into the handle, d(loss)/d(input) goes to input_grad_dev (N x input_width f32), the sum of the
 * per-sample losses is ADDED to *loss_sum_dev (may be NULL), predictions go to pred_dev (may be NULL). */
SXEN_API sxen_status sxen_mlp_forward_backward(sxen_mlp* mlp, const float* input_dev, const void* targets_dev,
                                               sxen_coord_type target_type, size_t n_samples, size_t global_batch,
                                               float* pred_dev, float* input_grad_dev, double* loss_sum_dev, void* stream);
/* The workspace of the last forward: [N x act_width] f32 rows, slot 0 = input, the output starts at output_offset. */
SXEN_API sxen_status sxen_mlp_activations_dev(sxen_mlp* mlp, float** out_dev, size_t* act_width, size_t* output_offset);
/* run_chunk's loss (src/trainer.cpp:26-44): e = pred - target, sample_loss = sum e^2, upstream = 2e / (global_batch*out_w).
 * pred_dev rows are pred_stride floats apart; targets N x out_w (f64 or f32); loss_sum_dev (may be NULL) receives the
 * deterministic sum of sample_loss. */
SXEN_API sxen_status sxen_mse_loss(const float* pred_dev, size_t pred_stride, const void* targets_dev,
                                   sxen_coord_type target_type, int32_t out_w, size_t n_samples, size_t global_batch,
                                   double* upstream_dev, double* sample_loss_dev, double* loss_sum_dev, void* stream);

/* ------------------------------------------------------------------ training step (src/trainer.cpp:94-136) */
typedef struct sxen_trainer sxen_trainer;
/* Binds an encoder and an MLP (not owned) with a gradient accumulator, SparseAdamState and AdamState (owned). */
SXEN_API sxen_status sxen_trainer_create(sxen_encoder* enc, sxen_mlp* mlp, sxen_trainer** out);
/* TrainConfig::aux_dims (include/sxen/trainer.hpp:18): aux_dims extra inputs per sample appended verbatim after the encoding
 * (src/trainer.cpp:32-35); the MLP's input width must be L*F + aux_dims (std::invalid_argument otherwise, :61-65).
 * sxen_trainer_set_aux names the caller-owned N x aux_dims array (f64 or f32) the NEXT accumulate / step calls read; it
 * must hold the batch those calls are given and stay valid until their stream work completes. */
SXEN_API sxen_status sxen_trainer_create_aux(sxen_encoder* enc, sxen_mlp* mlp, int32_t aux_dims, sxen_trainer** out);
SXEN_API sxen_status sxen_trainer_set_aux(sxen_trainer* trainer, const void* aux_dev, sxen_coord_type aux_type);
SXEN_API sxen_status sxen_trainer_destroy(sxen_trainer* trainer);
/* run_chunk over this rank's contiguous chunk: encode -> forward -> MSE -> backward -> encode_backward.  Table and MLP
 * gradients and the loss sum ACCUMULATE until sxen_trainer_update.  global_batch is the B of upstream = 2e/(B*out_w). */
SXEN_API sxen_status sxen_trainer_accumulate(sxen_trainer* trainer, const void* coords_dev, sxen_coord_type coord_type,
                                             const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                             size_t global_batch, void* stream);
/* Buffers a multi-GPU host all-reduces (SUM) between accumulate and update: the table-gradient accumulator, the MLP
 * gradient (sxen_mlp_grads_dev) and the loss sum. */
/* sxen_trainer_accumulate in two halves, for a multi-GPU host that overlaps the gradient exchange with the backward:
 * _head runs encode -> Mlp forward -> loss/upstream -> Mlp backward and leaves d(loss)/d(encoding) in the workspace;
 * _tables runs encode_backward for levels [first_level, first_level + level_count) of the same batch (call it once per
 * level chunk, all-reducing each chunk's slice of the accumulator while the next one runs).
 * _tables without a matching _head (same n_samples) is SXEN_LOGIC_ERROR. */
SXEN_API sxen_status sxen_trainer_accumulate_head(sxen_trainer* trainer, const void* coords_dev, sxen_coord_type coord_type,
                                                  const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                                  size_t global_batch, void* stream);
SXEN_API sxen_status sxen_trainer_accumulate_tables(sxen_trainer* trainer, const void* coords_dev,
                                                    sxen_coord_type coord_type, size_t n_samples, int32_t first_level,
                                                    int32_t level_count, void* stream);
SXEN_API sxen_status sxen_trainer_table_grad(sxen_trainer* trainer, sxen_grad** out);
SXEN_API sxen_status sxen_trainer_loss_dev(sxen_trainer* trainer, double** out_dev);
/* Synchronises; loss = sum / (global_batch*out_w).  SXEN_TRAINING_ERROR if non-finite (src/trainer.cpp:120-123);
 * SXEN_INVALID_ARGUMENT if a coordinate left the unit cube. */
SXEN_API sxen_status sxen_trainer_loss(sxen_trainer* trainer, size_t global_batch, double* loss_out, void* stream);
/* SparseAdamState::step + AdamState::step, then clears the accumulators for the next step (src/trainer.cpp:97-100,129-130). */
SXEN_API sxen_status sxen_trainer_update(sxen_trainer* trainer, const sxen_adam_config* table_adam,
                                         const sxen_adam_config* mlp_adam, void* stream);
SXEN_API sxen_status sxen_trainer_check(sxen_trainer* trainer, void* stream);  /* non-finite gradient -> SXEN_TRAINING_ERROR */
/* One whole single-GPU step: accumulate + loss + update + check -- one queued step (below) collected at once, so the loss and
 * the error words come back on a single stream synchronisation.  SXEN_LOGIC_ERROR while queued steps await their collect. */
SXEN_API sxen_status sxen_trainer_step(sxen_trainer* trainer, const void* coords_dev, sxen_coord_type coord_type,
                                       const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                       const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam,
                                       double* loss_out, void* stream);

/* train_field's loop body (src/trainer.cpp:94-136) WITHOUT a host round trip per step: queues the whole step
 * -- gradient pass, loss = sum/(B*out_w) into the step's slot of a device ring, both Adam updates -- and returns.  The
 * reference throws TrainingError before the optimizer steps when the loss is non-finite (:121-123); here the update
 * kernels of that and every later queued step return without writing (a device-side gate), and sxen_trainer_collect
 * reports it.  At most 4096 steps may be queued between two collects (SXEN_LOGIC_ERROR beyond).  One stream per trainer. */
SXEN_API sxen_status sxen_trainer_step_enqueue(sxen_trainer* trainer, const void* coords_dev, sxen_coord_type coord_type,
                                               const void* targets_dev, sxen_coord_type target_type, size_t n_samples,
                                               const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam,
                                               void* stream);
SXEN_API sxen_status sxen_trainer_pending(const sxen_trainer* trainer, size_t* out);
/* Synchronises the stream and returns the losses of the steps queued since the last collect, in order (*count_out of
 * them; capacity must hold them).  SXEN_TRAINING_ERROR when one was non-finite: *failed_out = its index in losses_out
 * (else -1), losses before it are valid, tables / MLP / moments are as they were before that step.  Also reports the
 * encoder's rejected-sample word and non-finite gradients like sxen_trainer_step. */
SXEN_API sxen_status sxen_trainer_collect(sxen_trainer* trainer, double* losses_out, size_t capacity, size_t* count_out,
                                          int64_t* failed_out, void* stream);

/* ------------------------------------------------------------------ multi-GPU: batch-sharded step (src/trainer.cpp:93-128) */
/* The reference fans a batch out over worker threads with private accumulators and merges them in worker order before the
 * optimizer steps (src/trainer.cpp:101-128).  Here ranks are the workers -- one per GPU, tables / MLP / moments replicated,
 * rank r takes the contiguous chunk [r*ceil(B/W), min(B, (r+1)*ceil(B/W))) of every batch (:93,107-108) -- and the merge is a
 * SUM all-reduce of the table-gradient accumulator, the MLP gradient and the loss sum.  (The in-band "touched" marker
 * survives a SUM: -0 + -0 = -0.)  A communicator is one rank's end of that exchange. */
typedef struct sxen_comm sxen_comm;
#define SXEN_COMM_ID_BYTES 128
typedef struct sxen_comm_id { char bytes[SXEN_COMM_ID_BYTES]; } sxen_comm_id; /* an ncclUniqueId */
/* NCCL transport, one process per GPU: rank 0 draws the id (ncclGetUniqueId), the host hands its bytes to the other ranks
 * (file, socket, MPI, torch.distributed ...), every rank calls sxen_comm_create (ncclCommInitRank; collective).  libnccl.so.2
 * is resolved at run time (an already loaded copy first, else the loader path, else $SXEN_NCCL_LIB). */
SXEN_API sxen_status sxen_comm_unique_id(sxen_comm_id* out);
SXEN_API sxen_status sxen_comm_create(const sxen_comm_id* id, int32_t world, int32_t rank, int32_t device, sxen_comm** out);
/* LOCAL transport, all ranks in one process with ONE HOST THREAD PER RANK (the reference's worker-thread layout): fills
 * out[0..world) with the ranks' handles; devices[r] is rank r's device (the same device may appear more than once).  The
 * exchange is this library's own kernel over peer-mapped memory: rank r sums slice r of every rank's buffer in rank order --
 * the reference's fixed merge order, so the result is bit-identical on all ranks and reproducible -- and stores it into
 * every buffer (P2P loads / stores over NVLink between devices).  Every rank must call each collective, from its own
 * thread; a rank that fails breaks the group (peers return SXEN_NCCL_ERROR instead of waiting). */
SXEN_API sxen_status sxen_comm_create_local(int32_t world, const int32_t* devices, sxen_comm** out);
SXEN_API sxen_status sxen_comm_destroy(sxen_comm* comm);
/* Marks the group broken: peers blocked in (or later entering) a collective return SXEN_NCCL_ERROR instead of waiting for a
 * rank that has failed.  LOCAL: immediate; NCCL: ncclCommAbort of this rank's communicator. */
SXEN_API sxen_status sxen_comm_abort(sxen_comm* comm);
/* any of the outputs may be NULL; kind: 0 = NCCL, 1 = LOCAL */
SXEN_API sxen_status sxen_comm_info(const sxen_comm* comm, int32_t* world, int32_t* rank, int32_t* device, int32_t* kind);
/* In-place SUM over the ranks of count elements (type: SXEN_COORD_F32 / SXEN_COORD_F64 / SXEN_ELEM_I64), stream-ordered. */
SXEN_API sxen_status sxen_comm_allreduce(sxen_comm* comm, void* buf_dev, size_t count, sxen_coord_type type, void* stream);

/* run_chunk as ONE kernel (csrc/sxen_train_fused.cu): gather warps encode the next tile straight into the tensor cores'
 * operand tile, the tcgen05 head runs, scatter warps take d loss / d encoding out of TMEM into encode_backward -- no feature or
 * gradient array in HBM.  Covers the simplex backend, F = 2, 16 levels, dim 2 or 3, head 32 -> 64 -> 64 -> <= 3 on the tensor
 * cores, no aux inputs, default accumulation.  mode 0 (default) = the three separate kernels -- measured faster: one CTA per SM
 * cannot hold enough warps to hide the lattice walk's latency next to the head's epilogue registers --,
 * 1 = the fused kernel or SXEN_INVALID_ARGUMENT, -1 = fused whenever the shapes allow.  Used by sxen_trainer_accumulate /
 * _step / _step_enqueue. */
SXEN_API sxen_status sxen_trainer_set_fused(sxen_trainer* trainer, int32_t mode);

/* Bit-reproducible training steps (opt-in): sxen_grad_set_reproducible on the trainer's accumulator, sxen_mlp_set_reproducible
 * on its MLP, and -- with the exact head -- d(loss)/d(encoding) handed to encode_backward as doubles.  Two runs of the same
 * steps then produce the same bits, on one GPU or sharded (the exchange sums the fixed-point words). */
SXEN_API sxen_status sxen_trainer_set_reproducible(sxen_trainer* trainer, int32_t on);

/* Attaches a communicator (not owned; NULL detaches) to a trainer.  The trainer's encoder, MLP and the communicator must
 * live on the same device; replicas on all ranks must have been initialised identically (same seeds). */
SXEN_API sxen_status sxen_trainer_set_comm(sxen_trainer* trainer, sxen_comm* comm);
/* The exchange between sxen_trainer_accumulate* and sxen_trainer_update, in the pieces a host overlaps with the backward:
 * _head sums the MLP gradient and the loss sum, _levels the accumulator slice of encoder levels [first_level,
 * first_level + level_count) (contiguous: level l starts at values + l*T*F).  No-ops without a communicator. */
SXEN_API sxen_status sxen_trainer_allreduce_head(sxen_trainer* trainer, void* stream);
SXEN_API sxen_status sxen_trainer_allreduce_levels(sxen_trainer* trainer, int32_t first_level, int32_t level_count, void* stream);
/* One whole batch-sharded step (train_field's loop body, src/trainer.cpp:94-136, with ranks as the workers).  coords_dev /
 * targets_dev hold the WHOLE batch of global_batch samples on every rank (the samplers are deterministic in (seed, step), so
 * nothing needs scattering); this rank runs its contiguous chunk, the exchange is overlapped with the backward -- the MLP
 * gradient and the loss go first, then encode_backward walks the levels in level_chunks ranges and each range's slice is
 * all-reduced on the trainer's second stream while the next range computes -- and every rank applies the identical update.
 * *loss_out = batch MSE before the update, the same on all ranks.  SXEN_TRAINING_ERROR (non-finite loss: nothing was updated,
 * on any rank) / SXEN_INVALID_ARGUMENT as sxen_trainer_step.  Without a communicator: a plain single-GPU step. */
SXEN_API sxen_status sxen_trainer_step_sharded(sxen_trainer* trainer, const void* coords_dev, sxen_coord_type coord_type,
                                               const void* targets_dev, sxen_coord_type target_type, size_t global_batch,
                                               const sxen_adam_config* table_adam, const sxen_adam_config* mlp_adam,
                                               int32_t level_chunks, double* loss_out, void* stream);

/* ------------------------------------------------------------------ noise-field task around the path (src/noise.cpp, src/tasks.cpp:139-194) */
typedef enum sxen_noise_kind { SXEN_NOISE_PERLIN = 0, SXEN_NOISE_SIMPLEX = 1 } sxen_noise_kind; /* include/sxen/noise.hpp:38 */
/* sxen::NoiseFieldSpec (include/sxen/noise.hpp:42-50), same defaults through sxen_noise_spec_default. */
typedef struct sxen_noise_spec {
  int32_t dim;       /* 1..8 */
  int32_t kind;      /* sxen_noise_kind */
  int32_t octaves;   /* >= 1 */
  int32_t reserved;
  uint64_t seed;
  double frequency;  /* lattice cells per unit of input space, > 0 */
} sxen_noise_spec;
SXEN_API sxen_status sxen_noise_spec_default(sxen_noise_spec* spec);
SXEN_API sxen_status sxen_noise_spec_validate(const sxen_noise_spec* spec);  /* NoiseFieldSpec::validate */
/* noise_field_value (src/noise.cpp:167-188) at n_points points: x_dev n_points x dim f64 -> out_dev n_points f64.
 * Vertex keys and subdivision order are the reference's; log/cos/sin are CUDA's, so values agree to rounding. */
SXEN_API sxen_status sxen_noise_field(const sxen_noise_spec* spec, const double* x_dev, size_t n_points, double* out_dev,
                                      void* stream);
/* fit_field's batch (src/tasks.cpp:156-166): coords = consecutive next_double() draws of CounterRng(seed, stream_id)
 * (or CounterRng(seed) when has_stream == 0: the hold-out stream, :173), targets = noise_field_value(coords). */
SXEN_API sxen_status sxen_sample_field_batch(const sxen_noise_spec* spec, uint64_t seed, int32_t has_stream,
                                             uint64_t stream_id, size_t n_samples, double* coords_dev,
                                             double* targets_dev, void* stream);

/* ------------------------------------------------------------------ image-fitting task around the path (src/tasks.cpp) */
/* fit_image's sampler (src/tasks.cpp:112-126): sample s of step k draws idx = CounterRng(seed, k).next_below(w*h);
 * coords = pixel centre ((idx%w)+0.5)/w, ((idx/w)+0.5)/h; targets = that pixel's RGB.  image_dev: h x w x 3 doubles in
 * [0,1] (ImageDataset::pixels, include/sxen/image.hpp).  coords_dev N x 2 f64, targets_dev N x 3 f64.  Bit-identical. */
SXEN_API sxen_status sxen_sample_image_batch(uint64_t seed, uint64_t step, const double* image_dev, int32_t width,
                                             int32_t height, size_t n_samples, double* coords_dev, double* targets_dev,
                                             void* stream);
/* The same sampler over make_test_image(width, height, image_seed) (src/image.cpp:68-96) WITHOUT the image in memory: the
 * drawn pixel's RGB is evaluated on the fly from the procedural definition (BASELINE configs[2]: 32768 x 32768 would be
 * 26 GB as doubles).  Fills samples [first_sample, first_sample + n_samples) of step `step`'s batch (draw s+1 of
 * CounterRng(train_seed, step) for sample s), so a rank of a batch-sharded run can generate its own chunk only.
 * coords_dev n_samples x 2 f64, targets_dev n_samples x 3 f64; coordinates and pixel indices bit-identical to
 * sxen_sample_image_batch, targets equal to the stored image's to rounding (libm). */
SXEN_API sxen_status sxen_sample_test_image_batch(uint64_t image_seed, int32_t width, int32_t height, uint64_t train_seed,
                                                  uint64_t step, size_t first_sample, size_t n_samples, double* coords_dev,
                                                  double* targets_dev, void* stream);
/* sxen_render_sq_error against the never-materialised test image: pred_dev count x 3 f32 for pixels [first_pixel, +count). */
SXEN_API sxen_status sxen_test_image_sq_error(uint64_t image_seed, int32_t width, int32_t height, const float* pred_dev,
                                              size_t first_pixel, size_t count, double* sum_dev, void* stream);
/* render_image's coordinates (src/tasks.cpp:69-71) for pixels [first_pixel, first_pixel + count), row-major. */
SXEN_API sxen_status sxen_pixel_centers(int32_t width, int32_t height, size_t first_pixel, size_t count, double* coords_dev,
                                        void* stream);
/* Adds sum over the pixel range and 3 channels of (clamp(pred, 0, 1) - pixel)^2 to *sum_dev (src/tasks.cpp:76-78, 35-46).
 * pred_dev: count x 3 f32. */
SXEN_API sxen_status sxen_render_sq_error(const float* pred_dev, const double* image_dev, size_t first_pixel, size_t count,
                                          double* sum_dev, void* stream);

/* ------------------------------------------------------------------ diagnostics (not part of the drop-in surface) */
/* (The tcgen05 hardware-convention probes of tests/test_gpu_tc.py are a test-only library, tests/cuda/sxen_tc_probe.cu; what
 * stays here are hooks INSIDE the product kernels: watchdog words, cycle counters, the A/B switch of the two training kernels.) */
/* The mbarrier waits of the tensor-core kernels trap after ~2 s instead of hanging the GPU; with two host-MAPPED words
 * registered here (NULL = off) the wait that gave up first notes its id and CTA in them (tools/mlp_watchdog_probe.py). */
SXEN_API sxen_status sxen_debug_tc_progress(unsigned int* mapped_host_words);
/* 16 device counters (NULL = off) the fused training kernel's roles add their cycles to: per role {cycles in the tile loop,
 * cycles of those spent waiting on each of up to three barriers} (tools/fused_step_bench.py). */
SXEN_API sxen_status sxen_debug_fused_timing(unsigned long long* counters_dev);
/* The same for the stand-alone tcgen05 training kernel, 8 counters: [0..2] epilogue thread 0 {cycles in the tile loop, waiting on
 * the chain MMAs, waiting on the weight-gradient MMAs}, [4..5] chain warp {cycles in the tile loop, waiting on the epilogue}. */
SXEN_API sxen_status sxen_debug_tc_timing(unsigned long long* counters_dev);
/* Which stand-alone tcgen05 training kernel runs (A/B measurements): 2 = two tiles in flight per SM (csrc/sxen_mlp_tc2.cu, the
 * default; launches of at most one tile per SM still take the other kernel), 1 = one tile in flight (csrc/sxen_mlp_tc.cu).  With variant 2 the timing counters read: [0..3] thread 0 of the first
 * epilogue group {cycles in the tile loop, waiting on the chain MMAs, on its own weight-gradient MMAs, on the other group's
 * phase-2 MMAs}, [4..5] chain warp {cycles in its loop, polling with nothing to issue}. */
SXEN_API sxen_status sxen_debug_tc_variant(int variant);

#ifdef __cplusplus
}
#endif
#endif /* SXEN_CUDA_H */
