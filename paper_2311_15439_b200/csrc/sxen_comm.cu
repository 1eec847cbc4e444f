// sxen_comm.cu -- the gradient exchange of the batch-sharded training step.
//
// Reference: train_field fans the batch out over worker threads, each with its own accumulators, and merges them into
// worker 0 in worker order before the optimizer steps (/root/reference/proj/src/trainer.cpp:101-128).  Here the workers
// are ranks, one per GPU, tables / MLP / moments replicated, and the merge is a SUM all-reduce of the table-gradient
// accumulator (level slices), the MLP gradient and the loss sum.  Two transports behind one handle:
//
//   NCCL   one process per GPU (the driver's torchrun layout, or any host that can hand an ncclUniqueId to its peers).
//          libnccl is resolved with dlopen at the first sxen_comm_* call -- an already loaded copy first (a Python host has
//          torch's) -- so libsxen_b200.so carries no link-time dependency and single-GPU hosts never touch it.
//   LOCAL  the ranks live in ONE process, one host thread each (the reference's own worker-thread layout), on any mix of
//          devices including the same device twice.  The exchange is this library's own kernel over peer-mapped memory:
//          rank r sums slice r of every rank's buffer in rank order (the reference's fixed merge order: the result is
//          bit-identical on every rank and from run to run) and stores the sum into every rank's buffer -- a one-hop
//          reduce-scatter + all-gather through NVLink P2P loads / stores; between devices the bytes on the wire equal a
//          ring all-reduce's 2 (W-1)/W * size.  Ordering is by CUDA events across the ranks' streams plus a host barrier
//          (no device-side spinning, so two ranks can share one GPU: that is how the one-GPU tests run it).
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <memory>
#include <mutex>
#include <thread>

#include "sxen_common.hpp"

using namespace sxen_host;

namespace {

// ---------------------------------------------------------------------------------------------- NCCL through dlopen
struct NcclApi {
  void* handle = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
  std::string why;
};

NcclApi& nccl_api() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {  // a copy the process already holds (torch's) wins: one NCCL per process
      api.handle = dlopen(n, RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
      if (api.handle) break;
    }
    if (!api.handle) {
      if (const char* env = std::getenv("SXEN_NCCL_LIB")) api.handle = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
      for (const char* n : names) {
        if (api.handle) break;
        api.handle = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      }
    }
    if (!api.handle) {
      api.why = std::string("libnccl.so.2 could not be loaded (") + (dlerror() ? dlerror() : "not found") +
                "); set SXEN_NCCL_LIB to its path";
      return;
    }
    auto sym = [&](const char* name) -> void* {
      void* p = dlsym(api.handle, name);
      if (!p && api.why.empty()) api.why = std::string("libnccl lacks ") + name;
      return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
  });
  return api;
}

sxen_status nccl_fail(ncclResult_t r, const char* what) {
  NcclApi& api = nccl_api();
  return fail(SXEN_NCCL_ERROR, "%s: %s", what, api.GetErrorString ? api.GetErrorString(r) : "NCCL error");
}

#define SXEN_NCCL(call)                                  \
  do {                                                   \
    ncclResult_t r__ = (call);                           \
    if (r__ != ncclSuccess) return nccl_fail(r__, #call); \
  } while (0)

// ---------------------------------------------------------------------------------------------- LOCAL transport
constexpr int kMaxLocalRanks = 16;

struct LocalGroup {
  int world = 0;
  std::vector<int> devices;
  // what each rank published for the exchange in flight
  void* buf[kMaxLocalRanks] = {};
  size_t count[kMaxLocalRanks] = {};
  int type[kMaxLocalRanks] = {};
  cudaEvent_t ready[kMaxLocalRanks] = {};  // rank's buffer holds its contribution (recorded on the rank's stream)
  cudaEvent_t done[kMaxLocalRanks] = {};   // rank's slice has been summed and stored into every buffer
  // sense-reversing host barrier over the ranks' threads
  std::atomic<int> arrived{0};
  std::atomic<unsigned> generation{0};
  std::atomic<int> broken{0};  // a rank failed or timed out: everyone leaves with an error instead of waiting for ever
  std::atomic<int> alive{0};   // handles not destroyed yet
  ~LocalGroup() {
    for (int r = 0; r < world; ++r) {
      DeviceGuard g(devices[static_cast<size_t>(r)]);
      if (ready[r]) cudaEventDestroy(ready[r]);
      if (done[r]) cudaEventDestroy(done[r]);
    }
  }
};

// false = the group is broken (a peer reported a failure or did not arrive within the time limit)
bool host_barrier(LocalGroup& g) {
  const unsigned gen = g.generation.load(std::memory_order_acquire);
  if (g.arrived.fetch_add(1, std::memory_order_acq_rel) + 1 == g.world) {
    g.arrived.store(0, std::memory_order_relaxed);
    g.generation.fetch_add(1, std::memory_order_release);
    return g.broken.load(std::memory_order_acquire) == 0;
  }
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (g.generation.load(std::memory_order_acquire) == gen) {
    if (g.broken.load(std::memory_order_acquire)) return false;
    if (++spins > 2000) {
      std::this_thread::yield();
      if ((spins & 0xfff) == 0 && std::chrono::steady_clock::now() - t0 > std::chrono::seconds(120)) {
        g.broken.store(1, std::memory_order_release);
        return false;
      }
    }
  }
  return g.broken.load(std::memory_order_acquire) == 0;
}

template <typename T>
struct PeerPtrs {
  T* p[kMaxLocalRanks];
};

// Slice [lo, hi) of every rank's buffer: sum in rank order (fixed, like the reference's worker-order merge,
// src/trainer.cpp:125-128), result stored into every rank's buffer.  IEEE adds: -0.0f + -0.0f = -0.0f keeps an untouched
// row untouched, anything + (+0.0f) marks it touched.  VEC elements per access (16 bytes).
template <typename T, int VEC>
__global__ void __launch_bounds__(256) peer_allreduce_kernel(const __grid_constant__ PeerPtrs<T> ptrs, int world, size_t lo,
                                                             size_t hi) {
  struct alignas(sizeof(T) * VEC) Pack {
    T v[VEC];
  };
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * VEC;
  for (size_t i = lo + (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * VEC; i < hi; i += stride) {
    if (i + VEC <= hi) {
      Pack acc = *reinterpret_cast<const Pack*>(ptrs.p[0] + i);
      for (int r = 1; r < world; ++r) {
        const Pack o = *reinterpret_cast<const Pack*>(ptrs.p[r] + i);
#pragma unroll
        for (int k = 0; k < VEC; ++k) acc.v[k] = acc.v[k] + o.v[k];
      }
      for (int r = 0; r < world; ++r) *reinterpret_cast<Pack*>(ptrs.p[r] + i) = acc;
    } else {
      for (size_t j = i; j < hi; ++j) {
        T acc = ptrs.p[0][j];
        for (int r = 1; r < world; ++r) acc = acc + ptrs.p[r][j];
        for (int r = 0; r < world; ++r) ptrs.p[r][j] = acc;
      }
    }
  }
}

}  // namespace

struct sxen_comm {
  int kind = 0;  // 0 NCCL, 1 LOCAL
  int world = 1, rank = 0, device = 0;
  ncclComm_t nccl = nullptr;
  std::shared_ptr<LocalGroup> group;
};

namespace {

template <typename T>
sxen_status local_allreduce(sxen_comm* c, void* buf, size_t count, int type_tag, cudaStream_t stream) {
  LocalGroup& g = *c->group;
  const int r = c->rank, W = c->world;
  auto broken = [&](const char* what) {
    g.broken.store(1, std::memory_order_release);
    return fail(SXEN_NCCL_ERROR, "local all-reduce: %s", what);
  };
  if (g.broken.load(std::memory_order_acquire)) return fail(SXEN_NCCL_ERROR, "local all-reduce: the group is broken (a peer failed)");
  g.buf[r] = buf;
  g.count[r] = count;
  g.type[r] = type_tag;
  if (cudaEventRecord(g.ready[r], stream) != cudaSuccess) return broken("cudaEventRecord failed");
  if (!host_barrier(g)) return fail(SXEN_NCCL_ERROR, "local all-reduce: a peer did not arrive");
  for (int p = 0; p < W; ++p)
    if (g.count[p] != count || g.type[p] != type_tag) return broken("ranks disagree on the element count or type of the buffer");
  for (int p = 0; p < W; ++p)
    if (p != r && cudaStreamWaitEvent(stream, g.ready[p], 0) != cudaSuccess) return broken("cudaStreamWaitEvent failed");
  // slice r, bounds on 16-byte packs
  constexpr int VEC = 16 / sizeof(T);
  const size_t packs = (count + VEC - 1) / VEC;
  const size_t per = (packs + static_cast<size_t>(W) - 1) / static_cast<size_t>(W);
  const size_t lo = std::min(count, per * static_cast<size_t>(r) * VEC), hi = std::min(count, per * static_cast<size_t>(r + 1) * VEC);
  bool aligned = true;
  PeerPtrs<T> ptrs{};
  for (int p = 0; p < W; ++p) {
    ptrs.p[p] = static_cast<T*>(g.buf[p]);
    aligned = aligned && (reinterpret_cast<uintptr_t>(g.buf[p]) % 16 == 0);
  }
  if (hi > lo) {
    const size_t work = (hi - lo + VEC - 1) / VEC;
    const unsigned blocks = static_cast<unsigned>(std::min<size_t>((work + 255) / 256, 148 * 8));
    if (aligned) peer_allreduce_kernel<T, VEC><<<blocks, 256, 0, stream>>>(ptrs, W, lo, hi);
    else peer_allreduce_kernel<T, 1><<<blocks, 256, 0, stream>>>(ptrs, W, lo, hi);
    if (cudaGetLastError() != cudaSuccess) return broken("kernel launch failed");
    count_launch();
  }
  if (cudaEventRecord(g.done[r], stream) != cudaSuccess) return broken("cudaEventRecord failed");
  if (!host_barrier(g)) return fail(SXEN_NCCL_ERROR, "local all-reduce: a peer did not arrive");
  for (int p = 0; p < W; ++p)
    if (p != r && cudaStreamWaitEvent(stream, g.done[p], 0) != cudaSuccess) return broken("cudaStreamWaitEvent failed");
  // (no third barrier: a rank can only publish its next exchange after this one's second barrier, by which time every
  // peer has read buf[] and queued its waits on ready[]; done[] is re-recorded only behind the NEXT first barrier)
  return SXEN_OK;
}

}  // namespace

extern "C" {

sxen_status sxen_comm_unique_id(sxen_comm_id* out) {
  SXEN_REQUIRE(out != nullptr, "null argument");
  static_assert(sizeof(ncclUniqueId) == SXEN_COMM_ID_BYTES, "sxen_comm_id must hold an ncclUniqueId");
  NcclApi& api = nccl_api();
  if (!api.why.empty()) return fail(SXEN_NCCL_ERROR, "%s", api.why.c_str());
  ncclUniqueId id;
  SXEN_NCCL(api.GetUniqueId(&id));
  std::memcpy(out->bytes, &id, sizeof(id));
  return SXEN_OK;
}

sxen_status sxen_comm_create(const sxen_comm_id* id, int32_t world, int32_t rank, int32_t device, sxen_comm** out) {
  SXEN_REQUIRE(id != nullptr && out != nullptr, "null argument");
  *out = nullptr;
  SXEN_REQUIRE(world >= 1 && rank >= 0 && rank < world, "comm: rank %d outside a world of %d", rank, world);
  NcclApi& api = nccl_api();
  if (!api.why.empty()) return fail(SXEN_NCCL_ERROR, "%s", api.why.c_str());
  DeviceGuard guard(device);
  if (!guard.ok) return fail(SXEN_CUDA_ERROR, "comm: cannot select device %d", device);
  ncclUniqueId nid;
  std::memcpy(&nid, id->bytes, sizeof(nid));
  ncclComm_t comm = nullptr;
  SXEN_NCCL(api.CommInitRank(&comm, world, nid, rank));
  sxen_comm* c = new sxen_comm();
  c->kind = 0;
  c->world = world;
  c->rank = rank;
  c->device = device;
  c->nccl = comm;
  *out = c;
  return SXEN_OK;
}

sxen_status sxen_comm_create_local(int32_t world, const int32_t* devices, sxen_comm** out) {
  SXEN_REQUIRE(devices != nullptr && out != nullptr, "null argument");
  SXEN_REQUIRE(world >= 1 && world <= kMaxLocalRanks, "comm: a local group holds 1..%d ranks", kMaxLocalRanks);
  for (int r = 0; r < world; ++r) out[r] = nullptr;
  int n_dev = 0;
  if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev < 1) return fail(SXEN_CUDA_ERROR, "comm: no CUDA device");
  for (int r = 0; r < world; ++r) SXEN_REQUIRE(devices[r] >= 0 && devices[r] < n_dev, "comm: device %d of rank %d does not exist", devices[r], r);
  auto g = std::make_shared<LocalGroup>();
  g->world = world;
  g->devices.assign(devices, devices + world);
  for (int r = 0; r < world; ++r) {
    DeviceGuard guard(devices[r]);
    SXEN_CUDA(cudaEventCreateWithFlags(&g->ready[r], cudaEventDisableTiming));
    SXEN_CUDA(cudaEventCreateWithFlags(&g->done[r], cudaEventDisableTiming));
    for (int p = 0; p < world; ++p) {  // the exchange kernel dereferences every rank's buffer from this rank's device
      if (devices[p] == devices[r]) continue;
      int can = 0;
      SXEN_CUDA(cudaDeviceCanAccessPeer(&can, devices[r], devices[p]));
      if (!can) return fail(SXEN_NCCL_ERROR, "comm: device %d cannot map device %d's memory (no P2P path)", devices[r], devices[p]);
      const cudaError_t e = cudaDeviceEnablePeerAccess(devices[p], 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
    }
  }
  g->alive.store(world);
  for (int r = 0; r < world; ++r) {
    sxen_comm* c = new sxen_comm();
    c->kind = 1;
    c->world = world;
    c->rank = r;
    c->device = devices[r];
    c->group = g;
    out[r] = c;
  }
  return SXEN_OK;
}

sxen_status sxen_comm_destroy(sxen_comm* c) {
  if (!c) return SXEN_OK;
  if (c->kind == 0 && c->nccl) {
    DeviceGuard guard(c->device);
    NcclApi& api = nccl_api();
    if (api.CommDestroy) api.CommDestroy(c->nccl);
  }
  if (c->group) c->group->alive.fetch_sub(1);
  delete c;
  return SXEN_OK;
}

sxen_status sxen_comm_abort(sxen_comm* c) {
  SXEN_REQUIRE(c != nullptr, "comm handle is null");
  if (c->kind == 1) {
    c->group->broken.store(1, std::memory_order_release);
  } else if (c->nccl) {
    DeviceGuard guard(c->device);
    NcclApi& api = nccl_api();
    if (api.CommAbort) api.CommAbort(c->nccl);
    c->nccl = nullptr;
  }
  return SXEN_OK;
}

sxen_status sxen_comm_info(const sxen_comm* c, int32_t* world, int32_t* rank, int32_t* device, int32_t* kind) {
  SXEN_REQUIRE(c != nullptr, "comm handle is null");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  if (device) *device = c->device;
  if (kind) *kind = c->kind;
  return SXEN_OK;
}

sxen_status sxen_comm_allreduce(sxen_comm* c, void* buf_dev, size_t count, sxen_coord_type type, void* stream) {
  SXEN_REQUIRE(c != nullptr, "comm handle is null");
  SXEN_REQUIRE(type == SXEN_COORD_F32 || type == SXEN_COORD_F64 || type == SXEN_ELEM_I64, "all-reduce: unknown element type %d",
               static_cast<int>(type));
  SXEN_REQUIRE(count == 0 || buf_dev != nullptr, "all-reduce: buffer is null");
  if (c->world == 1 && c->kind == 1) return SXEN_OK;
  DeviceGuard guard(c->device);
  if (c->kind == 0) {
    if (count == 0) return SXEN_OK;
    if (c->nccl == nullptr) return fail(SXEN_NCCL_ERROR, "all-reduce: the communicator was aborted");
    NcclApi& api = nccl_api();
    SXEN_NCCL(api.AllReduce(buf_dev, buf_dev, count,
                            type == SXEN_COORD_F32 ? ncclFloat32 : type == SXEN_COORD_F64 ? ncclFloat64 : ncclInt64, ncclSum,
                            c->nccl, as_stream(stream)));
    return SXEN_OK;
  }
  if (type == SXEN_ELEM_I64) return local_allreduce<long long>(c, buf_dev, count, 2, as_stream(stream));
  return type == SXEN_COORD_F32 ? local_allreduce<float>(c, buf_dev, count, 1, as_stream(stream))
                                : local_allreduce<double>(c, buf_dev, count, 0, as_stream(stream));
}

}  // extern "C"
