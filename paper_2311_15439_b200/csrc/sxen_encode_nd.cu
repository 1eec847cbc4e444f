// sxen_encode_nd.cu -- instantiates the encode kernels for ONE input dimension (compile with -DSXEN_ND=<1..8>).
// One translation unit per dimension keeps nvcc parallel and the per-file kernel count bounded.
#include "sxen_encode.cuh"

#ifndef SXEN_ND
#error "compile with -DSXEN_ND=<1..8>"
#endif

namespace sxen_dev {
namespace {

constexpr int ND = SXEN_ND;

template <int F, int LPT, int MODE, bool EXACT, bool GRID = false, bool REPRO = false>
cudaError_t go(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream) {
  a.groups = (a.n_levels + LPT - 1) / LPT;
  a.groups_shift = -1;
  a.span_groups = a.groups;
  int slices = 1;
  if (!a.level_major && ln.chunk_levels > 0 && ln.chunk_levels % LPT == 0 && ln.chunk_levels < a.n_levels) {
    const int cg = ln.chunk_levels / LPT;
    if ((cg & (cg - 1)) == 0) {
      a.span_groups = cg;
      slices = (a.groups + cg - 1) / cg;
    }
  }
  for (int sft = 0; sft < 31; ++sft)
    if ((1 << sft) == a.span_groups) a.groups_shift = sft;
  // out/upstream chunk alignment the kernel may rely on (base pointers are checked by the caller via a.vec)
  const int k = LPT * F;
  int vec = a.vec;
  while (vec > 1 && ((k % vec) != 0 || (a.row_width % vec) != 0 || ((a.level0 * F) % vec) != 0)) vec >>= 1;
  a.vec = vec;
  int block = ln.block_threads > 0 ? ln.block_threads : 256;
  const int max_block = (LPT >= 4 || GRID) ? 256 : 512;
  if (block > max_block) block = max_block;
  block = (block / 32) * 32;
  if (block < 32) block = 32;
  dim3 grid;
  if (a.level_major) {
    grid = dim3(static_cast<unsigned>((a.n_samples + block - 1) / block), static_cast<unsigned>(a.groups), 1);
  } else {
    const unsigned long long threads = a.n_samples * static_cast<unsigned long long>(a.span_groups);
    grid = dim3(static_cast<unsigned>((threads + block - 1) / block), static_cast<unsigned>(slices), 1);
  }
  encode_kernel<ND, F, LPT, MODE, EXACT, GRID, REPRO><<<grid, block, 0, stream>>>(a);
  return cudaGetLastError();
}

template <int F, int LPT, bool EXACT, bool GRID = false>
cudaError_t by_mode(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream) {
  switch (ln.mode) {
    case kModeFwd: return go<F, LPT, kModeFwd, EXACT, GRID>(ln, a, stream);
    case kModeBwd: return go<F, LPT, kModeBwd, EXACT, GRID>(ln, a, stream);
    default: return go<F, LPT, kModeBoth, EXACT, GRID>(ln, a, stream);
  }
}

template <int MODE, bool GRID>
cudaError_t go_generic(EncodeArgs& a, cudaStream_t stream) {
  const int block = 256;
  const unsigned long long threads = a.n_samples * static_cast<unsigned long long>(a.n_levels);
  encode_generic_kernel<ND, MODE, GRID><<<static_cast<unsigned>((threads + block - 1) / block), block, 0, stream>>>(a);
  return cudaGetLastError();
}

template <bool GRID>
cudaError_t generic_by_mode(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream) {
  switch (ln.mode) {
    case kModeFwd: return go_generic<kModeFwd, GRID>(a, stream);
    case kModeBwd: return go_generic<kModeBwd, GRID>(a, stream);
    default: return go_generic<kModeBoth, GRID>(a, stream);
  }
}

// Reproducible mode (sxen_grad_set_reproducible): fixed-point sums next to the fp32 atomics; F == 2, both backends at
// ND <= 3 for the grid (the tuned kernel), exact blend, one or two levels per thread.
template <bool GRID>
cudaError_t launch_f2_repro(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream, int* used) {
  if (ln.lpt >= 2) {
    *used = 2;
    return ln.mode == kModeBwd ? go<2, 2, kModeBwd, true, GRID, true>(ln, a, stream) : go<2, 2, kModeBoth, true, GRID, true>(ln, a, stream);
  }
  *used = 1;
  return ln.mode == kModeBwd ? go<2, 1, kModeBwd, true, GRID, true>(ln, a, stream) : go<2, 1, kModeBoth, true, GRID, true>(ln, a, stream);
}

// F == 2 is the configuration every BASELINE workload uses: full tuning surface.
cudaError_t launch_f2(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream, int* used) {
  int lpt = ln.lpt;
  if (ln.repro && (ln.mode & kModeBwd)) return launch_f2_repro<false>(ln, a, stream, used);
#if SXEN_ND == 2 || SXEN_ND == 3
  if (lpt >= 16) {
    *used = 16;
    return ln.exact ? by_mode<2, 16, true>(ln, a, stream) : by_mode<2, 16, false>(ln, a, stream);
  }
#endif
  if (lpt >= 4) {
    *used = 4;
    return ln.exact ? by_mode<2, 4, true>(ln, a, stream) : by_mode<2, 4, false>(ln, a, stream);
  }
  if (lpt >= 2) {
    *used = 2;
    return ln.exact ? by_mode<2, 2, true>(ln, a, stream) : by_mode<2, 2, false>(ln, a, stream);
  }
  *used = 1;
  return ln.exact ? by_mode<2, 1, true>(ln, a, stream) : by_mode<2, 1, false>(ln, a, stream);
}

// F in {1, 4, 8}: vectorised rows, exact blend only, one or two levels per thread.
template <int F>
cudaError_t launch_fx(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream, int* used) {
  if (ln.lpt >= 2) {
    *used = 2;
    return by_mode<F, 2, true>(ln, a, stream);
  }
  *used = 1;
  return by_mode<F, 1, true>(ln, a, stream);
}

}  // namespace

#define SXEN_CAT2(a, b) a##b
#define SXEN_CAT(a, b) SXEN_CAT2(a, b)

cudaError_t SXEN_CAT(launch_encode_nd, SXEN_ND)(const EncodeLaunch& ln, EncodeArgs& a, cudaStream_t stream,
                                                int* used_lpt) {
  if (ln.grid_backend) {
#if SXEN_ND == 2 || SXEN_ND == 3
    // the paper's comparator in its 2D / 3D settings: same tuned kernel, 2^ND corners instead of ND+1 vertices
    if (ln.features == 2) {
      if (ln.repro && (ln.mode & kModeBwd)) return launch_f2_repro<true>(ln, a, stream, used_lpt);
      if (ln.lpt >= 2) {
        *used_lpt = 2;
        return ln.exact ? by_mode<2, 2, true, true>(ln, a, stream) : by_mode<2, 2, false, true>(ln, a, stream);
      }
      *used_lpt = 1;
      return ln.exact ? by_mode<2, 1, true, true>(ln, a, stream) : by_mode<2, 1, false, true>(ln, a, stream);
    }
#endif
    *used_lpt = 1;
    return generic_by_mode<true>(ln, a, stream);
  }
  if (ln.repro && (ln.mode & kModeBwd) && ln.features != 2) {  // fixed-point sums for the other widths: the general kernel
    *used_lpt = 1;
    return generic_by_mode<false>(ln, a, stream);
  }
  switch (ln.features) {
    case 2: return launch_f2(ln, a, stream, used_lpt);
    case 1: return launch_fx<1>(ln, a, stream, used_lpt);
    case 4: return launch_fx<4>(ln, a, stream, used_lpt);
    case 8: return launch_fx<8>(ln, a, stream, used_lpt);
    default:
      *used_lpt = 1;
      return generic_by_mode<false>(ln, a, stream);
  }
}

cudaError_t SXEN_CAT(launch_fold_nd, SXEN_ND)(const EncodeArgs& a, cudaStream_t stream) {
  uint32_t most = 0;
  for (int l = 0; l < a.n_levels; ++l)
    if (a.cg.shift[l] >= 0) most = a.cg.verts[l] > most ? a.cg.verts[l] : most;
  if (most == 0 || a.coarse == nullptr) return cudaSuccess;
  const unsigned long long elems = static_cast<unsigned long long>(most) * static_cast<unsigned long long>(a.features);
  const dim3 grid(static_cast<unsigned>((elems + 255) / 256), static_cast<unsigned>(a.n_levels), 1);
  coarse_fold_kernel<ND><<<grid, 256, 0, stream>>>(a);
  return cudaGetLastError();
}

cudaError_t SXEN_CAT(launch_adam_walk_nd, SXEN_ND)(const EncodeArgs& a, const AdamWalkArgs& o, int grid_backend,
                                                    cudaStream_t stream) {
  const int block = 256;
  const unsigned long long threads = a.n_samples * static_cast<unsigned long long>(a.n_levels);
  const unsigned blocks = static_cast<unsigned>((threads + block - 1) / block);
  if (grid_backend) {
    sparse_adam_walk_kernel<ND, true><<<blocks, block, 0, stream>>>(a, o);
  } else {
    sparse_adam_walk_kernel<ND, false><<<blocks, block, 0, stream>>>(a, o);
  }
  return cudaGetLastError();
}

cudaError_t SXEN_CAT(launch_debug_nd, SXEN_ND)(EncodeArgs& a, int grid_backend, uint32_t* idx, double* w,
                                               int total_levels, cudaStream_t stream) {
  const int block = 256;
  const unsigned long long threads = a.n_samples * static_cast<unsigned long long>(a.n_levels);
  const unsigned blocks = static_cast<unsigned>((threads + block - 1) / block);
  if (grid_backend) {
    encode_debug_kernel<ND, true><<<blocks, block, 0, stream>>>(a, idx, w, total_levels);
  } else {
    encode_debug_kernel<ND, false><<<blocks, block, 0, stream>>>(a, idx, w, total_levels);
  }
  return cudaGetLastError();
}

}  // namespace sxen_dev
