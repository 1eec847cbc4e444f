// sxen_adam.cuh -- the Adam update's arithmetic, shared by the scanning kernels (sxen_optim.cu) and the batch-walking
// sparse step (sxen_encode.cuh).  Reference: adam_delta, /root/reference/proj/src/optimizer.cpp:9-15.
#pragma once

#include <cstdint>

#include "../../include/sxen_cuda.h"

namespace sxen_dev {

struct AdamScalars {
  double beta1, beta2, one_minus_beta1, one_minus_beta2, neg_lr, epsilon, bc1, bc2;
};

constexpr unsigned long long kAdamNoBad = ~0ULL;
constexpr uint32_t kUntouchedBits = 0x80000000u;  // -0.0f in feature 0 = "the accumulator never touched this row"

// fp64 with explicit round-to-nearest intrinsics: nvcc cannot contract what the reference's x86-64 build does not fuse
__device__ __forceinline__ double adam_delta(double g, double& m, double& v, const AdamScalars& c) {
  m = __dadd_rn(__dmul_rn(c.beta1, m), __dmul_rn(c.one_minus_beta1, g));
  v = __dadd_rn(__dmul_rn(c.beta2, v), __dmul_rn(__dmul_rn(c.one_minus_beta2, g), g));
  const double m_hat = __ddiv_rn(m, c.bc1);
  const double v_hat = __ddiv_rn(v, c.bc2);
  return __ddiv_rn(__dmul_rn(c.neg_lr, m_hat), __dadd_rn(__dsqrt_rn(v_hat), c.epsilon));
}

// What the batch-walking sparse step needs besides the encoder's argument block.
struct AdamWalkArgs {
  float2* tables;   // L x T rows
  float2* grads;    // same layout
  double2* m;
  double2* v;
  AdamScalars c;
  unsigned long long* status;        // first non-finite gradient element (TrainingError)
  const unsigned long long* gate;    // queued steps: non-~0 = skip
  longlong2* fixed;                  // reproducible mode: fixed-point sums (units of 2^-52), nullptr = off
};

}  // namespace sxen_dev

// host: beta/lr scalars and the global-t bias corrections of step t (src/optimizer.cpp:31-32,65-66), sxen_optim.cu
sxen_dev::AdamScalars sxen_adam_scalars(const sxen_adam_config& cfg, int64_t t);
