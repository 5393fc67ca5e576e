// devmath.cuh -- device helpers shared by the sm_100a kernels.
//
// Every fp64 operation that must reproduce the reference bit-for-bit is written with explicit
// round-to-nearest intrinsics so no FMA contraction can occur (the reference builds with
// -ffp-contract=off, CMakeLists.txt:11-13).
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kvc_core.hpp"

namespace kvc {
namespace dm {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double clamp1(double x) { return x < -1.0 ? -1.0 : (x > 1.0 ? 1.0 : x); }

__device__ __forceinline__ float ld_kv(const void* base, int64_t i, int bf16) {
  if (bf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[i]);
  return static_cast<const float*>(base)[i];
}

__device__ __forceinline__ void set_err(const DevTables& t, int bit) { atomicOr(t.err, bit); }

// (sim desc, key asc) "a better than b" -- the CandidateRef tie-break (index.hpp:27-33)
__device__ __forceinline__ bool better(double sa, long long ka, double sb, long long kb) {
  return sa > sb || (sa == sb && ka < kb);
}

// RN(a / b) for b > 0 given y = RN(1 / b): q1 = RN(a y) is within 2 ulps, one remainder
// correction makes it faithful, the second is Markstein's correctly rounded step -- bit-identical
// to __ddiv_rn (checked on the device by kvc_debug_div_check). One reciprocal serves every
// element of an Eq. 3/4 update (they share the divisor n + 1).
__device__ __forceinline__ double div_rcp(double a, double b, double y) {
  const double q1 = __dmul_rn(a, y);
  const double r1 = __fma_rn(-q1, b, a);
  const double q2 = __fma_rn(r1, y, q1);
  const double r2 = __fma_rn(-q2, b, a);
  return __fma_rn(r2, y, q2);
}

// Warp arg-best over (sim, key, payload).
__device__ __forceinline__ void warp_best(double& s, long long& k, int& p) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double so = __shfl_xor_sync(kFull, s, o);
    const long long ko = __shfl_xor_sync(kFull, k, o);
    const int po = __shfl_xor_sync(kFull, p, o);
    if (better(so, ko, s, k)) {
      s = so;
      k = ko;
      p = po;
    }
  }
}

}  // namespace dm
}  // namespace kvc
