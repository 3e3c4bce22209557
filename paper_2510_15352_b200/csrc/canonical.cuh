// canonical.cuh — correctly-rounded f32 ops that nvcc never contracts into
// FFMA.  Every integer decision of the path (cull, radius, tile rect, depth
// key bits) is computed with these in the operation order of DESIGN.md §2.1,
// so the GPU reproduces the canonical f32 sequence bit for bit.
#pragma once
#include <cuda_runtime.h>

namespace gg {
__device__ __forceinline__ float fm(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fa(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fs(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fd(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float fsq(float a) { return __fsqrt_rn(a); }
// (a*b + c*d) + e*f, each op rounded
__device__ __forceinline__ float dot3(float a0, float b0, float a1, float b1, float a2, float b2) {
  return fa(fa(fm(a0, b0), fm(a1, b1)), fm(a2, b2));
}
}  // namespace gg
