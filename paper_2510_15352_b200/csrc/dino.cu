// dino.cu — rendered frames -> DinoV2 input (SURVEY §8(f) row 4 "fused render
// -> DinoV2 input (224^2 resize, normalise, bf16 planar)"; PAPER.md:253;
// DESIGN.md reading R36).
//
// One thread per output pixel of one env: the 4 bilinear taps (half-pixel
// centres, no antialiasing) of the u8 frame, /255, ImageNet mean/std, bf16
// round-to-nearest-even, written channel-planar [E, 3, S, S] (each channel
// plane is written coalesced).  HBM-bound: ~12 B gathered (mostly L1/L2
// hits) and 6 B written per output pixel.
#include <cuda_bf16.h>

#include "gg_internal.cuh"

namespace gg {

// src = (d + 0.5) in/out - 0.5 = ((2d + 1) in - out) / (2 out), clamped at 0:
// the lower tap is an exact integer division and the weight the remainder
// over 2 out (one correctly rounded f32 division).
__device__ __forceinline__ void axis_taps(int d, int n_out, int n_in, int& lo, int& hi, float& w) {
  const int num = (2 * d + 1) * n_in - n_out, den = 2 * n_out;
  if (num <= 0) {
    lo = 0; w = 0.f;
  } else {
    lo = num / den;
    w = __fdiv_rn((float)(num - lo * den), (float)den);
  }
  if (lo >= n_in - 1) { lo = n_in - 1; w = 0.f; }
  hi = min(lo + 1, n_in - 1);
}

__global__ void __launch_bounds__(256) dino_input_kernel(int W, int H, int S, const uint8_t* __restrict__ rgb,
                                                         __nv_bfloat16* __restrict__ out) {
  const int e = blockIdx.y;
  const int n = S * S;
  const uint8_t* img = rgb + (size_t)e * H * W * 3;
  __nv_bfloat16* o = out + (size_t)e * 3 * n;
  const float mean[3] = {0.485f, 0.456f, 0.406f};
  const float istd[3] = {1.f / 0.229f, 1.f / 0.224f, 1.f / 0.225f};
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int dy = i / S, dx = i - dy * S;
    int x0, x1, y0, y1;
    float wx, wy;
    axis_taps(dx, S, W, x0, x1, wx);
    axis_taps(dy, S, H, y0, y1, wy);
    const uint8_t* r0 = img + (size_t)y0 * W * 3;
    const uint8_t* r1 = img + (size_t)y1 * W * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const float top = fmaf(wx, (float)r0[x1 * 3 + c] - (float)r0[x0 * 3 + c], (float)r0[x0 * 3 + c]);
      const float bot = fmaf(wx, (float)r1[x1 * 3 + c] - (float)r1[x0 * 3 + c], (float)r1[x0 * 3 + c]);
      const float v = fmaf(wy, bot - top, top) * (1.f / 255.f);
      o[(size_t)c * n + i] = __float2bfloat16_rn((v - mean[c]) * istd[c]);
    }
  }
}

void launch_dino_input(int E, int W, int H, int S, const uint8_t* rgb, void* out, cudaStream_t s) {
  const int n = S * S;
  dim3 grid((n + 255) / 256, E);
  dino_input_kernel<<<grid, 256, 0, s>>>(W, H, S, rgb, reinterpret_cast<__nv_bfloat16*>(out));
}

}  // namespace gg
