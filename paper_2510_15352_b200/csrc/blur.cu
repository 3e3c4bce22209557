// blur.cu — motion-blur sample poses and the in-order sample average
// (§3.3; readings R32-R34 in DESIGN.md).
#include "gg_internal.cuh"

namespace gg {

// One sample pose per (env, i) (R33): camera-to-world rotation Rwc = Rcw^T
// rotated by the axis-angle vector w*t_i (Rodrigues), centre C = -Rcw^T t
// moved by v*t_i.  Evaluated in f64 (a few hundred flops per env) so the f32
// view matrices are reproducible by an independent f64 implementation.
// Kc >= K poses per env: sample K (present when Kc > K) is the nominal pose
// t = 0, the depth sample of an even K (R34).  At t = 0 the pose is the
// input view matrix exactly (the translation-only branch subtracts R 0).
__global__ void blur_poses_kernel(int E, int K, int Kc, const float* __restrict__ viewmats,
                                  const float* __restrict__ lin, const float* __restrict__ ang, float shutter,
                                  float* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= E * Kc) return;
  const int e = idx / Kc, i = idx - e * Kc;
  const double t = i >= K ? 0.0 : (double)shutter * (((double)i + 0.5) / (double)K - 0.5);
  const float* V = viewmats + (size_t)e * 16;
  double Rcw[3][3], tc[3];
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) Rcw[r][c] = V[r * 4 + c];
    tc[r] = V[r * 4 + 3];
  }
  const double vx = lin[e * 3 + 0] * t, vy = lin[e * 3 + 1] * t, vz = lin[e * 3 + 2] * t;
  const double ax = ang[e * 3 + 0] * t, ay = ang[e * 3 + 1] * t, az = ang[e * 3 + 2] * t;
  const double th = sqrt(ax * ax + ay * ay + az * az);
  double Rn[3][3], tn[3];
  if (th == 0.0) {
    // translation only: R unchanged, t' = -R (C + v t) = t - R (v t); exact for v t = 0
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) Rn[r][c] = Rcw[r][c];
      tn[r] = tc[r] - (Rcw[r][0] * vx + Rcw[r][1] * vy + Rcw[r][2] * vz);
    }
  } else {
    double C[3];
    for (int k = 0; k < 3; ++k) C[k] = -(Rcw[0][k] * tc[0] + Rcw[1][k] * tc[1] + Rcw[2][k] * tc[2]);
    const double kx = ax / th, ky = ay / th, kz = az / th;
    const double s = sin(th), c = cos(th), oc = 1.0 - c;
    const double Q[3][3] = {{c + kx * kx * oc, kx * ky * oc - kz * s, kx * kz * oc + ky * s},
                            {ky * kx * oc + kz * s, c + ky * ky * oc, ky * kz * oc - kx * s},
                            {kz * kx * oc - ky * s, kz * ky * oc + kx * s, c + kz * kz * oc}};
    // Rwc' = Q Rwc  ->  Rcw' = Rcw Q^T
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) Rn[r][cc] = Rcw[r][0] * Q[cc][0] + Rcw[r][1] * Q[cc][1] + Rcw[r][2] * Q[cc][2];
    const double Cn[3] = {C[0] + vx, C[1] + vy, C[2] + vz};
    for (int r = 0; r < 3; ++r) tn[r] = -(Rn[r][0] * Cn[0] + Rn[r][1] * Cn[1] + Rn[r][2] * Cn[2]);
  }
  float* O = out + (size_t)idx * 16;
  for (int r = 0; r < 3; ++r) {
    for (int c = 0; c < 3; ++c) O[r * 4 + c] = (float)Rn[r][c];
    O[r * 4 + 3] = (float)tn[r];
  }
  O[12] = 0.f; O[13] = 0.f; O[14] = 0.f; O[15] = 1.f;
}

// Average the K colour samples of each env (R34; frames e*Kc + i, i < K):
// m = x0 + (sum_{i>=1} (x_i - x0)) / K, then u8 round-half-even or f32.
// Depth comes from the nominal-pose sample dk (t = 0).
__global__ void blur_average_kernel(int ec, int e0, int K, int Kc, int dk, size_t P, const float* __restrict__ srgb,
                                    const float* __restrict__ sdepth, const float* __restrict__ salpha,
                                    int rgb_format, void* __restrict__ rgb, float* __restrict__ depth,
                                    float* __restrict__ alpha) {
  const size_t n = (size_t)ec * P;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n; q += (size_t)gridDim.x * blockDim.x) {
    const size_t e = q / P, p = q - e * P;
    const size_t base = e * Kc * P + p;    // sample i of env e at frame e*Kc + i
    const size_t out = (size_t)(e0 + e) * P + p;
    if (rgb) {
      for (int ch = 0; ch < 3; ++ch) {
        const float x0 = srgb[base * 3 + ch];
        float s = 0.f;
        for (int i = 1; i < K; ++i) s += srgb[(base + (size_t)i * P) * 3 + ch] - x0;
        const float m = x0 + s / (float)K;
        if (rgb_format == 0)
          reinterpret_cast<uint8_t*>(rgb)[out * 3 + ch] = (uint8_t)__float2uint_rn(fminf(fmaxf(m, 0.f), 1.f) * 255.f);
        else
          reinterpret_cast<float*>(rgb)[out * 3 + ch] = m;
      }
    }
    if (alpha) {
      const float a0 = salpha[base];
      float s = 0.f;
      for (int i = 1; i < K; ++i) s += salpha[base + (size_t)i * P] - a0;
      alpha[out] = a0 + s / (float)K;
    }
    if (depth) depth[out] = sdepth[base + (size_t)dk * P];
  }
}

// replicate per-env ids / intrinsics K times (sample-major inside each env)
__global__ void blur_expand_kernel(int ec, int K, const int32_t* __restrict__ ids, const float* __restrict__ intr,
                                   int32_t* __restrict__ ids_k, float* __restrict__ intr_k) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ec * K) return;
  const int e = idx / K;
  ids_k[idx] = ids[e];
  for (int k = 0; k < 4; ++k) intr_k[idx * 4 + k] = intr[e * 4 + k];
}

void launch_blur_poses(int E, int K, int Kc, const float* viewmats, const float* lin, const float* ang,
                       float shutter, float* out, cudaStream_t s) {
  blur_poses_kernel<<<(E * Kc + 127) / 128, 128, 0, s>>>(E, K, Kc, viewmats, lin, ang, shutter, out);
}

void launch_blur_average(int ec, int e0, int K, int Kc, int dk, size_t P, const float* srgb, const float* sdepth,
                         const float* salpha, int rgb_format, void* rgb, float* depth, float* alpha, cudaStream_t s) {
  blur_average_kernel<<<148 * 8, 256, 0, s>>>(ec, e0, K, Kc, dk, P, srgb, sdepth, salpha, rgb_format, rgb, depth,
                                               alpha);
}

void launch_blur_expand(int ec, int K, const int32_t* ids, const float* intr, int32_t* ids_k, float* intr_k,
                        cudaStream_t s) {
  blur_expand_kernel<<<(ec * K + 127) / 128, 128, 0, s>>>(ec, K, ids, intr, ids_k, intr_k);
}

}  // namespace gg
