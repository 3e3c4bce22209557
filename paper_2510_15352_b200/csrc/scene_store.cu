// scene_store.cu — K0: validate and pack one scene into the 16-B SoA store.
//
// SPEC.md:28-34 (SplatPrimitive: quaternion normalised, scales > 0,
// opacity in [0,1], DC colour 0.2820948 c + 0.5 clamped) and SPEC.md:130
// (Sigma = R diag(s^2) R^T).  Sigma3 is computed once per Gaussian here in
// the canonical f32 order (DESIGN.md §2.1 "O1") and shared by every env
// bound to the scene ("shared, never copied per environment").
#include "gg_internal.cuh"
#include "canonical.cuh"

namespace gg {

__global__ void validate_kernel(int64_t n, int K, const float* __restrict__ means,
                                const float* __restrict__ scales, const float* __restrict__ quats,
                                const float* __restrict__ opac, const float* __restrict__ sh,
                                ValidateOut* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    bool fin = true;
    for (int k = 0; k < 3; ++k) fin &= isfinite(means[i * 3 + k]) && isfinite(scales[i * 3 + k]);
    for (int k = 0; k < 4; ++k) fin &= isfinite(quats[i * 4 + k]);
    fin &= isfinite(opac[i]);
    for (int k = 0; k < K * 3; ++k) fin &= isfinite(sh[i * K * 3 + k]);
    if (!fin) { atomicMin(&out->nonfinite, (unsigned long long)i); continue; }
    if (!(scales[i * 3] > 0.f && scales[i * 3 + 1] > 0.f && scales[i * 3 + 2] > 0.f))
      atomicMin(&out->bad_scale, (unsigned long long)i);
    if (!(opac[i] >= 0.f && opac[i] <= 1.f)) atomicMin(&out->bad_opacity, (unsigned long long)i);
    const float w = quats[i * 4], x = quats[i * 4 + 1], y = quats[i * 4 + 2], z = quats[i * 4 + 3];
    const float nrm = fsq(fa(fa(fa(fm(w, w), fm(x, x)), fm(y, y)), fm(z, z)));
    if (!(nrm > 0.f) || !isfinite(nrm)) atomicMin(&out->zero_quat, (unsigned long long)i);
  }
}

__global__ void pack_kernel(int64_t n, int K, int sh_stride, const float* __restrict__ means,
                            const float* __restrict__ scales, const float* __restrict__ quats,
                            const float* __restrict__ opac, const float* __restrict__ sh,
                            float4* pos_op, float4* cov_a, float4* cov_b, float2* aux, float* qmax,
                            float* sh_out) {
  const float SH_C0 = 0.28209479177387814f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // O1: q <- q/|q|
    float w = quats[i * 4], x = quats[i * 4 + 1], y = quats[i * 4 + 2], z = quats[i * 4 + 3];
    const float nrm = fsq(fa(fa(fa(fm(w, w), fm(x, x)), fm(y, y)), fm(z, z)));
    w = fd(w, nrm); x = fd(x, nrm); y = fd(y, nrm); z = fd(z, nrm);
    // R(q)
    float R[3][3];
    R[0][0] = fs(1.f, fm(2.f, fa(fm(y, y), fm(z, z))));
    R[0][1] = fm(2.f, fs(fm(x, y), fm(w, z)));
    R[0][2] = fm(2.f, fa(fm(x, z), fm(w, y)));
    R[1][0] = fm(2.f, fa(fm(x, y), fm(w, z)));
    R[1][1] = fs(1.f, fm(2.f, fa(fm(x, x), fm(z, z))));
    R[1][2] = fm(2.f, fs(fm(y, z), fm(w, x)));
    R[2][0] = fm(2.f, fs(fm(x, z), fm(w, y)));
    R[2][1] = fm(2.f, fa(fm(y, z), fm(w, x)));
    R[2][2] = fs(1.f, fm(2.f, fa(fm(x, x), fm(y, y))));
    const float s0 = scales[i * 3], s1 = scales[i * 3 + 1], s2 = scales[i * 3 + 2];
    float M[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      M[r][0] = fm(R[r][0], s0);
      M[r][1] = fm(R[r][1], s1);
      M[r][2] = fm(R[r][2], s2);
    }
    // Sigma3_ij = (M_i0 M_j0 + M_i1 M_j1) + M_i2 M_j2
    const float Sxx = dot3(M[0][0], M[0][0], M[0][1], M[0][1], M[0][2], M[0][2]);
    const float Sxy = dot3(M[0][0], M[1][0], M[0][1], M[1][1], M[0][2], M[1][2]);
    const float Sxz = dot3(M[0][0], M[2][0], M[0][1], M[2][1], M[0][2], M[2][2]);
    const float Syy = dot3(M[1][0], M[1][0], M[1][1], M[1][1], M[1][2], M[1][2]);
    const float Syz = dot3(M[1][0], M[2][0], M[1][1], M[2][1], M[1][2], M[2][2]);
    const float Szz = dot3(M[2][0], M[2][0], M[2][1], M[2][1], M[2][2], M[2][2]);
    // DC colour, used when rendering at degree 0
    float dc[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) dc[c] = fminf(1.f, fmaxf(0.f, SH_C0 * sh[i * K * 3 + c] + 0.5f));
    const float smax = fmaxf(s0, fmaxf(s1, s2));
    // log2(o) once per Gaussian: the blend works in the log2 domain (R30)
    pos_op[i] = make_float4(means[i * 3], means[i * 3 + 1], means[i * 3 + 2], log2f(opac[i]));
    cov_a[i] = make_float4(Sxx, Sxy, Sxz, Syy);
    cov_b[i] = make_float4(Syz, Szz, dc[0], dc[1]);
    aux[i] = make_float2(dc[2], smax * smax);
    // reading R35: q_max = f32(2 ln(255 o)) from an f64 log (once per Gaussian)
    qmax[i] = (float)__dmul_rn(2.0, log(__dmul_rn(255.0, (double)opac[i])));
    if (sh_out) {
      // float4 planes: plane q4 holds coefficients 4 q4 .. 4 q4 + 3 of every
      // Gaussian (a warp reading neighbouring Gaussians reads one line per plane)
      for (int k = 0; k < sh_stride; ++k)
        sh_out[((size_t)(k >> 2) * n + i) * 4 + (k & 3)] = k < K * 3 ? sh[i * K * 3 + k] : 0.f;
    }
  }
}

void launch_validate(int64_t n, int K, const float* means, const float* scales, const float* quats,
                     const float* opac, const float* sh, ValidateOut* out, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  validate_kernel<<<blocks, 256, 0, s>>>(n, K, means, scales, quats, opac, sh, out);
}

void launch_pack(int64_t n, int K, int sh_stride, const float* means, const float* scales,
                 const float* quats, const float* opac, const float* sh, float4* pos_op, float4* cov_a,
                 float4* cov_b, float2* aux, float* qmax, float* sh_out, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack_kernel<<<blocks, 256, 0, s>>>(n, K, sh_stride, means, scales, quats, opac, sh, pos_op, cov_a,
                                     cov_b, aux, qmax, sh_out);
}

}  // namespace gg
