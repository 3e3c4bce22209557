// scene_store.cu — K0: validate and pack one scene into the 16-B SoA store.
//
// SPEC.md:28-34 (SplatPrimitive: quaternion normalised, scales > 0,
// opacity in [0,1], DC colour 0.2820948 c + 0.5 clamped) and SPEC.md:130
// (Sigma = R diag(s^2) R^T).  Sigma3 is computed once per Gaussian here in
// the canonical f32 order (DESIGN.md §2.1 "O1") and shared by every env
// bound to the scene ("shared, never copied per environment").
//
// Storage order (per-scene spatial chunk culling): the
// Gaussians are stored in Morton order of their means (10 bits per axis over
// the scene's bounding box; a stable sort, so equal codes keep input order),
// with gid[i] = the input index of stored Gaussian i, and every storage block
// of PROJ_BLOCK Gaussians carries the bounding box of its means and its
// largest scale (bbox), which the cull kernel tests against each camera's
// widened frustum before touching the block's Gaussians.  The canonical list
// order (tile, depth bits, gid) does not depend on storage order: the depth
// sort's ties are put back in gid order (sort_bin.cu "tie fix-up").
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
                            const uint32_t* __restrict__ perm, float4* pos_op, float4* cov_a, float4* cov_b,
                            float2* aux, float* qmax, float* sh_out, uint32_t* gid_out) {
  const float SH_C0 = 0.28209479177387814f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    // storage slot i holds input Gaussian g (Morton order)
    const int64_t g = perm ? (int64_t)perm[i] : i;
    gid_out[i] = (uint32_t)g;
    // O1: q <- q/|q|
    float w = quats[g * 4], x = quats[g * 4 + 1], y = quats[g * 4 + 2], z = quats[g * 4 + 3];
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
    const float s0 = scales[g * 3], s1 = scales[g * 3 + 1], s2 = scales[g * 3 + 2];
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
    for (int c = 0; c < 3; ++c) dc[c] = fminf(1.f, fmaxf(0.f, SH_C0 * sh[g * K * 3 + c] + 0.5f));
    const float smax = fmaxf(s0, fmaxf(s1, s2));
    // log2(o) once per Gaussian: the blend works in the log2 domain (R30)
    pos_op[i] = make_float4(means[g * 3], means[g * 3 + 1], means[g * 3 + 2], log2f(opac[g]));
    cov_a[i] = make_float4(Sxx, Sxy, Sxz, Syy);
    cov_b[i] = make_float4(Syz, Szz, dc[0], dc[1]);
    aux[i] = make_float2(dc[2], smax * smax);
    // reading R35: q_max = f32(2 ln(255 o)) from an f64 log (once per Gaussian)
    qmax[i] = (float)__dmul_rn(2.0, log(__dmul_rn(255.0, (double)opac[g])));
    if (sh_out) {
      // float4 planes: plane q4 holds coefficients 4 q4 .. 4 q4 + 3 of every
      // Gaussian (a warp reading neighbouring Gaussians reads one line per plane)
      for (int k = 0; k < sh_stride; ++k)
        sh_out[((size_t)(k >> 2) * n + i) * 4 + (k & 3)] = k < K * 3 ? sh[g * K * 3 + k] : 0.f;
    }
  }
}

// ---- spatial order ---------------------------------------------------------
// order-preserving map of a finite float to u32 (for atomicMin / atomicMax)
__device__ __forceinline__ uint32_t f2ord(float f) {
  const uint32_t b = __float_as_uint(f);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// box[0..2] = min, box[3..5] = max of the means (ordered-int encoding)
__global__ void aabb_kernel(int64_t n, const float* __restrict__ means, uint32_t* box) {
  uint32_t lo[3] = {0xffffffffu, 0xffffffffu, 0xffffffffu}, hi[3] = {0u, 0u, 0u};
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    for (int k = 0; k < 3; ++k) {
      const uint32_t o = f2ord(means[i * 3 + k]);
      lo[k] = min(lo[k], o);
      hi[k] = max(hi[k], o);
    }
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&box[k], lo[k]);
      atomicMax(&box[3 + k], hi[k]);
    }
  }
}

__device__ __forceinline__ uint32_t spread3(uint32_t x) {   // 10 bits -> every third bit
  x &= 0x3ffu;
  x = (x | (x << 16)) & 0x030000ffu;
  x = (x | (x << 8)) & 0x0300f00fu;
  x = (x | (x << 4)) & 0x030c30c3u;
  x = (x | (x << 2)) & 0x09249249u;
  return x;
}

__global__ void morton_kernel(int64_t n, const float* __restrict__ means, const uint32_t* __restrict__ box,
                              uint32_t* __restrict__ code, uint32_t* __restrict__ idx) {
  float lo[3], sc[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = ord2f(box[k]);
    const float ext = ord2f(box[3 + k]) - lo[k];
    sc[k] = ext > 0.f ? 1023.f / ext : 0.f;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c = 0;
    for (int k = 0; k < 3; ++k) {
      const float t = (means[i * 3 + k] - lo[k]) * sc[k];
      c |= spread3((uint32_t)fminf(fmaxf(t, 0.f), 1023.f)) << k;
    }
    code[i] = c;
    idx[i] = (uint32_t)i;
  }
}

// Stable LSD radix sort of (code, idx) pairs, 4-bit digits, one element per
// thread (load time only: a few microseconds per pass per million elements).
constexpr int MS_THREADS = 256;
constexpr int MS_RADIX = 16;

__global__ void __launch_bounds__(MS_THREADS)
msort_up_kernel(int64_t n, const uint32_t* __restrict__ key, int shift, uint32_t* __restrict__ hist, int64_t nb) {
  __shared__ uint32_t h[MS_RADIX];
  if (threadIdx.x < MS_RADIX) h[threadIdx.x] = 0u;
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)MS_THREADS + threadIdx.x;
  if (i < n) atomicAdd(&h[(key[i] >> shift) & (MS_RADIX - 1)], 1u);
  __syncthreads();
  if (threadIdx.x < MS_RADIX) hist[threadIdx.x * nb + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of hist[0 .. m) in place (digit-major: the offsets of a stable scatter)
__global__ void __launch_bounds__(1024) msort_scan_kernel(uint32_t* hist, int64_t m) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t base = 0; base < m; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint32_t x = i < m ? hist[i] : 0u;
    uint32_t s = x;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane == 31) ws[warp] = s;
    __syncthreads();
    if (warp == 0) {
      uint32_t t = ws[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      ws[lane] = t;
    }
    __syncthreads();
    if (i < m) hist[i] = carry + (warp ? ws[warp - 1] : 0u) + s - x;
    __syncthreads();
    if (threadIdx.x == 0) carry += ws[31];
    __syncthreads();
  }
}

__global__ void __launch_bounds__(MS_THREADS)
msort_down_kernel(int64_t n, const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, int shift,
                  const uint32_t* __restrict__ hist, int64_t nb, uint32_t* __restrict__ kout,
                  uint32_t* __restrict__ vout) {
  __shared__ uint32_t wc[MS_THREADS / 32][MS_RADIX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * (int64_t)MS_THREADS + threadIdx.x;
  const bool ok = i < n;
  const uint32_t k = ok ? kin[i] : 0u;
  const uint32_t d = ok ? (k >> shift) & (MS_RADIX - 1) : MS_RADIX;   // MS_RADIX: no digit
  for (int q = threadIdx.x; q < (MS_THREADS / 32) * MS_RADIX; q += MS_THREADS) (&wc[0][0])[q] = 0u;
  __syncthreads();
  const uint32_t peers = __match_any_sync(0xffffffffu, d);
  const uint32_t lt = (1u << lane) - 1u;
  if (ok && (peers & lt) == 0u) wc[warp][d] = __popc(peers);
  __syncthreads();
  if (ok) {
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += wc[w][d];
    const uint32_t pos = hist[d * nb + blockIdx.x] + before + __popc(peers & lt);
    kout[pos] = k;
    vout[pos] = vin[i];
  }
}

__global__ void block_bounds_kernel(int n, const float4* __restrict__ pos_op, const float2* __restrict__ aux,
                                    float4* __restrict__ bbox) {
  __shared__ float red[7][PROJ_BLOCK / 32];
  const int i = blockIdx.x * PROJ_BLOCK + threadIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const float INF = __int_as_float(0x7f800000);
  float v[7] = {INF, INF, INF, -INF, -INF, -INF, 0.f};
  if (i < n) {
    const float4 p = pos_op[i];
    v[0] = v[3] = p.x; v[1] = v[4] = p.y; v[2] = v[5] = p.z;
    v[6] = sqrtf(aux[i].y);
  }
  for (int o = 16; o > 0; o >>= 1)
    for (int k = 0; k < 7; ++k) {
      const float y = __shfl_xor_sync(0xffffffffu, v[k], o);
      v[k] = k < 3 ? fminf(v[k], y) : fmaxf(v[k], y);
    }
  if (lane == 0)
    for (int k = 0; k < 7; ++k) red[k][warp] = v[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < PROJ_BLOCK / 32; ++w)
      for (int k = 0; k < 7; ++k) v[k] = k < 3 ? fminf(v[k], red[k][w]) : fmaxf(v[k], red[k][w]);
    bbox[2 * blockIdx.x] = make_float4(v[0], v[1], v[2], v[6]);
    bbox[2 * blockIdx.x + 1] = make_float4(v[3], v[4], v[5], 0.f);
  }
}

// Morton permutation of the means: perm[i] = input index of storage slot i.
// tmp: >= 4 n u32 of scratch; perm may alias neither.  Returns the launches.
int launch_spatial_order(int64_t n, const float* means, uint32_t* box, uint32_t* tmp, uint32_t* hist,
                         uint32_t* perm, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  const uint32_t init[6] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0u, 0u, 0u};
  cudaMemcpyAsync(box, init, sizeof init, cudaMemcpyHostToDevice, s);
  aabb_kernel<<<blocks, 256, 0, s>>>(n, means, box);
  uint32_t* k0 = tmp;
  uint32_t* v0 = tmp + n;
  uint32_t* k1 = tmp + 2 * n;
  uint32_t* v1 = perm;
  morton_kernel<<<blocks, 256, 0, s>>>(n, means, box, k0, v0);
  const int64_t nb = (n + MS_THREADS - 1) / MS_THREADS;
  int launches = 2;
  // 8 passes of 4 bits (30-bit codes): ping-pong so the last pass lands in perm
  uint32_t *ka = k0, *va = v0, *kb = k1, *vb = v1;
  for (int p = 0; p < 8; ++p) {
    msort_up_kernel<<<(unsigned)nb, MS_THREADS, 0, s>>>(n, ka, 4 * p, hist, nb);
    msort_scan_kernel<<<1, 1024, 0, s>>>(hist, nb * MS_RADIX);
    msort_down_kernel<<<(unsigned)nb, MS_THREADS, 0, s>>>(n, ka, va, 4 * p, hist, nb, kb, vb);
    launches += 3;
    uint32_t* t;
    t = ka; ka = kb; kb = t;
    t = va; va = vb; vb = t;
  }
  // after 8 (even) passes the sorted values are in v0: copy into perm
  cudaMemcpyAsync(perm, va, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
  return launches;
}

void launch_block_bounds(int n, const float4* pos_op, const float2* aux, float4* bbox, cudaStream_t s) {
  block_bounds_kernel<<<(n + PROJ_BLOCK - 1) / PROJ_BLOCK, PROJ_BLOCK, 0, s>>>(n, pos_op, aux, bbox);
}

void launch_validate(int64_t n, int K, const float* means, const float* scales, const float* quats,
                     const float* opac, const float* sh, ValidateOut* out, cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  validate_kernel<<<blocks, 256, 0, s>>>(n, K, means, scales, quats, opac, sh, out);
}

void launch_pack(int64_t n, int K, int sh_stride, const float* means, const float* scales,
                 const float* quats, const float* opac, const float* sh, const uint32_t* perm, float4* pos_op,
                 float4* cov_a, float4* cov_b, float2* aux, float* qmax, float* sh_out, uint32_t* gid_out,
                 cudaStream_t s) {
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  pack_kernel<<<blocks, 256, 0, s>>>(n, K, sh_stride, means, scales, quats, opac, sh, perm, pos_op, cov_a,
                                     cov_b, aux, qmax, sh_out, gid_out);
}

}  // namespace gg
