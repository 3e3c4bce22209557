// project.cu — per-env camera setup, K1a cull/count, K2 block scan, K1b projection.
//
// Operation defined by SPEC.md:117-135 (ProjectedGaussian, project_gaussian:
// Sigma' = J W Sigma W^T J^T, +0.3 px^2, cull at the near plane or when the
// 3-sigma footprint misses the image), with the readings of DESIGN.md §2
// (Jacobian clamp R4, eigenvalue floor R6, radius R7, rect R8, SH R16-R18).
// Every value that feeds an integer decision (p, 1/z, u, v, J, Sigma2, det,
// lambda1, r, rect, depth bits) is computed in the canonical f32 order of
// DESIGN.md §2.1 with non-contracting intrinsics (canonical.cuh).
//
// Work decomposition (DESIGN.md §4 K1): grid = (Gaussian blocks of 256,
// envs of the chunk).  Pass 1 (cull_count) does the exact near/far test and
// a CONSERVATIVE footprint test (never rejects a Gaussian the canonical rect
// keeps), writes one visibility bit per (env, Gaussian) and per-block counts.
// A per-env exclusive scan turns the counts into offsets, so pass 2
// (project) compacts the records deterministically in Gaussian order.
#include "gg_internal.cuh"
#include "canonical.cuh"

namespace gg {

__global__ void setup_envs_kernel(int E, const int32_t* __restrict__ scene_ids,
                                  const float* __restrict__ viewmats, const float* __restrict__ intr,
                                  const DevScene* __restrict__ scenes, int nscenes, int W, int H,
                                  int sh_degree, EnvConst* out, uint32_t* err) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  EnvConst c;
  const float* V = viewmats + (size_t)e * 16;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    c.R[r * 3 + 0] = V[r * 4 + 0];
    c.R[r * 3 + 1] = V[r * 4 + 1];
    c.R[r * 3 + 2] = V[r * 4 + 2];
    c.t[r] = V[r * 4 + 3];
  }
  c.fx = intr[e * 4 + 0]; c.fy = intr[e * 4 + 1]; c.cx = intr[e * 4 + 2]; c.cy = intr[e * 4 + 3];
  const float Wf = (float)W, Hf = (float)H;
  const float tan_x = fd(fm(0.5f, Wf), c.fx), tan_y = fd(fm(0.5f, Hf), c.fy);
  c.lim_xp = fa(fd(fs(Wf, c.cx), c.fx), fm(0.3f, tan_x));
  c.lim_xn = fa(fd(c.cx, c.fx), fm(0.3f, tan_x));
  c.lim_yp = fa(fd(fs(Hf, c.cy), c.fy), fm(0.3f, tan_y));
  c.lim_yn = fa(fd(c.cy, c.fy), fm(0.3f, tan_y));
#pragma unroll
  for (int k = 0; k < 3; ++k)
    c.C[k] = -(c.R[0 * 3 + k] * c.t[0] + c.R[1 * 3 + k] * c.t[1] + c.R[2 * 3 + k] * c.t[2]);
  const int sid = scene_ids[e];
  c.pad = 0;
  if (sid < 0 || sid >= nscenes || !scenes[sid].valid) {
    c.scene = -1; c.n = 0; c.degree = 0;
    atomicOr(err, (uint32_t)ERR_BAD_SCENE);
  } else {
    c.scene = sid;
    c.n = scenes[sid].n;
    const int d = scenes[sid].degree;
    c.degree = sh_degree < 0 ? d : min(sh_degree, d);
  }
  out[e] = c;
}

// p = R mu + t in the canonical order: ((R_k0 mu_x + R_k1 mu_y) + R_k2 mu_z) + t_k
__device__ __forceinline__ float3 to_cam(const EnvConst& c, float4 g) {
  float3 p;
  p.x = fa(dot3(c.R[0], g.x, c.R[1], g.y, c.R[2], g.z), c.t[0]);
  p.y = fa(dot3(c.R[3], g.x, c.R[4], g.y, c.R[5], g.z), c.t[1]);
  p.z = fa(dot3(c.R[6], g.x, c.R[7], g.y, c.R[8], g.z), c.t[2]);
  return p;
}

__global__ void __launch_bounds__(PROJ_BLOCK)
cull_count_kernel(int e0, const EnvConst* __restrict__ envs, const DevScene* __restrict__ scenes,
                  RenderParams rp, ChunkWS ws) {
  const int eloc = blockIdx.y;
  const EnvConst& c = envs[e0 + eloc];
  const int i = blockIdx.x * PROJ_BLOCK + threadIdx.x;
  bool keep = false;
  if (i < c.n) {
    const DevScene& sc = scenes[c.scene];
    const float4 g = __ldg(&sc.pos_op[i]);
    const float3 p = to_cam(c, g);
    if (p.z > rp.near_p && p.z <= rp.far_p) {
      const float rz = fd(1.f, p.z);
      const float u = fa(fm(fm(c.fx, p.x), rz), c.cx);
      const float v = fa(fm(fm(c.fy, p.y), rz), c.cy);
      // conservative radius bound: lambda1 <= a + c + sqrt(0.1) and
      // a + c <= s_max^2 |T|_F^2 + 0.6 (DESIGN.md §4 K1a); margins cover f32.
      const float txz = fminf(c.lim_xp, fmaxf(-c.lim_xn, p.x * rz));
      const float tyz = fminf(c.lim_yp, fmaxf(-c.lim_yn, p.y * rz));
      const float J00 = c.fx * rz, J11 = c.fy * rz;
      const float J02 = -c.fx * txz * rz, J12 = -c.fy * tyz * rz;
      float nT = 0.f;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const float t0 = J00 * c.R[j] + J02 * c.R[6 + j];
        const float t1 = J11 * c.R[3 + j] + J12 * c.R[6 + j];
        nT += t0 * t0 + t1 * t1;
      }
      const float smax2 = __ldg(&sc.aux[i]).y;
      const float lam_b = (smax2 * nT + 0.9163f) * 1.001f + 0.01f;
      const float rb = 3.f * sqrtf(lam_b) * 1.001f + 1.5f;
      keep = (u + rb > 0.f) && (u - rb < (float)(rp.TX * TILE)) && (v + rb > 0.f) &&
             (v - rb < (float)(rp.TY * TILE));
    }
  }
  const uint32_t word = __ballot_sync(0xffffffffu, keep);
  __shared__ uint32_t wc[PROJ_BLOCK / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wi = blockIdx.x * (PROJ_BLOCK / 32) + warp;
  if (lane == 0) {
    ws.flags[(size_t)eloc * ws.nwords + wi] = word;
    wc[warp] = __popc(word);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
#pragma unroll
    for (int w = 0; w < PROJ_BLOCK / 32; ++w) s += wc[w];
    ws.blkcnt[(size_t)eloc * ws.nblk + blockIdx.x] = s;
  }
}

// Exclusive scan of per-block counts, in place, one CTA per env.
__global__ void __launch_bounds__(1024) scan_blocks_kernel(uint32_t* data, int nblk, uint32_t* totals) {
  uint32_t* d = data + (size_t)blockIdx.x * nblk;
  __shared__ uint32_t ws[32];
  __shared__ uint32_t carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < nblk; base += 1024) {
    const int i = base + threadIdx.x;
    const uint32_t x = i < nblk ? d[i] : 0u;
    uint32_t s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane == 31) ws[warp] = s;
    __syncthreads();
    if (warp == 0) {
      uint32_t t = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      ws[lane] = t;
    }
    __syncthreads();
    const uint32_t excl = carry + (warp ? ws[warp - 1] : 0u) + s - x;
    if (i < nblk) d[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += ws[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[blockIdx.x] = carry;
}

// Real SH basis with the 3DGS sign convention (reading R17), f32.
__device__ __forceinline__ void sh_eval(int deg, float x, float y, float z, float* Y) {
  Y[0] = 0.28209479177387814f;
  if (deg < 1) return;
  Y[1] = -0.4886025119029199f * y;
  Y[2] = 0.4886025119029199f * z;
  Y[3] = -0.4886025119029199f * x;
  if (deg < 2) return;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[4] = 1.0925484305920792f * xy;
  Y[5] = -1.0925484305920792f * yz;
  Y[6] = 0.31539156525252005f * (2.f * zz - xx - yy);
  Y[7] = -1.0925484305920792f * xz;
  Y[8] = 0.5462742152960396f * (xx - yy);
  if (deg < 3) return;
  Y[9] = -0.5900435899266435f * y * (3.f * xx - yy);
  Y[10] = 2.890611442640554f * xy * z;
  Y[11] = -0.4570457994644658f * y * (4.f * zz - xx - yy);
  Y[12] = 0.3731763325901154f * z * (2.f * zz - 3.f * xx - 3.f * yy);
  Y[13] = -0.4570457994644658f * x * (4.f * zz - xx - yy);
  Y[14] = 1.445305721320277f * z * (xx - yy);
  Y[15] = -0.5900435899266435f * x * (xx - 3.f * yy);
}

__global__ void __launch_bounds__(PROJ_BLOCK)
project_kernel(int e0, const EnvConst* __restrict__ envs, const DevScene* __restrict__ scenes,
               RenderParams rp, ChunkWS ws) {
  const int eloc = blockIdx.y;
  const EnvConst& c = envs[e0 + eloc];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i = blockIdx.x * PROJ_BLOCK + threadIdx.x;
  const uint32_t word = ws.flags[(size_t)eloc * ws.nwords + blockIdx.x * (PROJ_BLOCK / 32) + warp];
  __shared__ uint32_t wc[PROJ_BLOCK / 32];
  __shared__ uint32_t ktot[PROJ_BLOCK / 32];
  if (lane == 0) wc[warp] = __popc(word);
  __syncthreads();
  uint32_t wpre = 0;
  for (int w = 0; w < warp; ++w) wpre += wc[w];
  uint32_t ntiles = 0;
  if ((word >> lane) & 1u) {
    const size_t r = ws.rec_base[eloc] + ws.blkcnt[(size_t)eloc * ws.nblk + blockIdx.x] + wpre +
                     __popc(word & lanemask_lt());
    const DevScene& sc = scenes[c.scene];
    const float4 g = __ldg(&sc.pos_op[i]);
    const float4 ca = __ldg(&sc.cov_a[i]);
    const float4 cb = __ldg(&sc.cov_b[i]);
    const float2 ax = __ldg(&sc.aux[i]);
    // O2.1 p = R mu + t, 1/z (canonical)
    const float3 p = to_cam(c, g);
    const float rz = fd(1.f, p.z);
    // O2.6 mean (unclamped p)
    const float u = fa(fm(fm(c.fx, p.x), rz), c.cx);
    const float v = fa(fm(fm(c.fy, p.y), rz), c.cy);
    // O2.2 clamped Jacobian
    const float txz = fminf(c.lim_xp, fmaxf(-c.lim_xn, fm(p.x, rz)));
    const float tyz = fminf(c.lim_yp, fmaxf(-c.lim_yn, fm(p.y, rz)));
    const float xc = fm(p.z, txz), yc = fm(p.z, tyz);
    const float J00 = fm(c.fx, rz), J11 = fm(c.fy, rz);
    const float J02 = -fm(fm(fm(c.fx, xc), rz), rz);
    const float J12 = -fm(fm(fm(c.fy, yc), rz), rz);
    // O2.3 T = J W ; U = T Sigma3 ; S = U T^T
    float T0[3], T1[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      T0[j] = fa(fm(J00, c.R[j]), fm(J02, c.R[6 + j]));
      T1[j] = fa(fm(J11, c.R[3 + j]), fm(J12, c.R[6 + j]));
    }
    const float S[3][3] = {{ca.x, ca.y, ca.z}, {ca.y, ca.w, cb.x}, {ca.z, cb.x, cb.y}};
    float U0[3], U1[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      U0[j] = dot3(T0[0], S[0][j], T0[1], S[1][j], T0[2], S[2][j]);
      U1[j] = dot3(T1[0], S[0][j], T1[1], S[1][j], T1[2], S[2][j]);
    }
    const float a = fa(dot3(U0[0], T0[0], U0[1], T0[1], U0[2], T0[2]), 0.3f);
    const float b = dot3(U0[0], T1[0], U0[1], T1[1], U0[2], T1[2]);
    const float cc = fa(dot3(U1[0], T1[0], U1[1], T1[1], U1[2], T1[2]), 0.3f);
    // O2.4 det, conic
    const float det = fs(fm(a, cc), fm(b, b));
    uint32_t x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    float cA = 0.f, cB = 0.f, cC = 0.f;
    if (det > 0.f) {
      cA = fd(cc, det); cB = fd(-b, det); cC = fd(a, det);
      // O2.5 radius
      const float mid = fm(0.5f, fa(a, cc));
      const float lam1 = fa(mid, fsq(fmaxf(0.1f, fs(fm(mid, mid), det))));
      const float rr = ceilf(fm(3.f, fsq(lam1)));
      // O2.7 tile rect
      const float fx0 = fminf(fmaxf(floorf(fm(fs(u, rr), 0.0625f)), 0.f), (float)rp.TX);
      const float fx1 = fminf(fmaxf(ceilf(fm(fa(u, rr), 0.0625f)), 0.f), (float)rp.TX);
      const float fy0 = fminf(fmaxf(floorf(fm(fs(v, rr), 0.0625f)), 0.f), (float)rp.TY);
      const float fy1 = fminf(fmaxf(ceilf(fm(fa(v, rr), 0.0625f)), 0.f), (float)rp.TY);
      if (fx0 < fx1 && fy0 < fy1) {
        x0 = (uint32_t)fx0; x1 = (uint32_t)fx1; y0 = (uint32_t)fy0; y1 = (uint32_t)fy1;
        ntiles = (x1 - x0) * (y1 - y0);
      }
    }
    // O2.8 colour
    float col[3];
    if (c.degree == 0) {
      col[0] = cb.z; col[1] = cb.w; col[2] = ax.x;
    } else {
      float dx = g.x - c.C[0], dy = g.y - c.C[1], dz = g.z - c.C[2];
      const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
      dx *= inv; dy *= inv; dz *= inv;
      float Y[16];
      sh_eval(c.degree, dx, dy, dz, Y);
      const int K = (c.degree + 1) * (c.degree + 1);
      const float* f = sc.sh + (size_t)i * sc.sh_stride;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f;
      for (int k = 0; k < K; ++k) {
        s0 += Y[k] * __ldg(&f[k * 3 + 0]);
        s1 += Y[k] * __ldg(&f[k * 3 + 1]);
        s2 += Y[k] * __ldg(&f[k * 3 + 2]);
      }
      col[0] = fminf(1.f, fmaxf(0.f, s0 + 0.5f));
      col[1] = fminf(1.f, fmaxf(0.f, s1 + 0.5f));
      col[2] = fminf(1.f, fmaxf(0.f, s2 + 0.5f));
    }
    // blend-side culling extents: alpha >= 1/255 needs q <= 2 ln(255 o);
    // the ellipse's half extents are sqrt(qmax * Sigma2_xx), sqrt(qmax * Sigma2_yy)
    // (+ margins, so the skip never changes a blend decision).
    const float o = g.w;
    float ex = -1.f, ey = -1.f;
    if (o * 255.f > 1.f) {
      const float qmax = 2.f * logf(255.f * o);
      ex = sqrtf(qmax * a) * 1.002f + 0.02f;
      ey = sqrtf(qmax * cc) * 1.002f + 0.02f;
    }
    ws.rec0[r] = make_float4(u, v, o, p.z);
    ws.rec1[r] = make_float4(cA, cB, cC, ex);
    ws.rec2[r] = make_float4(col[0], col[1], col[2], ey);
    ws.rect[r] = make_uint2(x0 | (x1 << 16), y0 | (y1 << 16));
    ws.zkey[r] = __float_as_uint(p.z);
    ws.gid[r] = (uint32_t)i;
  }
  // per-env key count (integer atomics: order-independent, deterministic)
  uint32_t s = ntiles;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) ktot[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int w = 0; w < PROJ_BLOCK / 32; ++w) t += ktot[w];
    if (t) atomicAdd(&ws.kcnt[eloc], t);
  }
}

void launch_setup_envs(int E, const int32_t* scene_ids, const float* viewmats, const float* intr,
                       const DevScene* scenes, int nscenes, int W, int H, int sh_degree, EnvConst* out,
                       uint32_t* err, cudaStream_t s) {
  setup_envs_kernel<<<(E + 127) / 128, 128, 0, s>>>(E, scene_ids, viewmats, intr, scenes, nscenes, W, H,
                                                    sh_degree, out, err);
}

void launch_cull_count(int e0, int ec, int nblk, const EnvConst* envs, const DevScene* scenes,
                       const RenderParams& rp, const ChunkWS& ws, cudaStream_t s) {
  cull_count_kernel<<<dim3(nblk, ec), PROJ_BLOCK, 0, s>>>(e0, envs, scenes, rp, ws);
}

void launch_scan_blocks(int ec, int nblk, uint32_t* data, uint32_t* totals, cudaStream_t s) {
  scan_blocks_kernel<<<ec, 1024, 0, s>>>(data, nblk, totals);
}

void launch_project(int e0, int ec, int nblk, const EnvConst* envs, const DevScene* scenes,
                    const RenderParams& rp, const ChunkWS& ws, cudaStream_t s) {
  project_kernel<<<dim3(nblk, ec), PROJ_BLOCK, 0, s>>>(e0, envs, scenes, rp, ws);
}

}  // namespace gg
