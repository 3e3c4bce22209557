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
// Work decomposition (DESIGN.md §4 K1).  Envs are processed scene-sorted and
// split into groups of <= 16 envs bound to one scene.  A CTA owns one block
// of 256 Gaussians x one env group, and the grid runs env groups fastest so
// consecutive CTAs reuse the same Gaussian block from L2 (the scene is read
// from HBM about once per chunk, not once per env):
//   K1a cull_count: each thread holds one Gaussian in registers and tests it
//       against every camera of the group — exact near/far test plus a
//       CONSERVATIVE footprint test that never rejects a Gaussian the
//       canonical rect keeps — one ballot word per (env, 32 Gaussians) and a
//       count per (env, block).
//   K2  scan: per-env exclusive scan of the block counts (compaction offsets).
//   K1b project: the CTA flattens the visible (env, Gaussian) pairs of the
//       group in (Gaussian, env) order (lanes that share a Gaussian read the
//       same scene lines through L1), projects them with full warps (SH at a
//       compile-time degree; optional R35 tight rect and R37 tile mask), and
//       writes each record at its compacted, Gaussian-ordered slot (its rank
//       among the env's visible Gaussians).
#include "gg_internal.cuh"
#include "canonical.cuh"

namespace gg {

__global__ void setup_envs_kernel(int E, const int32_t* __restrict__ perm, const int32_t* __restrict__ scene_ids,
                                  const float* __restrict__ viewmats, const float* __restrict__ intr,
                                  const DevScene* __restrict__ scenes, int nscenes, int W, int H,
                                  int sh_degree, EnvConst* out, uint32_t* err) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= E) return;
  const int e = perm ? perm[pos] : pos;
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
  {
    // sum_j (a R0j + b R2j)^2 <= (a^2 + b^2) lambda_max(Gram(R0, R2)) <= (a^2 + b^2)(max(|R0|^2,|R2|^2) + |R0.R2|)
    float a[3], cr[2];
#pragma unroll
    for (int r = 0; r < 3; ++r) a[r] = c.R[r * 3] * c.R[r * 3] + c.R[r * 3 + 1] * c.R[r * 3 + 1] + c.R[r * 3 + 2] * c.R[r * 3 + 2];
    cr[0] = c.R[0] * c.R[6] + c.R[1] * c.R[7] + c.R[2] * c.R[8];
    cr[1] = c.R[3] * c.R[6] + c.R[4] * c.R[7] + c.R[5] * c.R[8];
    c.rgram = fmaxf(fmaxf(a[0], a[2]) + fabsf(cr[0]), fmaxf(a[1], a[2]) + fabsf(cr[1])) * 1.0001f;
  }
  const int sid = scene_ids[e];
  c.out_index = e;
  if (sid < 0 || sid >= nscenes || !scenes[sid].valid) {
    c.scene = -1; c.n = 0; c.degree = 0;
    atomicOr(err, (uint32_t)ERR_BAD_SCENE);
  } else {
    c.scene = sid;
    c.n = scenes[sid].n;
    const int d = scenes[sid].degree;
    c.degree = sh_degree < 0 ? d : min(sh_degree, d);
  }
  out[pos] = c;
}

// Processing order of a sync-free render's envs (GG_ASYNC; the sync path
// sorts on the host, api.cu): by scene, then view cell (the forward axis's
// cube face and quadrant), then the Morton code of the camera centre in the
// batch's bounding box -- so the 16 envs of a projection group tend to share
// a scene and see the same storage blocks.  Only a work heuristic: every
// env's outputs go to its caller index, so any order gives the same frames.
// One CTA; (key << 32 | env) sorted by a shared-memory bitonic network
// (unique keys: deterministic); E <= ENV_ORDER_MAX, N = E rounded up to a
// power of two.
__device__ __forceinline__ float3 cam_centre(const float* V) {
  float c[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    const float x = -(V[0 * 4 + k] * V[3] + V[1 * 4 + k] * V[7] + V[2 * 4 + k] * V[11]);
    c[k] = isfinite(x) ? x : 0.f;
  }
  return make_float3(c[0], c[1], c[2]);
}

__global__ void __launch_bounds__(1024) env_order_kernel(int E, int N, const int32_t* __restrict__ scene_ids,
                                                         const float* __restrict__ viewmats, int nscenes,
                                                         const DevScene* __restrict__ scenes, int32_t* perm) {
  extern __shared__ unsigned long long so[];   // [N]
  __shared__ float red[6][32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  float lo[3] = {3.0e38f, 3.0e38f, 3.0e38f}, hi[3] = {-3.0e38f, -3.0e38f, -3.0e38f};
  for (int e = tid; e < E; e += 1024) {
    const float3 c = cam_centre(viewmats + (size_t)e * 16);
    lo[0] = fminf(lo[0], c.x); lo[1] = fminf(lo[1], c.y); lo[2] = fminf(lo[2], c.z);
    hi[0] = fmaxf(hi[0], c.x); hi[1] = fmaxf(hi[1], c.y); hi[2] = fmaxf(hi[2], c.z);
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = fminf(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = fmaxf(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 3; ++k) { red[k][warp] = lo[k]; red[3 + k][warp] = hi[k]; }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    float l = red[k][lane], h = red[3 + k][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      l = fminf(l, __shfl_xor_sync(0xffffffffu, l, o));
      h = fmaxf(h, __shfl_xor_sync(0xffffffffu, h, o));
    }
    lo[k] = l; hi[k] = h;
  }
  for (int e = tid; e < N; e += 1024) {
    if (e >= E) { so[e] = ~0ull; continue; }
    const float* V = viewmats + (size_t)e * 16;
    const float F[3] = {V[8], V[9], V[10]};   // forward axis (row 2 of R)
    int ax = 0;
    if (fabsf(F[1]) > fabsf(F[ax])) ax = 1;
    if (fabsf(F[2]) > fabsf(F[ax])) ax = 2;
    const float m = fabsf(F[ax]) > 0.f ? fabsf(F[ax]) : 1.f;
    const float a = F[(ax + 1) % 3] / m, b = F[(ax + 2) % 3] / m;
    const uint32_t face = (uint32_t)(2 * ax + (F[ax] < 0.f));
    const uint32_t cell = (a >= 0.f ? 1u : 0u) | (b >= 0.f ? 2u : 0u);
    const float3 c = cam_centre(V);
    const float cc[3] = {c.x, c.y, c.z};
    uint32_t pos = 0;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const float ext = hi[k] - lo[k];
      const uint32_t qk = ext > 0.f ? (uint32_t)fminf(15.f, fmaxf(0.f, (cc[k] - lo[k]) / ext * 16.f)) : 0u;
#pragma unroll
      for (int bb = 0; bb < 4; ++bb) pos |= ((qk >> bb) & 1u) << (3 * bb + k);
    }
    const int sid = scene_ids[e];
    const uint32_t sk = (sid < 0 || sid >= nscenes || !scenes[sid].valid) ? 0xffffu : (uint32_t)min(sid, 0xfffe);
    so[e] = ((unsigned long long)((sk << 16) | ((face * 4 + cell) << 12) | pos) << 32) | (uint32_t)e;
  }
  __syncthreads();
  for (int k = 2; k <= N; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < N / 2; i += 1024) {
        const int l = 2 * i - (i & (j - 1)), r = l + j;
        const bool up = (l & k) == 0;
        const unsigned long long x = so[l], y = so[r];
        if ((x > y) == up) { so[l] = y; so[r] = x; }
      }
      __syncthreads();
    }
  for (int p = tid; p < E; p += 1024) perm[p] = (int32_t)(uint32_t)so[p];
}

// p = R mu + t in the canonical order: ((R_k0 mu_x + R_k1 mu_y) + R_k2 mu_z) + t_k
__device__ __forceinline__ float3 to_cam(const EnvConst& c, float4 g) {
  float3 p;
  p.x = fa(dot3(c.R[0], g.x, c.R[1], g.y, c.R[2], g.z), c.t[0]);
  p.y = fa(dot3(c.R[3], g.x, c.R[4], g.y, c.R[5], g.z), c.t[1]);
  p.z = fa(dot3(c.R[6], g.x, c.R[7], g.y, c.R[8], g.z), c.t[2]);
  return p;
}

__device__ __forceinline__ void load_group_cams(EnvConst* cams, const EnvConst* __restrict__ envs, int e0,
                                                EnvGroup grp) {
  const int words = sizeof(EnvConst) / 4;
  const int* src = reinterpret_cast<const int*>(envs + e0 + grp.elo);
  int* dst = reinterpret_cast<int*>(cams);
  for (int i = threadIdx.x; i < grp.cnt * words; i += blockDim.x) dst[i] = src[i];
}

// single MUFU ops (no denormal range fix-ups): operands here are normal and
// the results only feed margin-protected tests
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqrt_approx(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// conservative footprint test (DESIGN.md §4 K1a): lambda1 <= a + c + sqrt(0.1)
// and a + c <= s_max^2 |T|_F^2 + 0.6; generous margins absorb f32 rounding.
__device__ __forceinline__ bool maybe_visible(const EnvConst& c, float4 g, float smax2, const RenderParams& rp) {
  // p_z in the canonical order (it decides near/far exactly); p_x, p_y only
  // feed the margin-protected footprint test
  const float pz = fa(dot3(c.R[6], g.x, c.R[7], g.y, c.R[8], g.z), c.t[2]);
  if (!(pz > rp.near_p && pz <= rp.far_p)) return false;
  const float px = fmaf(c.R[2], g.z, fmaf(c.R[1], g.y, fmaf(c.R[0], g.x, c.t[0])));
  const float py = fmaf(c.R[5], g.z, fmaf(c.R[4], g.y, fmaf(c.R[3], g.x, c.t[1])));
  const float rz = rcp_approx(pz);             // approximate: the test has margins
  const float u = c.fx * px * rz + c.cx;
  const float v = c.fy * py * rz + c.cy;
  const float txz = fminf(c.lim_xp, fmaxf(-c.lim_xn, px * rz));
  const float tyz = fminf(c.lim_yp, fmaxf(-c.lim_yn, py * rz));
  const float J00 = c.fx * rz, J11 = c.fy * rz;
  const float J02 = -c.fx * txz * rz, J12 = -c.fy * tyz * rz;
  // |T|_F^2 = |J00 R0 + J02 R2|^2 + |J11 R1 + J12 R2|^2 <= rgram (J00^2 + J02^2 + J11^2 + J12^2)
  const float nT = c.rgram * fmaf(J00, J00, fmaf(J02, J02, fmaf(J11, J11, J12 * J12)));
  const float lam_b = (smax2 * nT + 0.9163f) * 1.001f + 0.01f;
  const float rb = 3.f * (lam_b * rsqrt_approx(lam_b)) * 1.002f + 2.f;
  return (u + rb > 0.f) && (u - rb < (float)(rp.TX * TILE)) && (v + rb > 0.f) && (v - rb < (float)(rp.TY * TILE));
}

// Block test (per-scene spatial chunk culling): can any
// Gaussian of a storage block -- means in [lo, hi], scales <= smax -- have a
// non-empty canonical tile rect for this camera?  A NECESSARY condition, so
// a culled block never holds a visible Gaussian:
//   near < p_z <= far for some mean of the box, and the 4 screen-edge
//   conditions u + r > 0, u - r < 16 TX (v alike) with r = ceil(3 sqrt(l1))
//   < 3 sqrt(l1) + 1, l1 <= a + c + 0.32 <= smax^2 |T|_F^2 + 0.92 and
//   |T|_F^2 <= rgram |J|_F^2 <= rgram G / p_z^2, G = fx^2 (1 + limx^2) +
//   fy^2 (1 + limy^2) (clamped Jacobian).  Multiplied by p_z > 0 each edge
//   condition is linear in the mean: e.g. fx p_x + (cx + 3.88) p_z +
//   3 smax sqrt(rgram G) > 0, whose maximum over the box is exact.
// Evaluated in f32 with a relative tolerance that covers its rounding.
__device__ __forceinline__ bool block_may_see(const EnvConst& c, float4 b0, float4 b1, const RenderParams& rp) {
  const float lo[3] = {b0.x, b0.y, b0.z}, hi[3] = {b1.x, b1.y, b1.z};
  float mx[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) mx[k] = fmaxf(fabsf(lo[k]), fabsf(hi[k]));
  // max over the box of n . mu + d, and a bound on the magnitude of its terms
  auto maxlin = [&](float n0, float n1, float n2, float d, float& mag) {
    mag = fabsf(n0) * mx[0] + fabsf(n1) * mx[1] + fabsf(n2) * mx[2] + fabsf(d);
    return fmaxf(n0 * lo[0], n0 * hi[0]) + fmaxf(n1 * lo[1], n1 * hi[1]) + fmaxf(n2 * lo[2], n2 * hi[2]) + d;
  };
  const float rel = 1e-4f;
  float mag;
  const float zmax = maxlin(c.R[6], c.R[7], c.R[8], c.t[2], mag);
  if (zmax + rel * mag + 1e-6f <= rp.near_p) return false;
  const float zmin = -maxlin(-c.R[6], -c.R[7], -c.R[8], -c.t[2], mag);
  if (zmin - rel * mag - 1e-6f > rp.far_p) return false;
  const float limx = fmaxf(c.lim_xp, c.lim_xn), limy = fmaxf(c.lim_yp, c.lim_yn);
  const float G = c.fx * c.fx * (1.f + limx * limx) + c.fy * c.fy * (1.f + limy * limy);
  const float m = 3.f * b0.w * sqrtf(c.rgram * G) * 1.01f;   // 3 smax |J|_F p_z, with slack
  const float CR = 3.88f;                                     // 3 sqrt(0.92) + 1, rounded up
  const float Wp = (float)(rp.TX * TILE), Hp = (float)(rp.TY * TILE);
  // u + r > 0 ; u - r < Wp ; v + r > 0 ; v - r < Hp  (each times p_z)
  const float ax[4] = {c.fx, -c.fx, 0.f, 0.f}, ay[4] = {0.f, 0.f, c.fy, -c.fy};
  const float az[4] = {c.cx + CR, Wp - c.cx + CR, c.cy + CR, Hp - c.cy + CR};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float n0 = ax[e] * c.R[0] + ay[e] * c.R[3] + az[e] * c.R[6];
    const float n1 = ax[e] * c.R[1] + ay[e] * c.R[4] + az[e] * c.R[7];
    const float n2 = ax[e] * c.R[2] + ay[e] * c.R[5] + az[e] * c.R[8];
    const float d = ax[e] * c.t[0] + ay[e] * c.t[1] + az[e] * c.t[2];
    const float v = maxlin(n0, n1, n2, d, mag);
    if (v + m + rel * (mag + m) + 1e-3f <= 0.f) return false;
  }
  return true;
}

// A CTA handles `bpc` consecutive storage blocks of its env group (up to 16,
// api.cu cull_blocks_per_cta): the camera staging is shared and all the
// (env, block) frustum tests run in one step before the per-Gaussian tests.
constexpr int CULL_BPC_MAX = PROJ_BLOCK / ENV_GROUP;   // storage blocks per cull CTA (one test thread per env and block)
template <bool MULTI>   // false: one storage block per CTA (bpc = 1, full env groups)
#ifndef GG_CULL_MINB
#define GG_CULL_MINB 6   // 40 registers; measured: 5 (48 registers) 5.08 vs 4.69 ms per c3 step
#endif
__global__ void __launch_bounds__(PROJ_BLOCK, GG_CULL_MINB)
cull_count_kernel(int e0, const EnvGroup* __restrict__ groups, const EnvConst* __restrict__ envs,
                  const DevScene* __restrict__ scenes, RenderParams rp, ChunkWS ws, int bpc) {
  __shared__ EnvConst cams[ENV_GROUP];
  __shared__ uint32_t wc[2][ENV_GROUP][PROJ_BLOCK / 32];   // double-buffered per processed block
  __shared__ uint32_t bvis[CULL_BPC_MAX];   // bit k: env k may see some Gaussian of block b0 + j
  const EnvGroup grp = group_of(groups, blockIdx.x, ws.ec);
  if (grp.cnt <= 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b0 = MULTI ? blockIdx.y * bpc : blockIdx.y;
  const int b1 = MULTI ? min(ws.nblk, (int)(blockIdx.y + 1) * bpc) : b0 + 1;
  const int nb = b1 - b0;                     // <= CULL_BPC_MAX (launch_cull_count)
  load_group_cams(cams, envs, e0, grp);
  if (threadIdx.x < CULL_BPC_MAX) bvis[threadIdx.x] = 0u;
  __syncthreads();
  // the block tests of all the CTA's storage blocks at once: thread j * 16 + k
  // tests env k against block b0 + j (one barrier for the whole CTA)
  {
    const int j = threadIdx.x / ENV_GROUP, k = threadIdx.x % ENV_GROUP;
    if (j < nb && k < grp.cnt) {
      const EnvConst c = load_cam(&cams[k]);
      const int blk = b0 + j;
      if (c.n > blk * PROJ_BLOCK) {
        const DevScene& sc = scenes[c.scene];
        if (block_may_see(c, __ldg(&sc.bbox[2 * blk]), __ldg(&sc.bbox[2 * blk + 1]), rp))
          atomicOr(&bvis[j], 1u << k);
      }
    }
  }
  __syncthreads();
  int nproc = 0;   // processed (not skipped) blocks: selects the wc buffer
  for (int j = 0; j < nb; ++j) {
    const int blk = b0 + j;
    const uint32_t bv = bvis[j];
    if (bv == 0u) {   // the whole block is outside every camera of the group (CTA-uniform)
      if (lane < grp.cnt) ws.flags[(size_t)(grp.elo + lane) * ws.nwords + blk * (PROJ_BLOCK / 32) + warp] = 0u;
      if (threadIdx.x < grp.cnt) ws.blkcnt[(size_t)(grp.elo + threadIdx.x) * ws.nblk + blk] = 0u;
      continue;
    }
    const int i = blk * PROJ_BLOCK + threadIdx.x;
    int cur = -2;                       // scene whose Gaussian i is in registers
    float4 g = make_float4(0.f, 0.f, 0.f, 0.f);
    float smax2 = 0.f;
    const int wi = blk * (PROJ_BLOCK / 32) + warp;
    // lane k keeps env k's visibility word (no per-env branch in the loop;
    // ENV_GROUP <= 32)
    uint32_t my_word = 0u;
    for (uint32_t bm = bv; bm; bm &= bm - 1u) {   // only the envs whose block test passed (CTA-uniform)
      const int k = __ffs(bm) - 1;
      const EnvConst c = load_cam(&cams[k]);
      if (c.scene != cur) {             // uniform across the CTA
        cur = c.scene;
        if (i < c.n) {
          const DevScene& sc = scenes[c.scene];
          g = __ldg(&sc.pos_op[i]);
          smax2 = __ldg(&sc.aux[i]).y;
        }
      }
      const bool keep = i < c.n && maybe_visible(c, g, smax2, rp);
      const uint32_t word = __ballot_sync(0xffffffffu, keep);
      if (lane == k) my_word = word;
    }
    // two processed blocks that use the same wc buffer are separated by the
    // barrier of the processed block between them
    uint32_t (*w)[PROJ_BLOCK / 32] = wc[nproc & 1];
    ++nproc;
    if (lane < grp.cnt) {
      ws.flags[(size_t)(grp.elo + lane) * ws.nwords + wi] = my_word;
      w[lane][warp] = __popc(my_word);
    }
    __syncthreads();
    if (threadIdx.x < grp.cnt) {
      uint32_t s = 0;
#pragma unroll
      for (int q = 0; q < PROJ_BLOCK / 32; ++q) s += w[threadIdx.x][q];
      ws.blkcnt[(size_t)(grp.elo + threadIdx.x) * ws.nblk + blk] = s;
    }
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

// O2.8 colour at a compile-time SH degree D >= 1: 128-bit loads from the
// scene's float4 coefficient planes ((q, ch) order, zero-padded to a multiple
// of 4; plane q4 at sh4 + q4 n); each channel accumulates q = 0, 1, ... in order.
template <int D>
__device__ __forceinline__ void sh_colour(const float4* __restrict__ f4, int n, float x, float y, float z,
                                          float col[3]) {
  constexpr int KC = (D + 1) * (D + 1);
  constexpr int NF4 = (KC * 3 + 3) / 4;
  float Y[16];
  sh_eval(D, x, y, z, Y);
  float4 sh[NF4];
#pragma unroll
  for (int q4 = 0; q4 < NF4; ++q4) sh[q4] = __ldg(&f4[q4 * n]);
  float acc[3] = {0.f, 0.f, 0.f};
#pragma unroll
  for (int q4 = 0; q4 < NF4; ++q4) {
    const float xs[4] = {sh[q4].x, sh[q4].y, sh[q4].z, sh[q4].w};
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int idx = 4 * q4 + m;
      if (idx < KC * 3) acc[idx % 3] += Y[idx / 3] * xs[m];
    }
  }
#pragma unroll
  for (int ch = 0; ch < 3; ++ch) col[ch] = fminf(1.f, fmaxf(0.f, acc[ch] + 0.5f));
}

// Opacity-aware tile rect (GG_TIGHT_TILES, reading R35): the
// paper rect cut to the tiles whose pixel centres can reach the box of the
// alpha >= 1/255 ellipse {q <= qm} of the f32 conic.  Canonical f32 order
// with conservative rounding bounds (it decides integers: the tile lists).
// Returns q_m (R35), or +inf if the rect stays the paper's (no R37 pruning).
__device__ __forceinline__ float tight_rect(float u, float v, float A, float B, float C, float qmax,
                                            uint32_t& x0, uint32_t& x1, uint32_t& y0, uint32_t& y1) {
  const float INF = __int_as_float(0x7f800000);
  if (!(qmax >= 0.f)) { x0 = x1 = y0 = y1 = 0; return INF; }    // o < 1/255: no pixel blends
  const float AC = fm(A, C), BB = fm(B, B);
  const float Dlo = fs(fs(AC, BB), fm(9.5367431640625e-07f, fa(AC, BB)));   // D >= Dlo
  if (!(Dlo > 0.f) || !(A > 0.f) || !(C > 0.f)) return INF;     // degenerate: keep the paper rect
  const float rD = fd(1.f, Dlo);
  const float mag = fm(fm(qmax, rD), fa(fm(2.f, AC), fm(fm(2.f, fabsf(B)), fsq(AC))));
  const float qm = fa(fa(qmax, 1e-3f), fm(1e-5f, mag));
  const float grow = 1.0000038146972656f;                      // 1 + 2^-18
  const float ex = fm(fsq(fm(fm(qm, C), rD)), grow), ey = fm(fsq(fm(fm(qm, A), rD)), grow);
  const float sx = fa(fa(ex, 0.02f), fm(1e-5f, fabsf(u))), sy = fa(fa(ey, 0.02f), fm(1e-5f, fabsf(v)));
  const float lx = ceilf(fm(fs(fs(u, sx), 15.5f), 0.0625f));
  const float hx = fa(floorf(fm(fs(fa(u, sx), 0.5f), 0.0625f)), 1.f);
  const float ly = ceilf(fm(fs(fs(v, sy), 15.5f), 0.0625f));
  const float hy = fa(floorf(fm(fs(fa(v, sy), 0.5f), 0.0625f)), 1.f);
  const uint32_t nx0 = (uint32_t)fmaxf((float)x0, fminf((float)x1, lx));
  const uint32_t nx1 = (uint32_t)fmaxf((float)x0, fminf((float)x1, hx));
  const uint32_t ny0 = (uint32_t)fmaxf((float)y0, fminf((float)y1, ly));
  const uint32_t ny1 = (uint32_t)fmaxf((float)y0, fminf((float)y1, hy));
  if (nx0 >= nx1 || ny0 >= ny1) { x0 = x1 = y0 = y1 = 0; return qm; }
  x0 = nx0; x1 = nx1; y0 = ny0; y1 = ny1;
  return qm;
}

// R37: does tile (tx, ty)'s rectangle of pixel centres reach {q <= qm}?  The
// minimum of the convex quadratic over the rectangle: 0 if the mean is
// inside, else the least edge minimum.  Same f32 op order as the oracle.
__device__ __forceinline__ bool tile_keeps(float u, float v, float A, float B, float C, float qm, int tx, int ty) {
  const float dxl = fs(fa(fm(16.f, (float)tx), 0.5f), u), dxh = fs(fa(fm(16.f, (float)tx), 15.5f), u);
  const float dyl = fs(fa(fm(16.f, (float)ty), 0.5f), v), dyh = fs(fa(fm(16.f, (float)ty), 15.5f), v);
  if (dxl <= 0.f && dxh >= 0.f && dyl <= 0.f && dyh >= 0.f) return true;
  float best = __int_as_float(0x7f800000), mag = 0.f;
  const float B2 = fm(2.f, B), aA = fabsf(A), aB2 = fm(2.f, fabsf(B)), aC = fabsf(C);
  auto consider = [&](float dx, float dy) {
    const float q = fa(fa(fm(fm(A, dx), dx), fm(fm(B2, dx), dy)), fm(fm(C, dy), dy));
    if (q < best) {
      best = q;
      mag = fa(fa(fm(fm(aA, dx), dx), fm(fm(aB2, fabsf(dx)), fabsf(dy))), fm(fm(aC, dy), dy));
    }
  };
  consider(dxl, fminf(fmaxf(fd(fm(-B, dxl), C), dyl), dyh));
  consider(fminf(fmaxf(fd(fm(-B, dyl), A), dxl), dxh), dyl);
  consider(dxh, fminf(fmaxf(fd(fm(-B, dxh), C), dyl), dyh));
  consider(fminf(fmaxf(fd(fm(-B, dyh), A), dxl), dxh), dyh);
  return best <= fa(fa(qm, 1e-3f), fm(1e-5f, mag));
}

constexpr int SH_MAX = 48;              // floats per Gaussian at degree 3

// Cameras stored field-major (float2 pair q of env k at camT[q][k]): the lanes
// of a warp read the cameras of several envs at once, and a field-major
// 64-bit load of up to 16 envs is one contiguous 128-B row (no bank
// conflicts), where 128-bit loads of whole 112-B records conflicted.
typedef float2 CamWord;
constexpr int CAM_F2 = (int)(sizeof(EnvConst) / sizeof(CamWord));
__device__ __forceinline__ EnvConst load_cam_t(const CamWord (*camT)[ENV_GROUP], int k) {
  EnvConst c;
  CamWord* d = reinterpret_cast<CamWord*>(&c);
#pragma unroll
  for (int q = 0; q < CAM_F2; ++q) d[q] = camT[q][k];
  return c;
}

struct ProjSmem {
  CamWord camT[CAM_F2][ENV_GROUP];
  uint32_t fw[ENV_GROUP * PROJ_WPB];   // visibility words (env, word)
  uint32_t cnt[ENV_GROUP * PROJ_WPB];  // popc per (env, word), then exclusive prefix within the env
  uint32_t kacc[ENV_GROUP];
  uint32_t nunits;
  uint8_t units[ENV_GROUP * PROJ_WPB]; // non-empty (word, env) units, word-major: (w << 4) | k
  uint8_t bitpos[PROJ_BLOCK / 32][32]; // per warp: position of the word's l-th set bit
};

// Work decomposition (DESIGN.md §4 K1b).  A unit = one visibility word (32
// consecutive storage Gaussians) x one env of the group; a warp projects the
// unit's visible Gaussians, lane l taking the l-th set bit.  The unit's
// records are consecutive slots of its env (rank = the set bits before it),
// so a warp's stores are contiguous runs, its scene loads are consecutive
// Gaussians, its camera is warp-uniform, and the warps of the CTA walk the
// block word by word (all envs of word w before word w + 1), so the 32
// Gaussians being projected stay in L1.  With the Morton storage order a
// non-empty word is ~90% full (visibility is spatially coherent).
template <bool ELL, bool MULTI>   // GG_ELLIPSE_TILES (reading R37): per-record tile masks; bpc > 1
#ifndef GG_PROJ_MINB
#define GG_PROJ_MINB (1024 / PROJ_BLOCK)   // 4 CTAs x 256 threads at <= 64 registers
#endif
__global__ void __launch_bounds__(PROJ_BLOCK, GG_PROJ_MINB)
project_kernel(int e0, const EnvGroup* __restrict__ groups, const EnvConst* __restrict__ envs,
               const DevScene* __restrict__ scenes, RenderParams rp, ChunkWS ws, int bpc) {
  __shared__ ProjSmem sm;
  const EnvGroup grp = group_of(groups, blockIdx.x, ws.ec);
  if (grp.cnt <= 0 || !chunk_ok(ws.ok)) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gblk0 = MULTI ? blockIdx.y * bpc : blockIdx.y;
  const int gblk1 = MULTI ? min(ws.nblk, (int)(blockIdx.y + 1) * bpc) : gblk0 + 1;
  // the first block's visibility words are loaded before the camera staging
  // (their latencies overlap instead of adding up across the first barrier)
  static_assert(ENV_GROUP * PROJ_WPB <= PROJ_BLOCK, "one visibility word per thread");
  uint32_t wpre = 0;
  if (tid < ENV_GROUP * PROJ_WPB && tid / PROJ_WPB < grp.cnt)
    wpre = ws.flags[(size_t)(grp.elo + tid / PROJ_WPB) * ws.nwords + gblk0 * PROJ_WPB + tid % PROJ_WPB];
  {
    const CamWord* src = reinterpret_cast<const CamWord*>(envs + e0 + grp.elo);
    for (int i = threadIdx.x; i < grp.cnt * CAM_F2; i += blockDim.x) sm.camT[i % CAM_F2][i / CAM_F2] = src[i];
  }
  if (tid < ENV_GROUP) sm.kacc[tid] = 0;
  for (int gblk = gblk0; gblk < gblk1; ++gblk) {   // bpc storage blocks per CTA (cull_count_kernel)
  const int i0 = gblk * PROJ_BLOCK;
  __syncthreads();   // cameras staged; the previous block's units all processed
  if (tid < ENV_GROUP * PROJ_WPB) {
    const int k = tid / PROJ_WPB, w = tid % PROJ_WPB;
    uint32_t word = wpre;
    if (gblk != gblk0 && k < grp.cnt) word = ws.flags[(size_t)(grp.elo + k) * ws.nwords + gblk * PROJ_WPB + w];
    sm.fw[tid] = word;
    sm.cnt[tid] = __popc(word);
  }
  __syncthreads();
  if (tid < ENV_GROUP) {   // per env: exclusive prefix of its word counts
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < PROJ_WPB; ++w) {
      const uint32_t c = sm.cnt[tid * PROJ_WPB + w];
      sm.cnt[tid * PROJ_WPB + w] = run;
      run += c;
    }
  } else if (warp == 1) {  // non-empty units, word-major (w << 4 | k)
    uint32_t n = 0;
    for (int u0 = 0; u0 < ENV_GROUP * PROJ_WPB; u0 += 32) {
      const int u = u0 + lane, w = u / ENV_GROUP, k = u % ENV_GROUP;
      const bool live = u < ENV_GROUP * PROJ_WPB && sm.fw[k * PROJ_WPB + w] != 0u;
      const uint32_t m = __ballot_sync(0xffffffffu, live);
      if (live) sm.units[n + __popc(m & ((1u << lane) - 1u))] = (uint8_t)((w << 4) | k);
      n += __popc(m);
    }
    if (lane == 0) sm.nunits = n;
  }
  __syncthreads();
  const uint32_t nunits = sm.nunits;
  for (uint32_t j = warp; j < nunits; j += PROJ_BLOCK / 32) {
    const uint32_t unit = sm.units[j];
    const int w = (int)(unit >> 4), k = (int)(unit & 15u);
    const uint32_t word = sm.fw[k * PROJ_WPB + w];
    uint32_t ntiles = 0;
    // lane b with bit b set writes b at its rank among the set bits: lane l
    // then reads the position of the word's l-th visible Gaussian
    if ((word >> lane) & 1u) sm.bitpos[warp][__popc(word & ((1u << lane) - 1u))] = (uint8_t)lane;
    __syncwarp();
    const int bl = sm.bitpos[warp][lane];
    __syncwarp();
    if (lane < __popc(word)) {
      const int l = w * 32 + bl;                                 // the lane-th visible Gaussian of the word
    const EnvConst c = load_cam_t(sm.camT, k);
    const int eloc = grp.elo + k;
    const size_t r = ws.rec_base[eloc] + ws.blkcnt[(size_t)eloc * ws.nblk + gblk] + sm.cnt[k * PROJ_WPB + w] + lane;
    const DevScene& scn = scenes[c.scene];
    const int gi = i0 + l;
    // the scene is read through L1: lanes of a warp share few, adjacent
    // Gaussians (Gaussian-major pair list), reused by the group's envs
    const float4 g = __ldg(&scn.pos_op[gi]);
    const float4 ca = __ldg(&scn.cov_a[gi]);
    const float4 cb = __ldg(&scn.cov_b[gi]);
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
    float qm_r = __int_as_float(0x7f800000);   // R35 q_m (+inf: no R37 pruning)
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
        if (rp.tight) qm_r = tight_rect(u, v, cA, cB, cC, __ldg(&scn.qmax[gi]), x0, x1, y0, y1);
      }
    }
    ntiles = (x1 - x0) * (y1 - y0);
    if (ELL) {
      uint32_t m = 0xffffffffu;
      if (ntiles > 0u && ntiles <= 32u && qm_r < __int_as_float(0x7f800000)) {
        const uint32_t w = x1 - x0;
        m = 0u;
        for (uint32_t b = 0; b < ntiles; ++b) {
          const uint32_t ry = b / w, rx = b - ry * w;
          if (tile_keeps(u, v, cA, cB, cC, qm_r, (int)(x0 + rx), (int)(y0 + ry))) m |= 1u << b;
        }
        ntiles = __popc(m);
      }
      ws.rmask[r] = m;
    }
    // O2.8 colour
    float col[3] = {0.f, 0.f, 0.f};
    const int cdeg = c.degree;
    if (!rp.color) {
      // depth-only render: no colour is consumed
    } else if (cdeg == 0) {
      col[0] = cb.z; col[1] = cb.w; col[2] = __ldg(&scn.aux[gi]).x;
    } else {
      float dx = g.x - c.C[0], dy = g.y - c.C[1], dz = g.z - c.C[2];
      const float inv = rsqrtf(dx * dx + dy * dy + dz * dz);
      dx *= inv; dy *= inv; dz *= inv;
      const float4* f4 = scn.sh4 + gi;
      if (cdeg == 3) sh_colour<3>(f4, scn.n, dx, dy, dz, col);
      else if (cdeg == 2) sh_colour<2>(f4, scn.n, dx, dy, dz, col);
      else sh_colour<1>(f4, scn.n, dx, dy, dz, col);
    }
    // blend-side culling extents: alpha >= 1/255 needs q <= 2 ln(255 o); the
    // ellipse's half extents are sqrt(qmax Sigma2_xx), sqrt(qmax Sigma2_yy)
    // (+ margins, so the skip never changes a blend decision).
    const float L = g.w;                       // log2 opacity (scene store)
    float ex = -1.f, ey = -1.f;
    if (L > -7.99435343685885793f) {           // o > 1/255
      // q <= qmax = 2 ln 2 (log2 o + log2 255); half extents sqrt(qmax Sxx), sqrt(qmax Syy)
      const float qmax = 1.3862943611198906f * (L + 7.99435343685885793f);
      const float qa = qmax * a, qc = qmax * cc;
      ex = qa * rsqrtf(qa) * 1.002f + 0.02f;
      ey = qc * rsqrtf(qc) * 1.002f + 0.02f;
    }
    // record for the blend (DESIGN.md §4 K6): alpha = min(.99, 2^(A'dx^2 + B'dxdy + C'dy^2 + log2 o))
    const float kq = -0.72134752044448170f;   // -0.5 log2(e)
    ws.rec0[r] = make_float4(u, v, L, p.z);
    ws.rec1[r] = make_float4(cA * kq, 2.f * cB * kq, cC * kq, ex);
    ws.rec2[r] = make_float4(col[0], col[1], col[2], ey);
    ws.rect[r] = make_uint2(x0 | (x1 << 16), y0 | (y1 << 16));
    ws.zkey[r] = __float_as_uint(p.z);
    ws.gid[r] = __ldg(&scn.gid[gi]);                  // input index: the depth sort's tie-break
    if (ws.dconic) ws.dconic[r] = make_float4(cA, cB, cC, exp2f(L));
    }
    // the unit's tile keys -> its env's key count (one shared atomic per unit)
    ntiles = __reduce_add_sync(0xffffffffu, ntiles);   // REDUX.SUM: one instruction for the warp total
    if (lane == 0 && ntiles) atomicAdd(&sm.kacc[k], ntiles);
  }
  }   // storage blocks of this CTA
  __syncthreads();
  if (tid < grp.cnt && sm.kacc[tid]) atomicAdd(&ws.kcnt[grp.elo + tid], (unsigned long long)sm.kacc[tid]);
}

cudaError_t project_init() {
  return cudaFuncSetAttribute(env_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, ENV_ORDER_MAX * 8);
}

void launch_setup_envs(int E, const int32_t* perm, const int32_t* scene_ids, const float* viewmats,
                       const float* intr, const DevScene* scenes, int nscenes, int W, int H, int sh_degree,
                       EnvConst* out, uint32_t* err, cudaStream_t s) {
  setup_envs_kernel<<<(E + 127) / 128, 128, 0, s>>>(E, perm, scene_ids, viewmats, intr, scenes, nscenes, W, H,
                                                    sh_degree, out, err);
}

// returns false (no launch: identity order) above ENV_ORDER_MAX envs
bool launch_env_order(int E, const int32_t* scene_ids, const float* viewmats, int nscenes, const DevScene* scenes,
                      int32_t* perm, cudaStream_t s) {
  if (E < 2 || E > ENV_ORDER_MAX) return false;
  int N = 2;
  while (N < E) N <<= 1;
  env_order_kernel<<<1, 1024, (size_t)N * 8, s>>>(E, N, scene_ids, viewmats, nscenes, scenes, perm);
  return true;
}

void launch_cull_count(int e0, int ngroups, int nblk, int bpc, const EnvGroup* groups, const EnvConst* envs,
                       const DevScene* scenes, const RenderParams& rp, const ChunkWS& ws, cudaStream_t s) {
  bpc = std::min(bpc, CULL_BPC_MAX);
  if (bpc > 1)
    cull_count_kernel<true><<<dim3(ngroups, (nblk + bpc - 1) / bpc), PROJ_BLOCK, 0, s>>>(e0, groups, envs, scenes, rp,
                                                                                       ws, bpc);
  else
    cull_count_kernel<false><<<dim3(ngroups, nblk), PROJ_BLOCK, 0, s>>>(e0, groups, envs, scenes, rp, ws, 1);
}

void launch_scan_blocks(int ec, int nblk, uint32_t* data, uint32_t* totals, cudaStream_t s) {
  scan_blocks_kernel<<<ec, 1024, 0, s>>>(data, nblk, totals);
}

void launch_project(int e0, int ngroups, int nblk, int bpc, int max_degree, const EnvGroup* groups,
                    const EnvConst* envs, const DevScene* scenes, const RenderParams& rp, const ChunkWS& ws,
                    cudaStream_t s) {
  const dim3 grid(ngroups, (nblk + bpc - 1) / bpc);
  if (rp.ellipse)
    bpc > 1 ? project_kernel<true, true><<<grid, PROJ_BLOCK, 0, s>>>(e0, groups, envs, scenes, rp, ws, bpc)
            : project_kernel<true, false><<<grid, PROJ_BLOCK, 0, s>>>(e0, groups, envs, scenes, rp, ws, 1);
  else
    bpc > 1 ? project_kernel<false, true><<<grid, PROJ_BLOCK, 0, s>>>(e0, groups, envs, scenes, rp, ws, bpc)
            : project_kernel<false, false><<<grid, PROJ_BLOCK, 0, s>>>(e0, groups, envs, scenes, rp, ws, 1);
}

}  // namespace gg
