// gg_internal.cuh — device-side data layout shared by the kernels of libgg.
// (Product path only; shares nothing with the CPU checker.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace gg {

constexpr int TILE = 16;               // SPEC.md:183 "Tile size 16x16"
constexpr int TILE_PX = TILE * TILE;
#ifndef GG_PROJ_BLOCK
#define GG_PROJ_BLOCK 256   // measured: 512 gives project 8.50 vs 8.36 ms per 1024 envs
#endif
constexpr int PROJ_BLOCK = GG_PROJ_BLOCK;  // Gaussians per projection block (= threads of the cull/project CTAs)
constexpr int PROJ_WPB = PROJ_BLOCK / 32;  // visibility words per (env, block)
constexpr int PROJ_LB = PROJ_BLOCK == 512 ? 9 : 8;   // bits of a block-local Gaussian index
static_assert(PROJ_BLOCK == 256 || PROJ_BLOCK == 512, "projection block size");
constexpr int MAX_TILES = 8192;        // tile table limit (e.g. 1024x2048 px)
constexpr int ENV_ORDER_MAX = 16384;   // sync-free renders order their envs on the device up to this many

// Scene store (SoA, 16-B aligned; DESIGN.md §4 "HBM layout").  O1 results
// (Sigma3, DC colour) are precomputed at load (K0 scene_pack).
struct DevScene {
  const float4* pos_op;  // (x, y, z, log2 opacity)
  const float4* cov_a;   // (Sxx, Sxy, Sxz, Syy)
  const float4* cov_b;   // (Syz, Szz, dc_r, dc_g)
  const float2* aux;     // (dc_b, max_j s_j^2)
  const float* qmax;     // f32(2 ln(255 o)): alpha >= 1/255 <=> q <= qmax (reading R35)
  const float4* sh4;     // [sh_stride/4][n] float4 planes of the (k, ch) coefficients, zero padded; null if d = 0
  const uint32_t* gid;   // [n] input index of each stored Gaussian (storage is in Morton order of the means)
  const float4* bbox;    // [2 * nblk] per PROJ_BLOCK storage block: (lo.xyz, max scale), (hi.xyz, 0)
  int32_t n;
  int32_t degree;
  int32_t sh_stride;     // floats per Gaussian (multiple of 4) = 4 x planes
  int32_t valid;
};

// Per-env camera constants (setup_envs).  f32 values follow the canonical
// order of DESIGN.md §2.1 (they feed integer decisions).
struct __align__(16) EnvConst {
  float R[9];          // world->camera rotation, row-major
  float t[3];
  float fx, fy, cx, cy;
  float lim_xp, lim_xn, lim_yp, lim_yn;   // Jacobian clamp limits (reading R4)
  float C[3];          // camera centre -R^T t (SH view direction)
  int32_t scene;       // index into the scene table, -1 if invalid
  int32_t n;           // Gaussians in that scene (0 if invalid)
  int32_t degree;      // SH degree used at render
  int32_t out_index;   // caller's env index (outputs, counters); envs are processed scene-sorted
  float rgram;         // bound on the Gram matrices of R's row pairs (0,2), (1,2); 1 if R is orthonormal
};
static_assert(sizeof(EnvConst) == 112, "EnvConst: 7 x 16 B (its shared-memory stride avoids bank conflicts)");

// 128-bit loads of a camera from shared memory (7 x LDS.128 instead of 28 LDS)
__device__ __forceinline__ EnvConst load_cam(const EnvConst* p) {
  EnvConst c;
  const float4* s = reinterpret_cast<const float4*>(p);
  float4* d = reinterpret_cast<float4*>(&c);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(EnvConst) / 16); ++i) d[i] = s[i];
  return c;
}

// A run of <= ENV_GROUP chunk-local envs bound to the same scene; the
// projection kernels load each Gaussian once and test it against the group.
#ifndef GG_ENV_GROUP
#define GG_ENV_GROUP 16   // measured: project stage 45.4 (8), 42.9 (16), 46.6 (24) ms per c3 step
#endif
constexpr int ENV_GROUP = GG_ENV_GROUP;
static_assert(ENV_GROUP <= 32, "cull_count keeps one env per lane");
struct EnvGroup {
  int32_t elo;   // first chunk-local env
  int32_t cnt;   // envs in the group (1..ENV_GROUP)
};

struct RenderParams {
  int W, H, TX, TY, ntiles;
  float near_p, far_p;
  float bg[3];
  int rgb_format;
  int tight;             // GG_TIGHT_TILES: opacity-aware tile rects (reading R35)
  int color;             // 0 = depth-only render (rgb == null): no SH/colour work
  int ellipse;           // GG_ELLIPSE_TILES: per-record tile masks (reading R37)
  int blur_k, blur_kc, blur_dk;   // fused motion blur: K colour samples, Kc cameras per env, depth sample (0 = off)
};

// Workspace pointers for one env chunk (indices are chunk-local envs).
struct ChunkWS {
  // pass 1 / scan
  uint32_t* flags;      // [Ec][nwords]
  uint32_t* blkcnt;     // [Ec][nblk] -> exclusive offsets in place
  uint32_t* vcnt;       // [Ec]
  unsigned long long* kcnt;   // [Ec] keys per env (64-bit: a per-env total >= 2^32 is detected, not wrapped)
  // records (global index = rec_base[e] + local)
  const uint64_t* rec_base;  // [Ec]
  const uint64_t* k_base;    // [Ec]
  float4* rec0;         // (u, v, log2 opacity, z)
  float4* rec1;         // (A', B', C', ext_x): conic pre-scaled so -q/2 log2(e) = A'dx^2 + B'dxdy + C'dy^2
  float4* rec2;         // (r, g, b, ext_y)
  float4* dconic;       // debug only (null unless intermediates are kept): raw conic A, B, C, opacity
  uint2* rect;          // (x0 | x1<<16, y0 | y1<<16)
  uint32_t* rmask;      // [V] R37 kept-tile masks of <= 32-tile rects (null: variant off)
  uint32_t* zkey;       // f32 bits of z
  uint32_t zbase;       // f32 bits of the near plane: depth-sort key = z bits - zbase, in (0, bits(far) - zbase]
  uint32_t* gid;        // input (gid) index of each record: the tie-break of equal depth keys, debug dumps
  // depth-sort scratch [V]: packed (key - zmin) << 32 | record ping-pong, and
  // the last pass's output (records in depth order)
  uint64_t* dp0; uint64_t* dp1;
  uint32_t* order;
  uint32_t* sorted;     // [K] final record-local indices, tile-major
  uint2* ranges;        // [Ec][ntiles] [start,end) relative to k_base[e]
  const uint32_t* ok;   // chunk validity (async mode: 0 after a capacity overflow); null = always valid
  int nwords, nblk;
  int ec;               // envs in this chunk
};

// A group of envs for the Gaussian-major projection kernels: explicit table
// (sync mode, scene-sorted) or, when the table is null, the fixed groups
// [16 g, 16 g + 16) of the chunk (async mode).  Envs of one group may be
// bound to different scenes; the kernels reload a Gaussian per scene change.
__device__ __forceinline__ EnvGroup group_of(const EnvGroup* groups, int g, int ec) {
  if (groups) return groups[g];
  EnvGroup r;
  r.elo = g * ENV_GROUP;
  r.cnt = min(ENV_GROUP, ec - r.elo);
  return r;
}

__device__ __forceinline__ bool chunk_ok(const uint32_t* ok) { return ok == nullptr || *ok != 0u; }

// gg_load_scene validation: first offending record per class (atomicMin)
struct ValidateOut {
  unsigned long long nonfinite, bad_scale, bad_opacity, zero_quat;
};

// sticky error bits
enum { ERR_BAD_SCENE = 1, ERR_CAPACITY = 2 };

// Tiles of a record (R37): rects of <= 32 tiles may carry a row-major mask of
// kept tiles; ~0u = every tile of the rect.
__device__ __forceinline__ uint32_t rec_mask(const uint32_t* rmask, uint64_t r, uint32_t area) {
  return (rmask && area <= 32u) ? rmask[r] : 0xffffffffu;
}
__device__ __forceinline__ uint32_t rec_tiles(uint32_t mask, uint32_t area) {
  return area <= 32u ? (uint32_t)__popc(mask & (area == 32u ? 0xffffffffu : ((1u << area) - 1u))) : area;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace gg
