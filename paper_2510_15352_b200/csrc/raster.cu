// raster.cu — K6: per (env, 16x16 tile) front-to-back compositing.
//
// Per pixel (SPEC.md:145-153 composite_tile; DESIGN.md §2 O4-O5):
//   for each Gaussian i of the tile's depth-sorted list:
//     q = d^T Sigma2^-1 d (d = mean - pixel centre), q >= 0        (R1, R13)
//     alpha = min(0.99, o exp(-q/2)); skip if alpha < 1/255       (R10, R11)
//     T' = T (1 - alpha); stop (i not blended) if T' < 1e-4        (R12)
//     w = alpha T; C += w c; D += w z; A += w; T = T'
//   rgb = C + T bg (R15); depth = D / A or 0 (R14); alpha = A
//
// Decomposition: one CTA of 256 threads per (tile, env), one pixel per
// thread; warp w covers an 8x4 pixel block.  Records are staged in shared
// memory 256 at a time (3 x 128-bit loads each, gathered through the
// tile's sorted index list).  Each record carries the half extents of its
// alpha >= 1/255 ellipse (computed in K1b with safety margins), so a warp
// whose 8x4 block lies outside skips it with one uniform branch — this
// never changes a blend decision, it only avoids evaluating pixels whose
// alpha is below the cutoff.  Early-out: warp vote (__all_sync) ends a
// warp's walk; __syncthreads_count ends the tile.
#include "gg_internal.cuh"

namespace gg {

struct CounterOut {
  unsigned long long* env_counts;   // [E][4] (n_eval, n_contrib, V, K); null = off
  int32_t* dbg_neval;               // [H*W] per-pixel n_eval of the debug env, or null
  int dbg_eloc;                     // chunk-local debug env, -1 = none
};

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <bool COUNTERS>
__global__ void __launch_bounds__(TILE_PX)
raster_kernel(int e0, const EnvConst* __restrict__ envs, RenderParams rp, ChunkWS ws, void* __restrict__ rgb,
              float* __restrict__ depth, float* __restrict__ alpha_out, CounterOut co) {
  __shared__ float4 s0[TILE_PX], s1[TILE_PX], s2[TILE_PX];
  const int eloc = blockIdx.y;
  const int tile = blockIdx.x;
  const int e = envs[e0 + eloc].out_index;   // caller's env index
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tile % rp.TX, ty = tile / rp.TX;
  const int bx = warp & 1, by = warp >> 1;
  const int px = tx * TILE + bx * 8 + (lane & 7);
  const int py = ty * TILE + by * 4 + (lane >> 3);
  const bool inside = px < rp.W && py < rp.H;
  const float fpx = (float)px + 0.5f, fpy = (float)py + 0.5f;
  const float wx0 = (float)(tx * TILE + bx * 8) + 0.5f, wx1 = wx0 + 7.f;
  const float wy0 = (float)(ty * TILE + by * 4) + 0.5f, wy1 = wy0 + 3.f;

  const uint2 rg = ws.ranges[(size_t)eloc * rp.ntiles + tile];
  const uint64_t kb = ws.k_base[eloc];
  const uint64_t rb = ws.rec_base[eloc];
  const uint32_t* __restrict__ list = ws.sorted + kb;

  float T = 1.f, Cr = 0.f, Cg = 0.f, Cb = 0.f, Dn = 0.f, Aw = 0.f;
  bool done = !inside;
  uint32_t ne = 0, nc = 0;
  const float kExp = -0.72134752044448170f;   // -0.5 * log2(e)

  for (uint32_t b = rg.x; b < rg.y; b += TILE_PX) {
    const uint32_t n = min((uint32_t)TILE_PX, rg.y - b);
    __syncthreads();
    if (tid < n) {
      const uint64_t r = rb + __ldg(&list[b + tid]);
      s0[tid] = __ldg(&ws.rec0[r]);
      s1[tid] = __ldg(&ws.rec1[r]);
      s2[tid] = __ldg(&ws.rec2[r]);
    }
    __syncthreads();
    if (!__all_sync(0xffffffffu, done)) {
      for (uint32_t j = 0; j < n; ++j) {
        const float4 a0 = s0[j];
        const float4 a1 = s1[j];
        const float4 a2 = s2[j];
        if (COUNTERS && !done) ++ne;
        // warp-uniform: is this warp's 8x4 block outside the alpha >= 1/255 box?
        if (a1.w < 0.f || a0.x + a1.w < wx0 || a0.x - a1.w > wx1 || a0.y + a2.w < wy0 ||
            a0.y - a2.w > wy1)
          continue;
        if (!done) {
          const float dx = a0.x - fpx, dy = a0.y - fpy;
          float q = a1.x * dx * dx + 2.f * a1.y * dx * dy + a1.z * dy * dy;
          q = fmaxf(q, 0.f);
          const float al = fminf(0.99f, a0.z * ex2_approx(kExp * q));
          if (al >= (1.f / 255.f)) {
            const float Tn = T * (1.f - al);
            if (Tn < 1e-4f) {
              done = true;
            } else {
              const float w = al * T;
              Cr += w * a2.x; Cg += w * a2.y; Cb += w * a2.z;
              Dn += w * a0.w;
              Aw += w;
              T = Tn;
              if (COUNTERS) ++nc;
            }
          }
        }
        if ((j & 7) == 7 && __all_sync(0xffffffffu, done)) break;
      }
    }
    if (__syncthreads_count(done) == TILE_PX) break;
  }

  if (inside) {
    const size_t p = ((size_t)e * rp.H + py) * rp.W + px;
    const float r = Cr + T * rp.bg[0], g = Cg + T * rp.bg[1], bl = Cb + T * rp.bg[2];
    if (rgb) {
      if (rp.rgb_format == 0) {
        uint8_t* o = reinterpret_cast<uint8_t*>(rgb) + p * 3;
        o[0] = (uint8_t)__float2uint_rn(fminf(fmaxf(r, 0.f), 1.f) * 255.f);
        o[1] = (uint8_t)__float2uint_rn(fminf(fmaxf(g, 0.f), 1.f) * 255.f);
        o[2] = (uint8_t)__float2uint_rn(fminf(fmaxf(bl, 0.f), 1.f) * 255.f);
      } else {
        float* o = reinterpret_cast<float*>(rgb) + p * 3;
        o[0] = r; o[1] = g; o[2] = bl;
      }
    }
    if (depth) depth[p] = Aw > 0.f ? Dn / Aw : 0.f;
    if (alpha_out) alpha_out[p] = Aw;
  }
  if (COUNTERS) {
    if (co.dbg_neval && eloc == co.dbg_eloc && inside) co.dbg_neval[py * rp.W + px] = (int32_t)ne;
    unsigned long long a = ne, c = nc;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    if (lane == 0 && co.env_counts) {
      atomicAdd(&co.env_counts[(size_t)e * 4 + 0], a);
      atomicAdd(&co.env_counts[(size_t)e * 4 + 1], c);
    }
    if (tid == 0 && tile == 0 && co.env_counts) {
      co.env_counts[(size_t)e * 4 + 2] = ws.vcnt[eloc];
      co.env_counts[(size_t)e * 4 + 3] = ws.kcnt[eloc];
    }
  }
}

void launch_raster(int e0, int ec, const EnvConst* envs, const RenderParams& rp, const ChunkWS& ws, void* rgb,
                   float* depth, float* alpha, bool counters, unsigned long long* env_counts, int32_t* dbg_neval,
                   int dbg_eloc, cudaStream_t s) {
  CounterOut co{env_counts, dbg_neval, dbg_eloc};
  dim3 grid(rp.ntiles, ec);
  if (counters)
    raster_kernel<true><<<grid, TILE_PX, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha, co);
  else
    raster_kernel<false><<<grid, TILE_PX, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha, co);
}

}  // namespace gg
