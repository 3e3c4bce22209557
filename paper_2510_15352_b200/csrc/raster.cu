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
// Arithmetic in the log2 domain: the record carries the conic pre-scaled
// by -log2(e)/2 and log2(o), so x = A'dx^2 + B'dxdy + C'dy^2 + log2 o is the
// base-2 log of o exp(-q/2); the cutoff is the compare x < log2(1/255)
// BEFORE the exponential, and alpha = min(0.99, ex2(x)) (MUFU.EX2) only for
// Gaussians that can contribute.
//
// Two kernels compute the same images bit for bit:
//  * raster_kernel<COUNTERS> — the reference walk used for GG_COUNTERS (and
//    the per-pixel n_eval dump): one CTA of 256 threads per (tile, env), one
//    pixel per thread, records staged 256 at a time, every list entry counted
//    as the definition's n_eval;
//  * raster_warp_kernel<RGB> — the timed path (see its comment below): warps
//    walk the list independently for their 8x8 blocks, two pixels per lane in
//    packed f32x2, skipping records whose alpha >= 1/255 region cannot reach
//    the block (exact, conservative), branch-free blending.
// Skipping a record that cannot pass never changes a blend decision.
#include "gg_internal.cuh"
#include "f32x2.cuh"

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

constexpr float LOG2_CUTOFF = -7.99435343685885793f;   // log2(1/255)
constexpr float LOG2_099 = -0.014499569695115089f;      // log2(0.99): the alpha cap as an exponent bound

// The exponent x(d) = A'dx^2 + B'dxdy + C'dy^2 + log2 o (d = mean - pixel
// centre) expanded around the tile's first pixel centre (tox, toy): with
// D = mean - (tox, toy) and the pixel's offset (lx, ly) in the tile,
//   x = c0 + lx (c1 + A' lx) + ly (c2 + B' lx + C' ly),
//   c0 = x(D), c1 = -(2A'Dx + B'Dy), c2 = -(B'Dx + 2C'Dy).
// Both raster kernels evaluate exactly this sequence (bit-identical images).
// Returns (c0, -c1, -c2, w) with w = min(log2 o, log2 0.99): alpha = 2^min(x, w)
// is min(0.99, o e^(-q/2)) with q >= 0 enforced (R10, R13).  c1, c2 are kept
// negated: the walks add them with a negated FFMA operand (free, and exact),
// which saves the loader two negations.
template <bool NEG = true>   // false: (c0, c1, c2, w) (the blur walk: fewer spills there)
__device__ __forceinline__ float4 tile_coefs(const float4 a0, const float4 a1, float tox, float toy) {
  const float Dx = a0.x - tox, Dy = a0.y - toy;
  const float c0 = fmaf(Dx, fmaf(a1.x, Dx, a1.y * Dy), fmaf(a1.z * Dy, Dy, a0.z));
  const float c1n = fmaf(2.f * a1.x, Dx, a1.y * Dy);   // -c1
  const float c2n = fmaf(2.f * a1.z, Dy, a1.y * Dx);   // -c2
  return NEG ? make_float4(c0, c1n, c2n, fminf(a0.z, LOG2_099)) : make_float4(c0, -c1n, -c2n, fminf(a0.z, LOG2_099));
}

// One pixel-Gaussian step (R12-R15 with the R30 log2-domain cutoff).  s0 =
// (c0, -c1, -c2, w), s1 = (A', B', C', z), s2 = (r, g, b, -).  Alpha is not
// accumulated: A = 1 - T at the end (R15).
__device__ __forceinline__ void blend_step(const float4 s0, const float4 s1, const float4 s2, float lx, float ly,
                                           float& T, float& Cr, float& Cg, float& Cb, float& Dn,
                                           bool& done, uint32_t& nc) {
  const float P = fmaf(lx, fmaf(s1.x, lx, -s0.y), s0.x);
  const float Q = fmaf(s1.y, lx, -s0.z);
  const float x = fminf(fmaf(ly, fmaf(s1.z, ly, Q), P), s0.w);
  if (x >= LOG2_CUTOFF) {
    const float al = ex2_approx(x);
    const float w = al * T;
    const float Tn = T - w;
    if (Tn < 1e-4f) {
      done = true;
    } else {
      Cr = fmaf(w, s2.x, Cr);
      Cg = fmaf(w, s2.y, Cg);
      Cb = fmaf(w, s2.z, Cb);
      Dn = fmaf(w, s1.w, Dn);
      T = Tn;
      ++nc;
    }
  }
}

// Outputs of one pixel (O5): rgb = C + T bg; A = 1 - T (= sum of the weights,
// R15); depth = Dn / A, 0 where nothing was blended (T = 1 exactly).
__device__ __forceinline__ void write_pixel(const RenderParams& rp, void* rgb, float* depth, float* alpha_out,
                                            size_t p, float T, float Cr, float Cg, float Cb, float Dn) {
  const float r = fmaf(T, rp.bg[0], Cr), g = fmaf(T, rp.bg[1], Cg), bl = fmaf(T, rp.bg[2], Cb);
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
  const float A = 1.f - T;
  if (depth) depth[p] = A > 0.f ? Dn / A : 0.f;
  if (alpha_out) alpha_out[p] = A;
}

template <bool COUNTERS>
__global__ void __launch_bounds__(TILE_PX)
raster_kernel(int e0, const EnvConst* __restrict__ envs, RenderParams rp, ChunkWS ws, void* __restrict__ rgb,
              float* __restrict__ depth, float* __restrict__ alpha_out, CounterOut co) {
  __shared__ float4 srec[TILE_PX * 3];           // record j at srec[3j .. 3j+2]
  __shared__ uint8_t smask[TILE_PX];
  __shared__ uint8_t wlist[TILE_PX / 32][TILE_PX];   // per-warp relevant records
  const int eloc = blockIdx.y;
  const int tile = blockIdx.x;
  const int e = envs[e0 + eloc].out_index;   // caller's env index
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tile % rp.TX, ty = tile / rp.TX;
  const int bx = warp & 1, by = warp >> 1;
  const int px = tx * TILE + bx * 8 + (lane & 7);
  const int py = ty * TILE + by * 4 + (lane >> 3);
  const bool inside = px < rp.W && py < rp.H;
  const float lx = (float)(px - tx * TILE), ly = (float)(py - ty * TILE);   // offset in the tile
  // pixel-centre extents of the tile's warp blocks (columns: 2 x 8 px, rows: 4 x 4 px)
  const float tx0 = (float)(tx * TILE) + 0.5f, ty0 = (float)(ty * TILE) + 0.5f;

  const uint2 rg = chunk_ok(ws.ok) ? ws.ranges[(size_t)eloc * rp.ntiles + tile] : make_uint2(0u, 0u);
  const uint64_t kb = ws.k_base[eloc];
  const uint64_t rb = ws.rec_base[eloc];
  const uint32_t* __restrict__ list = ws.sorted + kb;

  float T = 1.f, Cr = 0.f, Cg = 0.f, Cb = 0.f, Dn = 0.f;
  bool done = !inside;
  uint32_t ne = 0, nc = 0;

  for (uint32_t b = rg.x; b < rg.y; b += TILE_PX) {
    const uint32_t n = min((uint32_t)TILE_PX, rg.y - b);
    __syncthreads();
    if (tid < n) {
      const uint64_t r = rb + __ldg(&list[b + tid]);
      const float4 a0 = __ldg(&ws.rec0[r]);
      const float4 a1 = __ldg(&ws.rec1[r]);
      const float4 a2 = __ldg(&ws.rec2[r]);
      srec[3 * tid] = tile_coefs(a0, a1, tx0, ty0);
      srec[3 * tid + 1] = make_float4(a1.x, a1.y, a1.z, a0.w);
      srec[3 * tid + 2] = a2;
      uint32_t m = 0;
      if (a1.w >= 0.f) {
        const float xl = a0.x - a1.w, xh = a0.x + a1.w, yl = a0.y - a2.w, yh = a0.y + a2.w;
        uint32_t cm = 0, rm = 0;
#pragma unroll
        for (int c = 0; c < 2; ++c)
          if (xh >= tx0 + 8.f * c && xl <= tx0 + 8.f * c + 7.f) cm |= 1u << c;
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4)
          if (yh >= ty0 + 4.f * r4 && yl <= ty0 + 4.f * r4 + 3.f) rm |= 1u << r4;
#pragma unroll
        for (int r4 = 0; r4 < 4; ++r4)
          if ((rm >> r4) & 1u) m |= cm << (2 * r4);
      }
      smask[tid] = (uint8_t)m;
    }
    __syncthreads();
    if (COUNTERS) {
      // reference walk: every record in order (counts n_eval exactly as defined)
      if (!__all_sync(0xffffffffu, done)) {
        for (uint32_t j = 0; j < n; ++j) {
          if (!done) ++ne;
          if (!((smask[j] >> warp) & 1u)) continue;
          if (!done) blend_step(srec[3 * j], srec[3 * j + 1], srec[3 * j + 2], lx, ly, T, Cr, Cg, Cb, Dn, done, nc);
          if ((j & 7) == 7 && __all_sync(0xffffffffu, done)) break;
        }
      }
    } else if (!__all_sync(0xffffffffu, done)) {
      // compact this warp's relevant records (order preserved)
      uint32_t cnt = 0;
      const uint32_t lt = (1u << lane) - 1u;
      for (uint32_t g = 0; g < n; g += 32) {
        const uint32_t j = g + lane;
        const bool mine = j < n && ((smask[j] >> warp) & 1u);
        const uint32_t m = __ballot_sync(0xffffffffu, mine);
        if (mine) wlist[warp][cnt + __popc(m & lt)] = (uint8_t)j;
        cnt += __popc(m);
      }
      __syncwarp();
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t j = wlist[warp][i];
        if (!done) blend_step(srec[3 * j], srec[3 * j + 1], srec[3 * j + 2], lx, ly, T, Cr, Cg, Cb, Dn, done, nc);
        if ((i & 15) == 15 && __all_sync(0xffffffffu, done)) break;
      }
    }
    if (__syncthreads_count(done) == TILE_PX) break;
  }

  if (inside) write_pixel(rp, rgb, depth, alpha_out, ((size_t)e * rp.H + py) * rp.W + px, T, Cr, Cg, Cb, Dn);
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

// ---------------------------------------------------------------------------
// Timed path: 128 threads per (tile, env); warp w covers an 8x8 block and
// lane (lx, ly) owns its pixels (lx, ly) and (lx, ly + 4), both evaluated
// with packed f32x2 arithmetic (FFMA2/FADD2/FMUL2) in the same per-pixel
// operation order as blend_step, so the images are bit-identical to the
// 256-thread walk above.  No CTA-wide batches: each warp streams the
// tile's sorted list 32 records at a time for its own 8x8 block, keeps the
// records whose alpha >= 1/255 box (the record's extents, with margins) meets
// the block (compacted in list order into a per-warp shared buffer), walks
// them, and leaves the tile as soon as its 64 pixels are saturated.  Warps
// never wait on each other.  A kept record that no pixel of the warp passes
// costs only the exponent and one vote (an exact ellipse-vs-block test in
// the loader was measured slower: 87.9 vs 85.5 ms per c3 step).
constexpr int RW_THREADS = 128;
#ifndef GG_RW_PF
#define GG_RW_PF 0   // 1: prefetch the next kept record's terms (A/B switch)
#endif

// The stop test looks at T' alone: a non-passing pixel has w = 0 and T' = T >=
// 1e-4, so only a passing pixel can stop; its weight is zeroed by a select.
// One warp's walk of one camera's tile list for its 8 x 8 block (the lane's
// pixels (lx, ly) and (lx, ly + 4)); `col` (runtime, warp-uniform) turns the
// colour accumulation off for a depth-only sample of a motion-blur render.
#ifdef GG_RW_STATS
__device__ unsigned long long g_rw_stats[8];
extern "C" int gg_debug_rw_stats(unsigned long long* out, int reset) {
  if (cudaMemcpyFromSymbol(out, g_rw_stats, sizeof(unsigned long long) * 8) != cudaSuccess) return 1;
  if (reset) {
    static const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_rw_stats, z, sizeof z);
  }
  return 0;
}
#endif
struct WarpGeom {
  float lx, tox, toy, bx0, by0;
  f2 LY;
  bool in0, in1;
};

// LEAN (the single-camera raster): unconditional gathers, a branch-free box
// test and negated tile coefficients (fewer loader instructions at 40
// registers); the blur raster, which keeps two pixels' sample sums live
// across its walks, uses the guarded form with plain coefficients (the lean
// one makes ptxas spill there: 224 vs 16 bytes of spill loads).  Both give
// the same bits (negation is exact).
template <bool RGB, bool LEAN = true>
__device__ __forceinline__ void warp_walk(const ChunkWS& ws, const RenderParams& rp, int eloc, int tile,
                                          const WarpGeom& g, bool col, float4* __restrict__ srec, f2& T, f2& Cr,
                                          f2& Cg, f2& Cb, f2& Dn) {
  const int lane = threadIdx.x & 31;
  constexpr float BW = 7.f, BH = 7.f;   // 8 x 8 blocks (16 x 4 bands measured 7% slower)
  const uint2 rg = chunk_ok(ws.ok) ? ws.ranges[(size_t)eloc * rp.ntiles + tile] : make_uint2(0u, 0u);
  const float4* __restrict__ R0 = ws.rec0 + ws.rec_base[eloc];
  const float4* __restrict__ R1 = ws.rec1 + ws.rec_base[eloc];
  const float4* __restrict__ R2 = ws.rec2 + ws.rec_base[eloc];
  const uint32_t* __restrict__ list = ws.sorted + ws.k_base[eloc];

  T = pk(1.f, 1.f); Cr = pk(0.f, 0.f); Cg = Cr; Cb = Cr; Dn = Cr;
  const float INF = __int_as_float(0x7f800000);
  float cut0 = g.in0 ? LOG2_CUTOFF : INF, cut1 = g.in1 ? LOG2_CUTOFF : INF;
  const uint32_t lt = (1u << lane) - 1u;

  // this batch's list entries are loaded one batch ahead
  uint32_t nidx = rg.x + lane < rg.y ? __ldg(&list[rg.x + lane]) : 0u;
  for (uint32_t b = rg.x; b < rg.y; b += 32) {
    if (__all_sync(0xffffffffu, cut0 == INF && cut1 == INF)) break;
    const float lx0 = g.bx0, lx1 = g.bx0 + BW, ly0 = g.by0, ly1 = g.by0 + BH;
    const bool valid = b + lane < rg.y;
    float4 a0, a1, a2;
    bool mine = false;
    if (LEAN) {
      // unconditional: an idle lane reads record 0 of the env (it exists: the list is not empty)
      a0 = __ldg(&R0[nidx]); a1 = __ldg(&R1[nidx]); a2 = __ldg(&R2[nidx]);
      // branch-free (bitwise &): one predicate chain instead of a branch around the box test
      const float xl = a0.x - a1.w, xh = a0.x + a1.w, yl = a0.y - a2.w, yh = a0.y + a2.w;
      mine = valid & (a1.w >= 0.f) & (a0.z >= LOG2_CUTOFF) & (xh >= lx0) & (xl <= lx1) & (yh >= ly0) & (yl <= ly1);
    } else {
      a0 = make_float4(0.f, 0.f, 0.f, 0.f); a1 = a0; a2 = a0;
      if (valid) { a0 = __ldg(&R0[nidx]); a1 = __ldg(&R1[nidx]); a2 = __ldg(&R2[nidx]); }
      nidx = b + 32 + lane < rg.y ? __ldg(&list[b + 32 + lane]) : 0u;
      if (valid && a1.w >= 0.f && a0.z >= LOG2_CUTOFF) {
        const float xl = a0.x - a1.w, xh = a0.x + a1.w, yl = a0.y - a2.w, yh = a0.y + a2.w;
        mine = xh >= lx0 && xl <= lx1 && yh >= ly0 && yl <= ly1;
      }
    }
    if (LEAN) nidx = b + 32 + lane < rg.y ? __ldg(&list[b + 32 + lane]) : 0u;
    const uint32_t m = __ballot_sync(0xffffffffu, mine);
    if (mine) {
      const int pos = __popc(m & lt);
      srec[3 * pos] = tile_coefs<LEAN>(a0, a1, g.tox, g.toy);
      srec[3 * pos + 1] = make_float4(a1.x, a1.y, a1.z, a0.w);
      srec[3 * pos + 2] = a2;
    }
    __syncwarp();
    const uint32_t cnt = __popc(m);
#if GG_RW_PF
    // the next kept record's exponent terms are read from shared memory one
    // record ahead, off the dependency chain of this record's vote
    float4 n0 = srec[0], n1 = srec[1];
    for (uint32_t i = 0; i < cnt; ++i) {
      const float4 r0 = n0, r1 = n1;
      n0 = srec[3 * (i + 1)];
      n1 = srec[3 * (i + 1) + 1];
#else
    for (uint32_t i = 0; i < cnt; ++i) {
      const float4 r0 = srec[3 * i], r1 = srec[3 * i + 1];
#endif
      // x = c0 + lx (c1 + A' lx) + ly (c2 + B' lx + C' ly)  (tile_coefs)
      const float P = fmaf(g.lx, fmaf(r1.x, g.lx, LEAN ? -r0.y : r0.y), r0.x);
      const float Q = fmaf(r1.y, g.lx, LEAN ? -r0.z : r0.z);
      float x0, x1;
      upk(fma2(g.LY, fma2(pk(r1.z, r1.z), g.LY, pk(Q, Q)), pk(P, P)), x0, x1);
#ifdef GG_RW_STATS   // instrumentation build: kept records, vote failures, geometric failures, live pixels
      if (LEAN) {
        const bool geo = __any_sync(0xffffffffu, (g.in0 && x0 >= LOG2_CUTOFF) || (g.in1 && x1 >= LOG2_CUTOFF));
        const bool any = __any_sync(0xffffffffu, x0 >= cut0 || x1 >= cut1);
        const uint32_t live = __popc(__ballot_sync(0xffffffffu, cut0 != INF)) + __popc(__ballot_sync(0xffffffffu, cut1 != INF));
        if ((threadIdx.x & 31) == 0) {
          atomicAdd(&g_rw_stats[0], 1ull);
          if (!any) atomicAdd(&g_rw_stats[1], 1ull);
          if (!geo) atomicAdd(&g_rw_stats[2], 1ull);
          atomicAdd(&g_rw_stats[3], (unsigned long long)live);
        }
      }
#endif
      // no pixel of the warp passes: nothing to blend, nothing stops (exact)
      if (!__any_sync(0xffffffffu, x0 >= cut0 || x1 >= cut1)) continue;
      const float al0 = x0 >= cut0 ? ex2_approx(fminf(x0, r0.w)) : 0.f;
      const float al1 = x1 >= cut1 ? ex2_approx(fminf(x1, r0.w)) : 0.f;
      f2 W = mul2(pk(al0, al1), T);
      float tn0, tn1, w0, w1;
      upk(sub2(T, W), tn0, tn1);
      upk(W, w0, w1);
      // T stays >= 1e-4, so only a passing pixel can stop; it is not blended
      const bool s0 = tn0 < 1e-4f, s1 = tn1 < 1e-4f;
      W = pk(s0 ? 0.f : w0, s1 ? 0.f : w1);
      cut0 = s0 ? INF : cut0;
      cut1 = s1 ? INF : cut1;
      if (RGB && col) {
        const float4 r2 = srec[3 * i + 2];
        Cr = fma2(W, pk(r2.x, r2.x), Cr);
        Cg = fma2(W, pk(r2.y, r2.y), Cg);
        Cb = fma2(W, pk(r2.z, r2.z), Cb);
      }
      Dn = fma2(W, pk(r1.w, r1.w), Dn);
      T = sub2(T, W);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ WarpGeom warp_geom(const RenderParams& rp, int tile, int& px, int& py0, int& py1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int tx = tile % rp.TX, ty = tile / rp.TX;
  const int bx = warp & 1, by = warp >> 1;
  px = tx * TILE + bx * 8 + (lane & 7);
  py0 = ty * TILE + by * 8 + (lane >> 3);
  py1 = py0 + 4;
  WarpGeom g;
  g.in0 = px < rp.W && py0 < rp.H;
  g.in1 = px < rp.W && py1 < rp.H;
  g.lx = (float)(px - tx * TILE);
  g.LY = pk((float)(py0 - ty * TILE), (float)(py1 - ty * TILE));
  g.tox = (float)(tx * TILE) + 0.5f;
  g.toy = (float)(ty * TILE) + 0.5f;
  g.bx0 = (float)(tx * TILE + bx * 8) + 0.5f;
  g.by0 = (float)(ty * TILE + by * 8) + 0.5f;
  return g;
}

template <bool RGB>   // false: depth-only render (no colour accumulation)
#ifndef GG_RW_MINB
#define GG_RW_MINB 12   // 40 registers, 48 warps/SM: measured best (10: 82.2, 11-12: 81.5, 14: 90.2 ms per c3 step)
#endif
__global__ void __launch_bounds__(RW_THREADS, GG_RW_MINB)
raster_warp_kernel(int e0, const EnvConst* __restrict__ envs, RenderParams rp, ChunkWS ws, void* __restrict__ rgb,
                      float* __restrict__ depth, float* __restrict__ alpha_out) {
  __shared__ float4 srec[RW_THREADS / 32][32 * 3 + 3];   // + 1 record of slack for the prefetch
  const int eloc = blockIdx.y;
  const int tile = blockIdx.x;
  const int e = envs[e0 + eloc].out_index;
  int px, py0, py1;
  const WarpGeom g = warp_geom(rp, tile, px, py0, py1);
  f2 T, Cr, Cg, Cb, Dn;
  warp_walk<RGB>(ws, rp, eloc, tile, g, true, srec[threadIdx.x >> 5], T, Cr, Cg, Cb, Dn);
  float t[2], cr[2], cg[2], cb[2], dn[2];
  upk(T, t[0], t[1]); upk(Cr, cr[0], cr[1]); upk(Cg, cg[0], cg[1]); upk(Cb, cb[0], cb[1]);
  upk(Dn, dn[0], dn[1]);
  const size_t p0 = ((size_t)e * rp.H + py0) * rp.W + px;
  if (g.in0) write_pixel(rp, RGB ? rgb : nullptr, depth, alpha_out, p0, t[0], cr[0], cg[0], cb[0], dn[0]);
  if (g.in1) write_pixel(rp, RGB ? rgb : nullptr, depth, alpha_out, p0 + (size_t)(py1 - py0) * rp.W, t[1], cr[1], cg[1], cb[1], dn[1]);
}

// Motion blur fused into the raster (reading
// R34): a CTA renders the Kc sample cameras of one env (consecutive
// chunk-local envs), keeps each pixel's f32 colour and alpha of sample 0 and
// the running sum of the later samples' differences, and writes the env's
// frame once: m = x0 + (sum_{i>=1} (x_i - x0)) / K (the same operations, in
// the same order, as averaging K rendered f32 frames), depth from sample dk
// (the nominal pose t = 0).  Sample K of an even K is that depth-only pose.
template <bool RGB>
__global__ void __launch_bounds__(RW_THREADS, 8)
raster_blur_kernel(int e0, const EnvConst* __restrict__ envs, RenderParams rp, ChunkWS ws, void* __restrict__ rgb,
                   float* __restrict__ depth, float* __restrict__ alpha_out) {
  __shared__ float4 srec[RW_THREADS / 32][32 * 3 + 3];
  const int K = rp.blur_k, Kc = rp.blur_kc, dk = rp.blur_dk;
  const int c0 = blockIdx.y * Kc;                      // chunk-local camera of sample 0
  const int tile = blockIdx.x;
  const int e = envs[e0 + c0].out_index / Kc;          // output env (relative to this render)
  int px, py0, py1;
  const WarpGeom g = warp_geom(rp, tile, px, py0, py1);
  float x0[2][4], sm[2][4], dep[2] = {0.f, 0.f};
  for (int k = 0; k < Kc; ++k) {
    f2 T, Cr, Cg, Cb, Dn;
    warp_walk<RGB, false>(ws, rp, c0 + k, tile, g, k < K, srec[threadIdx.x >> 5], T, Cr, Cg, Cb, Dn);
    float t[2], cr[2], cg[2], cb[2], dn[2];
    upk(T, t[0], t[1]); upk(Cr, cr[0], cr[1]); upk(Cg, cg[0], cg[1]); upk(Cb, cb[0], cb[1]);
    upk(Dn, dn[0], dn[1]);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      // this sample's f32 pixel (write_pixel's arithmetic): rgb = C + T bg, alpha = 1 - T
      const float x[4] = {fmaf(t[q], rp.bg[0], cr[q]), fmaf(t[q], rp.bg[1], cg[q]), fmaf(t[q], rp.bg[2], cb[q]),
                          1.f - t[q]};
      if (k == dk) dep[q] = x[3] > 0.f ? dn[q] / x[3] : 0.f;
      if (k == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) { x0[q][c] = x[c]; sm[q][c] = 0.f; }
      } else if (k < K) {
#pragma unroll
        for (int c = 0; c < 4; ++c) sm[q][c] += x[c] - x0[q][c];
      }
    }
  }
  const size_t p0 = ((size_t)e * rp.H + py0) * rp.W + px;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    if (!(q == 0 ? g.in0 : g.in1)) continue;
    const size_t p = p0 + (size_t)(q * (py1 - py0)) * rp.W;
    float m[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) m[c] = x0[q][c] + sm[q][c] / (float)K;
    if (RGB && rgb) {
      if (rp.rgb_format == 0) {
        uint8_t* o = reinterpret_cast<uint8_t*>(rgb) + p * 3;
#pragma unroll
        for (int c = 0; c < 3; ++c) o[c] = (uint8_t)__float2uint_rn(fminf(fmaxf(m[c], 0.f), 1.f) * 255.f);
      } else {
        float* o = reinterpret_cast<float*>(rgb) + p * 3;
        o[0] = m[0]; o[1] = m[1]; o[2] = m[2];
      }
    }
    if (alpha_out) alpha_out[p] = m[3];
    if (depth) depth[p] = dep[q];
  }
}

// ---------------------------------------------------------------------------
// Producer/consumer variant (GG_RASTER_PC): warp 4 of a
// 160-thread CTA loads each 32-record batch of the tile list ONCE per CTA,
// evaluates the four 8x8-block box tests, and publishes the batch (records in
// tile-relative form, plus a compacted index list per consumer warp) into a
// ring of PC_NS shared-memory slots guarded by mbarriers (full: producer ->
// consumers, empty: 4 consumer arrivals -> producer); warps 0-3 walk their
// lists exactly as raster_warp_kernel does, with no CTA-wide barrier.  A
// saturated consumer keeps releasing slots without work; once all four are
// saturated the producer publishes a stop slot.  Bit-identical images.
constexpr int PC_NS = 4;
constexpr int PC_THREADS = 160;
struct PcSlot {
  float4 rec[32 * 3];       // tile_coefs, (A', B', C', z), (r, g, b, -)
  uint8_t idx[4][32];       // per consumer warp: kept record indices, list order
  uint32_t cnt[4];
  uint32_t stop;
};
struct PcSmem {
  PcSlot slot[PC_NS];
  unsigned long long full[PC_NS], empty[PC_NS];
  uint32_t ndone;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}

template <bool RGB>
__global__ void __launch_bounds__(PC_THREADS, 9)
raster_pc_kernel(int e0, const EnvConst* __restrict__ envs, RenderParams rp, ChunkWS ws, void* __restrict__ rgb,
                 float* __restrict__ depth, float* __restrict__ alpha_out) {
  __shared__ PcSmem sm;
  const int eloc = blockIdx.y, tile = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint2 rg = chunk_ok(ws.ok) ? ws.ranges[(size_t)eloc * rp.ntiles + tile] : make_uint2(0u, 0u);
  const uint32_t nbatch = (rg.y - rg.x + 31u) / 32u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < PC_NS; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 4);
    }
    sm.ndone = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tx = tile % rp.TX, ty = tile / rp.TX;
  const float tox = (float)(tx * TILE) + 0.5f, toy = (float)(ty * TILE) + 0.5f;
  if (warp == 4) {   // ---- producer
    const float4* __restrict__ R0 = ws.rec0 + ws.rec_base[eloc];
    const float4* __restrict__ R1 = ws.rec1 + ws.rec_base[eloc];
    const float4* __restrict__ R2 = ws.rec2 + ws.rec_base[eloc];
    const uint32_t* __restrict__ list = ws.sorted + ws.k_base[eloc];
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t nidx = rg.x + lane < rg.y ? __ldg(&list[rg.x + lane]) : 0u;
    for (uint32_t bi = 0; bi < nbatch; ++bi) {
      const int sl = (int)(bi % PC_NS);
      const uint32_t ph = (bi / PC_NS) & 1u;
      const uint32_t b = rg.x + 32u * bi;
      const bool valid = b + lane < rg.y;
      // an idle lane reads record 0 (the list is not empty)
      const float4 a0 = __ldg(&R0[nidx]), a1 = __ldg(&R1[nidx]), a2 = __ldg(&R2[nidx]);
      nidx = b + 32 + lane < rg.y ? __ldg(&list[b + 32 + lane]) : 0u;
      const bool live = valid && a1.w >= 0.f && a0.z >= LOG2_CUTOFF;
      const float xl = a0.x - a1.w, xh = a0.x + a1.w, yl = a0.y - a2.w, yh = a0.y + a2.w;
      mbar_wait(&sm.empty[sl], ph ^ 1u);              // slot released by all four consumers
      PcSlot& S = sm.slot[sl];
      const bool stop = *((volatile uint32_t*)&sm.ndone) >= 4u;
      if (lane == 0) S.stop = stop ? 1u : 0u;
      if (!stop) {
        S.rec[3 * lane] = tile_coefs(a0, a1, tox, toy);
        S.rec[3 * lane + 1] = make_float4(a1.x, a1.y, a1.z, a0.w);
        S.rec[3 * lane + 2] = a2;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float bx0 = tox + 8.f * (w & 1), by0 = toy + 8.f * (w >> 1);
          const bool mine = live && xh >= bx0 && xl <= bx0 + 7.f && yh >= by0 && yl <= by0 + 7.f;
          const uint32_t m = __ballot_sync(0xffffffffu, mine);
          if (mine) S.idx[w][__popc(m & lt)] = (uint8_t)lane;
          if (lane == 0) S.cnt[w] = __popc(m);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.full[sl]);
      if (stop) break;
    }
    return;
  }
  // ---- consumers: warp w = 8 x 8 block (bx, by) of the tile
  int px, py0, py1;
  const WarpGeom g = warp_geom(rp, tile, px, py0, py1);
  f2 T = pk(1.f, 1.f), Cr = pk(0.f, 0.f), Cg = Cr, Cb = Cr, Dn = Cr;
  const float INF = __int_as_float(0x7f800000);
  float cut0 = g.in0 ? LOG2_CUTOFF : INF, cut1 = g.in1 ? LOG2_CUTOFF : INF;
  bool done = false;
  for (uint32_t bi = 0; bi < nbatch; ++bi) {
    const int sl = (int)(bi % PC_NS);
    mbar_wait(&sm.full[sl], (bi / PC_NS) & 1u);
    const PcSlot& S = sm.slot[sl];
    if (S.stop) break;
    if (!done) {
      const uint32_t cnt = S.cnt[warp];
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t j = S.idx[warp][i];
        const float4 r0 = S.rec[3 * j], r1 = S.rec[3 * j + 1];
        const float P = fmaf(g.lx, fmaf(r1.x, g.lx, -r0.y), r0.x);
        const float Q = fmaf(r1.y, g.lx, -r0.z);
        float x0, x1;
        upk(fma2(g.LY, fma2(pk(r1.z, r1.z), g.LY, pk(Q, Q)), pk(P, P)), x0, x1);
        if (!__any_sync(0xffffffffu, x0 >= cut0 || x1 >= cut1)) continue;
        const float al0 = x0 >= cut0 ? ex2_approx(fminf(x0, r0.w)) : 0.f;
        const float al1 = x1 >= cut1 ? ex2_approx(fminf(x1, r0.w)) : 0.f;
        f2 W = mul2(pk(al0, al1), T);
        float tn0, tn1, w0, w1;
        upk(sub2(T, W), tn0, tn1);
        upk(W, w0, w1);
        const bool s0 = tn0 < 1e-4f, s1 = tn1 < 1e-4f;
        W = pk(s0 ? 0.f : w0, s1 ? 0.f : w1);
        cut0 = s0 ? INF : cut0;
        cut1 = s1 ? INF : cut1;
        if (RGB) {
          const float4 r2 = S.rec[3 * j + 2];
          Cr = fma2(W, pk(r2.x, r2.x), Cr);
          Cg = fma2(W, pk(r2.y, r2.y), Cg);
          Cb = fma2(W, pk(r2.z, r2.z), Cb);
        }
        Dn = fma2(W, pk(r1.w, r1.w), Dn);
        T = sub2(T, W);
      }
      done = __all_sync(0xffffffffu, cut0 == INF && cut1 == INF);
      if (done && lane == 0) atomicAdd(&sm.ndone, 1u);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.empty[sl]);
  }
  float t[2], cr[2], cg[2], cb[2], dn[2];
  upk(T, t[0], t[1]); upk(Cr, cr[0], cr[1]); upk(Cg, cg[0], cg[1]); upk(Cb, cb[0], cb[1]);
  upk(Dn, dn[0], dn[1]);
  const int e = envs[e0 + eloc].out_index;
  const size_t p0 = ((size_t)e * rp.H + py0) * rp.W + px;
  if (g.in0) write_pixel(rp, RGB ? rgb : nullptr, depth, alpha_out, p0, t[0], cr[0], cg[0], cb[0], dn[0]);
  if (g.in1) write_pixel(rp, RGB ? rgb : nullptr, depth, alpha_out, p0 + (size_t)(py1 - py0) * rp.W, t[1], cr[1], cg[1], cb[1], dn[1]);
}

#ifndef GG_RASTER_PC
#define GG_RASTER_PC 0   // 1: the producer/consumer raster (A/B switch)
#endif

void launch_raster(int e0, int ec, const EnvConst* envs, const RenderParams& rp, const ChunkWS& ws, void* rgb,
                   float* depth, float* alpha, bool counters, unsigned long long* env_counts, int32_t* dbg_neval,
                   int dbg_eloc, cudaStream_t s) {
  CounterOut co{env_counts, dbg_neval, dbg_eloc};
  dim3 grid(rp.ntiles, ec);
  if (rp.blur_k > 0) {   // fused motion-blur average: one CTA per (tile, env) over the env's Kc cameras
    grid.y = ec / rp.blur_kc;
    if (rgb) raster_blur_kernel<true><<<grid, RW_THREADS, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha);
    else raster_blur_kernel<false><<<grid, RW_THREADS, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha);
    return;
  }
  if (counters)
    raster_kernel<true><<<grid, TILE_PX, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha, co);
  else if (GG_RASTER_PC && rgb)
    raster_pc_kernel<true><<<grid, PC_THREADS, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha);
  else if (GG_RASTER_PC)
    raster_pc_kernel<false><<<grid, PC_THREADS, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha);
  else if (rgb)
    raster_warp_kernel<true><<<grid, RW_THREADS, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha);
  else
    raster_warp_kernel<false><<<grid, RW_THREADS, 0, s>>>(e0, envs, rp, ws, rgb, depth, alpha);
}

}  // namespace gg
