// sort_bin.cu — K3-K5: per-env depth presort, stable tile placement and tile
// ranges, as massively parallel passes over a whole env chunk.
//
// Defines the per-tile lists of SPEC.md:136-144 (bin_and_sort: "each tile
// lists every gaussian whose 3-sigma footprint intersects it, sorted
// ascending by view_depth; ties broken by input index (stable)").  The
// canonical list (DESIGN.md §2 O3) is the triples (tile, depth bits, gid) in
// ascending order.  We produce it without ever materialising 64-bit keys:
//   1. stable LSD radix sort of every env's records (already in gid order)
//      by the f32 depth bits minus the env's minimum: ceil(span bits / 10)
//      passes of 10 bits (3 for a ~26-bit span)                -> (z, gid)
//   2. stable bucketing of the records' tiles (row-major) by tile id, the
//      records taken in depth order                          -> (tile, z, gid)
//   3. the per-env tile totals' exclusive scan is the range table (K5).
//
// Each pass is three launches over the chunk's records, split into blocks
// of SORT_BLK (6144) that never straddle an env segment (a per-block env table):
//   upsweep   — per-block histogram (digit or tile) -> global table
//   scan      — one CTA per env: exclusive prefix over (digit, block) in
//               digit-major order = each block's output offset per digit
//   downsweep — the block ranks its elements stably (warp-owned 256-element
//               slices; equal digits found with warp-private stamps and
//               peer masks; per-warp counters; prefix over warps), stages
//               them in shared memory in digit order, and writes contiguous
//               per-digit runs at the block's offsets.  The placement
//               downsweep walks per-warp segments and expands each record's
//               tiles 32 pairs at a time instead of staging.
// Thousands of independent blocks per pass keep HBM busy; staged runs keep
// the writes coalesced.  No float math, no order-dependent atomics:
// identical inputs give bit-identical lists.
#include "gg_internal.cuh"
#include <algorithm>
#include <cstdlib>

namespace gg {

constexpr int SB_THREADS = 512;                 // placement upsweep (1024 measured 13% slower)
constexpr int PS_THREADS = 1024;                // placement scan: one thread per tile of a 1024-tile slice
constexpr int PS_WARPS = PS_THREADS / 32;
#ifndef GG_PD_THREADS
#define GG_PD_THREADS 512   // measured: 256 threads (8 longer segments) 11.5 vs 6.3 ms per 1024 envs
#endif
constexpr int PD_THREADS = GG_PD_THREADS;        // placement downsweep: 16 warps = up to 16 segments
constexpr int PD_MINB = 1536 / PD_THREADS;       // resident CTAs per SM the smem budget below allows
constexpr int PD_SMEM = 216 * 1024 / PD_MINB;    // shared-memory budget per CTA
constexpr int PD_WARPS = PD_THREADS / 32;
#ifndef GG_PD_P1DEEP
#define GG_PD_P1DEEP 4   // placement phase 1 gathers 4 records per lane at once (measured: 0: 27.81, 2: 27.79, 4: 27.67, 8: 28.36 ms of placement per c3 step)
#endif
#ifndef GG_PD_OWNER
#define GG_PD_OWNER 1   // pair owners from a window bitmask (0: the shuffle binary search, 0.6 ms slower per c3 step)
#endif
#ifndef GG_SORT_BLK
#define GG_SORT_BLK 6144   // measured: sort stage 56.4 (4096), 54.9 (5120), 53.4 (6144), 53.7 (7168), 59.9 (8192) ms per c3 step;
                           // round 2 at HEAD (depth + placement): 54.67 (5120), 53.45 (6144), 55.26 (7168), 59.12 (8192)
#endif
constexpr int SORT_BLK = GG_SORT_BLK;                // records per sort block (depth and placement)
constexpr int DS_THREADS = 512;                 // depth passes: 16 warps x 8 elements
constexpr int DS_WARPS = DS_THREADS / 32;
constexpr int DS_IPT = SORT_BLK / DS_THREADS;
constexpr int DS_BITS = 10;                     // digit width of the depth passes
constexpr int DS_RADIX = 1 << DS_BITS;
constexpr int SORT_QCTR = 16;                   // async-mode work counters per chunk (2 per pass + 3)

// blocks of the chunk: env of block b is the e with blk_base[e] <= b < blk_base[e+1],
// tabulated once per chunk (blk_env_kernel) so a block finds it with one load
struct BlockTable {
  const uint32_t* blk_base;   // [ec + 1]
  const uint32_t* blk_env;    // [blk_base[ec]]
  int ec;
  uint32_t* q;                // async mode: this launch's work counter (zeroed before the launch)
};

// async mode: CTAs take blocks from a shared counter (dynamic balance, like
// the hardware's CTA scheduling in sync mode, within a bounded grid)
__device__ __forceinline__ uint32_t next_block(uint32_t* q) {
  __shared__ uint32_t b_s;
  __syncthreads();             // every thread has read the previous value
  if (threadIdx.x == 0) b_s = atomicAdd(q, 1u);
  __syncthreads();
  return b_s;
}

__device__ __forceinline__ int block_env(const BlockTable& bt, uint32_t b) { return (int)bt.blk_env[b]; }

__global__ void blk_env_kernel(const uint32_t* __restrict__ blk_base, int ec, uint32_t* __restrict__ blk_env) {
  const int e = blockIdx.x;
  const uint32_t end = blk_base[ec];
  const uint32_t b0 = blk_base[e], b1 = min(blk_base[e + 1], end);
  for (uint32_t b = b0 + threadIdx.x; b < b1; b += blockDim.x) blk_env[b] = (uint32_t)e;
}

__device__ __forceinline__ uint32_t peers_of(uint32_t v, int bits, uint32_t active) {
  uint32_t peers = active;
#pragma unroll 8
  for (int b = 0; b < bits; ++b) {
    const bool bit = (v >> b) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

// exclusive scan over the block (all threads call); *total = block sum
__device__ __forceinline__ uint32_t block_scan(uint32_t x, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  uint32_t s = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += y;
  }
  if (lane == 31) wsum[warp] = s;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < nw ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) wsum[lane] = t;
  }
  __syncthreads();
  const uint32_t excl = (warp ? wsum[warp - 1] : 0u) + s - x;
  *total = wsum[nw - 1];
  __syncthreads();
  return excl;
}

__device__ __forceinline__ void unpack_rect(uint2 r, uint32_t& x0, uint32_t& x1, uint32_t& y0, uint32_t& y1) {
  x0 = r.x & 0xffffu; x1 = r.x >> 16; y0 = r.y & 0xffffu; y1 = r.y >> 16;
}

// Input / output arrays of depth pass p (all indexed rec_base[e] + j).  The
// sort key is the f32 depth bits minus those of the near plane (a monotone map
// of the positive f32 bits; every record has near < z <= far), so the default
// [0.01, 1e10] span (29 bits) needs 3 passes of 10 bits.
// Between passes key and record travel as one 64-bit word (key << 32 |
// record): one load, one staging store and one scattered store per element.
struct DepthIO {
  const uint32_t* zin;   // first pass: f32 depth bits (records = identity j)
  const uint64_t* pin;   // later passes: packed (z bits - zbase) << 32 | record
  uint64_t* pout;        // packed out (null on the last pass)
  uint32_t* vout;        // last pass: records in depth order
  uint32_t* kout;        // last pass: their keys (the tie fix-up reads them)
};

__device__ __forceinline__ uint32_t depth_digit(uint32_t key, int shift) {
  return (key >> shift) & (DS_RADIX - 1);
}

// element i of the block as (z bits - zbase) << 32 | record
__device__ __forceinline__ uint64_t depth_elem(const DepthIO& io, uint64_t at, uint32_t j, uint32_t zmin) {
  return io.zin ? ((uint64_t)(io.zin[at] - zmin) << 32) | j : io.pin[at];
}

// ---- depth passes --------------------------------------------------------
__device__ __forceinline__ void depth_upsweep_block(uint32_t b, const BlockTable& bt, const ChunkWS& ws, const DepthIO& io, int shift, uint32_t* ghist, uint32_t* h) {
  const int e = block_env(bt, b);
  const uint32_t j0 = (b - bt.blk_base[e]) * SORT_BLK;
  const uint32_t n = min((uint32_t)SORT_BLK, ws.vcnt[e] - j0);
  const uint64_t rb = ws.rec_base[e];
  const uint32_t zmin = ws.zbase;
  for (int i = threadIdx.x; i < DS_RADIX; i += DS_THREADS) h[i] = 0;
  __syncthreads();
  uint32_t k[DS_IPT];                              // all of this thread's keys in flight first
#pragma unroll
  for (int j = 0; j < DS_IPT; ++j) {
    const uint32_t i = threadIdx.x + j * DS_THREADS;
    k[j] = i < n ? (io.zin ? io.zin[rb + j0 + i] - zmin : (uint32_t)(io.pin[rb + j0 + i] >> 32)) : 0u;
  }
#pragma unroll
  for (int j = 0; j < DS_IPT; ++j)
    if (threadIdx.x + j * DS_THREADS < n) atomicAdd(&h[depth_digit(k[j], shift)], 1u);
  __syncthreads();
  for (int i = threadIdx.x; i < DS_RADIX; i += DS_THREADS) ghist[(size_t)b * DS_RADIX + i] = h[i];
}

template <bool LOOP>
__global__ void __launch_bounds__(DS_THREADS)
depth_upsweep_kernel(BlockTable bt, ChunkWS ws, DepthIO io, int shift, uint32_t* ghist) {
  __shared__ uint32_t h[DS_RADIX];
  if (!chunk_ok(ws.ok)) return;
  const uint32_t nb = bt.blk_base[bt.ec];
  if (!LOOP) {                                     // one CTA per block (sync mode)
    if (blockIdx.x < nb) depth_upsweep_block(blockIdx.x, bt, ws, io, shift, ghist, h);
    return;
  }
  for (;;) {   // async mode: bounded grid, blocks taken dynamically
    const uint32_t b = next_block(bt.q);
    if (b >= nb) break;
    depth_upsweep_block(b, bt, ws, io, shift, ghist, h);
  }
}

// one CTA (1024 threads = digits) per env: ghist[b][d] -> output offset of
// (block b, digit d) relative to the env's segment (digit-major, block-minor)
__global__ void __launch_bounds__(DS_RADIX) depth_scan_kernel(BlockTable bt, uint32_t* ghist, const uint32_t* ok) {
  __shared__ uint32_t wsum[32];
  if (!chunk_ok(ok)) return;
  const int e = blockIdx.x;
  const uint32_t b0 = bt.blk_base[e], b1 = bt.blk_base[e + 1];
  const int d = threadIdx.x;
  uint32_t* col = ghist + d;
  // pass 1: the digit's total over the env's blocks (16 independent loads in flight)
  uint32_t run = 0;
  for (uint32_t b = b0; b < b1; b += 16) {
    uint32_t x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = b + u < b1 ? col[(size_t)(b + u) * DS_RADIX] : 0u;
#pragma unroll
    for (int u = 0; u < 16; ++u) run += x[u];
  }
  uint32_t total;
  uint32_t acc = block_scan(run, wsum, &total);   // digits below d, all blocks
  // pass 2: exclusive prefix over blocks, offset by the lower digits
  for (uint32_t b = b0; b < b1; b += 16) {
    uint32_t x[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) x[u] = b + u < b1 ? col[(size_t)(b + u) * DS_RADIX] : 0u;
#pragma unroll
    for (int u = 0; u < 16; ++u)
      if (b + u < b1) { col[(size_t)(b + u) * DS_RADIX] = acc; acc += x[u]; }
  }
}

struct DownSmem {
  union {
    struct {                                   // ranking
      uint32_t wcnt[DS_WARPS][DS_RADIX / 2];   // per-warp digit counts -> offsets, packed u16 pairs (32 KB)
      uint32_t pm[DS_WARPS][32];               // peer masks by representative lane
      uint8_t st[DS_WARPS][DS_RADIX];          // last lane that stamped each digit (warp-private)
    } r;
    struct {                                   // staging in digit order (after ranking)
      uint64_t sp[SORT_BLK];
    } o;
  } u;
  uint32_t dstart[DS_RADIX];
  uint32_t wsum[32];
};

// Stable block-local ranking: element (warp w, round j, lane l) has block
// index 32 DS_IPT w + 32 j + l and digit d[j].  lpos[j] = position in the block
// sorted stably by digit; sm.dstart = digit starts.  Equal digits among a
// warp's 32 lanes are found through a warp-private stamp per digit (the last
// lane to stamp it is the digits' representative) and one shared-memory OR
// into the representative's peer mask.  u.r is zero on entry; on exit it is
// free (the caller stages into u.o).
__device__ __forceinline__ void block_rank(const uint64_t (&x)[DS_IPT], int shift, uint32_t n,
                                           uint32_t (&lpos)[DS_IPT], DownSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = lanemask_lt();
  uint32_t* wc = sm.u.r.wcnt[warp];
  uint32_t* pm = sm.u.r.pm[warp];
  uint8_t* st = sm.u.r.st[warp];
  uint32_t rk[DS_IPT];
#pragma unroll
  for (int j = 0; j < DS_IPT; ++j) {
    const uint32_t e = warp * 32 * DS_IPT + j * 32 + lane;
    const bool ok = e < n;
    const uint32_t dd = depth_digit((uint32_t)(x[j] >> 32), shift);
    if (ok) st[dd] = (uint8_t)lane;
    __syncwarp();
    const uint32_t rep = ok ? st[dd] : 0u;
    if (ok) atomicOr(&pm[rep], 1u << lane);
    __syncwarp();
    const uint32_t peers = ok ? pm[rep] : 0u;
#ifdef GG_CHECK_PROTOCOLS   // race/protocol evidence build: the stamp protocol's peer mask = exact equal-digit set
    {
      const uint32_t ref = __match_any_sync(0xffffffffu, ok ? dd : 0xffffffffu);
      if (ok && peers != ref) __trap();
    }
#endif
    const uint32_t before = ok ? (wc[dd >> 1] >> (16 * (dd & 1))) & 0xffffu : 0u;
    __syncwarp();
    if (ok && lane == (int)rep) pm[rep] = 0u;
    if (ok && lane == __ffs(peers) - 1) atomicAdd(&wc[dd >> 1], __popc(peers) << (16 * (dd & 1)));
    __syncwarp();
    rk[j] = before + __popc(peers & lt);
  }
  __syncthreads();
  // per digit pair (one packed word per thread): prefix over warps; digit
  // totals -> block-wide exclusive scan
  static_assert(DS_RADIX == 2 * DS_THREADS, "one packed digit pair per thread");
  uint32_t run = 0;
#pragma unroll 4
  for (int w = 0; w < DS_WARPS; ++w) {
    const uint32_t x = sm.u.r.wcnt[w][tid];
    sm.u.r.wcnt[w][tid] = run;
    run += x;
  }
  const uint32_t c0 = run & 0xffffu, c1 = run >> 16;
  uint32_t total;
  const uint32_t ex = block_scan(c0 + c1, sm.wsum, &total);
  sm.dstart[2 * tid] = ex;
  sm.dstart[2 * tid + 1] = ex + c0;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < DS_IPT; ++j) {
    const uint32_t e = warp * 32 * DS_IPT + j * 32 + lane;
    const uint32_t dd = depth_digit((uint32_t)(x[j] >> 32), shift);
    lpos[j] = e < n ? sm.dstart[dd] + ((wc[dd >> 1] >> (16 * (dd & 1))) & 0xffffu) + rk[j] : 0u;
  }
  __syncthreads();
}

__device__ __forceinline__ void depth_downsweep_block(uint32_t b, const BlockTable& bt, const ChunkWS& ws, const DepthIO& io, int shift, const uint32_t* ghist, DownSmem& sm) {
  const int e = block_env(bt, b);
  const uint32_t j0 = (b - bt.blk_base[e]) * SORT_BLK;
  const uint32_t n = min((uint32_t)SORT_BLK, ws.vcnt[e] - j0);
  const uint64_t rb = ws.rec_base[e];
  const uint32_t zmin = ws.zbase;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < DS_WARPS * DS_RADIX / 2; i += DS_THREADS) (&sm.u.r.wcnt[0][0])[i] = 0u;
  for (int i = tid; i < DS_WARPS * 32; i += DS_THREADS) (&sm.u.r.pm[0][0])[i] = 0u;
  uint64_t x[DS_IPT];
  uint32_t lp[DS_IPT];
  // this block's output offset of its digits 2 tid, 2 tid + 1 (loaded early)
  const uint2 off = reinterpret_cast<const uint2*>(ghist + (size_t)b * DS_RADIX)[tid];
#pragma unroll
  for (int j = 0; j < DS_IPT; ++j) {
    const uint32_t i = warp * 32 * DS_IPT + j * 32 + lane;
    x[j] = i < n ? depth_elem(io, rb + j0 + i, j0 + i, zmin) : 0ull;
  }
  __syncthreads();
  block_rank(x, shift, n, lp, sm);
  // fold: dstart[d] <- (global offset of digit d) - (its start in the block),
  // so staged element q of digit d goes to rb + dstart[d] + q
  sm.dstart[2 * tid] = off.x - sm.dstart[2 * tid];
  sm.dstart[2 * tid + 1] = off.y - sm.dstart[2 * tid + 1];
#pragma unroll
  for (int j = 0; j < DS_IPT; ++j) {
    const uint32_t i = warp * 32 * DS_IPT + j * 32 + lane;
    if (i < n) sm.u.o.sp[lp[j]] = x[j];
  }
  __syncthreads();
#ifdef GG_CHECK_PROTOCOLS
  {  // the staged block is sorted by (key bits below this pass's top, record): stable, no element lost or doubled
    const uint32_t bits = (uint32_t)shift + DS_BITS;
    const uint64_t km = bits >= 32 ? 0xffffffffull : ((1ull << bits) - 1ull);
    for (uint32_t q = tid; q + 1 < n; q += DS_THREADS) {
      const uint64_t a = sm.u.o.sp[q], c = sm.u.o.sp[q + 1];
      const uint64_t ka = (a >> 32) & km, kc = (c >> 32) & km;
      if (!(ka < kc || (ka == kc && (uint32_t)a < (uint32_t)c))) __trap();
    }
  }
#endif
  if (io.pout) {
    uint64_t* pout = io.pout + rb;
    for (uint32_t q = tid; q < n; q += DS_THREADS) {
      const uint64_t xx = sm.u.o.sp[q];
      pout[sm.dstart[depth_digit((uint32_t)(xx >> 32), shift)] + q] = xx;
    }
  } else {
    uint32_t* vout = io.vout + rb;
    uint32_t* kout = io.kout + rb;
    for (uint32_t q = tid; q < n; q += DS_THREADS) {
      const uint64_t xx = sm.u.o.sp[q];
      const uint32_t at = sm.dstart[depth_digit((uint32_t)(xx >> 32), shift)] + q;
      vout[at] = (uint32_t)xx;
      kout[at] = (uint32_t)(xx >> 32);
    }
  }
}

template <bool LOOP>
#ifndef GG_DS_MINB
#define GG_DS_MINB 2   // 64 registers, no spills: measured best (2: 4.69, 3: 5.05, 4: 5.51 ms per 1024 envs)
#endif
__global__ void __launch_bounds__(DS_THREADS, GG_DS_MINB)
depth_downsweep_kernel(BlockTable bt, ChunkWS ws, DepthIO io, int shift, const uint32_t* ghist) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  DownSmem& sm = *reinterpret_cast<DownSmem*>(smem_raw);
  if (!chunk_ok(ws.ok)) return;
  const uint32_t nb = bt.blk_base[bt.ec];
  if (!LOOP) {                                     // one CTA per block (sync mode)
    if (blockIdx.x < nb) depth_downsweep_block(blockIdx.x, bt, ws, io, shift, ghist, sm);
    return;
  }
  for (;;) {   // async mode: bounded grid, blocks taken dynamically
    const uint32_t b = next_block(bt.q);
    if (b >= nb) break;
    depth_downsweep_block(b, bt, ws, io, shift, ghist, sm);
  }
}

// ---- tie fix-up ------------------------------------------------------------
// The records of an env are in storage order (Morton order of the means, not
// input order), so the stable depth sort leaves exactly-equal depth keys in
// storage order.  The canonical order breaks them by gid (SPEC.md:139
// "ties broken by input index"; DESIGN.md §2 O3): every run of equal keys
// (a few hundred short runs per env: coincident f32 depths) is re-sorted by
// gid in place, by the thread that owns the run's first position.
__device__ __noinline__ void sort_run_by_gid(uint32_t* __restrict__ o, uint32_t len, const uint32_t* __restrict__ gid) {
  if (len == 2) {                                   // the common run: one compare
    const uint32_t r0 = o[0], r1 = o[1];
    if (gid[r0] > gid[r1]) { o[0] = r1; o[1] = r0; }
    return;
  }
  // shell sort in place (a long run of exact ties, e.g. duplicated
  // Gaussians, stays O(len^1.3)); gaps 3h+1 below len
  uint32_t gap = 1;
  while (gap < len / 3) gap = 3 * gap + 1;
  for (; gap > 0; gap /= 3) {
    for (uint32_t i = gap; i < len; ++i) {
      const uint32_t r = o[i], g = gid[r];
      uint32_t k = i;
      while (k >= gap && gid[o[k - gap]] > g) {
        o[k] = o[k - gap];
        k -= gap;
      }
      o[k] = r;
    }
  }
}

// One CTA per sort block (its env's bounds are known): 8 keys per thread and
// step in two 128-bit loads; the rare tie (an equal successor) is resolved by
// the thread owning the run's first position.  (A warp per block measured
// slower: 0.95 vs 0.74 ms per 1,024 envs.)
#ifndef GG_TIES_THREADS
#define GG_TIES_THREADS 256
#endif
constexpr int TIES_THREADS = GG_TIES_THREADS;
__device__ __forceinline__ void ties_block(uint32_t b, const BlockTable& bt, const ChunkWS& ws, const uint32_t* keys) {
  const int e = block_env(bt, b);
  const uint32_t V = ws.vcnt[e];
  const uint32_t j0 = (b - bt.blk_base[e]) * SORT_BLK;
  const uint32_t n = min((uint32_t)SORT_BLK, V - j0);
  const uint64_t rb = ws.rec_base[e];
  const uint32_t* __restrict__ K = keys + rb;
  for (uint32_t q = threadIdx.x * 8; q < n; q += TIES_THREADS * 8) {
    const uint32_t j = j0 + q;
    uint32_t k[9];
    if (((rb + j) & 3u) == 0u && q + 8 <= n) {      // 16-B aligned: two 128-bit loads
      const uint4 a = *reinterpret_cast<const uint4*>(K + j), c = *reinterpret_cast<const uint4*>(K + j + 4);
      k[0] = a.x; k[1] = a.y; k[2] = a.z; k[3] = a.w; k[4] = c.x; k[5] = c.y; k[6] = c.z; k[7] = c.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) k[i] = q + i < n ? K[j + i] : 0u;
    }
    k[8] = j + 8 < V ? K[j + 8] : 0u;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t p = j + i;
      if (q + i >= n || p + 1 >= V || k[i + 1] != k[i]) continue;   // no equal successor (the common case)
      if (p > 0 && (i > 0 ? k[i - 1] : K[p - 1]) == k[i]) continue;  // not the run's first position
      uint32_t end = p + 2;
      while (end < V && K[end] == k[i]) ++end;
      sort_run_by_gid(ws.order + rb + p, end - p, ws.gid + rb);
    }
  }
}

template <bool LOOP>
__global__ void __launch_bounds__(TIES_THREADS) depth_ties_kernel(BlockTable bt, ChunkWS ws, const uint32_t* keys) {
  if (!chunk_ok(ws.ok)) return;
  const uint32_t nb = bt.blk_base[bt.ec];
  if (!LOOP) {
    if (blockIdx.x < nb) ties_block(blockIdx.x, bt, ws, keys);
    return;
  }
  for (;;) {
    const uint32_t b = next_block(bt.q);
    if (b >= nb) break;
    ties_block(b, bt, ws, keys);
  }
}

// ---- tile placement ------------------------------------------------------
// order[rb + j] = record (gid-ordered local index) of depth rank j
template <bool MASK>   // R37 tile masks present (GG_ELLIPSE_TILES)
__device__ __forceinline__ void place_upsweep_block(uint32_t b, const BlockTable& bt, const ChunkWS& ws, const uint32_t* order, int ntiles, int TX, uint32_t* thist, uint32_t* h) {
  const uint32_t* rmask = MASK ? ws.rmask : nullptr;
  const int e = block_env(bt, b);
  const uint32_t j0 = (b - bt.blk_base[e]) * SORT_BLK;
  const uint32_t n = min((uint32_t)SORT_BLK, ws.vcnt[e] - j0);
  const uint64_t rb = ws.rec_base[e];
  for (int i = threadIdx.x; i < ntiles; i += SB_THREADS) h[i] = 0u;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < n; i += SB_THREADS) {
    const uint32_t idx = order[rb + j0 + i];
    const uint2 r = ws.rect[rb + idx];
    uint32_t x0, x1, y0, y1;
    unpack_rect(r, x0, x1, y0, y1);
    const uint32_t w = x1 - x0, area = w * (y1 - y0);
    const uint32_t m = rec_mask(rmask, rb + idx, area);
    if (m != 0xffffffffu) {                       // R37 mask: the kept tiles only
      for (uint32_t mm = m; mm; mm &= mm - 1u) {
        const uint32_t bit = __ffs(mm) - 1, ry = bit / w;
        atomicAdd(&h[(y0 + ry) * TX + x0 + (bit - ry * w)], 1u);
      }
    } else {
      for (uint32_t ty = y0; ty < y1; ++ty)
        for (uint32_t tx = x0; tx < x1; ++tx) atomicAdd(&h[ty * TX + tx], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < ntiles; i += SB_THREADS) thist[(size_t)b * ntiles + i] = h[i];
}

template <bool LOOP, bool MASK>
__global__ void __launch_bounds__(SB_THREADS)
place_upsweep_kernel(BlockTable bt, ChunkWS ws, const uint32_t* order, int ntiles, int TX, uint32_t* thist) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* h = reinterpret_cast<uint32_t*>(smem_raw);
  if (!chunk_ok(ws.ok)) return;
  const uint32_t nb = bt.blk_base[bt.ec];
  if (!LOOP) {                                     // one CTA per block (sync mode)
    if (blockIdx.x < nb) place_upsweep_block<MASK>(blockIdx.x, bt, ws, order, ntiles, TX, thist, h);
    return;
  }
  for (;;) {   // async mode: bounded grid, blocks taken dynamically
    const uint32_t b = next_block(bt.q);
    if (b >= nb) break;
    place_upsweep_block<MASK>(b, bt, ws, order, ntiles, TX, thist, h);
  }
}

// one CTA per env: thist[b][t] -> output offset (relative to k_base[e]) of
// (block b, tile t); ranges[e][t] = [start, end)
__global__ void __launch_bounds__(PS_THREADS) place_scan_kernel(BlockTable bt, ChunkWS ws, uint32_t* thist,
                                                                int ntiles) {
  __shared__ uint32_t wsum[PS_WARPS];
  if (!chunk_ok(ws.ok)) return;
  const int e = blockIdx.x;
  const uint32_t b0 = bt.blk_base[e], b1 = bt.blk_base[e + 1];
  uint32_t carry = 0;
  for (int base = 0; base < ntiles; base += PS_THREADS) {
    const int t = base + threadIdx.x;
    uint32_t run = 0;
    uint32_t* col = thist + t;
    if (t < ntiles) {                               // pass 1: the tile's total (16 loads in flight)
      for (uint32_t b = b0; b < b1; b += 16) {
        uint32_t x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = b + u < b1 ? col[(size_t)(b + u) * ntiles] : 0u;
#pragma unroll
        for (int u = 0; u < 16; ++u) run += x[u];
      }
    }
    uint32_t total;
    const uint32_t ex = carry + block_scan(t < ntiles ? run : 0u, wsum, &total);
    if (t < ntiles) {                               // pass 2: exclusive prefix over blocks
      ws.ranges[(size_t)e * ntiles + t] = make_uint2(ex, ex + run);
      uint32_t acc = ex;
      for (uint32_t b = b0; b < b1; b += 16) {
        uint32_t x[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) x[u] = b + u < b1 ? col[(size_t)(b + u) * ntiles] : 0u;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (b + u < b1) { col[(size_t)(b + u) * ntiles] = acc; acc += x[u]; }
      }
    }
    carry += total;
  }
}

// Placement downsweep.  Warp w < S owns a contiguous segment of the block's
// records (in depth order).  Phase 1: per-warp tile histograms (u16 pairs
// packed in u32 words).  Phase 2: per tile, prefix over warps starting at
// the block's offset from place_scan -> per-warp cursors.  Phase 3: each
// warp walks its records in order, 32 (record, tile) pairs per step, ranks
// equal tiles among the lanes with a ballot multisplit and writes each
// record index at its final slot; no block barrier inside the walk.
template <int TB, bool MASK>   // tile-id bits (compile time: the multisplit fully unrolls); R37 masks
__device__ __forceinline__ void place_downsweep_block(uint32_t b, const BlockTable& bt, const ChunkWS& ws,
                                                      const uint32_t* order, const RenderParams& rp,
                                                      const uint32_t* thist, int S, unsigned char* smem_raw) {
  constexpr bool STAMP = TB <= 11;                   // warp-private tile stamps fit in shared memory
  const int nt = rp.ntiles;
  const int nw2 = (nt + 1) >> 1;                     // packed words per warp
  uint32_t* gb = reinterpret_cast<uint32_t*>(smem_raw);   // [nt] block offsets (rel. to k_base)
  uint32_t* wh = gb + nt;                                  // [S][nw2] packed u16 counters / cursors
  uint32_t* pmask = wh + (size_t)S * nw2;                  // [S][32] peer masks by representative lane
  uint8_t* stamps = reinterpret_cast<uint8_t*>(pmask + (STAMP ? S * 32 : 0));   // [S][nt] last lane per tile
  const int e = block_env(bt, b);
  const uint32_t j0 = (b - bt.blk_base[e]) * SORT_BLK;
  const uint32_t nrec = min((uint32_t)SORT_BLK, ws.vcnt[e] - j0);
  const uint64_t rb = ws.rec_base[e];
  uint32_t* out = ws.sorted + ws.k_base[e];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < nt; i += PD_THREADS) gb[i] = thist[(size_t)b * nt + i];
  for (int i = tid; i < S * nw2; i += PD_THREADS) wh[i] = 0u;
  if (STAMP)
    for (int i = tid; i < S * 32; i += PD_THREADS) pmask[i] = 0u;
  // segment of warp w: records [w*Ls, (w+1)*Ls) of the block, Ls multiple of 32
  const uint32_t Ls = ((nrec + S * 32 - 1) / (S * 32)) * 32;
  const uint32_t s0 = warp < S ? min(nrec, warp * Ls) : nrec;
  const uint32_t s1 = warp < S ? min(nrec, s0 + Ls) : nrec;
  __syncthreads();
  // phase 1: per-warp tile histogram over the warp's segment
  if (warp < S) {
    uint32_t* h = wh + (size_t)warp * nw2;
#if GG_PD_P1DEEP
    // the lane's records PD1 at a time: their order -> rect gathers in flight together
    constexpr int PD1 = GG_PD_P1DEEP;
    for (uint32_t jb = s0 + lane; jb < s1; jb += 32 * PD1) {
      uint32_t ix[PD1];
      uint2 rr[PD1];
#pragma unroll
      for (int u = 0; u < PD1; ++u) ix[u] = jb + 32 * u < s1 ? order[rb + j0 + jb + 32 * u] : 0u;
#pragma unroll
      for (int u = 0; u < PD1; ++u) rr[u] = jb + 32 * u < s1 ? ws.rect[rb + ix[u]] : make_uint2(0u, 0u);
#pragma unroll
      for (int u = 0; u < PD1; ++u) {
      if (jb + 32 * u >= s1) break;   // past the segment: no record (and no R37 mask lookup)
      const uint32_t idx = ix[u];
      const uint2 r = rr[u];
#else
    for (uint32_t j = s0 + lane; j < s1; j += 32) {
      const uint32_t idx = order[rb + j0 + j];
      const uint2 r = ws.rect[rb + idx];
#endif
      const uint32_t x0 = r.x & 0xffffu, x1 = r.x >> 16, y0 = r.y & 0xffffu, y1 = r.y >> 16;
      const uint32_t w = x1 - x0;
      const uint32_t m = rec_mask(MASK ? ws.rmask : nullptr, rb + idx, w * (y1 - y0));
      if (m != 0xffffffffu) {                     // R37 mask: the kept tiles only
        for (uint32_t mm = m; mm; mm &= mm - 1u) {
          const uint32_t bit = __ffs(mm) - 1, ry = bit / w;
          const uint32_t t = (y0 + ry) * rp.TX + x0 + (bit - ry * w);
          atomicAdd(&h[t >> 1], 1u << (16 * (t & 1)));
        }
      } else {
        for (uint32_t ty = y0; ty < y1; ++ty)
          for (uint32_t tx = x0; tx < x1; ++tx) {
            const uint32_t t = ty * rp.TX + tx;
            atomicAdd(&h[t >> 1], 1u << (16 * (t & 1)));
          }
      }
#if GG_PD_P1DEEP
      }
#endif
    }
  }
  __syncthreads();
  // phase 2: per-warp cursors relative to the block's run of each tile (one
  // thread per packed word; a warp-parallel scan over the segments measured
  // slower: 30.96 vs 29.8 ms of placement per c3 step)
  for (int q = tid; q < nw2; q += PD_THREADS) {
    uint32_t run0 = 0, run1 = 0;
    for (int w = 0; w < S; ++w) {
      const uint32_t c = wh[(size_t)w * nw2 + q];
      wh[(size_t)w * nw2 + q] = run0 | (run1 << 16);
      run0 += c & 0xffffu;
      run1 += c >> 16;
    }
  }
  __syncthreads();
  // phase 3: ordered walk, 32 records per step, their pairs 32 at a time
  if (warp >= S) return;
  uint32_t* h = wh + (size_t)warp * nw2;
  uint8_t* st = stamps + (size_t)warp * nt;
  uint32_t* pm = pmask + warp * 32;
  const uint32_t lt = lanemask_lt();
#if GG_PD_OWNER
  __shared__ uint8_t own_s[PD_WARPS][32];
  uint8_t* own = own_s[warp];
#endif
  for (uint32_t base = s0; base < s1; base += 32) {
    const uint32_t j = base + lane;
    uint32_t idx = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    if (j < s1) {
      idx = order[rb + j0 + j];
      const uint2 r = ws.rect[rb + idx];
      x0 = r.x & 0xffffu; x1 = r.x >> 16; y0 = r.y & 0xffffu; y1 = r.y >> 16;
    }
    const uint32_t w = x1 - x0;
    const uint32_t area = w * (y1 - y0);
    const uint32_t msk = j < s1 ? rec_mask(MASK ? ws.rmask : nullptr, rb + idx, area) : 0xffffffffu;
    const uint32_t np = msk != 0xffffffffu ? rec_tiles(msk, area) : area;
    uint32_t incl = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t excl = incl - np;
    const uint32_t xy0 = x0 | (y0 << 16);
#if GG_PD_OWNER
    int carry = 0;   // lane owning the first pair of the next window
#endif
    for (uint32_t f0 = 0; f0 < tot; f0 += 32) {
      const uint32_t f = f0 + lane;
      const bool ok = f < tot;
#if GG_PD_OWNER
      // lanes whose first pair falls in this window mark its position; pair f
      // belongs to the last mark at or before it, else to the carried owner
      const bool starts = np > 0 && excl >= f0 && excl < f0 + 32;
      const uint32_t M = __reduce_or_sync(0xffffffffu, starts ? 1u << (excl - f0) : 0u);
      if (starts) own[excl - f0] = (uint8_t)lane;
      __syncwarp();
      const uint32_t mm = M & ((2u << lane) - 1u);
      int src = mm ? (int)own[31 - __clz(mm)] : carry;
      __syncwarp();
      carry = __shfl_sync(0xffffffffu, src, 31);
#else
      int src = 0;   // first lane whose inclusive pair count exceeds f
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const uint32_t v = __shfl_sync(0xffffffffu, incl, src + step - 1);
        if (v <= f) src += step;
      }
#endif
      const uint32_t o_ex = __shfl_sync(0xffffffffu, excl, src);
      const uint32_t o_w = __shfl_sync(0xffffffffu, w, src);
      const uint32_t o_xy = __shfl_sync(0xffffffffu, xy0, src);
      const uint32_t o_idx = __shfl_sync(0xffffffffu, idx, src);
      const uint32_t o_msk = MASK ? __shfl_sync(0xffffffffu, msk, src) : 0xffffffffu;
      uint32_t t = 0;
      if (ok) {
        // the record's qq-th listed tile: the qq-th set bit of its R37 mask,
        // else the qq-th tile of the rect (row-major)
        uint32_t qq = f - o_ex;
        if (o_msk != 0xffffffffu) qq = __fns(o_msk, 0u, (int)qq + 1);
        // qq / o_w for small integers via the approximate f32 reciprocal: (qq + 0.5) / o_w lies
        // >= 0.5 / o_w from an integer and rcp.approx + the product err by <= (qq + 0.5) 2^-22 / o_w,
        // so the truncation is exact for qq < 2^21 (qq < MAX_TILES here)
        float rw;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rw) : "f"((float)o_w));
        const uint32_t row = (uint32_t)(((float)qq + 0.5f) * rw);
        t = ((o_xy >> 16) + row) * rp.TX + (o_xy & 0xffffu) + (qq - row * o_w);
      }
      uint32_t peers;
      if (STAMP) {
        // lanes sharing a tile agree on a representative (the last lane that
        // stamped it); one shared-memory OR per lane then yields the peer mask
        if (ok) st[t] = (uint8_t)lane;
        __syncwarp();
        const uint32_t rep = ok ? st[t] : 0u;
        if (ok) atomicOr(&pm[rep], 1u << lane);
        __syncwarp();
        peers = ok ? pm[rep] : 0u;
        __syncwarp();
        if (ok && lane == (int)rep) pm[rep] = 0u;
#ifdef GG_CHECK_PROTOCOLS
        {
          const uint32_t ref = __match_any_sync(0xffffffffu, ok ? t : 0xffffffffu);
          if (ok && peers != ref) __trap();
        }
#endif
      } else {
        peers = __ballot_sync(0xffffffffu, ok);
#pragma unroll
        for (int bb = 0; bb < TB; ++bb) {
          const bool bit = (t >> bb) & 1u;
          const uint32_t m = __ballot_sync(0xffffffffu, bit);
          peers &= bit ? m : ~m;
        }
      }
      const uint32_t before = ok ? (h[t >> 1] >> (16 * (t & 1))) & 0xffffu : 0u;
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) atomicAdd(&h[t >> 1], __popc(peers) << (16 * (t & 1)));
      __syncwarp();
#ifdef GG_CHECK_PROTOCOLS   // every list slot is written exactly once (the buffer is pre-filled with ~0)
      if (ok && atomicExch(&out[gb[t] + before + __popc(peers & lt)], o_idx) != 0xffffffffu) __trap();
#else
      if (ok) out[gb[t] + before + __popc(peers & lt)] = o_idx;
#endif
    }
  }
}

template <int TB, bool LOOP, bool MASK>
__global__ void __launch_bounds__(PD_THREADS, PD_MINB)
place_downsweep_kernel(BlockTable bt, ChunkWS ws, const uint32_t* order, RenderParams rp, const uint32_t* thist,
                       int S) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (!chunk_ok(ws.ok)) return;
  const uint32_t nb = bt.blk_base[bt.ec];
  if (!LOOP) {                                     // one CTA per block (sync mode)
    if (blockIdx.x < nb) place_downsweep_block<TB, MASK>(blockIdx.x, bt, ws, order, rp, thist, S, smem_raw);
    return;
  }
  for (;;) {   // async mode: bounded grid, blocks taken dynamically
    const uint32_t b = next_block(bt.q);
    if (b >= nb) break;
    place_downsweep_block<TB, MASK>(b, bt, ws, order, rp, thist, S, smem_raw);
  }
}

// ---- host side -------------------------------------------------------------
size_t depth_down_smem() { return sizeof(DownSmem); }
// placement segments per block: as many warps as the shared-memory budget
// allows (per segment: packed u16 counters, and for <= 2048 tiles the u8
// stamps and 32 peer masks of the warp-private ranking)
static size_t place_seg_bytes(int ntiles) {
  const size_t w = ((size_t)ntiles + 1) / 2 * 4;
  return ntiles <= 2048 ? w + 128 + (size_t)ntiles : w;
}
int place_segments(int ntiles) {
  const size_t budget = PD_SMEM - (size_t)ntiles * 4;
  const int s = (int)(budget / place_seg_bytes(ntiles));
  return s < 1 ? 1 : (s > PD_WARPS ? PD_WARPS : s);
}
size_t place_down_smem(int ntiles) {
  return (size_t)ntiles * 4 + (size_t)place_segments(ntiles) * place_seg_bytes(ntiles);
}

template <bool LOOP, bool MASK>
static cudaError_t place_init_variant() {
  cudaError_t e = cudaFuncSetAttribute(place_downsweep_kernel<8, LOOP, MASK>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, PD_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(place_downsweep_kernel<11, LOOP, MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PD_SMEM);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(place_downsweep_kernel<13, LOOP, MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           PD_SMEM);
  if (e != cudaSuccess) return e;
  return cudaFuncSetAttribute(place_upsweep_kernel<LOOP, MASK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)(MAX_TILES * 4));
}

template <bool LOOP>
static cudaError_t sort_bin_init_variant() {
  cudaError_t e = cudaFuncSetAttribute(depth_downsweep_kernel<LOOP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)depth_down_smem());
  if (e != cudaSuccess) return e;
  for (int mask = 0; mask < 2; ++mask) {
    e = mask ? place_init_variant<LOOP, true>() : place_init_variant<LOOP, false>();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

cudaError_t sort_bin_init() {
  cudaError_t e = sort_bin_init_variant<false>();
  return e != cudaSuccess ? e : sort_bin_init_variant<true>();
}

uint32_t sort_blocks(uint32_t V) { return (V + SORT_BLK - 1) / SORT_BLK; }
int sort_block_size() { return SORT_BLK; }
size_t sort_ghist_words() { return DS_RADIX; }

// number of depth passes for a key span (bits(far) - bits(near))
int depth_passes(uint32_t span) {
  int bits = 0;
  while (bits < 32 && (span >> bits) != 0) ++bits;
  const int p = (bits + DS_BITS - 1) / DS_BITS;
  return p < 1 ? 1 : p;
}

// Enqueue K3-K5 for a chunk.  blk_base: device [ec+1] block prefix; nb total
// blocks; ghist >= nb*DS_RADIX u32; thist >= nb*ntiles u32.  Returns launches.
template <bool LOOP>
static int launch_sort_bin_t(int ec, uint32_t nb, BlockTable bt, int passes, const RenderParams& rp,
                             const ChunkWS& ws, uint32_t* ghist, uint32_t* thist, cudaStream_t s, uint32_t* qctr,
                             cudaEvent_t after_depth) {
  // sync mode (LOOP = false): one CTA per block; async mode: nb is only a
  // capacity, so a bounded grid (a few waves of resident CTAs) takes the
  // blocks that exist from per-launch work counters
  const uint32_t g1 = LOOP ? std::min<uint32_t>(nb, 148u * 8u) : nb;
  const uint32_t g2 = LOOP ? std::min<uint32_t>(nb, 148u * 6u) : nb;
  int launches = 0;
  int qi = 0;
  if (LOOP) cudaMemsetAsync(qctr, 0, SORT_QCTR * sizeof(uint32_t), s);
  for (int p = 0; p < passes; ++p) {
    DepthIO io;
    io.zin = p == 0 ? ws.zkey : nullptr;
    io.pin = p == 0 ? nullptr : ((p & 1) ? ws.dp0 : ws.dp1);
    io.pout = p == passes - 1 ? nullptr : ((p & 1) ? ws.dp1 : ws.dp0);
    io.vout = ws.order;
    io.kout = reinterpret_cast<uint32_t*>((p & 1) ? ws.dp1 : ws.dp0);   // free on the last pass (it reads the other)
    if (LOOP) bt.q = qctr + qi++;
    depth_upsweep_kernel<LOOP><<<g1, DS_THREADS, 0, s>>>(bt, ws, io, DS_BITS * p, ghist);
    depth_scan_kernel<<<ec, DS_RADIX, 0, s>>>(bt, ghist, ws.ok);
    if (LOOP) bt.q = qctr + qi++;
    depth_downsweep_kernel<LOOP><<<g1, DS_THREADS, depth_down_smem(), s>>>(bt, ws, io, DS_BITS * p, ghist);
    launches += 3;
  }
  // gid order inside runs of equal depth keys (records are in storage order)
  if (LOOP) bt.q = qctr + qi++;
  depth_ties_kernel<LOOP><<<g1, TIES_THREADS, 0, s>>>(
      bt, ws, reinterpret_cast<const uint32_t*>(((passes - 1) & 1) ? ws.dp1 : ws.dp0));
  launches += 1;
  if (after_depth) cudaEventRecord(after_depth, s);   // stage timing: depth passes | placement
  const uint32_t* order = ws.order;   // records of the last depth pass
  if (LOOP) bt.q = qctr + qi++;
  const bool mask = ws.rmask != nullptr;
  if (mask)
    place_upsweep_kernel<LOOP, true><<<g2, SB_THREADS, rp.ntiles * 4, s>>>(bt, ws, order, rp.ntiles, rp.TX, thist);
  else
    place_upsweep_kernel<LOOP, false><<<g2, SB_THREADS, rp.ntiles * 4, s>>>(bt, ws, order, rp.ntiles, rp.TX, thist);
  place_scan_kernel<<<ec, PS_THREADS, 0, s>>>(bt, ws, thist, rp.ntiles);
  if (LOOP) bt.q = qctr + qi++;
  const size_t psm = place_down_smem(rp.ntiles);
  const int S = place_segments(rp.ntiles);
  if (rp.ntiles <= 256)
    mask ? place_downsweep_kernel<8, LOOP, true><<<g2, PD_THREADS, psm, s>>>(bt, ws, order, rp, thist, S)
         : place_downsweep_kernel<8, LOOP, false><<<g2, PD_THREADS, psm, s>>>(bt, ws, order, rp, thist, S);
  else if (rp.ntiles <= 2048)
    mask ? place_downsweep_kernel<11, LOOP, true><<<g2, PD_THREADS, psm, s>>>(bt, ws, order, rp, thist, S)
         : place_downsweep_kernel<11, LOOP, false><<<g2, PD_THREADS, psm, s>>>(bt, ws, order, rp, thist, S);
  else
    mask ? place_downsweep_kernel<13, LOOP, true><<<g2, PD_THREADS, psm, s>>>(bt, ws, order, rp, thist, S)
         : place_downsweep_kernel<13, LOOP, false><<<g2, PD_THREADS, psm, s>>>(bt, ws, order, rp, thist, S);
  return launches + 3;
}

// Enqueue K3-K5 for a chunk.  blk_base: device [ec+1] block prefix; nb total
// blocks; nb_is_capacity: nb is a capacity and the bounded-grid work-counter
// variants run (else one CTA per block of nb, surplus CTAs exit); ghist >= nb*DS_RADIX u32; thist >=
// nb*ntiles u32.  Returns the number of launches.
int launch_sort_bin(int ec, uint32_t nb, const uint32_t* blk_base, uint32_t* blk_env, int passes,
                    const RenderParams& rp, const ChunkWS& ws, uint32_t* ghist, uint32_t* thist, cudaStream_t s,
                    bool nb_is_capacity, uint32_t* qctr, cudaEvent_t after_depth) {
  if (nb == 0) {
    if (after_depth) cudaEventRecord(after_depth, s);
    cudaMemsetAsync(ws.ranges, 0, (size_t)ec * rp.ntiles * sizeof(uint2), s);
    return 0;
  }
  blk_env_kernel<<<ec, 128, 0, s>>>(blk_base, ec, blk_env);
  BlockTable bt{blk_base, blk_env, ec, nullptr};
  return 1 + (nb_is_capacity ? launch_sort_bin_t<true>(ec, nb, bt, passes, rp, ws, ghist, thist, s, qctr, after_depth)
                            : launch_sort_bin_t<false>(ec, nb, bt, passes, rp, ws, ghist, thist, s, nullptr,
                                                       after_depth));
}

}  // namespace gg
