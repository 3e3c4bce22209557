// sort_bin.cu — K3-K5: per-env depth presort, key emission, stable tile
// bucketing and tile ranges, one CTA per environment.
//
// Defines the per-tile lists of SPEC.md:136-144 (bin_and_sort: "each tile
// lists every gaussian whose 3-sigma footprint intersects it, sorted
// ascending by view_depth; ties broken by input index (stable)").  The
// canonical list (DESIGN.md §2 O3) is the triples (tile, depth bits, gid)
// in ascending order.  We produce it as:
//   1. stable LSD radix sort of the env's records (already in gid order) by
//      the f32 bits of the view depth (4 x 8-bit passes; a pass whose digit
//      is constant over the segment is skipped)          -> (z, gid) order
//   2. emission of (tile, record) pairs in that order, tiles of each record
//      row-major, with an exclusive-scan allocator; a shared-memory tile
//      histogram gives the tile ranges directly (K5)
//   3. stable LSD radix sort of the pairs by tile (8-bit digits)
//                                                          -> (tile, z, gid)
// which is the canonical order because each pass is stable.
//
// Stable ranking inside a 4096-element tile: each warp owns 256 consecutive
// elements processed in 8 rounds; __match_any_sync groups equal digits,
// per-warp digit counters accumulate across rounds, and a per-digit prefix
// over warps places the warps in input order.  Deterministic: no float
// math, no order-dependent atomics.
#include "gg_internal.cuh"

namespace gg {

constexpr int SB_THREADS = 512;
constexpr int SB_WARPS = SB_THREADS / 32;
constexpr int SB_IPT = 8;
constexpr int SB_TILE = SB_THREADS * SB_IPT;

struct SortSmem {
  uint32_t hist[256];
  uint32_t wcnt[SB_WARPS][256];
  uint32_t wsum[SB_WARPS];
  uint32_t flag;
  uint32_t thist[MAX_TILES];
};

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t x, uint32_t* wsum, uint32_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t s = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += y;
  }
  if (lane == 31) wsum[warp] = s;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = lane < SB_WARPS ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < SB_WARPS) wsum[lane] = t;
  }
  __syncthreads();
  const uint32_t excl = (warp ? wsum[warp - 1] : 0u) + s - x;
  *total = wsum[SB_WARPS - 1];
  __syncthreads();
  return excl;
}

// One stable counting pass on digit (key >> shift) & 255.
// vin == nullptr means identity values.  Writes keys only if kout != nullptr.
// Returns false (nothing written) if the digit is constant and !force.
__device__ bool radix_pass(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                           uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, uint32_t n,
                           int shift, bool force, SortSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 256; i += SB_THREADS) sm.hist[i] = 0;
  if (tid == 0) sm.flag = 0;
  __syncthreads();
  for (uint32_t i = tid; i < n; i += SB_THREADS) atomicAdd(&sm.hist[(kin[i] >> shift) & 255u], 1u);
  __syncthreads();
  for (int i = tid; i < 256; i += SB_THREADS)
    if (sm.hist[i] == n) sm.flag = 1;
  __syncthreads();
  if (sm.flag && !force) return false;
  // exclusive scan of the 256-bin histogram -> cursors (warps 0..7)
  if (warp < 8) {
    const uint32_t x = sm.hist[warp * 32 + lane];
    uint32_t s = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane == 31) sm.wsum[warp] = s;
    __syncwarp();
    sm.hist[warp * 32 + lane] = s - x;   // local exclusive; add warp offsets below
  }
  __syncthreads();
  if (tid < 256) {
    uint32_t off = 0;
    for (int w = 0; w < tid / 32; ++w) off += sm.wsum[w];
    sm.hist[tid] += off;
  }
  __syncthreads();

  for (uint32_t base = 0; base < n; base += SB_TILE) {
    const uint32_t wbase = base + warp * 32 * SB_IPT;
    uint32_t k[SB_IPT], v[SB_IPT], rk[SB_IPT];
#pragma unroll
    for (int j = 0; j < SB_IPT; ++j) {
      const uint32_t idx = wbase + j * 32 + lane;
      const bool valid = idx < n;
      k[j] = valid ? kin[idx] : 0u;
      v[j] = valid ? (vin ? vin[idx] : idx) : 0u;
    }
#pragma unroll
    for (int j = 0; j < SB_IPT; ++j) {
      const uint32_t idx = wbase + j * 32 + lane;
      const bool valid = idx < n;
      const uint32_t d = valid ? ((k[j] >> shift) & 255u) : 256u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t before = valid ? sm.wcnt[warp][d] : 0u;
      __syncwarp();
      if (valid && lane == __ffs(peers) - 1) sm.wcnt[warp][d] = before + __popc(peers);
      __syncwarp();
      rk[j] = before + __popc(peers & lanemask_lt());
    }
    __syncthreads();
    // per-digit prefix over warps, starting at the global cursor
    if (tid < 256) {
      uint32_t run = sm.hist[tid];
#pragma unroll
      for (int w = 0; w < SB_WARPS; ++w) {
        const uint32_t t = sm.wcnt[w][tid];
        sm.wcnt[w][tid] = run;
        run += t;
      }
      sm.hist[tid] = run;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < SB_IPT; ++j) {
      const uint32_t idx = wbase + j * 32 + lane;
      if (idx < n) {
        const uint32_t d = (k[j] >> shift) & 255u;
        const uint32_t pos = sm.wcnt[warp][d] + rk[j];
        if (kout) kout[pos] = k[j];
        vout[pos] = v[j];
      }
    }
    __syncthreads();
    for (int i = tid; i < SB_WARPS * 256; i += SB_THREADS) (&sm.wcnt[0][0])[i] = 0u;
    __syncthreads();
  }
  return true;
}

__global__ void __launch_bounds__(SB_THREADS)
sort_bin_kernel(RenderParams rp, ChunkWS ws, int tile_passes) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
  const int eloc = blockIdx.x;
  const int tid = threadIdx.x;
  const uint64_t rb = ws.rec_base[eloc];
  const uint64_t kb = ws.k_base[eloc];
  const uint32_t V = ws.vcnt[eloc];
  const uint32_t K = ws.kcnt[eloc];
  for (int i = tid; i < SB_WARPS * 256; i += SB_THREADS) (&sm.wcnt[0][0])[i] = 0u;
  for (int i = tid; i < rp.ntiles; i += SB_THREADS) sm.thist[i] = 0u;
  __syncthreads();

  // ---- 1. stable depth sort of the env's records ----------------------
  const uint32_t* ck = ws.zkey + rb;
  const uint32_t* cv = nullptr;   // identity
  uint32_t* bufk[2] = {ws.dk0 + rb, ws.dk1 + rb};
  uint32_t* bufv[2] = {ws.dv0 + rb, ws.dv1 + rb};
  int nb = 0;
  for (int pass = 0; pass < 4; ++pass) {
    if (radix_pass(ck, cv, bufk[nb], bufv[nb], V, pass * 8, false, sm)) {
      ck = bufk[nb];
      cv = bufv[nb];
      nb ^= 1;
    }
    __syncthreads();
  }

  // ---- 2. emit (tile, record) pairs in (z, gid) order + tile histogram --
  uint32_t* tk[2] = {ws.tk0 + kb, ws.tk1 + kb};
  uint32_t* tv[2] = {ws.tv0 + kb, ws.tv1 + kb};
  uint32_t running = 0;
  for (uint32_t base = 0; base < V; base += SB_THREADS) {
    const uint32_t j = base + tid;
    uint32_t idx = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0, nt = 0;
    if (j < V) {
      idx = cv ? cv[j] : j;
      const uint2 r = ws.rect[rb + idx];
      x0 = r.x & 0xffffu; x1 = r.x >> 16; y0 = r.y & 0xffffu; y1 = r.y >> 16;
      nt = (x1 - x0) * (y1 - y0);
    }
    uint32_t total;
    uint32_t pos = running + block_excl_scan(nt, sm.wsum, &total);
    for (uint32_t ty = y0; ty < y1; ++ty)
      for (uint32_t tx = x0; tx < x1; ++tx) {
        const uint32_t t = ty * rp.TX + tx;
        tk[0][pos] = t;
        tv[0][pos] = idx;
        ++pos;
        atomicAdd(&sm.thist[t], 1u);
      }
    running += total;
  }
  __syncthreads();
  // ---- K5 ranges: exclusive scan of the tile histogram ------------------
  {
    uint32_t carry = 0;
    for (int base = 0; base < rp.ntiles; base += SB_THREADS) {
      const int t = base + tid;
      const uint32_t c = t < rp.ntiles ? sm.thist[t] : 0u;
      uint32_t total;
      const uint32_t ex = carry + block_excl_scan(c, sm.wsum, &total);
      if (t < rp.ntiles) ws.ranges[(size_t)eloc * rp.ntiles + t] = make_uint2(ex, ex + c);
      carry += total;
    }
  }
  __syncthreads();

  // ---- 3. stable tile bucketing: LSD passes on the tile index -----------
  int cur = 0;
  for (int pass = 0; pass < tile_passes; ++pass) {
    const bool last = pass == tile_passes - 1;
    if (last) {
      radix_pass(tk[cur], tv[cur], nullptr, ws.sorted + kb, K, pass * 8, true, sm);
    } else if (radix_pass(tk[cur], tv[cur], tk[cur ^ 1], tv[cur ^ 1], K, pass * 8, false, sm)) {
      cur ^= 1;
    }
    __syncthreads();
  }
}

size_t sort_bin_smem() { return sizeof(SortSmem); }

cudaError_t sort_bin_init() {
  return cudaFuncSetAttribute(sort_bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sizeof(SortSmem));
}

void launch_sort_bin(int ec, const RenderParams& rp, const ChunkWS& ws, int tile_passes, cudaStream_t s) {
  sort_bin_kernel<<<ec, SB_THREADS, sizeof(SortSmem), s>>>(rp, ws, tile_passes);
}

}  // namespace gg
