// sort_bin.cu — K3-K5: per-env depth presort, stable tile placement and tile
// ranges, one CTA per environment.
//
// Defines the per-tile lists of SPEC.md:136-144 (bin_and_sort: "each tile
// lists every gaussian whose 3-sigma footprint intersects it, sorted
// ascending by view_depth; ties broken by input index (stable)").  The
// canonical list (DESIGN.md §2 O3) is the triples (tile, depth bits, gid) in
// ascending order.  We produce it without ever materialising 64-bit keys:
//   0. one pass over the env's records builds the four 8-bit digit
//      histograms of the depth bits and the tile histogram; an exclusive
//      scan of the latter IS the tile-range table (K5)
//   1. stable LSD radix sort of the records (already in gid order) by the
//      f32 depth bits, skipping passes whose digit is constant  -> (z, gid)
//   2. walk the records in that order; each record's tiles are appended to
//      a shared-memory list in record order, and ONE warp places the list
//      32 entries at a time: __match_any_sync groups equal tiles, the group
//      leader advances that tile's cursor.  Every tile's entries therefore
//      land in (z, gid) order at their final position: (tile, z, gid).
// Deterministic: no float math, no order-dependent atomics.
#include "gg_internal.cuh"

namespace gg {

constexpr int SB_THREADS = 256;
constexpr int SB_WARPS = SB_THREADS / 32;
constexpr int SB_IPT = 8;
constexpr int SB_TILE = SB_THREADS * SB_IPT;
constexpr int SB_CAP = 2048;     // placement list capacity (pairs)

struct SortSmem {
  uint32_t hist[4][256];
  uint32_t wcnt[SB_WARPS][256];
  uint32_t wsum[SB_WARPS];
  uint32_t cur[256];
  uint2 list[SB_CAP];             // (tile, record)
  uint32_t tcur[1];               // [ntiles] tile cursors (dynamic tail)
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

// One stable counting pass on digit (key >> shift) & 255 with a precomputed
// histogram.  vin == nullptr means identity values; kout == nullptr skips
// writing keys (last pass).
__device__ void radix_pass(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                           uint32_t* __restrict__ kout, uint32_t* __restrict__ vout, uint32_t n, int shift,
                           const uint32_t* hist, SortSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // exclusive scan of the 256-bin histogram -> cursors
  {
    const uint32_t x = hist[tid];
    uint32_t total;
    const uint32_t ex = block_excl_scan(x, sm.wsum, &total);
    sm.cur[tid] = ex;
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
    {   // per-digit prefix over warps, starting at the global cursor
      uint32_t run = sm.cur[tid];
#pragma unroll
      for (int w = 0; w < SB_WARPS; ++w) {
        const uint32_t t = sm.wcnt[w][tid];
        sm.wcnt[w][tid] = run;
        run += t;
      }
      sm.cur[tid] = run;
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
#pragma unroll
    for (int w = 0; w < SB_WARPS; ++w) sm.wcnt[w][tid] = 0u;
    __syncthreads();
  }
}

__device__ __forceinline__ void unpack_rect(uint2 r, uint32_t& x0, uint32_t& x1, uint32_t& y0, uint32_t& y1) {
  x0 = r.x & 0xffffu; x1 = r.x >> 16; y0 = r.y & 0xffffu; y1 = r.y >> 16;
}

__global__ void __launch_bounds__(SB_THREADS)
sort_bin_kernel(RenderParams rp, ChunkWS ws) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem& sm = *reinterpret_cast<SortSmem*>(smem_raw);
  const int eloc = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t rb = ws.rec_base[eloc];
  const uint64_t kb = ws.k_base[eloc];
  const uint32_t V = ws.vcnt[eloc];
  for (int i = tid; i < 4 * 256; i += SB_THREADS) (&sm.hist[0][0])[i] = 0u;
  for (int w = 0; w < SB_WARPS; ++w) sm.wcnt[w][tid] = 0u;
  for (int i = tid; i < rp.ntiles; i += SB_THREADS) sm.tcur[i] = 0u;
  __syncthreads();

  // ---- 0. digit histograms of the depth bits + tile histogram ----------
  const uint32_t* zk = ws.zkey + rb;
  const uint2* rect = ws.rect + rb;
  for (uint32_t j = tid; j < V; j += SB_THREADS) {
    const uint32_t z = zk[j];
    atomicAdd(&sm.hist[0][z & 255u], 1u);
    atomicAdd(&sm.hist[1][(z >> 8) & 255u], 1u);
    atomicAdd(&sm.hist[2][(z >> 16) & 255u], 1u);
    atomicAdd(&sm.hist[3][z >> 24], 1u);
    uint32_t x0, x1, y0, y1;
    unpack_rect(rect[j], x0, x1, y0, y1);
    for (uint32_t ty = y0; ty < y1; ++ty)
      for (uint32_t tx = x0; tx < x1; ++tx) atomicAdd(&sm.tcur[ty * rp.TX + tx], 1u);
  }
  __syncthreads();
  // ---- K5: tile ranges = exclusive scan of the tile histogram ----------
  {
    uint32_t carry = 0;
    for (int base = 0; base < rp.ntiles; base += SB_THREADS) {
      const int t = base + tid;
      const uint32_t c = t < rp.ntiles ? sm.tcur[t] : 0u;
      uint32_t total;
      const uint32_t ex = carry + block_excl_scan(c, sm.wsum, &total);
      if (t < rp.ntiles) {
        ws.ranges[(size_t)eloc * rp.ntiles + t] = make_uint2(ex, ex + c);
        sm.tcur[t] = ex;          // becomes the placement cursor
      }
      carry += total;
    }
  }
  // which depth digits vary?  (a constant digit leaves the order unchanged)
  __shared__ uint32_t live_mask;
  if (tid == 0) live_mask = 0;
  __syncthreads();
#pragma unroll
  for (int p = 0; p < 4; ++p)
    if (sm.hist[p][tid] == V && V > 0) atomicOr(&live_mask, 1u << (4 + p));   // bit 4+p: constant
  __syncthreads();
  const uint32_t constant = live_mask >> 4;

  // ---- 1. stable LSD depth sort ------------------------------------------
  const uint32_t* ck = zk;
  const uint32_t* cv = nullptr;   // identity (records are in gid order)
  uint32_t* bufk[2] = {ws.dk0 + rb, ws.dk1 + rb};
  uint32_t* bufv[2] = {ws.dv0 + rb, ws.dv1 + rb};
  int last = -1;
  for (int p = 0; p < 4; ++p)
    if (!((constant >> p) & 1u)) last = p;
  int nb = 0;
  for (int p = 0; p < 4; ++p) {
    if ((constant >> p) & 1u) continue;
    radix_pass(ck, cv, p == last ? nullptr : bufk[nb], bufv[nb], V, p * 8, sm.hist[p], sm);
    ck = bufk[nb];
    cv = bufv[nb];
    nb ^= 1;
  }

  // ---- 2. stable placement in (z, gid) order ------------------------------
  uint32_t* out = ws.sorted + kb;
  for (uint32_t base = 0; base < V; base += SB_THREADS) {
    const uint32_t j = base + tid;
    uint32_t idx = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
    if (j < V) {
      idx = cv ? cv[j] : j;
      unpack_rect(rect[idx], x0, x1, y0, y1);
    }
    const uint32_t w = x1 - x0;
    const uint32_t n = w * (y1 - y0);
    uint32_t total;
    const uint32_t excl = block_excl_scan(n, sm.wsum, &total);
    for (uint32_t w0 = 0; w0 < total; w0 += SB_CAP) {
      // this thread's pairs with flattened position in [w0, w0 + CAP)
      const uint32_t qa = excl >= w0 ? 0u : w0 - excl;
      const uint32_t qb = min(n, w0 + SB_CAP > excl ? w0 + SB_CAP - excl : 0u);
      for (uint32_t q = qa; q < qb; ++q) {
        const uint32_t ty = y0 + q / w, tx = x0 + q % w;
        sm.list[excl + q - w0] = make_uint2(ty * rp.TX + tx, idx);
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t m = min((uint32_t)SB_CAP, total - w0);
        for (uint32_t g = 0; g < m; g += 32) {
          const bool valid = g + lane < m;
          const uint2 e = valid ? sm.list[g + lane] : make_uint2(0xffffffffu, 0u);
          const uint32_t peers = __match_any_sync(0xffffffffu, e.x);
          const uint32_t before = valid ? sm.tcur[e.x] : 0u;
          __syncwarp();
          if (valid && lane == __ffs(peers) - 1) sm.tcur[e.x] = before + __popc(peers);
          __syncwarp();
          if (valid) out[before + __popc(peers & lanemask_lt())] = e.y;
        }
      }
      __syncthreads();
    }
  }
}

size_t sort_bin_smem(int ntiles) {
  size_t base = offsetof(SortSmem, tcur);
  return base + (size_t)ntiles * 4;
}

cudaError_t sort_bin_init() {
  return cudaFuncSetAttribute(sort_bin_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)sort_bin_smem(MAX_TILES));
}

void launch_sort_bin(int ec, const RenderParams& rp, const ChunkWS& ws, cudaStream_t s) {
  sort_bin_kernel<<<ec, SB_THREADS, sort_bin_smem(rp.ntiles), s>>>(rp, ws);
}

}  // namespace gg
