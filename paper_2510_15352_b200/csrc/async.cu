// async.cu — device-side offset tables of the sync-free render mode
// (GG_ASYNC; SURVEY §8(f) row 2 "graph-capturable gg_render").  The
// host-synchronising mode reads the per-env visible/key counts back to size
// the workspace; this mode keeps everything on the device: exclusive scans
// over the chunk's envs give record offsets, key offsets and the sort block
// table, checked against the capacities reserved by gg_reserve_async.  On
// overflow the chunk is marked invalid (kernels skip it, its frames are
// background) and a sticky GG_E_CAPACITY is raised for gg_check_errors.
#include "gg_internal.cuh"

namespace gg {

constexpr int TB_THREADS = 1024;

__device__ __forceinline__ uint64_t block_excl_scan64(uint64_t x, uint64_t* wsum, uint64_t* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t s = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s += y;
  }
  if (lane == 31) wsum[warp] = s;
  __syncthreads();
  if (warp == 0) {
    uint64_t t = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    wsum[lane] = t;
  }
  __syncthreads();
  const uint64_t ex = (warp ? wsum[warp - 1] : 0ull) + s - x;
  *total = wsum[31];
  __syncthreads();
  return ex;
}

// rec_base = excl-scan(vcnt); overflow -> chunk invalid
__global__ void __launch_bounds__(TB_THREADS)
tables_v_kernel(int ec, const uint32_t* __restrict__ vcnt, uint64_t* __restrict__ rbase, uint64_t vcap,
                uint32_t* ok, uint32_t* err) {
  __shared__ uint64_t wsum[32];
  uint64_t carry = 0;
  for (int base = 0; base < ec; base += TB_THREADS) {
    const int e = base + threadIdx.x;
    const uint64_t x = e < ec ? vcnt[e] : 0ull;
    uint64_t tot;
    const uint64_t ex = carry + block_excl_scan64(x, wsum, &tot);
    if (e < ec) rbase[e] = ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && carry > vcap) {
    *ok = 0u;
    atomicOr(err, (uint32_t)ERR_CAPACITY);
  }
}

// k_base = excl-scan(kcnt); blk_base = excl-scan(ceil(vcnt / sort_blk)) (ec+1 entries)
__global__ void __launch_bounds__(TB_THREADS)
tables_k_kernel(int ec, const uint32_t* __restrict__ vcnt, const unsigned long long* __restrict__ kcnt,
                uint64_t* __restrict__ kbase, uint32_t* __restrict__ blkbase, int sort_blk, uint64_t kcap,
                uint64_t nbcap, uint32_t* ok, uint32_t* err) {
  __shared__ uint64_t wsum[32];
  uint64_t ck = 0, cb = 0;
  __shared__ uint32_t wide;   // an env with >= 2^32 keys (u32 list offsets)
  if (threadIdx.x == 0) wide = 0u;
  __syncthreads();
  for (int base = 0; base < ec; base += TB_THREADS) {
    const int e = base + threadIdx.x;
    const uint64_t k = e < ec ? kcnt[e] : 0ull;
    if (k > 0xffffffffull) wide = 1u;
    const uint64_t nb = e < ec ? (vcnt[e] + (uint64_t)sort_blk - 1) / (uint64_t)sort_blk : 0ull;
    uint64_t tk, tb;
    const uint64_t exk = ck + block_excl_scan64(k, wsum, &tk);
    const uint64_t exb = cb + block_excl_scan64(nb, wsum, &tb);
    if (e < ec) {
      kbase[e] = exk;
      blkbase[e] = (uint32_t)exb;
    }
    ck += tk;
    cb += tb;
  }
  if (threadIdx.x == 0) {
    blkbase[ec] = (uint32_t)(cb <= nbcap ? cb : nbcap);
    if (ck > kcap || cb > nbcap || wide) {
      *ok = 0u;
      atomicOr(err, (uint32_t)ERR_CAPACITY);
    }
  }
}

void launch_tables_v(int ec, const uint32_t* vcnt, uint64_t* rbase, uint64_t vcap, uint32_t* ok, uint32_t* err,
                     cudaStream_t s) {
  tables_v_kernel<<<1, TB_THREADS, 0, s>>>(ec, vcnt, rbase, vcap, ok, err);
}

void launch_tables_k(int ec, const uint32_t* vcnt, const unsigned long long* kcnt, uint64_t* kbase, uint32_t* blkbase,
                     int sort_blk, uint64_t kcap, uint64_t nbcap, uint32_t* ok, uint32_t* err, cudaStream_t s) {
  tables_k_kernel<<<1, TB_THREADS, 0, s>>>(ec, vcnt, kcnt, kbase, blkbase, sort_blk, kcap, nbcap, ok, err);
}

}  // namespace gg
