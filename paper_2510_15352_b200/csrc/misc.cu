#include <algorithm>
// misc.cu — K7 checksum and K8 debug extraction kernels.
#include "gg_internal.cuh"

namespace gg {

__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL;
  x ^= x >> 33;
  return x;
}

// K7: per-env digest = sum over elements of mix64(position, value bits).
// Integer sums are order-independent, so the digest is deterministic.
__global__ void checksum_kernel(int W, int H, const uint8_t* __restrict__ rgb8,
                                const float* __restrict__ rgbf, const float* __restrict__ depth,
                                unsigned long long* out) {
  const int e = blockIdx.y;
  const size_t P = (size_t)W * H;
  unsigned long long acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < P; i += (size_t)gridDim.x * blockDim.x) {
    const size_t p = (size_t)e * P + i;
    unsigned long long v = 0;
    if (rgb8) v = (unsigned long long)rgb8[p * 3] | ((unsigned long long)rgb8[p * 3 + 1] << 8) |
                  ((unsigned long long)rgb8[p * 3 + 2] << 16);
    if (rgbf) v ^= mix64(__float_as_uint(rgbf[p * 3]) ^ ((unsigned long long)__float_as_uint(rgbf[p * 3 + 1]) << 32)) ^
                   (unsigned long long)__float_as_uint(rgbf[p * 3 + 2]);
    if (depth) v ^= (unsigned long long)__float_as_uint(depth[p]) << 24;
    acc += mix64(v * 0x9E3779B97F4A7C15ULL + i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&out[e], acc);
}

void launch_checksum(int E, int W, int H, const uint8_t* rgb8, const float* rgbf, const float* depth,
                     unsigned long long* out, cudaStream_t s) {
  checksum_kernel<<<dim3(64, E), 256, 0, s>>>(W, H, rgb8, rgbf, depth, out);
}

// K8: intermediates of one env for gg_debug_dump (test only).
__global__ void debug_records_kernel(uint32_t V, uint64_t rb, const ChunkWS ws, int32_t* tile_counts,
                                     float* proj) {
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < V; j += gridDim.x * blockDim.x) {
    const uint64_t r = rb + j;
    const uint2 rc = ws.rect[r];
    const uint32_t x0 = rc.x & 0xffffu, x1 = rc.x >> 16, y0 = rc.y & 0xffffu, y1 = rc.y >> 16;
    const uint32_t area = (x1 - x0) * (y1 - y0);
    const uint32_t nt = rec_tiles(rec_mask(ws.rmask, r, area), area);
    const uint32_t g = ws.gid[r];
    tile_counts[g] = (int32_t)nt;
    if (nt) {
      const float4 a = ws.rec0[r], b = ws.dconic[r], c = ws.rec2[r];
      float* d = proj + (size_t)g * 16;
      d[0] = 1.f; d[1] = a.x; d[2] = a.y; d[3] = b.x; d[4] = b.y; d[5] = b.z; d[6] = a.w;
      d[7] = 0.f;   // radius is not stored by the product path
      d[8] = (float)x0; d[9] = (float)x1; d[10] = (float)y0; d[11] = (float)y1;
      d[12] = c.x; d[13] = c.y; d[14] = c.z; d[15] = b.w;
    }
  }
}

__global__ void debug_sorted_kernel(int ntiles, const uint2* __restrict__ ranges, uint64_t kb, uint64_t rb,
                                    const ChunkWS ws, int32_t* s_tile, uint32_t* s_z, int32_t* s_gid) {
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint2 rg = ranges[t];
    for (uint32_t k = rg.x + threadIdx.x; k < rg.y; k += blockDim.x) {
      const uint64_t r = rb + ws.sorted[kb + k];
      s_tile[k] = t;
      s_z[k] = ws.zkey[r];
      s_gid[k] = (int32_t)ws.gid[r];
    }
  }
}

void launch_debug_records(uint32_t V, uint64_t rb, const ChunkWS& ws, int32_t* tile_counts, float* proj,
                          cudaStream_t s) {
  debug_records_kernel<<<256, 256, 0, s>>>(V, rb, ws, tile_counts, proj);
}

void launch_debug_sorted(int ntiles, const uint2* ranges, uint64_t kb, uint64_t rb, const ChunkWS& ws,
                         int32_t* s_tile, uint32_t* s_z, int32_t* s_gid, cudaStream_t s) {
  debug_sorted_kernel<<<min(ntiles, 1024), 256, 0, s>>>(ntiles, ranges, kb, rb, ws, s_tile, s_z, s_gid);
}


// Small host<->device table transfers for the sync-mode host loop.  Pinned
// host memory is UVA-mapped, so a one-block kernel moves the words over the
// bus without touching a copy engine: the per-chunk readbacks never queue
// behind large frame copies (gg_render_host) issued on other streams.
__global__ void copy_words_kernel(uint32_t* __restrict__ dst, const uint32_t* __restrict__ src, size_t n) {
  for (size_t i = threadIdx.x + (size_t)blockIdx.x * blockDim.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

int launch_copy_words(void* dst, const void* src, size_t bytes, cudaStream_t s) {
  const size_t n = bytes / 4;
  if (!n) return 0;
  const int grid = (int)std::min<size_t>((n + 255) / 256, 64);
  copy_words_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<uint32_t*>(dst), reinterpret_cast<const uint32_t*>(src), n);
  return 1;
}

}  // namespace gg
