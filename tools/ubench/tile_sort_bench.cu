// tile_sort_bench.cu — feasibility microbenchmark for a "tile-first" binning:
// per-tile lists (record indices in arbitrary order) sorted by the 64-bit key
// (f32 depth bits << 32 | gid) with a shared-memory bitonic network, one CTA
// per list, lists classed by length.  List lengths follow the c3 distribution
// measured with the oracle (opacity-aware lists: 64-24k entries, ~440 mean).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tile_sort_bench tile_sort_bench.cu
//   ./tile_sort_bench [n_tiles=1228800]   -> one JSON line (ms per class, keys/s)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t key_of(const uint32_t* __restrict__ z, const uint32_t* __restrict__ g, uint32_t r) {
  return ((uint64_t)z[r] << 32) | g[r];
}

// one CTA of T threads sorts list w (length n <= NMAX) in shared memory
template <int T, int NMAX>
__global__ void __launch_bounds__(T) sort_class(const uint32_t* __restrict__ work, const uint2* __restrict__ ranges,
                                                uint32_t* __restrict__ list, const uint32_t* __restrict__ z,
                                                const uint32_t* __restrict__ g) {
  extern __shared__ __align__(16) unsigned char sm_raw[];
  uint64_t* K = reinterpret_cast<uint64_t*>(sm_raw);
  uint32_t* V = reinterpret_cast<uint32_t*>(K + NMAX);
  const uint2 rg = ranges[work[blockIdx.x]];
  const uint32_t n = rg.y - rg.x;
  uint32_t N = 2;
  while (N < n) N <<= 1;
  for (uint32_t i = threadIdx.x; i < N; i += T) {
    if (i < n) {
      const uint32_t r = list[rg.x + i];
      K[i] = key_of(z, g, r);
      V[i] = r;
    } else {
      K[i] = ~0ull;
      V[i] = 0u;
    }
  }
  __syncthreads();
  for (uint32_t k = 2; k <= N; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < N / 2; t += T) {
        const uint32_t i = 2 * t - (t & (j - 1));   // lower index of the pair (bit j clear)
        const uint32_t l = i + j;
        const bool up = (i & k) == 0;
        const uint64_t a = K[i], b = K[l];
        if ((a > b) == up) {
          K[i] = b; K[l] = a;
          const uint32_t va = V[i];
          V[i] = V[l]; V[l] = va;
        }
      }
      __syncthreads();
    }
  }
  for (uint32_t i = threadIdx.x; i < n; i += T) list[rg.x + i] = V[i];
}

int main(int argc, char** argv) {
  const int ntile = argc > 1 ? atoi(argv[1]) : 1228800;   // 1024 envs x 1200 tiles
  // c3 opacity-aware list-length distribution (log2 bins 5..15, oracle, 16 envs)
  const int bins[11] = {96, 3175, 4607, 3996, 3294, 2041, 1188, 533, 223, 40, 7};
  const int tot = 19200;
  std::vector<uint32_t> len(ntile);
  uint64_t s = 12345;
  auto rnd = [&]() { s = s * 6364136223846793005ull + 1442695040888963407ull; return (uint32_t)(s >> 33); };
  uint64_t K = 0;
  for (int t = 0; t < ntile; ++t) {
    int x = rnd() % tot, b = 0;
    while (x >= bins[b]) x -= bins[b++];
    const uint32_t lo = b == 0 ? 1u : (1u << (b + 4)) + 1u, hi = 1u << (b + 5);
    len[t] = lo + rnd() % (hi - lo + 1);
    K += len[t];
  }
  const uint32_t NREC = 250000;
  std::vector<uint2> rg(ntile);
  std::vector<uint32_t> list(K);
  uint64_t off = 0;
  for (int t = 0; t < ntile; ++t) {
    rg[t] = make_uint2((uint32_t)off, (uint32_t)(off + len[t]));
    for (uint32_t i = 0; i < len[t]; ++i) list[off + i] = rnd() % NREC;
    off += len[t];
  }
  std::vector<uint32_t> zh(NREC), gh(NREC);
  for (uint32_t r = 0; r < NREC; ++r) { zh[r] = 0x3c000000u + rnd() % (1u << 26); gh[r] = r; }
  // classes by length
  const int NC = 4;
  const uint32_t cmax[NC] = {256, 2048, 16384, 0xffffffffu};
  std::vector<uint32_t> work[NC];
  for (int t = 0; t < ntile; ++t)
    for (int c = 0; c < NC; ++c)
      if (len[t] <= cmax[c]) { work[c].push_back(t); break; }
  uint2* d_rg; uint32_t *d_list, *d_z, *d_g, *d_work[NC];
  cudaMalloc(&d_rg, ntile * sizeof(uint2));
  cudaMalloc(&d_list, K * 4);
  cudaMalloc(&d_z, NREC * 4);
  cudaMalloc(&d_g, NREC * 4);
  cudaMemcpy(d_rg, rg.data(), ntile * sizeof(uint2), cudaMemcpyHostToDevice);
  cudaMemcpy(d_z, zh.data(), NREC * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(d_g, gh.data(), NREC * 4, cudaMemcpyHostToDevice);
  for (int c = 0; c < NC; ++c) {
    cudaMalloc(&d_work[c], std::max<size_t>(1, work[c].size()) * 4);
    cudaMemcpy(d_work[c], work[c].data(), work[c].size() * 4, cudaMemcpyHostToDevice);
  }
  cudaFuncSetAttribute(sort_class<1024, 16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 * 12);
  cudaEvent_t e[NC + 1];
  for (auto& x : e) cudaEventCreate(&x);
  float ms[NC] = {0, 0, 0, 0};
  for (int rep = 0; rep < 3; ++rep) {
    cudaMemcpy(d_list, list.data(), K * 4, cudaMemcpyHostToDevice);
    cudaEventRecord(e[0]);
    if (work[0].size()) sort_class<128, 256><<<work[0].size(), 128, 256 * 12>>>(d_work[0], d_rg, d_list, d_z, d_g);
    cudaEventRecord(e[1]);
    if (work[1].size()) sort_class<512, 2048><<<work[1].size(), 512, 2048 * 12>>>(d_work[1], d_rg, d_list, d_z, d_g);
    cudaEventRecord(e[2]);
    if (work[2].size()) sort_class<1024, 16384><<<work[2].size(), 1024, 16384 * 12>>>(d_work[2], d_rg, d_list, d_z, d_g);
    cudaEventRecord(e[3]);
    cudaEventRecord(e[4]);
    cudaEventSynchronize(e[4]);
    for (int c = 0; c < 3; ++c) cudaEventElapsedTime(&ms[c], e[c], e[c + 1]);
  }
  // verify sortedness of a few lists
  std::vector<uint32_t> out(K);
  cudaMemcpy(out.data(), d_list, K * 4, cudaMemcpyDeviceToHost);
  uint64_t bad = 0;
  for (int t = 0; t < ntile; t += 97) {
    if (len[t] > 16384) continue;
    for (uint32_t i = 1; i < len[t]; ++i) {
      const uint32_t a = out[rg[t].x + i - 1], b = out[rg[t].x + i];
      if ((((uint64_t)zh[a] << 32) | gh[a]) > (((uint64_t)zh[b] << 32) | gh[b])) ++bad;
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"tiles\": %d, \"keys\": %llu, \"class_tiles\": [%zu, %zu, %zu, %zu], \"ms\": [%.3f, %.3f, %.3f], "
         "\"total_ms\": %.3f, \"keys_per_s\": %.3e, \"unsorted_pairs\": %llu, \"err\": \"%s\"}\n",
         ntile, (unsigned long long)K, work[0].size(), work[1].size(), work[2].size(), work[3].size(), ms[0], ms[1],
         ms[2], ms[0] + ms[1] + ms[2], K / ((ms[0] + ms[1] + ms[2]) * 1e-3), (unsigned long long)bad,
         cudaGetErrorString(err));
  return 0;
}
