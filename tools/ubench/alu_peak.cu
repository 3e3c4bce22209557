// alu_peak.cu — measured FP32 / FFMA2 / MUFU.EX2 throughput of this B200
// ("verify both with microbenchmarks, including FFMA2").
// The raster (K6) reports its roofline fraction against the FP32 pipe; this
// program measures that denominator instead of assuming 148 x 128 x 2 x clk.
//
// Each kernel runs NCH independent dependency chains per thread (enough ILP
// to cover the pipe latency), a grid of 148 x 8 CTAs x 256 threads, and
// reports lane-ops per SM per cycle (cycles from clock64 on SM 0's CTAs and
// the wall time from CUDA events) and the absolute rate.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_peak alu_peak.cu
//   ./alu_peak            -> one JSON line
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int NCH = 8;
constexpr int ITERS = 4096;
constexpr int THREADS = 256;

__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo(uint64_t v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a + b;
}

__global__ void __launch_bounds__(THREADS) k_ffma(float* out, float a, float b, long long* cyc) {
  float x[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) x[c] = threadIdx.x * 1e-3f + c;
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) x[c] = fmaf(x[c], a, b);
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(THREADS) k_ffma2(float* out, float a, float b, long long* cyc) {
  uint64_t x[NCH];
  const uint64_t A = pk(a, a), B = pk(b, b);
#pragma unroll
  for (int c = 0; c < NCH; ++c) x[c] = pk(threadIdx.x * 1e-3f + c, c * 0.5f);
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(x[c]) : "l"(A), "l"(B));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += lo(x[c]);
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(THREADS) k_ex2(float* out, float a, float b, long long* cyc) {
  float x[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) x[c] = -(threadIdx.x * 1e-4f + c * 0.01f);
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < NCH; ++c) s += x[c];
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the raster's mix: per step 2 FFMA2 + 3 FFMA + 1 EX2 (as in the K6 inner loop)
__global__ void __launch_bounds__(THREADS) k_mix(float* out, float a, float b, long long* cyc) {
  float x[4];
  uint64_t y[4];
  const uint64_t A = pk(a, a), B = pk(b, b);
#pragma unroll
  for (int c = 0; c < 4; ++c) { x[c] = -(threadIdx.x * 1e-4f + c); y[c] = pk(c * 0.1f, c * 0.2f); }
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[c]) : "l"(A), "l"(B));
      asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(y[c]) : "l"(A), "l"(B));
      x[c] = fmaf(x[c], a, b);
      x[c] = fmaf(x[c], a, b);
      x[c] = fmaf(x[c], a, b);
      asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += x[c] + lo(y[c]);
  if (s == 1234.5f) out[0] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

typedef void (*kfn)(float*, float, float, long long*);

static void run(const char* name, kfn k, double lane_ops_per_iter, int blocks, float* out, long long* cyc,
                bool last) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) k<<<blocks, THREADS>>>(out, 0.999f, 1e-6f, cyc);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) k<<<blocks, THREADS>>>(out, 0.999f, 1e-6f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[4096];
  cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double cmax = 0;
  for (int i = 0; i < blocks; ++i) cmax = h[i] > cmax ? h[i] : cmax;
  const double ops = (double)blocks * THREADS * ITERS * lane_ops_per_iter * reps;
  const double rate = ops / (ms * 1e-3);                       // lane-ops/s
  const double sec_per_launch = ms * 1e-3 / reps;
  const double mhz = cmax / sec_per_launch / 1e6;              // effective SM clock (upper bound on the CTA's window)
  const double per_sm_clk = rate / 148.0 / (mhz * 1e6);
  printf("\"%s\": {\"lane_ops_per_s\": %.4e, \"ms_per_launch\": %.4f, \"sm_mhz_est\": %.1f, "
         "\"lane_ops_per_sm_per_clk\": %.2f}%s",
         name, rate, ms / reps, mhz, per_sm_clk, last ? "" : ", ");
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 16);
  const int blocks = 148 * 8;
  cudaMalloc(&cyc, sizeof(long long) * blocks);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"threads\": %d, \"blocks\": %d, \"chains\": %d, ", p.name,
         p.multiProcessorCount, THREADS, blocks, NCH);
  // lane-ops per iteration per thread: FFMA = 1 lane-op (2 flops); FFMA2 = 2 lane-ops (4 flops)
  run("ffma", k_ffma, NCH, blocks, out, cyc, false);
  run("ffma2", k_ffma2, 2.0 * NCH, blocks, out, cyc, false);
  run("ex2", k_ex2, NCH, blocks, out, cyc, false);
  // mix: 4 chains x (2 FFMA2 = 4 lane-ops, 3 FFMA = 3 lane-ops, 1 EX2) -> count FP32 lane-ops only
  run("mix_fp32_lane_ops", k_mix, 4 * 7.0, blocks, out, cyc, true);
  printf("}\n");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    fprintf(stderr, "CUDA error: %s\n", cudaGetErrorString(e));
    return 1;
  }
  return 0;
}
