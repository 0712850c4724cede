// FP32 FMA-pipe microbenchmark for sm_100a: scalar FFMA (uniform-register tap
// operand), FFMA2 with a broadcast uniform-register tap, FFMA2 with a register
// pair, and FFMA2 interleaved with LDS.128 at fixed ratios. Reports achieved
// TFLOP/s and the SM clock measured inside the kernel (clock64 vs globaltimer).
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float c_taps[64];

#define NACC 16
#define ITERS 2048

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t;
}

__global__ void k_ffma_ur(float* out, float seed, unsigned long long* clk) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = seed * (threadIdx.x + i);
  float x = seed + threadIdx.x;
  unsigned long long c0 = clock64(), t0 = gtime();
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 8; d++)
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = fmaf(x, c_taps[d], acc[i]);
  }
  unsigned long long c1 = clock64(), t1 = gtime();
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) { clk[0] = c1 - c0; clk[1] = t1 - t0; }
}

__global__ void k_ffma_rrr(float* out, float seed, unsigned long long* clk) {
  float acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = seed * (threadIdx.x + i);
  float x = seed + threadIdx.x, y = seed - threadIdx.x;
  float w[8];
#pragma unroll
  for (int d = 0; d < 8; d++) w[d] = y * d;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 8; d++)
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = fmaf(x, w[d], acc[i]);
    x += 1e-7f;
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2_ur(float* out, float seed, unsigned long long* clk) {
  float2 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = make_float2(seed * (threadIdx.x + i), seed * i);
  float2 x = make_float2(seed + threadIdx.x, seed - threadIdx.x);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 8; d++) {
      float2 w = make_float2(c_taps[d], c_taps[d]);
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = __ffma2_rn(x, w, acc[i]);
    }
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2_rr(float* out, float seed, unsigned long long* clk) {
  float2 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = make_float2(seed * (threadIdx.x + i), seed * i);
  float2 x = make_float2(seed + threadIdx.x, seed - threadIdx.x);
  float2 w[8];
#pragma unroll
  for (int d = 0; d < 8; d++) w[d] = make_float2(seed * d, seed * d + 1);
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 8; d++)
#pragma unroll
      for (int i = 0; i < NACC; i++) acc[i] = __ffma2_rn(x, w[d], acc[i]);
    x.x += 1e-7f;
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FFMA2 (UR tap) with one LDS.128 per RATIO FFMA2s; data varies per load
template <int RATIO>
__global__ void k_ffma2_lds(float* out, float seed, unsigned long long* clk) {
  __shared__ float4 sm[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = make_float4(seed * i, seed, seed + i, seed - i);
  __syncthreads();
  float2 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; i++) acc[i] = make_float2(seed * (threadIdx.x + i), seed * i);
  int base = threadIdx.x;
  for (int it = 0; it < ITERS; it++) {
#pragma unroll
    for (int d = 0; d < 128 / RATIO; d++) {
      float4 v = sm[(base + d * 32) & 2047];
      float2 a = make_float2(v.x, v.y), b = make_float2(v.z, v.w);
#pragma unroll
      for (int i = 0; i < RATIO; i++) {
        float2 w = make_float2(c_taps[(d * RATIO + i) & 63], c_taps[(d * RATIO + i) & 63]);
        acc[i % NACC] = __ffma2_rn((i & 1) ? a : b, w, acc[i % NACC]);
      }
    }
    base += 7;
  }
  float s = 0; for (int i = 0; i < NACC; i++) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

typedef void (*kfn)(float*, float, unsigned long long*);

static void run(const char* name, kfn k, double fma_per_thread, int blocks, int threads, float* d_out, unsigned long long* d_clk) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int w = 0; w < 3; w++) k<<<blocks, threads>>>(d_out, 1e-3f, d_clk);
  cudaEventRecord(a);
  const int reps = 5;
  for (int w = 0; w < reps; w++) k<<<blocks, threads>>>(d_out, 1e-3f, d_clk);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double flops = 2.0 * fma_per_thread * blocks * threads * reps;
  unsigned long long h[2] = {0, 0};
  cudaMemcpy(h, d_clk, sizeof h, cudaMemcpyDeviceToHost);
  printf("{\"kernel\": \"%s\", \"blocks\": %d, \"threads\": %d, \"ms\": %.4f, \"tflops\": %.3f, \"sm_mhz_in_kernel\": %.0f}\n",
         name, blocks, threads, ms / reps, flops / (ms * 1e-3) / 1e12, h[1] ? 1e3 * (double)h[0] / (double)h[1] : 0.0);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("{\"sms\": %d, \"clock_rate_khz\": %d, \"peak_tflops_at_clock\": %.2f}\n", sms, clk, sms * 128.0 * 2 * clk * 1e3 / 1e12);
  float taps[64]; for (int i = 0; i < 64; i++) taps[i] = 1.0f / (1 + i);
  cudaMemcpyToSymbol(c_taps, taps, sizeof taps);
  float* d_out; unsigned long long* d_clk;
  cudaMalloc(&d_out, sizeof(float) * sms * 8 * 1024); cudaMalloc(&d_clk, 16);
  cudaMemset(d_clk, 0, 16);
  const double per = (double)ITERS * 8 * NACC;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (2048 / tpb) * 2;
    run("ffma_ur", k_ffma_ur, per, blocks, tpb, d_out, d_clk);
    run("ffma_rrr", k_ffma_rrr, per, blocks, tpb, d_out, d_clk);
    run("ffma2_ur", k_ffma2_ur, 2 * per, blocks, tpb, d_out, d_clk);
    run("ffma2_rr", k_ffma2_rr, 2 * per, blocks, tpb, d_out, d_clk);
  }
  for (int tpb : {256, 512}) {
    int blocks = sms * (2048 / tpb);
    run("ffma2_lds_r4", k_ffma2_lds<4>, 2.0 * ITERS * 128, blocks, tpb, d_out, d_clk);
    run("ffma2_lds_r8", k_ffma2_lds<8>, 2.0 * ITERS * 128, blocks, tpb, d_out, d_clk);
    run("ffma2_lds_r16", k_ffma2_lds<16>, 2.0 * ITERS * 128, blocks, tpb, d_out, d_clk);
    run("ffma2_lds_r32", k_ffma2_lds<32>, 2.0 * ITERS * 128, blocks, tpb, d_out, d_clk);
  }
  return 0;
}
