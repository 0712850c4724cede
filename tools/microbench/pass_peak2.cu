// dev tool: row-pass FFMA2 efficiency vs outputs per thread (PO) and warps, R=15.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 15;
struct Taps { float t[R + 1]; };
__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) { return __ffma2_rn(a, make_float2(w, w), c); }

template <int PO>
__global__ void __launch_bounds__(1024, 1) k(const Taps tp, float* out, int iters) {
  extern __shared__ __align__(16) float2 sm[];
  constexpr int ROWW = 290;  // float2 per row, ROWW/2 odd: conflict-free LDS.128 across q
  for (int i = threadIdx.x; i < 8 * ROWW * 4; i += blockDim.x) sm[i] = make_float2(i * 1e-3f, 1.f);
  __syncthreads();
  const int q = threadIdx.x % 8, xc = threadIdx.x / 8;
  float2 tot = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; ++it) {
    const float4* gin = reinterpret_cast<const float4*>(sm + (q + 8 * (it & 3)) * ROWW + (xc * PO) % 256);
    float2 acc[PO];
#pragma unroll
    for (int o = 0; o < PO; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
    for (int j = 0; j < (PO + 2 * R) / 2; ++j) {
      const float4 v4 = gin[j];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = 2 * j + h;
        const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
        for (int o = 0; o < PO; ++o) {
          const int d = jj - o;
          if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, tp.t[d >= R ? d - R : R - d], acc[o]);
        }
      }
    }
#pragma unroll
    for (int o = 0; o < PO; ++o) { tot.x += acc[o].x; tot.y += acc[o].y; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = tot.x + tot.y;
}

int main() {
  Taps tp; for (int j = 0; j <= R; j++) tp.t[j] = 1.f / (1 + j);
  float* out; cudaMalloc(&out, 148 * 1024 * 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int threads, int po, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100000);
    const int iters = 4000;
    kern<<<148, threads, 80000>>>(tp, out, 10);
    cudaEventRecord(a); kern<<<148, threads, 80000>>>(tp, out, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 148.0 * threads * iters * (double)po * (2 * R + 1) * 4;
    printf("%s threads %4d: %.1f%% of 74.45 %s\n", name, threads, flops / ms / 1e9 / 74.45 * 100, cudaGetErrorString(cudaGetLastError()));
  };
  for (int t : {128, 224, 448, 896}) { run(k<8>, t, 8, "PO=8 "); run(k<16>, t, 16, "PO=16"); run(k<4>, t, 4, "PO=4 "); }
}
