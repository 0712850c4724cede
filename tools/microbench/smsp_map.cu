// Which warps of a CTA share an SM sub-partition? Warp `a` and warp `b` both run an
// FFMA2 loop that alone fills its sub-partition's FMA pipe; if they share a
// sub-partition each takes ~2x as long. Prints, per base warp, the partners that slow it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o smsp_map smsp_map.cu && ./smsp_map [threads]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void probe(unsigned mask, int iters, long long* cyc, float* sink) {
  const int w = threadIdx.x / 32;
  if (!((mask >> w) & 1)) return;
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, i);
  const float2 m = make_float2(1.0001f, 0.9999f);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], m, m);
  }
  const long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 12345.f) sink[0] = s;
  if ((threadIdx.x & 31) == 0 && blockIdx.x == 0) cyc[w] = t1 - t0;
}
int main(int argc, char** argv) {
  const int threads = argc > 1 ? atoi(argv[1]) : 512, W = threads / 32;
  long long* cyc; float* sink;
  cudaMallocManaged(&cyc, 32 * sizeof(long long)); cudaMalloc(&sink, 4);
  const int iters = 20000;
  auto run = [&](unsigned mask, int w) { probe<<<148, threads>>>(mask, iters, cyc, sink); cudaDeviceSynchronize(); return (double)cyc[w] / (iters * 64.0); };
  run(1, 0);
  for (int a = 0; a < W; ++a) {
    const double alone = run(1u << a, a);
    printf("warp %2d alone %.2f cyc/FFMA2; shares with:", a, alone);
    for (int b = 0; b < W; ++b) {
      if (b == a) continue;
      const double t = run((1u << a) | (1u << b), a);
      if (t > 1.5 * alone) printf(" %d", b);
    }
    printf("\n");
  }
  return 0;
}
