// dev tool: FFMA2 efficiency of the row and column passes alone (R=15, c1 shape),
// on static shared-memory data, no synchronisation: the ceiling of the hot loops.
#define FBF_Q 8
#include <cstdio>
#include <cstdlib>
#include "../../paper_1811_02168_b200/csrc/fbf_kernel.cuh"
using namespace fbf_dev;
constexpr int R = 15;
using G = Geometry<R>;

template <int MODE>  // 0 row only, 1 col only, 2 both (half warps each)
__global__ void __launch_bounds__(1024, 1) k(const Params p, float* out, int iters, int np) {
  extern __shared__ __align__(128) unsigned char sm[];
  float2* gen = reinterpret_cast<float2*>(sm);
  float2* ring = gen + (size_t)np * kQ * G::GS;
  for (int i = threadIdx.x; i < np * kQ * G::GS + np * G::RROWS * G::RS; i += blockDim.x) gen[i] = make_float2(i * 1e-3f, 1.f);
  __syncthreads();
  const int nrole = np * 32;
  const int role = MODE == 2 ? (threadIdx.x >= nrole) : MODE;
  const int tid = threadIdx.x % nrole;
  float sink = 0.f;
  for (int it = 0; it < iters; ++it) {
    const int blk = it % G::RBX;
    if (role == 0) {
      const int q = tid % kQ, xc = (tid / kQ) % (kTW / kP), pr = tid / (kQ * (kTW / kP));
      const float4* gin = reinterpret_cast<const float4*>(gen + ((size_t)pr * kQ + q) * G::GS + xc * kP);
      float2 accp[kP];
#pragma unroll
      for (int o = 0; o < kP; ++o) accp[o] = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < (kP + 2 * R) / 2; ++j) {
        const float4 v4 = gin[j];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int jj = 2 * j + h;
          const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
          for (int o = 0; o < kP; ++o) {
            const int d = jj - o;
            if (d >= 0 && d <= 2 * R) accp[o] = ffma2(v, p.taps[d >= R ? d - R : R - d], accp[o]);
          }
        }
      }
      float4* hout = reinterpret_cast<float4*>(ring + ((size_t)pr * G::RROWS + ((it + 3) % G::RBX) * kQ + q) * G::RS + xc * kP);
#pragma unroll
      for (int o = 0; o < kP / 2; ++o) hout[o] = make_float4(accp[2 * o].x, accp[2 * o].y, accp[2 * o + 1].x, accp[2 * o + 1].y);
    } else {
      const int x = tid % kTW, pr = tid / kTW;
      float* oc = reinterpret_cast<float*>(gen) + (((size_t)pr % 4) * kQ * kTW + x) * 4;
      column_pass<R, 0>(ring + (size_t)pr * G::RROWS * G::RS, blk, x, p.taps, oc, pr & 1, 2 + (pr & 1));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = gen[5].x + sink;
}

int main(int argc, char** argv) {
  const int np = 7, iters = 2000;
  Params p{};
  for (int j = 0; j <= R; j++) p.taps[j] = 1.f / (1 + j);
  float* out; cudaMalloc(&out, 4096 * 4);
  size_t smem = sizeof(float2) * (np * kQ * G::GS + np * G::RROWS * G::RS);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int threads, const char* name, double ffma2_per_thread_iter) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    kern<<<148, threads, smem>>>(p, out, 10, np);
    cudaEventRecord(a); kern<<<148, threads, smem>>>(p, out, iters, np); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 148.0 * threads * iters * ffma2_per_thread_iter * 4;
    printf("%-10s threads %4d: %.3f ms  %.1f TFLOP/s  (%.1f%% of 74.45)  %s\n", name, threads, ms, flops / ms / 1e9, flops / ms / 1e9 / 74.45 * 100, cudaGetErrorString(cudaGetLastError()));
  };
  for (int mult = 1; mult <= 4; mult *= 2) {
    const int n = np * mult;
    smem = sizeof(float2) * (n * kQ * G::GS + n * G::RROWS * G::RS);
    if (smem > 220000) break;
    printf("np=%d\n", n);
    auto run2 = [&](auto kern, int threads, const char* name) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220000);
      kern<<<148, threads, smem>>>(p, out, 10, n);
      cudaEventRecord(a); kern<<<148, threads, smem>>>(p, out, iters, n); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double flops = 148.0 * threads * iters * 248.0 * 4;
      printf("  %-8s threads %4d: %.1f%% of 74.45 %s\n", name, threads, flops / ms / 1e9 / 74.45 * 100, cudaGetErrorString(cudaGetLastError()));
    };
    run2(k<0>, n * 32, "row");
    run2(k<1>, n * 32, "col");
    if (2 * n * 32 <= 1024) run2(k<2>, 2 * n * 32, "row+col");
  }
  return 0;
}
