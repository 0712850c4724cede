// Does bar.arrive block? Warp 0 (fast producer) arrives on barrier 1 and then waits on
// barrier 2; warp 1 (slow producer, `work` cycles) arrives on barrier 1 too; warp 2
// (consumer) syncs on barrier 1 and releases barrier 2. Prints the cycles warp 0 spends
// in bar.arrive and in the following bar.sync, per iteration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bar_arrive bar_arrive.cu && ./bar_arrive
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ long long clk() {  // ordered against the barrier instructions (memory clobber)
  long long t;
  asm volatile("mov.u64 %0, %%clock64;\n" : "=l"(t)::"memory");
  return t;
}
// clock read that cannot issue before `dep` (a value loaded after the barrier) is available:
// BAR.SYNC is DEFER_BLOCKING -- an independent CS2R right after it issues before the barrier completes
__device__ __forceinline__ long long clk_after(unsigned dep) {
  long long t;
  asm volatile("{\n.reg .u32 z;\nand.b32 z, %1, 0;\n.reg .u64 zz;\ncvt.u64.u32 zz, z;\nmov.u64 %0, %%clock64;\nadd.u64 %0, %0, zz;\n}\n" : "=l"(t) : "r"(dep) : "memory");
  return t;
}
__device__ __forceinline__ void spin(long long cycles) {
  const long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
__global__ void probe(int iters, long long work, long long* out) {
  const int w = threadIdx.x / 32;
  long long t_arr = 0, t_sync = 0, t_sync2 = 0;
  __shared__ unsigned flag;
  if (threadIdx.x == 0) flag = 0;
  __syncthreads();
  for (int i = 0; i < iters; ++i) {
    if (w == 0) {
      const long long a = clk();
      asm volatile("bar.arrive 1, 96;\n" ::: "memory");
      const long long b = clk();
      asm volatile("bar.sync 2, 96;\n" ::: "memory");
      const long long c = clk();
      const unsigned v = *(volatile unsigned*)&flag;  // shared-memory load ordered after the barrier
      const long long d = clk_after(v);
      t_arr += b - a;
      t_sync += c - b;
      t_sync2 += d - b;
    } else if (w == 1) {
      spin(work);
      asm volatile("bar.arrive 1, 96;\n" ::: "memory");
      asm volatile("bar.sync 2, 96;\n" ::: "memory");
    } else {
      asm volatile("bar.sync 1, 96;\n" ::: "memory");
      asm volatile("bar.sync 2, 96;\n" ::: "memory");
    }
  }
  if (threadIdx.x == 0) { out[0] = t_arr / iters; out[1] = t_sync / iters; out[2] = t_sync2 / iters; }
}
int main() {
  long long* out; cudaMallocManaged(&out, 32);
  for (long long work : {0LL, 1000LL, 5000LL}) {
    probe<<<1, 96>>>(200, work, out); cudaDeviceSynchronize();
    printf("slow producer %5lld cycles: fast producer spends %lld cycles in bar.arrive, %lld in the next bar.sync by a plain clock read, %lld by a clock read behind a shared load  (%s)\n", work,
           out[0], out[1], out[2], cudaGetErrorString(cudaGetLastError()));
  }
}
