// Minimal TMA check (dev tool): loads one (FSW x 8) box through the fbf_kernel.cuh helpers.
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cudaTypedefs.h>
#include "../../paper_1811_02168_b200/csrc/fbf_kernel.cuh"
using namespace fbf_dev;

template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tmap, float* out, int x, int y, int boxw) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* buf = (float*)sm;
  uint64_t* bar = (uint64_t*)(sm + 8 * 1024);
  if (threadIdx.x == 0) { mbar_init(bar, 1); if (V & 1) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (V & 2) fence_proxy_async();
    mbar_arrive_expect_tx(bar, boxw * 8 * 4);
    if (V & 4)
      asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
        :: "r"(smem_u32(buf)), "l"(&tmap), "r"(x), "r"(y), "r"(0), "r"(smem_u32(bar)) : "memory");
    else
      tma_load_3d(buf, &tmap, x, y, 0, bar);
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < boxw * 8; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int W = 200, H = 150, boxw = 44;
  float* h = new float[W * H];
  for (int i = 0; i < W * H; i++) h[i] = i;
  float *d, *o;
  cudaMalloc(&d, W * H * 4); cudaMalloc(&o, boxw * 8 * 4);
  cudaMemcpy(d, h, W * H * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t dims[3] = {W, H, 1}; cuuint64_t str[2] = {W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {boxw, 8, 1}, es[3] = {1, 1, 1};
  CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc=%d sizeof(CUtensorMap)=%zu\n", (int)rc, sizeof(CUtensorMap));
  cudaError_t e;
  #define RUN(V) k<V><<<1, 128, 16 * 1024>>>(m, o, 10, 20, boxw); e = cudaDeviceSynchronize(); printf("variant %d: %s\n", V, cudaGetErrorString(e)); if (e) return 1;
  int v = argc > 1 ? atoi(argv[1]) : 0;
  switch (v) { case 0: RUN(0) break; case 1: RUN(1) break; case 2: RUN(2) break; case 3: RUN(3) break; case 4: RUN(4) break; case 5: RUN(5) break; case 6: RUN(6) break; case 7: RUN(7) break; }
  float r[boxw * 8]; cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
  int bad = 0; for (int yy = 0; yy < 8; yy++) for (int xx = 0; xx < boxw; xx++) bad += r[yy * boxw + xx] != (float)((20 + yy) * W + 10 + xx);
  printf("mismatches %d\n", bad);
}
