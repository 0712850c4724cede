// TMA variants (dev tool)
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cudaTypedefs.h>
#include "../../paper_1811_02168_b200/csrc/fbf_kernel.cuh"
using namespace fbf_dev;

__device__ __forceinline__ void tma2d(float* dst, const void* map, int x, int y, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
    :: "r"(smem_u32(dst)), "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}

// V: 0 = 3d param map, 1 = 3d global map, 2 = 2d param map, 3 = 1d bulk copy
template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tmap, const CUtensorMap* gmap, const float* src, float* out, int x, int y, int bytes) {
  extern __shared__ __align__(1024) unsigned char sm[];
  float* buf = (float*)sm;
  uint64_t* bar = (uint64_t*)(sm + 8 * 1024);
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, bytes);
    if (V == 0) tma_load_3d(buf, &tmap, x, y, 0, bar);
    if (V == 1) tma_load_3d(buf, gmap, x, y, 0, bar);
    if (V == 2) tma2d(buf, &tmap, x, y, bar);
    if (V == 4) asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n"
                             :: "r"(smem_u32(buf)), "l"(&tmap), "r"(x), "r"(y), "r"(0), "r"(smem_u32(bar)) : "memory");
    if (V == 5) asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6;\n"
                             :: "r"(smem_u32(buf)), "l"(&tmap), "r"(x), "r"(y), "r"(0), "r"(smem_u32(bar)), "l"(0x12F0000000000000ull) : "memory");
    if (V == 3) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                             :: "r"(smem_u32(buf)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
  }
  mbar_wait(bar, 0);
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  const int W = 200, H = 150;
  int boxw = argc > 2 ? atoi(argv[2]) : 44;
  int V = argc > 1 ? atoi(argv[1]) : 0;
  float* h = new float[W * H];
  for (int i = 0; i < W * H; i++) h[i] = i;
  float *d, *o; CUtensorMap* gm;
  cudaMalloc(&d, W * H * 4); cudaMalloc(&o, 64 * 1024); cudaMalloc(&gm, sizeof(CUtensorMap));
  cudaMemcpy(d, h, W * H * 4, cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  if (argc > 3) cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  else cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  int dv = 0; cudaDriverGetVersion(&dv); int rv = 0; cudaRuntimeGetVersion(&rv); printf("driver %d runtime %d q=%d fn=%p\n", dv, rv, (int)q, fn);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap m; memset(&m, 0, sizeof m);
  cuuint64_t dims[3] = {W, H, 1}; cuuint64_t str[2] = {W * 4, (cuuint64_t)W * H * 4};
  cuuint32_t box[3] = {(cuuint32_t)boxw, 8, 1}, es[3] = {1, 1, 1};
  CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, V == 2 ? 2 : 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
  int bytes = V == 3 ? 1024 : boxw * 8 * 4;
  cudaError_t e;
  switch (V) {
    case 0: k<0><<<1, 128, 16 * 1024>>>(m, gm, d, o, 10, 20, bytes); break;
    case 1: k<1><<<1, 128, 16 * 1024>>>(m, gm, d, o, 10, 20, bytes); break;
    case 2: k<2><<<1, 128, 16 * 1024>>>(m, gm, d, o, 10, 20, bytes); break;
    case 4: k<4><<<1, 128, 16 * 1024>>>(m, gm, d, o, 10, 20, bytes); break;
    case 5: k<5><<<1, 128, 16 * 1024>>>(m, gm, d, o, 10, 20, bytes); break;
    case 3: k<3><<<1, 128, 16 * 1024>>>(m, gm, d, o, 10, 20, bytes); break;
  }
  e = cudaDeviceSynchronize();
  float r[16384]; cudaMemcpy(r, o, bytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  if (V == 3) { for (int i = 0; i < bytes / 4; i++) bad += r[i] != (float)i; }
  else for (int yy = 0; yy < 8; yy++) for (int xx = 0; xx < boxw; xx++) bad += r[yy * boxw + xx] != (float)((20 + yy) * W + 10 + xx);
  printf("V=%d boxw=%d encode=%d kernel=%s mismatches=%d\n", V, boxw, (int)rc, cudaGetErrorString(e), bad);
}
