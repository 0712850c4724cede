// dev tool: 2-D tensor-map TMA (cp.async.bulk.tensor.2d) of a Q x W float tile into
// shared memory on sm_100a, tensor map encoded with the driver API (-lcuda) and
// passed as a __grid_constant__ kernel parameter. Prints mismatches per tile.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

constexpr int BW = 64, BH = 16;

__global__ void load_tile(const __grid_constant__ CUtensorMap tmap, float* out, int x, int y) {
    __shared__ __align__(1024) float buf[BH * BW];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned sd = (unsigned)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(BH * BW * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(sd),
            "l"(reinterpret_cast<unsigned long long>(&tmap)), "r"(x), "r"(y), "r"(sb)
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WAIT_%=;\n}" ::"r"(sb)
        : "memory");
    for (int i = threadIdx.x; i < BH * BW; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                            const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                            CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    // argv[1]: 0 = cuTensorMapEncodeTiled linked from libcuda, 1 = cudaGetDriverEntryPoint,
    // 2 = cudaGetDriverEntryPointByVersion(12000), 3 = (13000)
    const int how = argc > 1 ? argv[1][0] - '0' : 0;
    const int W = 300, H = 200;
    float* h = new float[W * H];
    for (int i = 0; i < W * H; ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, W * H * 4);
    cudaMalloc(&o, BH * BW * 4);
    cudaMemcpy(d, h, W * H * 4, cudaMemcpyHostToDevice);
    int drv = 0;
    cudaDriverGetVersion(&drv);
    CUtensorMap m;
    std::memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H};
    cuuint64_t strides[1] = {(cuuint64_t)W * 4};
    cuuint32_t box[2] = {BW, BH}, es[2] = {1, 1};
    EncodeFn enc = cuTensorMapEncodeTiled;
    if (how > 0) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        cudaError_t ge = how == 1 ? cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q)
                                  : cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn,
                                                                     how == 2 ? 12000 : 13000, cudaEnableDefault, &q);
        printf("entry point (%d): %s q=%d fn=%p linked=%p\n", how, cudaGetErrorString(ge), (int)q, fn,
               (void*)&cuTensorMapEncodeTiled);
        enc = (EncodeFn)fn;
    }
    CUresult rc = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("driver %d encode rc=%d\n", drv, (int)rc);
    int fails = 0;
    for (int t = 0; t < 3; ++t) {
        const int x = t == 2 ? W - 20 : 8 + 40 * t, y = t == 2 ? H - 5 : 3 + 30 * t;
        load_tile<<<1, 128>>>(m, o, x, y);
        cudaError_t e = cudaDeviceSynchronize();
        float r[BH * BW];
        cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int yy = 0; yy < BH; ++yy)
            for (int xx = 0; xx < BW; ++xx) {
                const int gx = x + xx, gy = y + yy;
                const float want = (gx < W && gy < H) ? (float)(gy * W + gx) : 0.f;
                bad += r[yy * BW + xx] != want;
            }
        printf("tile (%d,%d): %s mismatches=%d\n", x, y, cudaGetErrorString(e), bad);
        fails += bad != 0 || e != cudaSuccess;
    }
    return fails;
}
