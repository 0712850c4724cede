// dev tool: minimal 2-D tensor-map TMA load (cp.async.bulk.tensor) of a 16 x 64
// float tile into shared memory, compared element by element.
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

template <int V>
__global__ void k(const __grid_constant__ CUtensorMap tmap, const CUtensorMap* gmap, float* out, int x, int y) {
    __shared__ __align__(128) float buf[16 * 64];
    __shared__ __align__(8) unsigned long long bar;
    const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
    const unsigned sd = (unsigned)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(16 * 64 * 4) : "memory");
        const unsigned long long desc = V == 1 ? (unsigned long long)gmap : (unsigned long long)&tmap;
        if (V == 1) asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;" ::"l"(desc) : "memory");
        if (V == 2)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(sd), "l"(desc), "r"(x), "r"(y), "r"(sb) : "memory");
        else
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                ::"r"(sd), "l"(desc), "r"(x), "r"(y), "r"(sb) : "memory");
    }
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(sb) : "memory");
    for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
    const int VSEL = argc > 1 ? atoi(argv[1]) : 0;
    const int W = 300, H = 200;
    float* h = new float[W * H];
    for (int i = 0; i < W * H; ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, W * H * 4);
    cudaMalloc(&o, 16 * 64 * 4);
    cudaMemcpy(d, h, W * H * 4, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    CUtensorMap m;
    memset(&m, 0, sizeof m);
    cuuint64_t dims[2] = {W, H};
    cuuint64_t str[1] = {W * 4};
    cuuint32_t box[2] = {64, 16}, es[2] = {1, 1};
    CUresult rc = ((PFN_cuTensorMapEncodeTiled_v12000)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es,
                                                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                          CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* gm = nullptr;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
    for (int V = VSEL; V <= VSEL; ++V)
    for (int t = 0; t < 3; ++t) {
        const int x = t == 2 ? W - 20 : 7 + 40 * t, y = t == 2 ? H - 5 : 3 + 30 * t;  // t = 2: partly outside (zero fill)
        if (V == 0) k<0><<<1, 128>>>(m, gm, o, x, y);
        if (V == 1) k<1><<<1, 128>>>(m, gm, o, x, y);
        if (V == 2) k<2><<<1, 128>>>(m, gm, o, x, y);
        cudaError_t e = cudaDeviceSynchronize();
        float r[16 * 64];
        cudaMemcpy(r, o, sizeof r, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int yy = 0; yy < 16; ++yy)
            for (int xx = 0; xx < 64; ++xx) {
                const int gx = x + xx, gy = y + yy;
                const float want = (gx < W && gy < H) ? (float)(gy * W + gx) : 0.f;
                bad += r[yy * 64 + xx] != want;
            }
        printf("V=%d encode=%d query=%d launch=%s tile(%d,%d) mismatches=%d\n", V, (int)rc, (int)q, cudaGetErrorString(e), x, y, bad);
    }
    return 0;
}
