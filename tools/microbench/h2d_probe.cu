// dev tool: PCIe transfer paths for the host-buffer API. Copy engine
// (cudaMemcpyAsync, pinned) vs SM-driven zero-copy kernels that read / write
// mapped pinned host memory directly, alone and with both directions at once.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/h2d_probe tools/microbench/h2d_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void pull(const float4* __restrict__ h, float4* __restrict__ d, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        d[i] = h[i];
}
__global__ void push(const float4* __restrict__ d, float4* __restrict__ h, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        h[i] = d[i];
}

int main() {
    const size_t bytes = 16u << 20, n4 = bytes / 16;
    float *h_in, *h_out, *d_in, *d_out;
    cudaHostAlloc(&h_in, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h_out, bytes, cudaHostAllocMapped);
    cudaMalloc(&d_in, bytes);
    cudaMalloc(&d_out, bytes);
    for (size_t i = 0; i < bytes / 4; ++i) h_in[i] = (float)i;
    cudaStream_t s1, s2;
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto time = [&](auto f) {
        for (int i = 0; i < 3; ++i) f();
        cudaDeviceSynchronize();
        cudaEventRecord(a, 0);
        const int reps = 20;
        for (int i = 0; i < reps; ++i) f();
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        return ms / reps;
    };
    auto gbs = [&](float ms, double mult = 1.0) { return mult * bytes / (ms * 1e-3) / 1e9; };
    float t = time([&] { cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, 0); });
    printf("copy engine H2D        %6.1f GB/s\n", gbs(t));
    t = time([&] { cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, 0); });
    printf("copy engine D2H        %6.1f GB/s\n", gbs(t));
    for (int blocks : {sms, 2 * sms, 4 * sms, 8 * sms}) {
        t = time([&] { pull<<<blocks, 512>>>((const float4*)h_in, (float4*)d_in, n4); });
        printf("kernel pull H2D %4d CTAs %6.1f GB/s\n", blocks, gbs(t));
    }
    for (int blocks : {sms, 4 * sms}) {
        t = time([&] { push<<<blocks, 512>>>((const float4*)d_out, (float4*)h_out, n4); });
        printf("kernel push D2H %4d CTAs %6.1f GB/s\n", blocks, gbs(t));
    }
    // both directions at once: copy engines vs kernel pull + copy-engine D2H
    cudaEvent_t e1;
    cudaEventCreateWithFlags(&e1, cudaEventDisableTiming);
    auto both_ce = [&] {
        cudaEventRecord(e1, 0);
        cudaStreamWaitEvent(s1, e1, 0);
        cudaStreamWaitEvent(s2, e1, 0);
        cudaMemcpyAsync(d_in, h_in, bytes, cudaMemcpyHostToDevice, s1);
        cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(e1, s1);
        cudaStreamWaitEvent(0, e1, 0);
        cudaEventRecord(e1, s2);
        cudaStreamWaitEvent(0, e1, 0);
    };
    t = time(both_ce);
    printf("both, copy engines      %6.1f GB/s total (%.3f ms)\n", gbs(t, 2.0), t);
    auto both_k = [&] {
        cudaEventRecord(e1, 0);
        cudaStreamWaitEvent(s1, e1, 0);
        cudaStreamWaitEvent(s2, e1, 0);
        pull<<<2 * sms, 512, 0, s1>>>((const float4*)h_in, (float4*)d_in, n4);
        cudaMemcpyAsync(h_out, d_out, bytes, cudaMemcpyDeviceToHost, s2);
        cudaEventRecord(e1, s1);
        cudaStreamWaitEvent(0, e1, 0);
        cudaEventRecord(e1, s2);
        cudaStreamWaitEvent(0, e1, 0);
    };
    t = time(both_k);
    printf("both, pull + CE D2H     %6.1f GB/s total (%.3f ms)\n", gbs(t, 2.0), t);
    auto both_kk = [&] {
        cudaEventRecord(e1, 0);
        cudaStreamWaitEvent(s1, e1, 0);
        cudaStreamWaitEvent(s2, e1, 0);
        pull<<<sms, 512, 0, s1>>>((const float4*)h_in, (float4*)d_in, n4);
        push<<<sms, 512, 0, s2>>>((const float4*)d_out, (float4*)h_out, n4);
        cudaEventRecord(e1, s1);
        cudaStreamWaitEvent(0, e1, 0);
        cudaEventRecord(e1, s2);
        cudaStreamWaitEvent(0, e1, 0);
    };
    t = time(both_kk);
    printf("both, pull + push       %6.1f GB/s total (%.3f ms)\n", gbs(t, 2.0), t);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
