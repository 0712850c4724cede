// dev tool: concurrent H2D + D2H copy-engine rate vs host buffer size and
// allocation flags (default / write-combined source), 16 MiB chunks streamed
// through large pinned buffers like the pipelined batch call does.
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t chunk = 16u << 20;
    cudaStream_t si, so;
    cudaStreamCreateWithFlags(&si, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&so, cudaStreamNonBlocking);
    float *d_in, *d_out;
    cudaMalloc(&d_in, chunk);
    cudaMalloc(&d_out, chunk);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int wc = 0; wc < 2; ++wc)
        for (size_t nchunks : {1, 4, 20}) {
            char *h_in, *h_out;
            cudaHostAlloc(&h_in, chunk * nchunks, cudaHostAllocPortable | (wc ? cudaHostAllocWriteCombined : 0));
            cudaHostAlloc(&h_out, chunk * nchunks, cudaHostAllocPortable);
            for (size_t i = 0; i < chunk * nchunks; i += 4096) h_in[i] = 1, h_out[i] = 1;
            float best = 1e9;
            for (int rep = 0; rep < 4; ++rep) {
                cudaDeviceSynchronize();
                cudaEventRecord(a, 0);
                cudaStreamWaitEvent(si, a, 0);
                cudaStreamWaitEvent(so, a, 0);
                for (int r = 0; r < 20; ++r) {
                    const size_t off = (r % nchunks) * chunk;
                    cudaMemcpyAsync(d_in, h_in + off, chunk, cudaMemcpyHostToDevice, si);
                    cudaMemcpyAsync(h_out + off, d_out, chunk, cudaMemcpyDeviceToHost, so);
                }
                cudaEventRecord(b, si);
                cudaStreamWaitEvent(so, b, 0);
                cudaEventRecord(b, so);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("%s source, %2zu x 16 MiB host buffers: %.3f ms per 16 MiB each way (%.1f GB/s total)\n",
                   wc ? "write-combined" : "default       ", nchunks, best / 20, 2.0 * 20 * chunk / (best * 1e-3) / 1e9);
            cudaFreeHost(h_in);
            cudaFreeHost(h_out);
        }
    return 0;
}
