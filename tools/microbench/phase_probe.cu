// dev tool: per-phase cycle breakdown of the fused kernel (c1-like: R=15, K=4)
#define FBF_PHASES 1
#ifndef FBF_Q
#define FBF_Q 8
#endif
#include <cstdio>
#include <cmath>
#include <vector>
#include <algorithm>
#include <cstdlib>
#include "../../paper_1811_02168_b200/csrc/fbf_kernel.cuh"
using namespace fbf_dev;
template cudaError_t fbf_dev::launch_fused<15, 3>(const Params&, int, cudaStream_t);
int main(int argc, char** argv) {
  const int W = 2048, H = 2048, R = 15;
  int grid = argc > 1 ? atoi(argv[1]) : 148;
  std::vector<float> h((size_t)W * H);
  for (size_t i = 0; i < h.size(); i++) h[i] = (float)((i * 2654435761u) % 256);
  float *d, *o; cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, h.size() * 4);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  Params p{}; p.src = d; p.src_pitch = W; p.src_rows = H; p.dst = o; p.dst_pitch = W; p.width = W; p.height = H;
  p.n_frames = 1; p.out_rows = H; p.k_lo = 0; p.n_pairs = 7; p.k_first = 1; p.first_chunk = 1; p.last_chunk = 1;
  p.n_strips = W / 32; p.use_tma = argc > 2 ? atoi(argv[2]) : 1; p.total_units = (long long)p.n_strips * H;
  for (int j = 0; j <= R; j++) p.taps[j] = expf(-j * j / 50.f);
  float c[4] = {0.2f, 0.3f, 0.2f, 0.1f}; for (int k = 0; k < 4; k++) p.coeff[k] = c[k];
  p.inv_period = 1.f / 407.f;
  launch_fused<15, 3>(p, grid, 0); cudaDeviceSynchronize();
  unsigned long long z[16] = {0}; cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  std::vector<float> tms;
  for (int rep = 0; rep < 21; rep++) {
    if (rep == 20) cudaMemcpyToSymbol(g_phase_cycles, z, sizeof z);
    cudaEventRecord(a); launch_fused<15, 3>(p, grid, 0); cudaEventRecord(b); cudaEventSynchronize(b);
    float t; cudaEventElapsedTime(&t, a, b); tms.push_back(t);
  }
  std::sort(tms.begin(), tms.end()); float ms = tms[10];
  unsigned long long r[16]; cudaMemcpyFromSymbol(r, g_phase_cycles, sizeof r);
  int occ=0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fbf_fused_kernel<15,3>, kRoles*7*kItemsPerPair+kExtraThreads, Geometry<15>::smem_bytes(7)); printf("occupancy %d blocks/SM\n", occ);
  printf("grid %d: %.3f ms (%s)\n", grid, ms, cudaGetErrorString(cudaGetLastError()));
  const char* names[16] = {"G:loop", "G:waits", "P:loop", "P:gen wait", "G:gen", "G:arrive",
                           "P:row", "P:colbuf wait", "-", "-", "P:col", "P:arrive", "C:wait", "C:combine", "", ""};
  double tp = 0, tc = 0; for (int i = 0; i < 8; i++) tp += r[i]; for (int i = 8; i < 14; i++) tc += r[i];
  printf("max CTA cycles %llu (%.3f ms at 1965 MHz); mean SM clock in kernel %.0f MHz; mean per-step (115) %.0f\n", r[14], r[14] / 1.965e6, (double)r[15] / grid, (double)r[14] / 115);
  { unsigned long long cc[1024]; cudaMemcpyFromSymbol(cc, g_cta_cycles, sizeof cc);
    printf("per-CTA kcycles:"); for (int i = 0; i < grid && i < 1024; i++) printf(" %llu", cc[i] / 1000); printf("\n"); }
  for (int i = 0; i < 14; i++) printf("  %-20s %6.1f%%  %.0f cyc/step\n", names[i], 100.0 * r[i] / (i < 8 ? tp : tc), r[i] / (grid * 115.0));
}
