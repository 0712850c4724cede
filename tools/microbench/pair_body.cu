#include <vector>
#include <cstdlib>
// dev tool: FFMA2 efficiency of the pair-warp body (row pass into a ring, column
// pass out of it) for step heights Q (= outputs per lane P), sequential or
// interleaved passes, and warps per SM. No inter-warp synchronisation: the
// ceiling of the body alone. R = 15 (config c1).
#include <cstdio>
#include <cuda_runtime.h>
constexpr int R = 15, TW = 32;
struct Taps { float t[R + 1]; };
__device__ __forceinline__ float2 ffma2(float2 a, float w, float2 c) { return __ffma2_rn(a, make_float2(w, w), c); }

template <int Q>
struct Geo {
  static constexpr int GW = TW + 2 * R;
  static constexpr int GS = GW + ((2 - GW % 4) + 4) % 4;
  static constexpr int RB = 1 + (2 * R + Q - 1) / Q;
  static constexpr int RS = TW + 2;
  static constexpr int floats2 = Q * GS + (RB + 1) * Q * RS + Q * TW;
};

// row pass of Q rows: lane = (q, chunk of P=32/(32/Q)... ) -> P = Q outputs
template <int Q>
__device__ __forceinline__ void row_pass(const float2* gen, float2* ring_blk, int lane, const Taps& tp) {
  using G = Geo<Q>;
  constexpr int P = Q * TW / 32;
  const int q = lane % Q, xc = lane / Q;
  const float4* gin = reinterpret_cast<const float4*>(gen + q * G::GS + xc * P);
  float2 acc[P];
#pragma unroll
  for (int o = 0; o < P; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < (P + 2 * R) / 2; ++j) {
    const float4 v4 = gin[j];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int jj = 2 * j + h;
      const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
      for (int o = 0; o < P; ++o) {
        const int d = jj - o;
        if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, tp.t[d >= R ? d - R : R - d], acc[o]);
      }
    }
  }
  float4* hout = reinterpret_cast<float4*>(ring_blk + q * G::RS + xc * P);
#pragma unroll
  for (int o = 0; o < P / 2; ++o) hout[o] = make_float4(acc[2 * o].x, acc[2 * o].y, acc[2 * o + 1].x, acc[2 * o + 1].y);
}

template <int Q, int NB>
__device__ __forceinline__ void col_pass(const float2* ring, int blk, int lane, const Taps& tp, float2* out) {
  using G = Geo<Q>;
  constexpr int RB = G::RB, RS = G::RS;
  const float2* bptr[RB];
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    int bb = blk - b;
    bb += bb < 0 ? NB : 0;
    bptr[b] = ring + bb * Q * RS + lane;
  }
  float2 acc[Q];
#pragma unroll
  for (int o = 0; o < Q; ++o) acc[o] = make_float2(0.f, 0.f);
#pragma unroll
  for (int i = 0; i < Q + 2 * R; ++i) {
    const int jr = i - 2 * R;
    const int b = jr >= 0 ? 0 : (-jr + Q - 1) / Q;
    const float2 v = bptr[b][(jr + b * Q) * RS];
#pragma unroll
    for (int o = 0; o < Q; ++o) {
      const int d = i - o;
      if (d >= 0 && d <= 2 * R) acc[o] = ffma2(v, tp.t[d >= R ? d - R : R - d], acc[o]);
    }
  }
#pragma unroll
  for (int o = 0; o < Q; ++o) out[o * TW + lane] = acc[o];
}

// interleaved Q=8 body (the v11 pair_iter)
__device__ __forceinline__ void inter8(const float2* gen, float2* ring, int blk_row, int blk_col, int lane, const Taps& tp,
                                       float2* out) {
  using G = Geo<8>;
  constexpr int RB = G::RB, NB = G::RB + 1, RS = G::RS, P = 8, Q = 8;
  const int q = lane % Q, xc = lane / Q;
  const float4* gin = reinterpret_cast<const float4*>(gen + q * G::GS + xc * P);
  float2 accr[P], accc[P];
  const float2* bptr[RB];
#pragma unroll
  for (int o = 0; o < P; ++o) { accr[o] = make_float2(0.f, 0.f); accc[o] = make_float2(0.f, 0.f); }
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    int bb = blk_col - b;
    bb += bb < 0 ? NB : 0;
    bptr[b] = ring + bb * Q * RS + lane;
  }
#pragma unroll
  for (int j = 0; j < (P + 2 * R) / 2; ++j) {
    const float4 v4 = gin[j];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int jj = 2 * j + h;
      const float2 v = h ? make_float2(v4.z, v4.w) : make_float2(v4.x, v4.y);
#pragma unroll
      for (int o = 0; o < P; ++o) {
        const int d = jj - o;
        if (d >= 0 && d <= 2 * R) accr[o] = ffma2(v, tp.t[d >= R ? d - R : R - d], accr[o]);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = 2 * j + h;
      const int jr = i - 2 * R;
      const int b = jr >= 0 ? 0 : (-jr + Q - 1) / Q;
      const float2 v = bptr[b][(jr + b * Q) * RS];
#pragma unroll
      for (int o = 0; o < P; ++o) {
        const int d = i - o;
        if (d >= 0 && d <= 2 * R) accc[o] = ffma2(v, tp.t[d >= R ? d - R : R - d], accc[o]);
      }
    }
  }
  float4* hout = reinterpret_cast<float4*>(ring + (blk_row * Q + q) * RS + xc * P);
#pragma unroll
  for (int o = 0; o < P / 2; ++o) hout[o] = make_float4(accr[2 * o].x, accr[2 * o].y, accr[2 * o + 1].x, accr[2 * o + 1].y);
#pragma unroll
  for (int o = 0; o < P; ++o) out[o * TW + lane] = accc[o];
}

// scatter column pass over Q new rows (state st[2R] in registers)
template <int Q>
__device__ __forceinline__ void col_scatter(const float2* hin, float2 (&st)[2 * R], float2* out, const Taps& tp) {
  constexpr int RS = TW + 2;
#pragma unroll
  for (int r = 0; r < Q; ++r) {
    const float2 v = hin[r * RS];
    const float2 o = ffma2(v, tp.t[R], st[0]);
#pragma unroll
    for (int i = 0; i < 2 * R - 1; ++i) {
      const int d = R - 1 - i;
      st[i] = ffma2(v, tp.t[d >= 0 ? d : -d], st[i + 1]);
    }
    st[2 * R - 1] = __fmul2_rn(v, make_float2(tp.t[R], tp.t[R]));
    out[r * TW] = o;
  }
}

// MODE 0: interleaved Q=8; 1: sequential Q; 2: sequential Q with scatter column pass
template <int Q, int MODE, int SYNC = 0>
__global__ void __launch_bounds__(384, 1) body(const Taps tp, float* sink, int steps) {
  using G = Geo<Q>;
  extern __shared__ __align__(16) float2 sm[];
  const int w = threadIdx.x / 32, lane = threadIdx.x & 31;
  float2* gen = sm + (size_t)w * G::floats2;
  float2* ring = gen + Q * G::GS;
  float2* out = ring + (G::RB + 1) * Q * G::RS;
  for (int i = lane; i < G::floats2; i += 32) gen[i] = make_float2(1e-3f * i, 1.f);
  __syncwarp();
  float2 st[2 * R];
  for (int i = 0; i < 2 * R; ++i) st[i] = make_float2(0.f, 0.f);
  for (int t = 0; t < steps; ++t) {
    if (MODE == 2) {
      row_pass<Q>(gen, ring, lane, tp);
      __syncwarp();
      col_scatter<Q>(ring + lane, st, out + lane, tp);
      if (SYNC == 1) asm volatile("bar.sync 1;" ::: "memory");
      if (SYNC == 2 && (t & 1)) asm volatile("bar.sync 1;" ::: "memory");
    } else if (MODE == 0) {
      inter8(gen, ring, t % (G::RB + 1), (t + G::RB) % (G::RB + 1), lane, tp, out);
    } else {
      const int blk = t % G::RB;
      row_pass<Q>(gen, ring + blk * Q * G::RS, lane, tp);
      __syncwarp();
      col_pass<Q, G::RB>(ring, blk, lane, tp, out);
    }
    __syncwarp();
  }
  if (out[lane].x == 12345.f) sink[0] = 1.f;
}

int main(int argc, char** argv) {
  Taps tp; for (int j = 0; j <= R; j++) tp.t[j] = 1.f / (1 + j);
  float* sink; cudaMalloc(&sink, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto run = [&](auto kern, int q, int warps, size_t per_warp, const char* name) {
    const size_t smem = per_warp * warps;
    if (smem > 232448) { printf("%s warps %d: smem %zu too big\n", name, warps, smem); return; }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    const int steps = 8000 / q;
    kern<<<148, warps * 32, smem>>>(tp, sink, 4);
    cudaEventRecord(a); kern<<<148, warps * 32, smem>>>(tp, sink, steps); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 148.0 * warps * steps * 2.0 * (q * TW) * (2 * R + 1) * 4;
    printf("%s warps %2d: %.1f%% of 74.45 TF  (%s)\n", name, warps, flops / ms / 1e9 / 74.45 * 100, cudaGetErrorString(cudaGetLastError()));
  };
  // warps per CTA from the command line (default 7): 4 = one FFMA2 warp per sub-partition
  std::vector<int> wlist; for (int i = 1; i < argc; ++i) wlist.push_back(atoi(argv[i]));
  if (wlist.empty()) wlist.push_back(7);
  for (int wps : wlist) {
    run(body<16, 2>, 16, wps, sizeof(float2) * Geo<16>::floats2, "scat  Q=16");
    run(body<16, 2, 1>, 16, wps, sizeof(float2) * Geo<16>::floats2, "scat  Q=16 sync");
    run(body<16, 2, 2>, 16, wps, sizeof(float2) * Geo<16>::floats2, "scat  Q=16 sync/2");
    run(body<8, 2>, 8, wps, sizeof(float2) * Geo<8>::floats2, "scat  Q=8 ");
    run(body<8, 2, 1>, 8, wps, sizeof(float2) * Geo<8>::floats2, "scat  Q=8 sync");
  }
}
