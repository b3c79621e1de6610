// Microbenchmark: compact 32x32 dense-layer formulations for thread/warp-per-sample
// MLPs on sm_100a (decides the taped-pass decoder design).
//   0: fully unrolled FFMA, weights from __constant__ float4 (current kernels)
//   1: FFMA with a runtime output-quad loop (uniform constant index), outputs staged
//      to a per-thread shared-memory row, next layer reloads with LDS.128
//   2: mma.sync m16n8k8 TF32, 1 pass, warp = 32 samples, D fragments chained as A
//   3: same, 3xTF32 (hi*hi + hi*lo + lo*hi)
// Each thread/warp runs `iters` layers; reports effective fp32 FMA/s.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__constant__ float4 c_w[32 * 8 + 8];

__device__ __forceinline__ uint32_t tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ void mma(float* d, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int MODE>
__global__ void __launch_bounds__(128) k_layers(const float* __restrict__ gw, float* out, int iters) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x & 31;
  if (MODE <= 1) {
    float x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = (threadIdx.x + j) * 1e-3f;
    float* row = sm + threadIdx.x * 36;
    for (int it = 0; it < iters; ++it) {
      if (MODE == 0) {
        float acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.f;
#pragma unroll
        for (int i = 0; i < 32; ++i)
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            float4 w = c_w[i * 8 + j4];
            acc[4 * j4] = fmaf(x[i], w.x, acc[4 * j4]);
            acc[4 * j4 + 1] = fmaf(x[i], w.y, acc[4 * j4 + 1]);
            acc[4 * j4 + 2] = fmaf(x[i], w.z, acc[4 * j4 + 2]);
            acc[4 * j4 + 3] = fmaf(x[i], w.w, acc[4 * j4 + 3]);
          }
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = fmaxf(acc[j], 0.f) * 0.5f + 1e-3f;
      } else {
#pragma unroll 1
        for (int j4 = 0; j4 < 8; ++j4) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float4 w = c_w[i * 8 + j4];
            a0 = fmaf(x[i], w.x, a0);
            a1 = fmaf(x[i], w.y, a1);
            a2 = fmaf(x[i], w.z, a2);
            a3 = fmaf(x[i], w.w, a3);
          }
          reinterpret_cast<float4*>(row)[j4] = make_float4(a0, a1, a2, a3);
        }
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          float4 v = reinterpret_cast<float4*>(row)[j4];
          x[4 * j4] = fmaxf(v.x, 0.f) * 0.5f + 1e-3f;
          x[4 * j4 + 1] = fmaxf(v.y, 0.f) * 0.5f + 1e-3f;
          x[4 * j4 + 2] = fmaxf(v.z, 0.f) * 0.5f + 1e-3f;
          x[4 * j4 + 3] = fmaxf(v.w, 0.f) * 0.5f + 1e-3f;
        }
      }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 32; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  } else {
    // B fragments (weights) in registers: 4 k-steps x 4 n-tiles x 2 regs, hi and lo
    uint32_t bh[4][4][2], bl[4][4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          float w = gw[(k * 8 + (lane & 3) + 4 * r) * 32 + n * 8 + (lane >> 2)];
          bh[k][n][r] = tf32(w);
          bl[k][n][r] = tf32(w - __uint_as_float(bh[k][n][r]));
        }
    // activations as D fragments: [m-tile 2][n-tile 4][4]
    float x[2][4][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int r = 0; r < 4; ++r) x[m][n][r] = (threadIdx.x + m + n + r) * 1e-3f;
    for (int it = 0; it < iters; ++it) {
      float d[2][4][4];
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int r = 0; r < 4; ++r) d[m][n][r] = 0.f;
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // D fragment of n-tile k (cols 2c,2c+1 at rows g, g+8) is the A fragment of
          // k-step k under the K permutation slot c <-> 2c, slot c+4 <-> 2c+1.
          float av[4] = {x[m][k][0], x[m][k][2], x[m][k][1], x[m][k][3]};
          uint32_t ah[4], al[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            ah[r] = tf32(av[r]);
            al[r] = tf32(av[r] - __uint_as_float(ah[r]));
          }
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            mma(d[m][n], ah, bh[k][n][0], bh[k][n][1]);
            if (MODE == 3) {
              mma(d[m][n], ah, bl[k][n][0], bl[k][n][1]);
              mma(d[m][n], al, bh[k][n][0], bh[k][n][1]);
            }
          }
        }
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
          for (int r = 0; r < 4; ++r) x[m][n][r] = fmaxf(d[m][n][r], 0.f) * 0.5f + 1e-3f;
    }
    float s = 0.f;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n)
#pragma unroll
        for (int r = 0; r < 4; ++r) s += x[m][n][r];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  }
}

int main() {
  float* gw;
  float* out;
  const int NW = (32 * 8 + 8) * 4;
  cudaMalloc(&gw, NW * 4);
  cudaMalloc(&out, 1 << 26);
  static float h[NW];
  for (int i = 0; i < NW; ++i) h[i] = 0.01f * ((i * 37) % 11 - 5);
  cudaMemcpy(gw, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_w, h, sizeof(h));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64;
  const char* names[4] = {"ffma-unrolled-const", "ffma-quadloop-smem", "mma-tf32-1x", "mma-tf32-3x"};
  void (*ks[4])(const float*, float*, int) = {k_layers<0>, k_layers<1>, k_layers<2>, k_layers<3>};
  const int smem = 128 * 36 * 4;
  for (int m = 0; m < 4; ++m) cudaFuncSetAttribute(ks[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int blocksPerSm : {1, 2, 3, 4, 8}) {
    int grid = sms * blocksPerSm;
    for (int mode = 0; mode < 4; ++mode) {
      auto k = ks[mode];
      k<<<grid, 128, smem>>>(gw, out, iters);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k<<<grid, 128, smem>>>(gw, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      // samples processed: threads (modes 0,1) or 32 per warp (modes 2,3) -> same count
      double fma = 5.0 * grid * 128.0 * iters * 1024.0;
      printf("blocks/SM=%d %-20s %.3f ms  %6.1f TFMA/s (%3.0f%% of 128 FFMA/clk/SM @1.965GHz)\n",
             blocksPerSm, names[mode], ms, fma / (ms * 1e-3) / 1e12,
             100.0 * fma / (ms * 1e-3) / (sms * 128.0 * 1.965e9));
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
