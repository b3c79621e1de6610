// Microbenchmark: feeding MLP weights to thread-per-sample FFMA layers on sm_100a.
//   A: weights in shared memory, 16-byte broadcast loads (LDS.128)
//   B: weights in __constant__, float4 reads with compile-time indices (LDCU)
// Each thread runs L dense 32x32 layers (ReLU) on its own 32-vector.
#include <cstdio>
#include <cuda_runtime.h>

__constant__ float4 c_w[32 * 8 + 8];

template <int MODE>
__global__ void __launch_bounds__(128) k_layers(const float* __restrict__ gw, float* out, int iters) {
  __shared__ float4 sw[32 * 8 + 8];
  for (int t = threadIdx.x; t < 32 * 8 + 8; t += blockDim.x) sw[t] = reinterpret_cast<const float4*>(gw)[t];
  __syncthreads();
  float x[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) x[j] = (threadIdx.x + j) * 1e-3f;
  for (int it = 0; it < iters; ++it) {
    float acc[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) acc[j] = 0.f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
#pragma unroll
      for (int j4 = 0; j4 < 8; ++j4) {
        float4 w = MODE == 0 ? sw[i * 8 + j4] : c_w[i * 8 + j4];
        acc[4 * j4] = fmaf(x[i], w.x, acc[4 * j4]);
        acc[4 * j4 + 1] = fmaf(x[i], w.y, acc[4 * j4 + 1]);
        acc[4 * j4 + 2] = fmaf(x[i], w.z, acc[4 * j4 + 2]);
        acc[4 * j4 + 3] = fmaf(x[i], w.w, acc[4 * j4 + 3]);
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = fmaxf(acc[j], 0.f) * 0.5f + 1e-3f;
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 32; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* gw;
  float* out;
  cudaMalloc(&gw, (32 * 8 + 8) * 16);
  cudaMemset(gw, 0, (32 * 8 + 8) * 16);
  cudaMalloc(&out, 1 << 26);
  float h[(32 * 8 + 8) * 4];
  for (int i = 0; i < (32 * 8 + 8) * 4; ++i) h[i] = 0.01f * ((i * 37) % 11 - 5);
  cudaMemcpy(gw, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_w, h, sizeof(h));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64;
  for (int blocksPerSm : {1, 2, 4, 8}) {
    int grid = sms * blocksPerSm;
    for (int mode = 0; mode < 2; ++mode) {
      auto k = mode == 0 ? k_layers<0> : k_layers<1>;
      k<<<grid, 128>>>(gw, out, iters);
      cudaEventRecord(a);
      for (int r = 0; r < 5; ++r) k<<<grid, 128>>>(gw, out, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      double fma = 5.0 * grid * 128.0 * iters * 1024.0;
      printf("blocks/SM=%d mode=%s  %.3f ms  %.1f TFMA/s (%.0f%% of 128 FMA/clk/SM @1.965GHz)\n",
             blocksPerSm, mode == 0 ? "smem-LDS128" : "const-LDCU", ms, fma / (ms * 1e-3) / 1e12,
             100.0 * fma / (ms * 1e-3) / (sms * 128.0 * 1.965e9));
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
