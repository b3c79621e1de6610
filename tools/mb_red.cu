// Microbenchmark: L2 reduction throughput for the grid-gradient scatter.
// A 95 MB float array (the c2 finest level), N updates at random 16-byte
// aligned rows; variants: red.global.add.v4.f32, 4 x scalar red.add.f32,
// plain st.global.v4 (no reduction), and pairs of z-adjacent rows (32 B) as
// two v4 reds vs one cp.reduce.async.bulk of 32 B from shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_red tools/mb_red.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
  return x;
}
__device__ __forceinline__ void red_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}
template <int MODE>
__global__ void k(float* buf, uint32_t rows, int per_thread, int locality) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ __align__(128) float stage[256 * 8];
  for (int i = 0; i < per_thread; ++i) {
    uint32_t h = hash32(t * 977u + i * 131u);
    // locality: consecutive lanes hit nearby rows (a ray's samples), else random
    uint32_t r = locality ? (hash32(t / 32 + i * 7919u) % rows + (threadIdx.x & 31) * 3) % (rows - 2)
                          : h % (rows - 2);
    float* p = buf + (size_t)r * 4;
    if (MODE == 0) {
      red_v4(p, 1.f, 2.f, 3.f, 4.f);
    } else if (MODE == 1) {
      atomicAdd(p, 1.f); atomicAdd(p + 1, 2.f); atomicAdd(p + 2, 3.f); atomicAdd(p + 3, 4.f);
    } else if (MODE == 2) {
      *reinterpret_cast<float4*>(p) = make_float4(1.f, 2.f, 3.f, (float)i);
    } else if (MODE == 3) {  // two adjacent rows, two v4 reds (counts as 2 updates)
      red_v4(p, 1.f, 2.f, 3.f, 4.f);
      red_v4(p + 4, 1.f, 2.f, 3.f, 4.f);
    } else if (MODE == 4) {  // two adjacent rows, one 32 B bulk reduction from smem
      float* s = stage + threadIdx.x * 8;
      *reinterpret_cast<float4*>(s) = make_float4(1.f, 2.f, 3.f, 4.f);
      *reinterpret_cast<float4*>(s + 4) = make_float4(1.f, 2.f, 3.f, 4.f);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint32_t sa = (uint32_t)__cvta_generic_to_shared(s);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 32;" ::"l"(p), "r"(sa)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
  }
}

int main() {
  const uint32_t rows = 95u * 1024 * 1024 / 16;
  float* buf;
  cudaMalloc(&buf, (size_t)rows * 16 + 64);
  cudaMemset(buf, 0, (size_t)rows * 16 + 64);
  const int threads = 256, blocks = 148 * 8, per = 48;
  const double n = (double)threads * blocks * per;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"red.v4 (16 B)", "4 x red.f32", "st.v4 (no red)", "2 x red.v4 adjacent (32 B)",
                         "bulk reduce 32 B"};
  for (int loc = 0; loc < 2; ++loc)
    for (int m = 0; m < 5; ++m) {
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(a);
        switch (m) {
          case 0: k<0><<<blocks, threads>>>(buf, rows, per, loc); break;
          case 1: k<1><<<blocks, threads>>>(buf, rows, per, loc); break;
          case 2: k<2><<<blocks, threads>>>(buf, rows, per, loc); break;
          case 3: k<3><<<blocks, threads>>>(buf, rows, per, loc); break;
          case 4: k<4><<<blocks, threads>>>(buf, rows, per, loc); break;
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep == 2)
          printf("%-28s locality=%d: %8.3f ms  %7.2f G updates/s  (%.1f M updates)\n", names[m], loc, ms,
                 n / ms / 1e6, n / 1e6);
      }
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
