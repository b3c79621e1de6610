// tcgen05 feasibility for the decoders: a CTA of 128 threads (one sample per
// thread) runs 32-wide MLP layers as tcgen05.mma kind::tf32 (3xTF32 split,
// M=128 samples, N=32, K=32), operands in shared memory in the canonical
// K-major no-swizzle layout, accumulator in TMEM, epilogue via
// tcgen05.ld.32x32b (thread = TMEM lane = sample).
//   mode 1: one layer, checked against fp64 on the host
//   mode 2: throughput of chained layers (ld -> relu -> split -> st.shared ->
//           fence -> mma), several CTAs per SM
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// element (r, k) of an [R x K] fp32 tile: core matrices of 8 rows x 4 k (16 B
// rows), K-chunks adjacent (LBO = 128 B), 8-row groups after K/4 chunks (SBO)
__host__ __device__ __forceinline__ int kmaj(int r, int k, int K) {
  return (r >> 3) * (K / 4) * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100)
  return d;                // base offset 0, SWIZZLE_NONE
}

// kind::tf32, D f32, A/B tf32 K-major, N = 32, M = 128
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(s32(bar)), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  const uint32_t h = (__float_as_uint(x) + 0x1000u) & 0xffffe000u;
  hi = __uint_as_float(h);
  lo = x - hi;
}

struct Smem {
  float a[2][128 * 32];  // A hi / lo  (samples x features, K-major)
  float b[2][32 * 32];   // B hi / lo  (out x in, K-major)
  uint64_t bar;
  uint32_t tmem;
};

// 3xTF32: D = Ahi Bhi + Ahi Blo + Alo Bhi over K = 32 (4 k-steps of 8)
__device__ __forceinline__ void layer_mma(Smem& S, uint32_t tmem) {
  const uint32_t a0 = s32(S.a[0]), a1 = s32(S.a[1]), b0 = s32(S.b[0]), b1 = s32(S.b[1]);
  uint32_t acc = 0;
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const uint32_t off = kk * 256;  // 2 K-chunks of 128 B per k-step
    mma_tf32(tmem, sdesc(a1 + off, 128, 1024), sdesc(b0 + off, 128, 1024), acc);
    acc = 1;
    mma_tf32(tmem, sdesc(a0 + off, 128, 1024), sdesc(b1 + off, 128, 1024), 1);
    mma_tf32(tmem, sdesc(a0 + off, 128, 1024), sdesc(b0 + off, 128, 1024), 1);
  }
}

__global__ void __launch_bounds__(128) k_test(const float* A, const float* W, float* D, int iters) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(s32(&S.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&S.bar);
  // weights: B[n][k] = W[k][n]
  for (int i = t; i < 32 * 32; i += 128) {
    const int k = i / 32, n = i % 32;
    float hi, lo;
    split(W[i], hi, lo);
    S.b[0][kmaj(n, k, 32)] = hi;
    S.b[1][kmaj(n, k, 32)] = lo;
  }
  float x[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = A[((size_t)blockIdx.x * 128 + t) * 32 + k];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = S.tmem;
  const uint32_t my = tmem + ((uint32_t)(warp * 32) << 16);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k4 = 0; k4 < 32; k4 += 4) {
      float h[4], l[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) split(x[k4 + q], h[q], l[q]);
      *reinterpret_cast<float4*>(&S.a[0][kmaj(t, k4, 32)]) = make_float4(h[0], h[1], h[2], h[3]);
      *reinterpret_cast<float4*>(&S.a[1][kmaj(t, k4, 32)]) = make_float4(l[0], l[1], l[2], l[3]);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
      layer_mma(S, tmem);
      commit(&S.bar);
    }
    mbar_wait(&S.bar, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    float y[32];
    ld32(my, y);
    if (iters == 1) {
#pragma unroll
      for (int n = 0; n < 32; ++n) x[n] = y[n];
    } else {
#pragma unroll
      for (int n = 0; n < 32; ++n) x[n] = fmaxf(y[n], 0.f) * 0.5f + 1e-3f;
    }
  }
#pragma unroll
  for (int n = 0; n < 32; ++n) D[((size_t)blockIdx.x * 128 + t) * 32 + n] = x[n];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

__device__ __forceinline__ void mma_tf32_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(b), "r"(IDESC), "r"(acc));
}
#define U(i) "r"(__float_as_uint(v[i]))
__device__ __forceinline__ void st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      U(0), U(1), U(2), U(3), U(4), U(5), U(6), U(7), U(8), U(9), U(10), U(11), U(12), U(13), U(14), U(15),
      U(16), U(17), U(18), U(19), U(20), U(21), U(22), U(23), U(24), U(25), U(26), U(27), U(28), U(29), U(30),
      U(31));
}
#undef U

// TS chain: activations hi/lo live in TMEM columns [32,64) / [64,96); D in [0,32)
__global__ void __launch_bounds__(128) k_test_ts(const float* A, const float* W, float* D, int iters) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(s32(&S.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&S.bar);
  for (int i = t; i < 32 * 32; i += 128) {
    const int k = i / 32, n = i % 32;
    float hi, lo;
    split(W[i], hi, lo);
    S.b[0][kmaj(n, k, 32)] = hi;
    S.b[1][kmaj(n, k, 32)] = lo;
  }
  float x[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) x[k] = A[((size_t)blockIdx.x * 128 + t) * 32 + k];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = S.tmem;
  const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
  const uint32_t b0 = s32(S.b[0]), b1 = s32(S.b[1]);
  for (int it = 0; it < iters; ++it) {
    float h[32], l[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) split(x[k], h[k], l[k]);
    st32(tmem + lane_off + 32, h);
    st32(tmem + lane_off + 64, l);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
      uint32_t acc = 0;
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t off = kk * 256;
        mma_tf32_ts(tmem, tmem + 64 + kk * 8, sdesc(b0 + off, 128, 1024), acc);
        acc = 1;
        mma_tf32_ts(tmem, tmem + 32 + kk * 8, sdesc(b1 + off, 128, 1024), 1);
        mma_tf32_ts(tmem, tmem + 32 + kk * 8, sdesc(b0 + off, 128, 1024), 1);
      }
      commit(&S.bar);
    }
    mbar_wait(&S.bar, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    float y[32];
    ld32(tmem + lane_off, y);
    if (iters == 1) {
#pragma unroll
      for (int n = 0; n < 32; ++n) x[n] = y[n];
    } else {
#pragma unroll
      for (int n = 0; n < 32; ++n) x[n] = fmaxf(y[n], 0.f) * 0.5f + 1e-3f;
    }
  }
#pragma unroll
  for (int n = 0; n < 32; ++n) D[((size_t)blockIdx.x * 128 + t) * 32 + n] = x[n];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  const int blocks1 = 4;
  std::vector<float> A(blocks1 * 128 * 32), W(32 * 32), D(blocks1 * 128 * 32);
  srand(1);
  for (auto& v : A) v = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
  for (auto& v : W) v = (rand() / (float)RAND_MAX - 0.5f) * 0.5f;
  float *dA, *dW, *dD;
  cudaMalloc(&dA, 1 << 28);
  cudaMalloc(&dW, W.size() * 4);
  cudaMalloc(&dD, 1 << 28);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
  const int smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_test_ts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int variant = 0; variant < 2; ++variant) {
    auto kern = variant == 0 ? k_test : k_test_ts;
    const char* nm = variant == 0 ? "SS (A via smem)" : "TS (A in TMEM)";
    kern<<<blocks1, 128, smem>>>(dA, dW, dD, 1);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int r = 0; r < blocks1 * 128; ++r)
      for (int n = 0; n < 32; ++n) {
        double ref = 0;
        for (int k = 0; k < 32; ++k) ref += (double)A[r * 32 + k] * W[k * 32 + n];
        maxerr = fmax(maxerr, fabs(ref - D[r * 32 + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("%s: %s  rel err %.3e\n", nm, cudaGetErrorString(e), maxerr / maxref);
    for (int per_sm : {1, 2, 4}) {
      const int grid = sms * per_sm, iters = 64;
      kern<<<grid, 128, smem>>>(dA, dW, dD, iters);
      cudaEventRecord(a);
      kern<<<grid, 128, smem>>>(dA, dW, dD, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double fma = (double)grid * 128 * iters * 1024;
      printf("  %s CTAs/SM=%d  %.3f ms  %.1f TFMA/s effective (%.0f%% of fp32 FFMA peak); %s\n", nm, per_sm,
             ms, fma / (ms * 1e-3) / 1e12, 100.0 * fma / (ms * 1e-3) / (sms * 128.0 * 1.965e9),
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
