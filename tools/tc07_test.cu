// tcgen05 weight-gradient GEMM with transposed activations: D = X^T Y over
// K = 128 samples, both operands K-major with the 128-byte swizzle, written
// by the sample threads themselves (thread s writes column s of every row:
// one warp covers a whole 128-byte swizzle row, so the stores are
// bank-conflict-free).  This is the operand form a tcgen05 backward needs for
// dW = sum_s a_s (x) delta_s (tools/tc06_test.cu showed MN-major tf32 operands
// are not accepted).  Checks 1xTF32 and 3xTF32 against fp64, then times the
// write + 3xTF32 MMA of one tile.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SM100 shared-memory descriptor: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
// version 1 at bit 46, layout type [61,64): 2 = SWIZZLE_128B
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;  // LBO (unused for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mma_ss(uint32_t tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s32(bar))
               : "memory");
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
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
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
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void split(float x, float& hi, float& lo) {
  hi = __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
  lo = x - hi;
}

// element (row r, k) of an [R x 128] K-major operand, 128B swizzle: k-block
// kb = k / 32 is its own [R x 32] tile (R/8 atoms of 8 rows x 128 B, SBO 1024 B)
__device__ __forceinline__ int sw128(int r, int k, int R) {
  const int kb = k >> 5, kk = k & 31;
  const int chunk = (kk >> 2) ^ (r & 7);
  return kb * R * 32 + (r >> 3) * 256 + (r & 7) * 32 + chunk * 4 + (kk & 3);
}

constexpr int MROWS = 64, NCOLS = 32, KS = 128;
struct __align__(1024) Smem {
  float ah[MROWS * KS], al[MROWS * KS];  // X^T hi / lo
  float bh[NCOLS * KS], bl[NCOLS * KS];  // Y^T hi / lo
  uint64_t bar;
  uint32_t tmem;
};

// thread s = sample s writes its X row (64 features) and Y row (32)
__global__ void __launch_bounds__(128) k_dw(const float* X, const float* Y, float* D, int three, int iters) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~(uintptr_t)1023);
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(s32(&S.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&S.bar)) : "memory");
  // M = 64 rows of D land in TMEM lanes 0-15, 32-47, 64-79, 96-111 (tc06)
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NCOLS >> 3) << 17) |
                         ((uint32_t)(MROWS >> 4) << 24);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = S.tmem;
  float xr[MROWS], yr[NCOLS];  // the activations a backward kernel holds in registers
#pragma unroll
  for (int m = 0; m < MROWS; ++m) xr[m] = X[t * MROWS + m];
#pragma unroll
  for (int n = 0; n < NCOLS; ++n) yr[n] = Y[t * NCOLS + n];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < MROWS; ++m) {
      float h, l;
      split(xr[m] + 1e-30f * it, h, l);
      S.ah[sw128(m, t, MROWS)] = h;
      S.al[sw128(m, t, MROWS)] = l;
    }
#pragma unroll
    for (int n = 0; n < NCOLS; ++n) {
      float h, l;
      split(yr[n], h, l);
      S.bh[sw128(n, t, NCOLS)] = h;
      S.bl[sw128(n, t, NCOLS)] = l;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (t == 0) {
      for (int kk = 0; kk < KS / 8; ++kk) {
        const int kb = kk >> 2, ko = (kk & 3) * 32;  // k-block tile, 32 B per k-step inside the atom
        const uint32_t oa = kb * MROWS * 128 + ko, ob = kb * NCOLS * 128 + ko;
        mma_ss(tmem, sdesc_sw128(s32(S.ah) + oa, 1024), sdesc_sw128(s32(S.bh) + ob, 1024), idesc, kk > 0);
        if (three) {
          mma_ss(tmem, sdesc_sw128(s32(S.ah) + oa, 1024), sdesc_sw128(s32(S.bl) + ob, 1024), idesc, 1);
          mma_ss(tmem, sdesc_sw128(s32(S.al) + oa, 1024), sdesc_sw128(s32(S.bh) + ob, 1024), idesc, 1);
        }
      }
      commit(&S.bar);
    }
    mbar_wait(&S.bar, it & 1);
    asm volatile("tcgen05.fence::after_thread_sync;");
    __syncthreads();
  }
  float v[32];
  ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 32; ++n) D[(size_t)blockIdx.x * 128 * 32 + t * 32 + n] = v[n];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  std::vector<float> X(KS * MROWS), Y(KS * NCOLS), D(128 * 32 * 148 * 4);
  srand(7);
  for (auto& v : X) v = (rand() / (float)RAND_MAX - 0.5f);
  for (auto& v : Y) v = (rand() / (float)RAND_MAX - 0.5f);
  std::vector<double> ref(MROWS * NCOLS);
  for (int m = 0; m < MROWS; ++m)
    for (int n = 0; n < NCOLS; ++n) {
      double a = 0;
      for (int s = 0; s < KS; ++s) a += (double)X[s * MROWS + m] * Y[s * NCOLS + n];
      ref[m * NCOLS + n] = a;
    }
  float *dX, *dY, *dD;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dY, Y.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  const int smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(k_dw, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int three = 0; three < 2; ++three) {
    cudaMemset(dD, 0, D.size() * 4);
    k_dw<<<1, 128, smem>>>(dX, dY, dD, three, 1);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, 128 * 32 * 4, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int m = 0; m < MROWS; ++m) {
      const int lane = (m >> 4) * 32 + (m & 15);  // M = 64 TMEM lane map
      for (int n = 0; n < NCOLS; ++n) {
        err = fmax(err, fabs(D[lane * 32 + n] - ref[m * NCOLS + n]));
        mx = fmax(mx, fabs(ref[m * NCOLS + n]));
      }
    }
    printf("%s-TF32 SW128 K-major dW tile (M=64, N=32, K=128): %s, max rel err %.3e\n", three ? "3x" : "1x",
           cudaGetErrorString(e), err / mx);
  }
  // throughput: 4 CTAs/SM, each repeating write + 3xTF32 MMA of one tile
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 64, grid = 148 * 2;
  k_dw<<<grid, 128, smem>>>(dX, dY, dD, 1, iters);
  cudaEventRecord(a);
  k_dw<<<grid, 128, smem>>>(dX, dY, dD, 1, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double tiles = (double)grid * iters;
  printf("write + 3xTF32 dW tile: %.3f us per tile per CTA, %.1f M samples/s of dW(64x32) per GPU; %s\n",
         ms * 1e3 / iters, tiles * 128 / (ms * 1e-3) / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
