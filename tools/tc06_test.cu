// tcgen05 weight-gradient layout probe: D = X^T Y over K = 128 samples with
// BOTH operands MN-major in shared memory (each thread = one sample writes its
// feature row as 16-byte chunks into the interleaved core-matrix layout), the
// form a fused backward needs for dW = sum_s a_s (x) delta_s.
//   X: 128 x M (features), Y: 128 x 32.  M = 64 or 128.  kind::tf32, 1 pass.
// Probes which descriptor field (LBO / SBO) is the MN-direction stride, and
// where the M = 64 accumulator rows land in TMEM.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t s32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
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

// MN-major interleaved: element (mn, k) of an [MN x 128] operand:
//   core (mn >> 2, k >> 3) holds 8 k-rows of 16 bytes (4 mn elements)
//   mode 0: mn-core stride = 128 B * 16 (= all k-cores of one mn chunk contiguous), k-core stride = 128 B
//   mode 1: k-core stride = 128 B * (MN / 4), mn-core stride = 128 B
__host__ __device__ __forceinline__ int mnmaj(int mn, int k, int MN, int mode) {
  const int mc = mn >> 2, kc = k >> 3;
  const int core = mode == 0 ? mc * 16 + kc : kc * (MN / 4) + mc;
  return core * 32 + (k & 7) * 4 + (mn & 3);
}

// K-major: element (r, k) of an [R x 128] operand (core: 8 rows x 16 B of k)
__host__ __device__ __forceinline__ int kmaj(int r, int k) {
  return (r >> 3) * 32 * 32 + (k >> 2) * 32 + (r & 7) * 4 + (k & 3);
}

struct Smem {
  float a[128 * 128];
  float b[32 * 128];
  uint64_t bar;
  uint32_t tmem;
};

// one CTA of 128 threads; thread t = sample t
__global__ void __launch_bounds__(128) k_probe(const float* X, const float* Y, float* D, int M, int mode,
                                               uint32_t lbo_a, uint32_t sbo_a, uint32_t lbo_b, uint32_t sbo_b,
                                               int ta, int tb) {
  extern __shared__ __align__(1024) unsigned char raw[];
  Smem& S = *reinterpret_cast<Smem*>(raw);
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(s32(&S.tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s32(&S.bar)) : "memory");
  for (int m = 0; m < M; ++m) S.a[ta ? mnmaj(m, t, M, mode) : kmaj(m, t)] = X[t * M + m];
  for (int n = 0; n < 32; ++n) S.b[tb ? mnmaj(n, t, 32, mode) : kmaj(n, t)] = Y[t * 32 + n];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = S.tmem;
  // kind::tf32, D f32, A/B MN-major (bits 15, 16), N = 32, M
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)ta << 15) | ((uint32_t)tb << 16) |
                         ((32u >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  if (t == 0) {
    for (int kk = 0; kk < 16; ++kk) {  // K = 128 in steps of 8 (one k-core)
      const uint32_t koff = !ta ? kk * 256 : (mode == 0 ? kk * 128 : kk * 128 * (M / 4));
      const uint32_t koffb = !tb ? kk * 256 : (mode == 0 ? kk * 128 : kk * 128 * 8);
      mma_ss(tmem, sdesc(s32(S.a) + koff, lbo_a, sbo_a), sdesc(s32(S.b) + koffb, lbo_b, sbo_b), idesc, kk > 0);
    }
    commit(&S.bar);
  }
  mbar_wait(&S.bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  float v[32];
  ld32(tmem + ((uint32_t)(warp * 32) << 16), v);
  for (int n = 0; n < 32; ++n) D[t * 32 + n] = v[n];  // TMEM lane t, column n
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  std::vector<float> X(128 * 128), Y(128 * 32), D(128 * 32);
  srand(3);
  auto tf = [](float x) {  // tf32-representable values: exact products
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
  };
  for (auto& v : Y) v = tf((rand() / (float)RAND_MAX - 0.5f));
  float *dX, *dY, *dD;
  cudaMalloc(&dX, X.size() * 4);
  cudaMalloc(&dY, Y.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dY, Y.data(), Y.size() * 4, cudaMemcpyHostToDevice);
  const int smem = sizeof(Smem) + 1024;
  cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int M : {64, 128}) {
    for (auto& v : X) v = 0.f;
    for (int s = 0; s < 128; ++s)
      for (int m = 0; m < M; ++m) X[s * M + m] = tf((rand() / (float)RAND_MAX - 0.5f));
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    std::vector<double> ref(M * 32);
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < 32; ++n) {
        double a = 0;
        for (int s = 0; s < 128; ++s) a += (double)X[s * M + m] * Y[s * 32 + n];
        ref[m * 32 + n] = a;
      }
    for (int variant = 0; variant < 10; ++variant) {
      // variant 0: both K-major (harness check); 1..: MN-major A and/or B with (mode, swap)
      const int ta = variant == 0 ? 0 : (variant <= 4 ? 1 : (variant <= 8 ? 0 : 1));
      const int tb = variant == 0 ? 0 : (variant <= 4 ? 0 : 1);
      const int mode = ((variant - 1) >> 1) & 1, swap = (variant - 1) & 1;
      {
        const uint32_t mn_a = mode == 0 ? 2048 : 128, mn_b = mode == 0 ? 2048 : 128;
        const uint32_t k_a = mode == 0 ? 128 : 128 * (M / 4), k_b = mode == 0 ? 128 : 128 * 8;
        uint32_t lbo_a = swap ? k_a : mn_a, sbo_a = swap ? mn_a : k_a;
        uint32_t lbo_b = swap ? k_b : mn_b, sbo_b = swap ? mn_b : k_b;
        if (!ta) { lbo_a = 128; sbo_a = 4096; }
        if (!tb) { lbo_b = 128; sbo_b = 4096; }
        cudaMemset(dD, 0, D.size() * 4);
        k_probe<<<1, 128, smem>>>(dX, dY, dD, M, mode, lbo_a, sbo_a, lbo_b, sbo_b, ta, tb);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        // find where row m landed: lane L with best match
        int rows_ok = 0;
        double worst = 0;
        int lane_of[128];
        for (int m = 0; m < M; ++m) {
          lane_of[m] = -1;
          for (int L = 0; L < 128; ++L) {
            double err = 0, mx = 0;
            for (int n = 0; n < 32; ++n) {
              err = fmax(err, fabs(D[L * 32 + n] - ref[m * 32 + n]));
              mx = fmax(mx, fabs(ref[m * 32 + n]));
            }
            if (err <= 1e-4 * mx) {
              lane_of[m] = L;
              break;
            }
          }
          if (lane_of[m] >= 0) ++rows_ok;
        }
        printf("M=%d ta=%d tb=%d mode=%d swap=%d A(lbo %u sbo %u) B(lbo %u sbo %u): %s rows matched %d/%d", M, ta, tb, mode, swap,
               lbo_a, sbo_a, lbo_b, sbo_b,
               cudaGetErrorString(e), rows_ok, M);
        if (rows_ok) {
          printf("  lanes:");
          for (int m = 0; m < M; m += 8) printf(" %d->%d", m, lane_of[m]);
        }
        printf("\n");
        (void)worst;
        if (false) {  // dumps for offline analysis
          char fn[64];
          snprintf(fn, sizeof fn, "gpurun_out/tc06_D_m%d.bin", mode);
          FILE* f = fopen(fn, "wb");
          fwrite(D.data(), 4, D.size(), f);
          fclose(f);
          f = fopen("gpurun_out/tc06_X.bin", "wb");
          fwrite(X.data(), 4, 128 * 128, f);
          fwrite(Y.data(), 4, 128 * 32, f);
          fclose(f);
        }
      }
    }
  }
  return 0;
}
