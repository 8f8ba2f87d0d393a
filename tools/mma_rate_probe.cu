// mma_rate_probe.cu -- issue rate of back-to-back tcgen05.mma.cta_group::2
// kind::f16 (M = 256, fp32 accumulate, both operands in shared memory) as a
// function of N, with and without the A-collector reuse the SCREEN kernel's
// three-product K step uses.  No loads, no epilogue: one elected thread per
// CTA pair issues MMAs on a fixed shared-memory stage.  Profiling aid for
// the SCREEN engine's tile shape (adg_screen_kernel.cuh), not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_rate_probe.cu
//   /tmp/mma_probe
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                 \
  do {                                                                        \
    cudaError_t e = (x);                                                      \
    if (e != cudaSuccess) {                                                   \
      std::printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); \
      return 1;                                                               \
    }                                                                         \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

// mode 0: one product per K16 step; mode 1: three products per K16 step with
// collector::a fill / lastuse on the first two (the screen's pattern); mode 2:
// three plain products per K16 step
template <int N, int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
mma_probe(int steps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  __shared__ uint64_t bar, bar2, ring[3];
  __shared__ uint32_t tslot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar2)));
    for (int q = 0; q < 3; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&ring[q])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (rank == 0 && threadIdx.x == 0) {
    const uint64_t a_hi = sw128_desc(smem_u32(base)), a_lo = sw128_desc(smem_u32(base + 16384));
    const uint64_t b_hi = sw128_desc(smem_u32(base + 32768)), b_lo = sw128_desc(smem_u32(base + 49152));
    const unsigned long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      const uint64_t o = (uint64_t)(2 * (s & 3));
      if (MODE == 0) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(a_hi + o), "l"(b_hi + o), "r"(IDESC), "r"(s)
            : "memory");
      } else if (MODE == 1) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %3, %5, p;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %4, %5, 1;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, 1;\n\t}\n" ::"r"(tmem),
            "l"(a_hi + o), "l"(a_lo + o), "l"(b_hi + o), "l"(b_lo + o), "r"(IDESC), "r"(s)
            : "memory");
      } else if (MODE == 5 || MODE == 6) {
        // a ring of STG stages of 4 K16 steps (mode 5: 3 stages, mode 6: 2): before
        // reusing a stage wait for the commit of its previous use
        constexpr int STG = MODE == 5 ? 3 : 2;
        const int stage = (s >> 2) % STG;
        const int use = (s >> 2) / STG;
        if ((s & 3) == 0 && use > 0) {
          asm volatile(
              "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}\n" ::"r"(
                  smem_u32(&ring[stage])),
              "r"((uint32_t)((use - 1) & 1))
              : "memory");
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %3, %5, p;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %4, %5, 1;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, 1;\n\t}\n" ::"r"(tmem),
            "l"(a_hi + o), "l"(a_lo + o), "l"(b_hi + o), "l"(b_lo + o), "r"(IDESC), "r"(s)
            : "memory");
        if ((s & 3) == 3)
          asm volatile(
              "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                  smem_u32(&ring[stage])),
              "h"((uint16_t)0x3)
              : "memory");
      } else if (MODE >= 3) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %3, %5, p;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %4, %5, 1;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, 1;\n\t}\n" ::"r"(tmem),
            "l"(a_hi + o), "l"(a_lo + o), "l"(b_hi + o), "l"(b_lo + o), "r"(IDESC), "r"(s)
            : "memory");
        // a commit every 4 K16 steps (12 MMAs), as the screen's ring stages;
        // mode 4 multicasts it to both CTAs, mode 3 arrives in the leader only
        if ((s & 3) == 3) {
          if (MODE == 4)
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&bar2)),
                "h"((uint16_t)0x3)
                : "memory");
          else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&bar2))
                         : "memory");
        }
      } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %3, %5, p;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %4, %5, 1;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, 1;\n\t}\n" ::"r"(tmem),
            "l"(a_hi + o), "l"(a_lo + o), "l"(b_hi + o), "l"(b_lo + o), "r"(IDESC), "r"(s)
            : "memory");
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)0x3)
        : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x >> 1] = clock64() - t0;
  } else if (rank == 1 && threadIdx.x == 0) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// cta_group::1 kind::tf32, M = 128, N = NN, K = 8: A from shared memory
// (TS = 0) or from TMEM (TS = 1); three products per step into two
// accumulators as the embedding's 3xTF32 split does
template <int NN, int TS>
__global__ void __launch_bounds__(128, 1) tf32_probe(int steps, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(NN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint64_t a_hi = sw128_desc(smem_u32(base)), a_lo = sw128_desc(smem_u32(base + 16384));
    const uint64_t b_hi = sw128_desc(smem_u32(base + 32768)), b_lo = sw128_desc(smem_u32(base + 49152));
    const uint32_t dmain = tmem, dcross = tmem + NN, ta = tmem + 256;
    const unsigned long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      const uint64_t o = (uint64_t)(2 * (s & 3));
      if (TS) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %7, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %4, %6, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%1], [%2], %5, %6, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %4, %6, 1;\n\t}\n" ::"r"(dmain),
            "r"(dcross), "r"(ta + 8u * (s & 3)), "r"(ta + 32u + 8u * (s & 3)), "l"(b_hi + o), "l"(b_lo + o),
            "r"(IDESC), "r"(s)
            : "memory");
      } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %7, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %2, %4, %6, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%1], %2, %5, %6, p;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%1], %3, %4, %6, 1;\n\t}\n" ::"r"(dmain),
            "r"(dcross), "l"(a_hi + o), "l"(a_lo + o), "l"(b_hi + o), "l"(b_lo + o), "r"(IDESC), "r"(s)
            : "memory");
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile(
        "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}\n" ::"r"(
            smem_u32(&bar))
        : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

template <int NN, int TS>
static int run_tf32() {
  const int steps = 20000, grid = 148;
  unsigned long long* d;
  CK(cudaMalloc(&d, sizeof(unsigned long long) * grid));
  auto k = tf32_probe<NN, TS>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024));
  k<<<grid, 128, 66 * 1024>>>(steps, d);
  CK(cudaDeviceSynchronize());
  k<<<grid, 128, 66 * 1024>>>(steps, d);
  CK(cudaDeviceSynchronize());
  unsigned long long h[148];
  CK(cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost));
  double cyc = 0;
  for (int i = 0; i < grid; ++i) cyc += (double)h[i];
  cyc /= grid;
  std::printf("tf32 M=128 N=%3d A from %s: %6.1f cyc/MMA (floor %5.1f)\n", NN, TS ? "TMEM" : "SMEM",
              cyc / (3.0 * steps), 128.0 * NN / 256.0);
  cudaFree(d);
  return 0;
}

template <int N, int MODE>
static int run(int grid) {
  const int steps = 20000;
  unsigned long long* d;
  CK(cudaMalloc(&d, sizeof(unsigned long long) * grid));
  auto k = mma_probe<N, MODE>;
  CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024));
  k<<<grid, 128, 66 * 1024>>>(steps, d);  // warm
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<grid, 128, 66 * 1024>>>(steps, d);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  CK(cudaMemcpy(h, d, sizeof(unsigned long long) * (grid / 2), cudaMemcpyDeviceToHost));
  double cyc = 0;
  for (int i = 0; i < grid / 2; ++i) cyc += (double)h[i];
  cyc /= grid / 2;
  const int per_step = MODE == 0 ? 1 : 3;  // modes 1-4: three products per step
  const double mmas = (double)steps * per_step;
  const double flop = mmas * 2.0 * 256 * N * 16 * (grid / 2);
  std::printf("N=%3d mode=%d grid=%3d: %6.1f cyc/MMA (floor %5.1f)  %.0f TF/s  (%.3f ms)\n", N, MODE, grid,
              cyc / mmas, 256.0 * N / 512.0, flop / (ms * 1e-3) / 1e12, ms);
  cudaFree(d);
  return 0;
}

int main() {
  run_tf32<64, 0>();
  run_tf32<64, 1>();
  run_tf32<128, 0>();
  run_tf32<128, 1>();
  run_tf32<256, 0>();
  for (int grid : {2, 148}) {
    run<128, 0>(grid);
    run<160, 0>(grid);
    run<192, 0>(grid);
    run<256, 0>(grid);
    run<160, 1>(grid);
    run<160, 2>(grid);
    run<256, 1>(grid);
    run<160, 3>(grid);
    run<160, 4>(grid);
    run<160, 5>(grid);
    run<160, 6>(grid);
  }
  return 0;
}
