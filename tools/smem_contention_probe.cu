// smem_contention_probe.cu -- does TMA traffic into shared memory slow the
// tensor core's shared-memory operand reads?  One CTA pair per two SMs: the
// leader issues the SCREEN kernel's MMA pattern (cta_group::2, M=256, N=160,
// three f16 products per K16 step, A-collector reuse) on a fixed stage, while
// one thread per CTA streams 1-D bulk copies (L2-resident source) into a
// separate shared-memory ring, as fast as they complete.  Reports cycles per
// MMA and bulk-copy bytes per cycle per SM, with and without the copies.
// Profiling aid for the SCREEN engine, not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/smem_probe tools/smem_contention_probe.cu -lcuda
// Measured (profiles/r02_screen_limits.md): MMA at 80 cycles with none / 1-D
// bulk (62 B/cycle/SM) / 2-D boxes (37 B/cycle/SM) streaming in.
#include <cuda.h>
#include <cudaTypedefs.h>
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

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}

constexpr int RMAX = 4, SLOT = 24 * 1024;  // copy ring: 4 x 24 KB per CTA

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
contention_kernel(const __grid_constant__ CUtensorMap map, const __grid_constant__ CUtensorMap map2, int steps, int copy_on, int RING, const char* __restrict__ src,
                  long long src_bytes, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024u - (smem_u32(sm) & 1023u)) & 1023u);
  uint8_t* ring = base + 64 * 1024;
  __shared__ uint64_t done_bar, cbar[RMAX];
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done_bar)));
    for (int s = 0; s < RING; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cbar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    stop = 0;
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
  constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(160 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
  if (warp == 0 && (threadIdx.x & 31) == 0 && copy_on) {
    // bulk copies, up to RING in flight, until the MMAs are done
    unsigned long long bytes = 0, q = 0;
    long long off = ((long long)blockIdx.x * 7919 * SLOT) % (src_bytes - SLOT);
    const unsigned long long t0 = clock64();
    while (!stop) {
      const int s = (int)(q % RING);
      if (q >= RING)
        while (!try_wait(smem_u32(&cbar[s]), (uint32_t)(((q / RING) - 1) & 1))) {
        }
      const uint32_t bar = smem_u32(&cbar[s]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(SLOT) : "memory");
      if (copy_on == 1) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(ring + s * SLOT)),
                     "l"(src + off), "r"(SLOT), "r"(bar)
                     : "memory");
      } else {
        // the screen's pattern: 2-D boxes of 64 fp16 (128 B) x rows, SWIZZLE_128B:
        // a 128-row box + an 64-row box = 24 KB, rows walked over the source
        const int row = (int)((off / 128) % (src_bytes / 1024 - 192));
        const int col = (int)(q % 8) * 64;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(ring + s * SLOT)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(bar), "r"(col), "r"(row)
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                smem_u32(ring + s * SLOT) + 16384),
            "l"(reinterpret_cast<uint64_t>(&map2)), "r"(bar), "r"(col), "r"(row + 128)
            : "memory");
      }
      off += SLOT;
      if (off + SLOT > src_bytes) off = 0;
      bytes += SLOT;
      ++q;
    }
    for (unsigned long long k = (q > RING ? q - RING : 0); k < q; ++k)  // drain
      while (!try_wait(smem_u32(&cbar[k % RING]), (uint32_t)((k / RING) & 1))) {
      }
    out[2 * blockIdx.x + 1] = bytes;
    out[2 * gridDim.x + blockIdx.x] = clock64() - t0;
  }
  if (rank == 0 && threadIdx.x == 32) {
    const uint64_t a_hi = sw128_desc(smem_u32(base)), a_lo = sw128_desc(smem_u32(base + 16384));
    const uint64_t b_hi = sw128_desc(smem_u32(base + 32768)), b_lo = sw128_desc(smem_u32(base + 49152));
    const unsigned long long t0 = clock64();
    for (int s = 0; s < steps; ++s) {
      const uint64_t o = (uint64_t)(2 * (s & 3));
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %6, 0;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16.collector::a::fill [%0], %1, %3, %5, p;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16.collector::a::lastuse [%0], %1, %4, %5, 1;\n\t"
          "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %3, %5, 1;\n\t}\n" ::"r"(tmem),
          "l"(a_hi + o), "l"(a_lo + o), "l"(b_hi + o), "l"(b_lo + o), "r"(IDESC), "r"(s)
          : "memory");
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&done_bar)),
        "h"((uint16_t)0x3)
        : "memory");
    while (!try_wait(smem_u32(&done_bar), 0)) {
    }
    out[2 * blockIdx.x] = clock64() - t0;
  } else if (rank == 1 && threadIdx.x == 32) {
    while (!try_wait(smem_u32(&done_bar), 0)) {
    }
  }
  // both CTAs: stop the copier once the MMAs are done
  if (threadIdx.x == 32) stop = 1;
  __syncthreads();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

int main() {
  const int grid = 148, steps = 30000;
  const long long src_bytes = 48ll << 20;  // L2-resident source
  char* src;
  unsigned long long* out;
  CK(cudaMalloc(&src, src_bytes));
  CK(cudaMemset(src, 0, src_bytes));
  CK(cudaMalloc(&out, sizeof(unsigned long long) * 3 * grid));
  // source viewed as rows of 512 fp16 (1 KB): box 64 x 128 rows (16 KB) and 64 x 64 rows (8 KB)
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap maps[2];
  for (int m = 0; m < 2; ++m) {
    cuuint64_t dims[2] = {512, (cuuint64_t)(src_bytes / 1024)};
    cuuint64_t str[1] = {1024};
    cuuint32_t box[2] = {64, m == 0 ? 128u : 64u};
    cuuint32_t es[2] = {1, 1};
    CUresult rc = enc(&maps[m], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, src, dims, str, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rc != CUDA_SUCCESS) std::printf("encode failed %d\n", (int)rc);
  }
  const int smem = 1024 + 64 * 1024 + RMAX * SLOT;
  CK(cudaFuncSetAttribute(contention_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int rep = 0; rep < 2; ++rep)
    for (int copy_on = 0; copy_on < 3; ++copy_on) {
      const int RING = RMAX;
      CK(cudaMemset(out, 0, sizeof(unsigned long long) * 3 * grid));
      contention_kernel<<<grid, 128, smem>>>(maps[0], maps[1], steps, copy_on, RING, src, src_bytes, out);
      CK(cudaDeviceSynchronize());
      unsigned long long h[3 * 148];
      CK(cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost));
      double mma = 0, bytes = 0, cyc = 0;
      int np = 0, nc = 0;
      for (int i = 0; i < grid; ++i) {
        if (h[2 * i]) mma += (double)h[2 * i], ++np;
        if (h[2 * i + 1]) bytes += (double)h[2 * i + 1], cyc += (double)h[2 * grid + i], ++nc;
      }
      const char* nm[3] = {"none", "1-D bulk", "2-D boxes"};
      std::printf("copies %-9s: %.1f cycles per MMA (floor 80)%s", nm[copy_on], mma / np / (3.0 * steps),
                  copy_on ? "" : "\n");
      if (copy_on) std::printf(", %.1f B/cycle/SM into shared memory\n", bytes / cyc);
    }
  return 0;
}
