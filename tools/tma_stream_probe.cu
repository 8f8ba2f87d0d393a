// tma_stream_probe.cu -- how fast can one persistent CTA per SM stream the C3
// cloud (60000 x 784 fp32) into shared memory, per access pattern?  No math:
// the consumer releases each stage as soon as it lands.  Profiling aid for
// the embedding kernel (adg_embed.cu), not product code.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_probe tools/tma_stream_probe.cu
//   /tmp/tma_probe
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdint>
#include <vector>

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
__device__ __forceinline__ void wait_bar(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

// mode 0: box (32 fp32) x BR rows, tiles of 128 rows strided over the grid, K chunks inner
// mode 1: same, but each CTA owns a contiguous balanced row range (boxes of BR rows)
// mode 2: 1-D bulk copies of CH contiguous bytes, CTA owns a contiguous byte range
// extra W: + wbytes per stage from a small L2-resident buffer (2-D box 32 x 64, two of them)
struct Args {
  int mode, stages, br, d, n, wboxes;
  long long chunk;
};

__global__ void __launch_bounds__(64, 1) probe_kernel(const __grid_constant__ CUtensorMap xmap,
                                                      const __grid_constant__ CUtensorMap wmap,
                                                      const char* __restrict__ xraw, Args a,
                                                      unsigned long long* sink) {
  extern __shared__ unsigned char raw[];
  unsigned char* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  const int S = a.stages;
  const int XB = (a.mode == 2) ? (int)a.chunk : 128 * 128;  // bytes of X per stage
  const int WB = a.wboxes * 8192;
  const int STAGE = XB + WB;
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * STAGE);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nk = (a.d + 31) / 32;
  // build the work list: (row0, rows, kc) per stage
  long long units = 0;
  long long r_begin = 0, r_end = 0;
  if (a.mode == 0) {
    const long long tiles = (a.n + 127) / 128;
    units = 0;
    for (long long t = blockIdx.x; t < tiles; t += gridDim.x) units += nk;
  } else if (a.mode == 1) {
    r_begin = (long long)a.n * blockIdx.x / gridDim.x;
    r_end = (long long)a.n * (blockIdx.x + 1) / gridDim.x;
    units = ((r_end - r_begin + 127) / 128) * nk;
  } else {
    const long long total = (long long)a.n * a.d * 4;
    r_begin = (total * blockIdx.x / gridDim.x) & ~15LL;
    r_end = blockIdx.x + 1 == gridDim.x ? total : ((total * (blockIdx.x + 1) / gridDim.x) & ~15LL);
    units = (r_end - r_begin + a.chunk - 1) / a.chunk;
  }
  if (warp == 0) {
    if (lane == 0) {
      const long long tiles = (a.n + 127) / 128;
      long long t = blockIdx.x;
      int kc = 0;
      long long tile_row = r_begin;
      for (long long q = 0; q < units; ++q) {
        const int s = (int)(q % S);
        wait_bar(smem_u32(&empty[s]), (uint32_t)(((q / S) & 1) ^ 1));
        const uint32_t bar = smem_u32(&full[s]);
        const uint32_t dst = smem_u32(base + s * STAGE);
        uint32_t bytes = WB;
        if (a.mode == 0 || a.mode == 1) {
          long long row0 = a.mode == 0 ? t * 128 : tile_row;
          long long rows = a.mode == 0 ? 128 : (r_end - tile_row < 128 ? r_end - tile_row : 128);
          int boxes = (int)((rows + a.br - 1) / a.br);
          bytes += (uint32_t)(boxes * a.br * 128);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                       : "memory");
          for (int b = 0; b < boxes; ++b)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst + b * a.br * 128),
                "l"(reinterpret_cast<uint64_t>(&xmap)), "r"(bar), "r"(kc * 32), "r"((int)(row0 + b * a.br))
                : "memory");
          if (++kc == nk) {
            kc = 0;
            if (a.mode == 0) {
              t += gridDim.x;
            } else {
              tile_row += 128;
            }
          }
          (void)tiles;
        } else {
          const long long off = r_begin + q * a.chunk;
          long long len = r_end - off < a.chunk ? r_end - off : a.chunk;
          len &= ~15LL;
          bytes += (uint32_t)len;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                       : "memory");
          if (len)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dst),
                "l"(xraw + off), "r"((uint32_t)len), "r"(bar)
                : "memory");
        }
        for (int w = 0; w < a.wboxes; ++w)
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst + XB + w * 8192),
              "l"(reinterpret_cast<uint64_t>(&wmap)), "r"(bar), "r"((int)((q % nk) * 32)), "r"(w * 64)
              : "memory");
      }
    }
  } else {
    unsigned long long acc = 0;
    for (long long q = 0; q < units; ++q) {
      const int s = (int)(q % S);
      wait_bar(smem_u32(&full[s]), (uint32_t)((q / S) & 1));
      acc += base[s * STAGE + lane * 4];
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    }
    if (lane == 0 && acc == 0xFFFFFFFFFFFFull) *sink = acc;
  }
}


// mode 3: plain LDG.128 grid-stride stream (U loads in flight per thread)
template <int U>
__global__ void ldg_stream_kernel(const float4* __restrict__ X, long long n4, unsigned long long* sink) {
  float acc = 0.f;
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(X + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) {
    float4 v = __ldcs(X + i);
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 123.f) *sink = 1;
}

// mode 4: the embedding's tile pattern with LDG: 128-row tiles strided over
// the grid, K chunks of 32 floats (128 B per row); each warp loads 16 rows x
// 128 B per chunk (4 LDG.128 per lane), D chunks in flight per thread.
template <int D>
__global__ void __launch_bounds__(256, 1) ldg_tile_kernel(const float* __restrict__ X, int n, int d,
                                                          unsigned long long* sink) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nk = d / 32;
  const int tiles = (n + 127) / 128;
  float acc = 0.f;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int row0 = t * 128 + warp * 16 + lane / 8;
    const int col = (lane % 8) * 4;
    for (int kc = 0; kc < nk; kc += D) {
      float4 v[D][4];
#pragma unroll
      for (int dd = 0; dd < D; ++dd)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int row = row0 + 4 * q;
          v[dd][q] = (kc + dd < nk && row < n)
                         ? __ldcs(reinterpret_cast<const float4*>(X + (long long)row * d + (kc + dd) * 32 + col))
                         : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
      for (int dd = 0; dd < D; ++dd)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc += v[dd][q].x + v[dd][q].y + v[dd][q].z + v[dd][q].w;
    }
  }
  if (acc == 123.f) *sink = 1;
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
}

static CUtensorMap map2d(const void* p, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t str[1] = {inner * 4};
  cuuint32_t box[2] = {bi, bo};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = enc()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(p), dims, str, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) std::printf("encode failed %d\n", (int)rc);
  return m;
}

int main() {
  const int n = 60000, d = 784;
  float *X, *W;
  void* flush;
  unsigned long long* sink;
  CK(cudaMalloc(&X, (size_t)n * d * 4));
  CK(cudaMalloc(&W, (size_t)128 * 800 * 4));
  CK(cudaMalloc(&flush, 512u << 20));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemset(X, 1, (size_t)n * d * 4));
  CK(cudaMemset(W, 0, (size_t)128 * 800 * 4));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  CK(cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = (double)n * d * 4;
  struct Cfg {
    int mode, stages, br, wboxes;
    long long chunk;
    int grid_mult;
  };
  std::vector<Cfg> cfgs = {
      {0, 4, 128, 2, 0, 1}, {0, 4, 128, 0, 0, 1}, {0, 8, 128, 0, 0, 1}, {0, 12, 128, 0, 0, 1},
      {0, 8, 32, 0, 0, 1},  {1, 4, 128, 0, 0, 1}, {1, 8, 128, 0, 0, 1}, {1, 12, 128, 0, 0, 1},
      {1, 8, 32, 0, 0, 1},  {1, 12, 32, 0, 0, 1}, {1, 8, 32, 2, 0, 1},  {1, 6, 32, 2, 0, 1},
      {2, 4, 0, 0, 16384, 1}, {2, 8, 0, 0, 16384, 1}, {2, 12, 0, 0, 16384, 1}, {2, 6, 0, 0, 32768, 1},
      {2, 16, 0, 0, 8192, 1}, {2, 24, 0, 0, 8192, 1}, {2, 8, 0, 2, 8192, 1}, {2, 6, 0, 2, 16384, 1},
      {2, 4, 0, 0, 32768, 1}, {2, 3, 0, 0, 65536, 1},
  };
  CUtensorMap wmap = map2d(W, 800, 128, 32, 64);
  for (auto c : cfgs) {
    CUtensorMap xmap = map2d(X, d, n, 32, c.mode == 2 ? 128 : c.br);
    Args a{c.mode, c.stages, c.br, d, n, c.wboxes, c.chunk};
    const int XB = c.mode == 2 ? (int)c.chunk : 128 * 128;
    const int smem = 1024 + c.stages * (XB + c.wboxes * 8192) + 2 * c.stages * 8;
    if (smem > 227 * 1024) {
      std::printf("skip (smem)\n");
      continue;
    }
    const int grid = sms * c.grid_mult;
    float best = 1e30f, tot = 0.f;
    const int reps = 10;
    for (int r = 0; r < reps + 2; ++r) {
      cudaMemsetAsync(flush, r, 512u << 20);
      cudaEventRecord(e0);
      probe_kernel<<<grid, 64, smem>>>(xmap, wmap, (const char*)X, a, sink);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) {
        tot += ms;
        if (ms < best) best = ms;
      }
    }
    CK(cudaGetLastError());
    const float avg = tot / reps;
    std::printf("mode %d stages %2d box_rows %3d wboxes %d chunk %6lld : avg %.4f ms (%.0f GB/s X)  best %.4f ms\n",
                c.mode, c.stages, c.br, c.wboxes, c.chunk, avg, bytes / (avg * 1e6), best);
  }

  auto timeit = [&](auto launch, const char* name) {
    float tot = 0.f;
    for (int r = 0; r < 12; ++r) {
      cudaMemsetAsync(flush, r, 512u << 20);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2) tot += ms;
    }
    const float avg = tot / 10;
    std::printf("%-44s: avg %.4f ms (%.0f GB/s X)  err=%s\n", name, avg, bytes / (avg * 1e6),
                cudaGetErrorString(cudaGetLastError()));
  };
  const long long n4 = (long long)n * d / 4;
  for (int bpsm : {1, 2, 4, 8}) {
    char nm[96];
    std::snprintf(nm, sizeof nm, "ldg stream U=4 256thr x %d/SM", bpsm);
    timeit([&] { ldg_stream_kernel<4><<<sms * bpsm, 256>>>((const float4*)X, n4, sink); }, nm);
    std::snprintf(nm, sizeof nm, "ldg stream U=8 256thr x %d/SM", bpsm);
    timeit([&] { ldg_stream_kernel<8><<<sms * bpsm, 256>>>((const float4*)X, n4, sink); }, nm);
  }
  timeit([&] { ldg_tile_kernel<1><<<sms, 256>>>(X, n, d, sink); }, "ldg tile D=1 (16 KB/CTA in flight)");
  timeit([&] { ldg_tile_kernel<2><<<sms, 256>>>(X, n, d, sink); }, "ldg tile D=2");
  timeit([&] { ldg_tile_kernel<4><<<sms, 256>>>(X, n, d, sink); }, "ldg tile D=4");
  timeit([&] { ldg_tile_kernel<7><<<sms, 256>>>(X, n, d, sink); }, "ldg tile D=7");
  timeit([&] { ldg_tile_kernel<4><<<sms * 2, 256>>>(X, n, d, sink); }, "ldg tile D=4, 2 CTA/SM");
  return 0;
}
