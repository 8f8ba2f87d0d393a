// adg_prep.cuh -- one row of the SCREEN engine's operand prep
// (prep_vec_kernel, adg_screen.cu), as a device function any kernel can run
// on its rows with bit-identical planes and metadata (a fused embed + prep
// kernel was built on it and measured: profiles/r02_embed_prep_fusion.md).
//
// One warp per row: centre by the screen's shift (fp32, staged in shared
// memory by the caller), scale by the power of two that puts the row max in
// [2^14, 2^15), split into fp16 hi + lo, and the squared norm of the
// represented row in fp64 -- the original side vectorised (a lane owns 4
// consecutive columns per step; its slice stays in registers between the max
// and the split), the embedded side scalar.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstdint>
#include <type_traits>

namespace adg {

__device__ __forceinline__ void note_lo(bool nonzero, int* lo_flag) {
  if (__any_sync(0xffffffffu, nonzero) && (threadIdx.x & 31) == 0 &&
      *reinterpret_cast<volatile int*>(lo_flag) == 0)
    atomicOr(lo_flag, 1);
}
__device__ __forceinline__ bool half_nonzero(__half h) { return (__half_as_ushort(h) & 0x7fffu) != 0; }

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) {
  if constexpr (std::is_same<T, float>::value)
    return __ldg(p);
  else
    return __bfloat162float(*p);
}

template <typename T>
__device__ __forceinline__ float4 ld4(const T* p) {
  if constexpr (std::is_same<T, float>::value) {
    return __ldg(reinterpret_cast<const float4*>(p));
  } else {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    return make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                       __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
  }
}

// Row `row` of the planes ([rows][ktot]: original at [0, d) padded to kp,
// embedded at [kp, kp + r) padded to ktot) from xrow (d values) and yrow (r
// values); rows past n (xrow == nullptr) are zero.  msx4: the shift as float4
// (d padded to 4), msy: r floats.  Returns whether an original-side lo entry
// is non-zero (for ScreenParams::lo_flag).
template <typename TO, typename TE, int NV>
__device__ __forceinline__ bool prep_row(const TO* __restrict__ xrow, const TE* __restrict__ yrow,
                                         int64_t d, int64_t r, int64_t kp, int64_t ktot,
                                         const float4* __restrict__ msx4, const float* __restrict__ msy,
                                         __half* __restrict__ hrow, __half* __restrict__ lrow,
                                         float4* __restrict__ meta_row, int lane) {
  if (xrow == nullptr) {
    for (int64_t t = lane; t < ktot / 4; t += 32) {
      reinterpret_cast<uint2*>(hrow)[t] = make_uint2(0u, 0u);
      reinterpret_cast<uint2*>(lrow)[t] = make_uint2(0u, 0u);
    }
    if (lane == 0) *meta_row = make_float4(0.f, 0.f, 0.f, 0.f);
    return false;
  }
  float4 m4;
  bool lnz = false;
  {  // original side, vectorised
    const int64_t d4 = d / 4, kp4 = kp / 4;
    float4 v[NV];
    float amax = 0.0f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t t = lane + 32 * i;
      v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (t < d4) {
        const float4 x = ld4(xrow + 4 * t);
        const float4 m = msx4[t];
        v[i] = make_float4(x.x - m.x, x.y - m.y, x.z - m.z, x.w - m.w);
        amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v[i].x), fabsf(v[i].y)), fmaxf(fabsf(v[i].z), fabsf(v[i].w))));
      }
    }
    for (int s = 16; s; s >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, s));
    int ex = 0;
    if (amax > 0.0f) frexpf(amax, &ex);
    const int e = amax > 0.0f ? 15 - ex : 0;
    const float scale = ldexpf(1.0f, e);
    double nrm = 0.0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int64_t t = lane + 32 * i;
      if (t < kp4) {
        const float sv[4] = {v[i].x * scale, v[i].y * scale, v[i].z * scale, v[i].w * scale};
        __half h[4], l[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          h[c] = __float2half_rn(sv[c]);
          l[c] = __float2half_rn(sv[c] - __half2float(h[c]));
          lnz = lnz || half_nonzero(l[c]);
          const double rep = (double)(__half2float(h[c]) + __half2float(l[c]));
          nrm = fma(rep, rep, nrm);
        }
        reinterpret_cast<uint2*>(hrow)[t] =
            make_uint2(__half_as_ushort(h[0]) | ((uint32_t)__half_as_ushort(h[1]) << 16),
                       __half_as_ushort(h[2]) | ((uint32_t)__half_as_ushort(h[3]) << 16));
        reinterpret_cast<uint2*>(lrow)[t] =
            make_uint2(__half_as_ushort(l[0]) | ((uint32_t)__half_as_ushort(l[1]) << 16),
                       __half_as_ushort(l[2]) | ((uint32_t)__half_as_ushort(l[3]) << 16));
      }
    }
    for (int s = 16; s; s >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, s);
    const double inv = ldexp(1.0, -e);
    m4.x = (float)(nrm * inv * inv);
    m4.z = (float)inv;
  }
  {  // embedded side, scalar
    float amax = 0.0f;
    for (int64_t t = lane; t < r; t += 32) amax = fmaxf(amax, fabsf(ld_f(yrow + t) - msy[t]));
    for (int s = 16; s; s >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, s));
    int ex = 0;
    if (amax > 0.0f) frexpf(amax, &ex);
    const int e = amax > 0.0f ? 15 - ex : 0;
    const float scale = ldexpf(1.0f, e);
    double nrm = 0.0;
    for (int64_t t = lane; t < ktot - kp; t += 32) {
      const float vv = t < r ? ld_f(yrow + t) - msy[t] : 0.0f;
      const float sv = vv * scale;
      const __half h = __float2half_rn(sv);
      const __half l = __float2half_rn(sv - __half2float(h));
      hrow[kp + t] = h;
      lrow[kp + t] = l;
      const double rep = (double)(__half2float(h) + __half2float(l));
      nrm = fma(rep, rep, nrm);
    }
    for (int s = 16; s; s >>= 1) nrm += __shfl_xor_sync(0xffffffffu, nrm, s);
    const double inv = ldexp(1.0, -e);
    m4.y = (float)(nrm * inv * inv);
    m4.w = (float)inv;
  }
  if (lane == 0) *meta_row = m4;
  return lnz;
}

}  // namespace adg
