// The tensor-core gather's trace format (kk_gather_tc.cu): every trace sample
// x of frame f scaled by a power of two s_f and split into two fp16 halves,
// x s_f = hi + lo, stored as four planes (re hi, im hi, re lo, im lo) laid out
// [plane][frame group of 8][pair][sample][8 frames] — a sample of 8 frames is
// one 16-byte row, so a pair's window for 64 frames is a single TMA box.
// s_f = 2^(14 - floor(log2 m_f)) for a bound m_f >= max |x| over the frame
// (its exact maximum, or an upper bound): |x s_f| < 2^15 fits fp16.
#pragma once

#include <cuda_fp16.h>

namespace kkb {

__device__ __forceinline__ float frame_scale(unsigned maxbits) {
    if (maxbits == 0u) return 1.0f;
    const int e = (int)((maxbits >> 23) & 0xff) - 127;
    const int s = min(max(14 - e, -120), 120);
    return __uint_as_float((unsigned)(127 + s) << 23);
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

__device__ __forceinline__ void split_h(float x, __half &hi, __half &lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}

// split_h of (a, b) with packed conversions (two F2FP instead of four F2F):
// hi = pack_h2(hi(a), hi(b)), lo = pack_h2(lo(a), lo(b)), bit for bit
__device__ __forceinline__ void split_h2(float a, float b, uint32_t &hi, uint32_t &lo) {
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = pack_h2(__low2half(h), __high2half(h));
    lo = pack_h2(__low2half(l), __high2half(l));
}

}  // namespace kkb
