// Shared helpers of libkkb (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/kkb.h"

namespace kkb {

// ------------------------------------------------------------- error state
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);
void count_launch(int n = 1);

#define KKB_CHECK_LAUNCH(what)                                  \
    do {                                                        \
        ::kkb::count_launch();                                  \
        cudaError_t _e = cudaGetLastError();                    \
        if (_e != cudaSuccess) return ::kkb::cuda_status(_e, what); \
    } while (0)

#define KKB_TRY_CUDA(call, what)                                \
    do {                                                        \
        cudaError_t _e = (call);                                \
        if (_e != cudaSuccess) return ::kkb::cuda_status(_e, what); \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline long long ceil_div(long long a, long long b) { return (a + b - 1) / b; }

int sm_count();

// ------------------------------------------------------------- device math
// floor(fi) without a float->int conversion: RD(fi + 1.5*2^52) = 1.5*2^52 + floor(fi)
// exactly for |fi| < 2^51; the low word is floor(fi) (two's complement) and the
// high word is 0x43380000 iff 0 <= floor(fi) < 2^32.
#define KKB_FLOOR_MAGIC 6755399441055744.0
#define KKB_MAGIC_HI 0x43380000

// Fractional part in [0,1) as float (truncated to 23 bits) given fi and
// y = RD(fi + MAGIC).  Uses z = fi - (floor(fi) - 1) in [1, 2): its mantissa
// bits are the fraction.
__device__ __forceinline__ float frac_from_floor(double fi, double y) {
    double fl1 = __dsub_rn(y, KKB_FLOOR_MAGIC + 1.0);  // floor(fi) - 1, exact
    double z = __dsub_rd(fi, fl1);  // 1 + frac, rounded down so it stays < 2
    unsigned lo = (unsigned)__double2loint(z);
    unsigned hi = (unsigned)__double2hiint(z);
    unsigned bits = (__funnelshift_l(lo, hi, 3) & 0x007FFFFFu) | 0x3F800000u;
    return __uint_as_float(bits) - 1.0f;
}

}  // namespace kkb
