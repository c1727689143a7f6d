// Compile-time Stockham FFT building blocks shared by K1 / K3 (fft_ct.cu) and
// the fused stage-1 kernel (stage1_fused.cu): radix butterflies with
// compile-time twiddles, the per-length plans, one Stockham stage in
// registers, and stages 1-2 of a plan through one shared buffer.
#pragma once

#include "common.cuh"

namespace kkb {
namespace ct {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }

// compile-time exp(-2 pi i m / N), evaluated in double (Taylor series on the
// angle reduced to [-pi, pi]) and rounded once to float
__host__ __device__ constexpr double cx_cos(double x) {
    double term = 1.0, sum = 1.0;
    for (int n = 1; n < 40; ++n) {
        term *= -x * x / ((2.0 * n - 1.0) * (2.0 * n));
        sum += term;
    }
    return sum;
}
__host__ __device__ constexpr double cx_sin(double x) {
    double term = x, sum = x;
    for (int n = 1; n < 40; ++n) {
        term *= -x * x / ((2.0 * n) * (2.0 * n + 1.0));
        sum += term;
    }
    return sum;
}
template <int N>
struct TwTab {
    float re[N], im[N];
    __host__ __device__ constexpr TwTab() : re(), im() {
        constexpr double pi = 3.14159265358979323846;
        for (int m = 0; m < N; ++m) {
            double a = 2.0 * pi * (double)m / (double)N;  // [0, 2 pi)
            if (a > pi) a -= 2.0 * pi;
            re[m] = (float)cx_cos(a);
            im[m] = (float)(-cx_sin(a));
        }
    }
};

// x * exp(-2 pi i m / N) with m a compile-time constant after unrolling
template <int N>
__device__ __forceinline__ float2 twc(float2 x, int m) {
    constexpr TwTab<N> tab{};
    m %= N;
    if (m == 0) return x;
    if (4 * m == N) return mul_mi(x);
    if (2 * m == N) return make_float2(-x.x, -x.y);
    if (4 * m == 3 * N) return make_float2(-x.y, x.x);
    return cmul(x, make_float2(tab.re[m], tab.im[m]));
}

template <int R>
struct Dft;

template <>
struct Dft<2> {
    __device__ __forceinline__ static void run(float2 *v) {
        float2 t = v[0];
        v[0] = cadd(t, v[1]);
        v[1] = csub(t, v[1]);
    }
};
template <>
struct Dft<3> {
    __device__ __forceinline__ static void run(float2 *v) {
        const float s = 0.86602540378443864676f;
        float2 t1 = cadd(v[1], v[2]);
        float2 t2 = make_float2(fmaf(-0.5f, t1.x, v[0].x), fmaf(-0.5f, t1.y, v[0].y));
        float2 t3 = csub(v[1], v[2]);
        float2 t4 = make_float2(s * t3.y, -s * t3.x);
        v[0] = cadd(v[0], t1);
        v[1] = cadd(t2, t4);
        v[2] = csub(t2, t4);
    }
};
template <>
struct Dft<4> {
    __device__ __forceinline__ static void run(float2 *v) {
        float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
        float2 a2 = cadd(v[1], v[3]), a3 = mul_mi(csub(v[1], v[3]));
        v[0] = cadd(a0, a2);
        v[2] = csub(a0, a2);
        v[1] = cadd(a1, a3);
        v[3] = csub(a1, a3);
    }
};
template <>
struct Dft<8> {
    __device__ __forceinline__ static void run(float2 *v) {
        const float r = 0.70710678118654752440f;
        float2 e[4] = {v[0], v[2], v[4], v[6]};
        float2 o[4] = {v[1], v[3], v[5], v[7]};
        Dft<4>::run(e);
        Dft<4>::run(o);
        o[1] = make_float2(r * (o[1].x + o[1].y), r * (o[1].y - o[1].x));
        o[2] = mul_mi(o[2]);
        o[3] = make_float2(r * (o[3].y - o[3].x), -r * (o[3].x + o[3].y));
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            v[k] = cadd(e[k], o[k]);
            v[k + 4] = csub(e[k], o[k]);
        }
    }
};
// composite N = N1 x N2 (Cooley-Tukey, n = N2 n1 + n2, k = k1 + N1 k2)
template <int N1, int N2>
struct DftComp {
    __device__ __forceinline__ static void run(float2 *v) {
        constexpr int N = N1 * N2;
        float2 a[N2][N1];
#pragma unroll
        for (int n2 = 0; n2 < N2; ++n2) {
#pragma unroll
            for (int n1 = 0; n1 < N1; ++n1) a[n2][n1] = v[N2 * n1 + n2];
            Dft<N1>::run(a[n2]);
#pragma unroll
            for (int k1 = 0; k1 < N1; ++k1) a[n2][k1] = twc<N>(a[n2][k1], n2 * k1);
        }
#pragma unroll
        for (int k1 = 0; k1 < N1; ++k1) {
            float2 t[N2];
#pragma unroll
            for (int n2 = 0; n2 < N2; ++n2) t[n2] = a[n2][k1];
            Dft<N2>::run(t);
#pragma unroll
            for (int k2 = 0; k2 < N2; ++k2) v[k1 + N1 * k2] = t[k2];
        }
    }
};
template <>
struct Dft<6> : DftComp<2, 3> {};
template <>
struct Dft<12> : DftComp<4, 3> {};
template <>
struct Dft<16> : DftComp<4, 4> {};

template <int T>
struct Plan;
template <>
struct Plan<1024> { static constexpr int NT = 64, R0 = 16, R1 = 8, R2 = 8, R3 = 1; };
template <>
#ifndef KKB_FFT1536_NT
#define KKB_FFT1536_NT 128
#endif
struct Plan<1536> { static constexpr int NT = KKB_FFT1536_NT, R0 = 16, R1 = 12, R2 = 8, R3 = 1; };
template <>
struct Plan<2048> { static constexpr int NT = 128, R0 = 16, R1 = 16, R2 = 8, R3 = 1; };
template <>
struct Plan<4096> { static constexpr int NT = 256, R0 = 16, R1 = 16, R2 = 16, R3 = 1; };

// registers of one stage: lane j handles butterflies j, j + NT, ... (< T/R);
// butterfly j reads inputs j + r T/R and writes outputs base + r NS,
// base = (j - j % NS) R + j % NS (Stockham, natural order after the last stage)
template <int T, int NT, int R>
struct Stage {
    static constexpr int TR = T / R;
    static constexpr int ITER = (TR + NT - 1) / NT;
    float2 v[ITER][R];

    // NT is a power of two; a CTA may run several transforms side by side
    // (k_c2c_planes: threads [i NT, (i + 1) NT) take transform i)
    __device__ __forceinline__ static int lane_j(int t) { return (int)(threadIdx.x & (NT - 1)) + t * NT; }
    __device__ __forceinline__ static bool ok(int j) { return TR % NT == 0 || j < TR; }
    __device__ __forceinline__ static int swz(int e) { return e ^ ((e >> 4) & 15); }

    template <bool SW>
    __device__ __forceinline__ void load(const float2 *buf) {
#pragma unroll
        for (int t = 0; t < ITER; ++t) {
            const int j = lane_j(t);
            if (ok(j)) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[t][r] = buf[SW ? swz(j + r * TR) : j + r * TR];
            }
        }
    }
    // twiddles from the stage-ordered table (entry OFF + (r-1) NS + k), then DFT_R
    template <int NS, int OFF>
    __device__ __forceinline__ void compute(const float2 *__restrict__ tw) {
#pragma unroll
        for (int t = 0; t < ITER; ++t) {
            const int j = lane_j(t);
            if (ok(j)) {
                if (NS > 1) {
                    const int k = j % NS;
#pragma unroll
                    for (int r = 1; r < R; ++r)
                        v[t][r] = cmul(v[t][r], __ldg(tw + OFF + (r - 1) * NS + k));
                }
                Dft<R>::run(v[t]);
            }
        }
    }
    template <int NS, bool SW>
    __device__ __forceinline__ void store(float2 *buf) const {
#pragma unroll
        for (int t = 0; t < ITER; ++t) {
            const int j = lane_j(t);
            if (ok(j)) {
                const int k = j % NS;
                const int base = (j - k) * R + k;
#pragma unroll
                for (int r = 0; r < R; ++r) buf[SW ? swz(base + r * NS) : base + r * NS] = v[t][r];
            }
        }
    }
};

// barrier of one transform's NT threads: the CTA-wide __syncthreads (BAR 0)
// for one transform per CTA, named barrier 1 + i for transform i of several
template <int NT>
__device__ __forceinline__ void xform_sync(int bar) {
    if (bar == 0)
        __syncthreads();
    else
        asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(NT) : "memory");
}

// stages 1 and 2 of the plan on `buf` holding stage 0's swizzled output;
// returns with stage 2's outputs (bins j + r T/R2) in `c`
template <int T, typename S2>
__device__ __forceinline__ void stages12(float2 *buf, const float2 *__restrict__ tw, S2 &c, int bar = 0) {
    using P = Plan<T>;
    Stage<T, P::NT, P::R1> b;
    b.template load<true>(buf);
    xform_sync<P::NT>(bar);
    b.template compute<P::R0, 0>(tw);
    b.template store<P::R0, false>(buf);
    xform_sync<P::NT>(bar);
    c.template load<false>(buf);
    c.template compute<P::R0 * P::R1, (P::R1 - 1) * P::R0>(tw);
}

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(short x) { return (float)x; }  // exact

}  // namespace ct
}  // namespace kkb
