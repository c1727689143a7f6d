// K1 / K3 specialised for the trace lengths of the five workloads
// (T = 1024, 1536, 2048, 4096): the radix plan, thread count and every index
// are compile-time constants, so the Stockham stages are straight-line code.
//
// One CTA = one complex transform of length T (two real traces packed as
// re/im for the forward real FFT).  The transform lives in ONE shared buffer;
// each stage reads all of a thread's butterfly inputs into registers, barriers,
// then writes the outputs in place (no ping-pong buffer: 8 B x T of shared
// memory per CTA, so many CTAs per SM overlap their global loads with other
// CTAs' arithmetic).  Stages whose output stride Ns < 16 would hit the same
// shared-memory banks from neighbouring lanes write through an XOR swizzle
// (index ^ ((index >> 3) & 15)), which the next stage reads back.
// Twiddles exp(-2 pi i k / T): float64-accurate table in global memory (L1).
//
// Measured (r1, config 4): a persistent cp.async-pipelined variant of the
// real FFT was 22% slower than one CTA per pair (register cap -> fewer
// resident CTAs), and a multi-pair CTA with cp.async double-buffered input
// staging was 53% slower (237 registers uncapped; 64 capped -> 512 B spills),
// so the simple form is the one kept.

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"

namespace kkb {
namespace ct {

__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(fmaf(a.x, b.x, -a.y * b.y), fmaf(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }

template <int R>
__device__ __forceinline__ void dft(float2 *v);

template <>
__device__ __forceinline__ void dft<2>(float2 *v) {
    float2 t = v[0];
    v[0] = cadd(t, v[1]);
    v[1] = csub(t, v[1]);
}
template <>
__device__ __forceinline__ void dft<4>(float2 *v) {
    float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    float2 a2 = cadd(v[1], v[3]), a3 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(a0, a2);
    v[2] = csub(a0, a2);
    v[1] = cadd(a1, a3);
    v[3] = csub(a1, a3);
}
template <>
__device__ __forceinline__ void dft<8>(float2 *v) {
    const float r = 0.70710678118654752440f;
    float2 e[4] = {v[0], v[2], v[4], v[6]};
    float2 o[4] = {v[1], v[3], v[5], v[7]};
    dft<4>(e);
    dft<4>(o);
    o[1] = make_float2(r * (o[1].x + o[1].y), r * (o[1].y - o[1].x));
    o[2] = mul_mi(o[2]);
    o[3] = make_float2(r * (o[3].y - o[3].x), -r * (o[3].x + o[3].y));
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[k] = cadd(e[k], o[k]);
        v[k + 4] = csub(e[k], o[k]);
    }
}
template <>
__device__ __forceinline__ void dft<3>(float2 *v) {
    const float s = 0.86602540378443864676f;
    float2 t1 = cadd(v[1], v[2]);
    float2 t2 = make_float2(fmaf(-0.5f, t1.x, v[0].x), fmaf(-0.5f, t1.y, v[0].y));
    float2 t3 = csub(v[1], v[2]);
    float2 t4 = make_float2(s * t3.y, -s * t3.x);
    v[0] = cadd(v[0], t1);
    v[1] = cadd(t2, t4);
    v[2] = csub(t2, t4);
}

template <bool SW>
__device__ __forceinline__ int swz(int e) {
    return SW ? (e ^ ((e >> 3) & 15)) : e;
}

// One Stockham stage, in place: radix R, input sub-transform length NS.
// Twiddles come from the stage-ordered table (see stage_twiddles): entry
// OFF + (r-1)*NS + k = exp(-2 pi i r k / (NS R)), so the lanes of a warp read
// consecutive k for each r (two 128 B wavefronts) instead of r*k-strided
// entries of a length-T table (up to 32 wavefronts per load).
template <int T, int NT, int R, int NS, int OFF, bool SW_IN, bool SW_OUT>
__device__ __forceinline__ void stage(float2 *buf, const float2 *__restrict__ tw) {
    constexpr int TR = T / R;
    constexpr int ITER = (TR + NT - 1) / NT;
    float2 v[ITER][R];
#pragma unroll
    for (int t = 0; t < ITER; ++t) {
        const int j = threadIdx.x + t * NT;
        if (TR % NT == 0 || j < TR) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[t][r] = buf[swz<SW_IN>(j + r * TR)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < ITER; ++t) {
        const int j = threadIdx.x + t * NT;
        if (TR % NT == 0 || j < TR) {
            const int k = j % NS;
            if (NS > 1) {
#pragma unroll
                for (int r = 1; r < R; ++r) v[t][r] = cmul(v[t][r], __ldg(tw + OFF + (r - 1) * NS + k));
            }
            dft<R>(v[t]);
            const int base = (j - k) * R + k;
#pragma unroll
            for (int r = 0; r < R; ++r) buf[swz<SW_OUT>(base + r * NS)] = v[t][r];
        }
    }
    __syncthreads();
}

// Full transform: radices R0..R3 (R3 == 1: three stages).  Output natural order.
template <int T, int NT, int R0, int R1, int R2, int R3>
__device__ __forceinline__ void fft(float2 *buf, const float2 *__restrict__ tw) {
    constexpr int N1 = R0, N2 = R0 * R1, N3 = R0 * R1 * R2;
    constexpr int O2 = (R1 - 1) * N1, O3 = O2 + (R2 - 1) * N2;
    static_assert(R0 * R1 * R2 * R3 == T, "radix plan must multiply to T");
    // stage s writes at stride NS_s: swizzle its output when NS_s < 16
    stage<T, NT, R0, 1, 0, false, true>(buf, tw);
    stage<T, NT, R1, N1, 0, true, (N1 < 16)>(buf, tw);
    if constexpr (R3 == 1) {
        static_assert(N2 >= 16, "last stage must write in natural order");
        stage<T, NT, R2, N2, O2, (N1 < 16), false>(buf, tw);
    } else {
        stage<T, NT, R2, N2, O2, (N1 < 16), (N2 < 16)>(buf, tw);
        static_assert(N3 >= 16, "last stage must write in natural order");
        stage<T, NT, R3, N3, O3, (N2 < 16), false>(buf, tw);
    }
}

template <int T>
struct Plan;
template <>
struct Plan<1024> { static constexpr int NT = 64, R0 = 8, R1 = 8, R2 = 4, R3 = 4; };
template <>
struct Plan<1536> {
#ifndef KKB_FFT1536_NT
#define KKB_FFT1536_NT 128  // measured: 128 threads beat 64 / 192 (fewer registers, more CTAs)
#endif
    static constexpr int NT = KKB_FFT1536_NT, R0 = 8, R1 = 8, R2 = 8, R3 = 3;
};
template <>
struct Plan<2048> { static constexpr int NT = 128, R0 = 8, R1 = 8, R2 = 8, R3 = 4; };
template <>
struct Plan<4096> { static constexpr int NT = 192, R0 = 8, R1 = 8, R2 = 8, R3 = 8; };

template <int T>
__device__ __forceinline__ void run_fft(float2 *buf, const float2 *tw) {
    using P = Plan<T>;
    fft<T, P::NT, P::R0, P::R1, P::R2, P::R3>(buf, tw);
}

// four consecutive samples as float (float32 rows: one 16 B load; int16 rows:
// one 8 B load, converted exactly — the reference consumes q.astype(float32))
__device__ __forceinline__ float4 load4(const float *p) { return __ldg(reinterpret_cast<const float4 *>(p)); }
__device__ __forceinline__ float4 load4(const short *p) {
    const int2 u = __ldg(reinterpret_cast<const int2 *>(p));
    return make_float4((float)(short)(u.x & 0xFFFF), (float)(short)(u.x >> 16),
                       (float)(short)(u.y & 0xFFFF), (float)(short)(u.y >> 16));
}

// Real-pair forward FFT: rows 2p, 2p+1 of `in` (length T) -> bins [0, K) of
// each row's spectrum at out + row*out_stride, times bin_scale[k].
template <int T, typename InT>
__global__ void __launch_bounds__(Plan<T>::NT)
k_r2c(const InT *__restrict__ in, long long ntraces, float2 *__restrict__ out,
      long long out_stride, int K, const float *__restrict__ bin_scale,
      const float2 *__restrict__ tw) {
    constexpr int NT = Plan<T>::NT;
    __shared__ __align__(16) float2 buf[T];
    const long long r0 = 2 * (long long)blockIdx.x;
    const bool l1 = r0 + 1 < ntraces;
    const InT *x0 = in + r0 * T;
    const InT *x1 = in + (l1 ? r0 + 1 : r0) * T;
#pragma unroll
    for (int i = threadIdx.x; i < T / 4; i += NT) {
        const float4 u = load4(x0 + 4 * i);
        float4 w = load4(x1 + 4 * i);
        if (!l1) w = make_float4(0.f, 0.f, 0.f, 0.f);
        buf[4 * i] = make_float2(u.x, w.x);
        buf[4 * i + 1] = make_float2(u.y, w.y);
        buf[4 * i + 2] = make_float2(u.z, w.z);
        buf[4 * i + 3] = make_float2(u.w, w.w);
    }
    __syncthreads();
    run_fft<T>(buf, tw);
    float2 *o0 = out + r0 * out_stride;
    float2 *o1 = out + (r0 + 1) * out_stride;
    for (int k = threadIdx.x; k < K; k += NT) {
        const float2 zk = buf[k];
        const float2 zn = buf[k == 0 ? 0 : T - k];
        const float s = 0.5f * (bin_scale ? bin_scale[k] : 1.0f);
        // X0 = (Z_k + conj(Z_-k)) / 2 ; X1 = (Z_k - conj(Z_-k)) / (2i)
        o0[k] = make_float2(s * (zk.x + zn.x), s * (zk.y - zn.y));
        if (l1) o1[k] = make_float2(s * (zk.y + zn.y), -s * (zk.x - zn.x));
    }
}

// Complex FFT of rows: input bins [0, in_len) (rest zero), output the first
// out_len points times `scale`; INV selects exp(+) via conjugation.
template <int T, bool INV>
__global__ void __launch_bounds__(Plan<T>::NT)
k_c2c(const float2 *__restrict__ in, long long in_stride, int in_len, float2 *__restrict__ out,
      long long out_stride, int out_len, float scale, const float2 *__restrict__ tw) {
    constexpr int NT = Plan<T>::NT;
    __shared__ __align__(16) float2 buf[T];
    const long long row = blockIdx.x;
    const float2 *src = in + row * in_stride;
    const float sg = INV ? -1.f : 1.f;
#pragma unroll
    for (int t = threadIdx.x; t < T; t += NT) {
        float2 v = make_float2(0.f, 0.f);
        if (t < in_len) v = __ldg(src + t);
        buf[t] = make_float2(v.x, sg * v.y);
    }
    __syncthreads();
    run_fft<T>(buf, tw);
    float2 *dst = out + row * out_stride;
    const float sy = sg * scale;
#pragma unroll
    for (int t = threadIdx.x; t < out_len; t += NT) {
        const float2 v = buf[t];
        dst[t] = make_float2(v.x * scale, v.y * sy);
    }
}

}  // namespace ct

bool fft_ct_supported(int T) { return T == 1024 || T == 1536 || T == 2048 || T == 4096; }

// Stage-ordered twiddle table of plan P, in the order fft<> reads it:
// for stages 1.. (input length NS, radix R): (R-1) x NS entries
// exp(-2 pi i r k / (NS R)), evaluated in double as the length-T table was.
template <int T>
static void stage_twiddles(std::vector<float2> &out) {
    using P = ct::Plan<T>;
    const int radix[4] = {P::R0, P::R1, P::R2, P::R3};
    int ns = radix[0];
    for (int s = 1; s < 4 && radix[s] > 1; ++s) {
        const int R = radix[s];
        for (int r = 1; r < R; ++r)
            for (int k = 0; k < ns; ++k) {
                const double a = -2.0 * M_PI * (double)(r * k * (T / (ns * R))) / (double)T;
                out.push_back(make_float2((float)cos(a), (float)sin(a)));
            }
        ns *= R;
    }
}

void fft_ct_twiddles(int T, std::vector<float2> &out) {
    out.clear();
    switch (T) {
        case 1024: stage_twiddles<1024>(out); break;
        case 1536: stage_twiddles<1536>(out); break;
        case 2048: stage_twiddles<2048>(out); break;
        case 4096: stage_twiddles<4096>(out); break;
    }
}

template <int T>
static int launch_r2c(const void *in, int in_kind, long long ntraces, float2 *out,
                      long long out_stride, int K, const float *bin_scale, const float2 *tw,
                      cudaStream_t s) {
    const unsigned npairs = (unsigned)((ntraces + 1) / 2);
    if (in_kind)
        ct::k_r2c<T, short><<<npairs, ct::Plan<T>::NT, 0, s>>>(
            reinterpret_cast<const short *>(in), ntraces, out, out_stride, K, bin_scale, tw);
    else
        ct::k_r2c<T, float><<<npairs, ct::Plan<T>::NT, 0, s>>>(
            reinterpret_cast<const float *>(in), ntraces, out, out_stride, K, bin_scale, tw);
    KKB_CHECK_LAUNCH("k_fft_r2c_ct");
    return KKB_OK;
}

template <int T>
static int launch_c2c(const float2 *in, long long in_stride, int in_len, float2 *out,
                      long long out_stride, int out_len, long long ntraces, bool inverse,
                      float scale, const float2 *tw, cudaStream_t s) {
    if (inverse)
        ct::k_c2c<T, true><<<(unsigned)ntraces, ct::Plan<T>::NT, 0, s>>>(
            in, in_stride, in_len, out, out_stride, out_len, scale, tw);
    else
        ct::k_c2c<T, false><<<(unsigned)ntraces, ct::Plan<T>::NT, 0, s>>>(
            in, in_stride, in_len, out, out_stride, out_len, scale, tw);
    KKB_CHECK_LAUNCH("k_fft_c2c_ct");
    return KKB_OK;
}

int fft_r2c_ct(const void *in, int in_kind, long long ntraces, int T, float2 *out,
               long long out_stride, int K, const float *bin_scale, const float2 *tw,
               cudaStream_t s) {
    if (ntraces <= 0) return KKB_OK;
    if ((ntraces + 1) / 2 > 0x7fffffffLL) return KKB_ERR_UNSUPPORTED;
    switch (T) {
        case 1024: return launch_r2c<1024>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s);
        case 1536: return launch_r2c<1536>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s);
        case 2048: return launch_r2c<2048>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s);
        case 4096: return launch_r2c<4096>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s);
    }
    return KKB_ERR_UNSUPPORTED;
}

int fft_c2c_ct(const float2 *in, long long in_stride, int in_len, float2 *out, long long out_stride,
               int out_len, long long ntraces, int T, bool inverse, float scale, const float2 *tw,
               cudaStream_t s) {
    if (ntraces <= 0) return KKB_OK;
    if (ntraces > 0x7fffffffLL) return KKB_ERR_UNSUPPORTED;
    switch (T) {
        case 1024: return launch_c2c<1024>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s);
        case 1536: return launch_c2c<1536>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s);
        case 2048: return launch_c2c<2048>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s);
        case 4096: return launch_c2c<4096>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s);
    }
    return KKB_ERR_UNSUPPORTED;
}

}  // namespace kkb
