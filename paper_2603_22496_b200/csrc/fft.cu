// K1 / K3: batched length-T FFTs along time, in shared memory (sm_100a).
//
// Replaces the numpy/scipy pocketfft calls of the reference hot path
// (spectral.py:90,92; compress.py:75,81; bench.py:128,138): full-length DFTs,
// no padding — the circular-shear wrap position depends on T exactly
// (compress.py:21-26, spectral.py:8-10).
//
// Algorithm: Stockham autosort, mixed radix (8, 4, 2, 3, 5, direct odd
// radices <= 31), ping-pong between two shared-memory buffers, one or more
// traces per CTA.  Stage s with radix R and sub-transform length Ns:
//   j in [0, T/R):  k = j mod Ns
//   v[r] = a[j + r T/R] * W_T^{r k T/(Ns R)}        (r = 0..R-1)
//   b[(j/Ns) Ns R + k + r Ns] = DFT_R(v)[r]
// Twiddles W_T^i = exp(-2 pi i/T) are computed in float64 on the host and
// rounded once to float32, so the float32 transform error stays ~eps*log T.
// Inverse transforms run the forward stages on conj(x) and conjugate again.
// Lengths whose largest prime factor exceeds 31 use a direct O(T^2) DFT
// kernel (still on the GPU; correctness path for odd sizes only).

#include <map>
#include <mutex>
#include <vector>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "fft.cuh"

namespace kkb {

namespace {

std::mutex g_fft_mu;
std::map<int, FftPlan> g_fft_plans;  // keyed by (T, device)

}  // namespace

int get_fft_plan(int T, FftPlan *out) {
    std::lock_guard<std::mutex> lock(g_fft_mu);
    int dev = 0;
    cudaGetDevice(&dev);
    int key = T * 64 + dev;
    auto it = g_fft_plans.find(key);
    if (it != g_fft_plans.end()) {
        *out = it->second;
        return KKB_OK;
    }
    if (T < 1 || T > KKB_FFT_MAX_T_TOTAL) {
        set_error("FFT length %d outside [1, %d]", T, KKB_FFT_MAX_T_TOTAL);
        return KKB_ERR_UNSUPPORTED;
    }
    FftPlan p{};
    p.T = T;
    int t = T;
    if (T > KKB_FFT_MAX_T) {
        // four-step split T = T1 x T2, both single-CTA lengths, T1 as close to
        // sqrt(T) as the divisors allow; no such split -> direct DFT
        for (int a = (int)std::sqrt((double)T); a >= 2; --a) {
            if (T % a) continue;
            const int b = T / a;
            if (a <= KKB_FFT_MAX_T && b <= KKB_FFT_MAX_T) {
                p.T1 = b;  // the larger factor first (rows of length T1)
                p.T2 = a;
                break;
            }
        }
        p.large = p.T1 > 0 ? 1 : 0;
        p.direct = p.large ? 0 : 1;
        t = 1;
    }
    const int order[] = {8, 4, 2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31};
    for (int r : order) {
        while (t % r == 0) {
            if (p.nstages >= KKB_FFT_MAX_STAGES) break;
            p.radix[p.nstages++] = r;
            t /= r;
        }
    }
    if (T <= KKB_FFT_MAX_T) p.direct = (t != 1) ? 1 : 0;
    if (p.direct || p.large) p.nstages = 0;
    std::vector<float2> tw(T);
    for (int k = 0; k < T; ++k) {
        // exp(-2 pi i k / T) in double, reduced exactly by symmetry
        double a = -2.0 * M_PI * (double)k / (double)T;
        tw[k] = make_float2((float)cos(a), (float)sin(a));
    }
    cudaError_t e = cudaMalloc(&p.tw, sizeof(float2) * T);
    if (e == cudaSuccess)
        e = cudaMemcpy(p.tw, tw.data(), sizeof(float2) * T, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && fft_ct_supported(T)) {
        std::vector<float2> tws;
        fft_ct_twiddles(T, tws);
        e = cudaMalloc(&p.tws, sizeof(float2) * tws.size());
        if (e == cudaSuccess)
            e = cudaMemcpy(p.tws, tws.data(), sizeof(float2) * tws.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {  // nothing cached: free what was allocated
        cudaFree(p.tw);
        cudaFree(p.tws);
        return cuda_status(e, "FFT plan twiddles");
    }
    g_fft_plans[key] = p;
    *out = p;
    return KKB_OK;
}

// ------------------------------------------------------------- small DFTs
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ float2 cmul(float2 a, float2 b) {
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ float2 mul_mi(float2 a) { return make_float2(a.y, -a.x); }  // * (-i)

__device__ __forceinline__ void dft2(float2 &a, float2 &b) {
    float2 t = a;
    a = cadd(t, b);
    b = csub(t, b);
}

__device__ __forceinline__ void dft4(float2 *v) {
    float2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]);
    float2 a2 = cadd(v[1], v[3]), a3 = mul_mi(csub(v[1], v[3]));
    v[0] = cadd(a0, a2);
    v[2] = csub(a0, a2);
    v[1] = cadd(a1, a3);
    v[3] = csub(a1, a3);
}

__device__ __forceinline__ void dft8(float2 *v) {
    const float r = 0.70710678118654752440f;
    float2 e[4] = {v[0], v[2], v[4], v[6]};
    float2 o[4] = {v[1], v[3], v[5], v[7]};
    dft4(e);
    dft4(o);
    // twiddle o[k] by W8^k
    o[1] = make_float2(r * (o[1].x + o[1].y), r * (o[1].y - o[1].x));
    o[2] = mul_mi(o[2]);
    o[3] = make_float2(r * (o[3].y - o[3].x), -r * (o[3].x + o[3].y));
    for (int k = 0; k < 4; ++k) {
        v[k] = cadd(e[k], o[k]);
        v[k + 4] = csub(e[k], o[k]);
    }
}

__device__ __forceinline__ void dft3(float2 *v) {
    const float s = 0.86602540378443864676f;  // sin(2pi/3)
    float2 t1 = cadd(v[1], v[2]);
    float2 t2 = make_float2(v[0].x - 0.5f * t1.x, v[0].y - 0.5f * t1.y);
    float2 t3 = csub(v[1], v[2]);
    // -i*s*t3
    float2 t4 = make_float2(s * t3.y, -s * t3.x);
    v[0] = cadd(v[0], t1);
    v[1] = cadd(t2, t4);
    v[2] = csub(t2, t4);
}

__device__ __forceinline__ void dft5(float2 *v) {
    const float c1 = 0.30901699437494742410f;   // cos(2pi/5)
    const float c2 = -0.80901699437494742410f;  // cos(4pi/5)
    const float s1 = 0.95105651629515357212f;   // sin(2pi/5)
    const float s2 = 0.58778525229247312917f;   // sin(4pi/5)
    float2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
    float2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
    float2 x0 = v[0];
    float2 p1 = make_float2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
    float2 p2 = make_float2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
    // q = -i (s1 b1 + s2 b2),  r = -i (s2 b1 - s1 b2)
    float2 q1 = make_float2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
    float2 q2 = make_float2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
    q1 = mul_mi(q1);
    q2 = mul_mi(q2);
    v[0] = make_float2(x0.x + a1.x + a2.x, x0.y + a1.y + a2.y);
    v[1] = cadd(p1, q1);
    v[4] = csub(p1, q1);
    v[2] = cadd(p2, q2);
    v[3] = csub(p2, q2);
}

// generic odd radix (<= 31) by direct summation with table twiddles
__device__ __noinline__ void dft_generic(float2 *v, int R, const float2 *__restrict__ tw, int T) {
    float2 out[KKB_FFT_MAX_RADIX];
    int step = T / R;
    for (int p = 0; p < R; ++p) {
        float2 acc = make_float2(0.f, 0.f);
        for (int q = 0; q < R; ++q) {
            float2 w = tw[(size_t)step * ((p * q) % R)];
            acc = cadd(acc, cmul(v[q], w));
        }
        out[p] = acc;
    }
    for (int p = 0; p < R; ++p) v[p] = out[p];
}

// Run every Stockham stage on G traces laid out back to back (stride T) in
// buffer `a`; `b` is scratch of the same size; `tw` is the twiddle table in
// shared memory.  Each thread walks butterfly indices j and applies them to
// all G traces, so a twiddle is fetched once per j.  Ns is a power of two in
// every stage that precedes the first odd radix (radices run 8,4,2 first),
// so k = j mod Ns is a mask there.  Returns the buffer holding the result.
__device__ float2 *stockham(float2 *a, float2 *b, int G, const FftPlan &p, const float2 *tw) {
    const int T = p.T;
    const int sw = (T & 15) == 0 ? 15 : 0;  // XOR swizzle of the low 4 index bits (bank spread)
#define SW(e) ((e) ^ (((e) >> 3) & sw))
    int Ns = 1;
    for (int s = 0; s < p.nstages; ++s) {
        const int R = p.radix[s];
        const int TR = T / R;
        const int tws = T / (Ns * R);
        const bool pow2 = (Ns & (Ns - 1)) == 0;
        for (int j = threadIdx.x; j < TR; j += blockDim.x) {
            const int k = pow2 ? (j & (Ns - 1)) : (j % Ns);
            const int base = (j - k) * R + k;
            if (R == 8) {
                float2 w[8];
#pragma unroll
                for (int r = 1; r < 8; ++r) w[r] = tw[r * k * tws];
                for (int g = 0; g < G; ++g) {
                    const float2 *src = a + g * T;
                    float2 *dst = b + g * T;
                    float2 v[8];
#pragma unroll
                    for (int r = 0; r < 8; ++r) v[r] = src[SW(j + r * TR)];
#pragma unroll
                    for (int r = 1; r < 8; ++r) v[r] = cmul(v[r], w[r]);
                    dft8(v);
#pragma unroll
                    for (int r = 0; r < 8; ++r) dst[SW(base + r * Ns)] = v[r];
                }
            } else if (R == 4) {
                float2 w[4];
#pragma unroll
                for (int r = 1; r < 4; ++r) w[r] = tw[r * k * tws];
                for (int g = 0; g < G; ++g) {
                    const float2 *src = a + g * T;
                    float2 *dst = b + g * T;
                    float2 v[4];
#pragma unroll
                    for (int r = 0; r < 4; ++r) v[r] = src[SW(j + r * TR)];
#pragma unroll
                    for (int r = 1; r < 4; ++r) v[r] = cmul(v[r], w[r]);
                    dft4(v);
#pragma unroll
                    for (int r = 0; r < 4; ++r) dst[SW(base + r * Ns)] = v[r];
                }
            } else if (R == 2) {
                const float2 w1 = tw[k * tws];
                for (int g = 0; g < G; ++g) {
                    const float2 *src = a + g * T;
                    float2 *dst = b + g * T;
                    float2 v0 = src[SW(j)], v1 = cmul(src[SW(j + TR)], w1);
                    dft2(v0, v1);
                    dst[SW(base)] = v0;
                    dst[SW(base + Ns)] = v1;
                }
            } else if (R == 3) {
                const float2 w1 = tw[k * tws], w2 = tw[2 * k * tws];
                for (int g = 0; g < G; ++g) {
                    const float2 *src = a + g * T;
                    float2 *dst = b + g * T;
                    float2 v[3] = {src[SW(j)], cmul(src[SW(j + TR)], w1), cmul(src[SW(j + 2 * TR)], w2)};
                    dft3(v);
#pragma unroll
                    for (int r = 0; r < 3; ++r) dst[SW(base + r * Ns)] = v[r];
                }
            } else if (R == 5) {
                float2 w[5];
#pragma unroll
                for (int r = 1; r < 5; ++r) w[r] = tw[r * k * tws];
                for (int g = 0; g < G; ++g) {
                    const float2 *src = a + g * T;
                    float2 *dst = b + g * T;
                    float2 v[5];
#pragma unroll
                    for (int r = 0; r < 5; ++r) v[r] = src[SW(j + r * TR)];
#pragma unroll
                    for (int r = 1; r < 5; ++r) v[r] = cmul(v[r], w[r]);
                    dft5(v);
#pragma unroll
                    for (int r = 0; r < 5; ++r) dst[SW(base + r * Ns)] = v[r];
                }
            } else {
                for (int g = 0; g < G; ++g) {
                    const float2 *src = a + g * T;
                    float2 *dst = b + g * T;
                    float2 v[KKB_FFT_MAX_RADIX];
                    for (int r = 0; r < R; ++r) v[r] = cmul(src[SW(j + r * TR)], tw[r * k * tws]);
                    dft_generic(v, R, tw, T);
                    for (int r = 0; r < R; ++r) dst[SW(base + r * Ns)] = v[r];
                }
            }
        }
        __syncthreads();
        float2 *t = a;
        a = b;
        b = t;
        Ns *= R;
    }
#undef SW
    return a;
}

// Index of logical element t of a trace buffer (the swizzle stockham uses).
__device__ __forceinline__ int fft_sw(int t, int T) { return (T & 15) == 0 ? t ^ ((t >> 3) & 15) : t; }

// ------------------------------------------------------------- kernels
__device__ __forceinline__ void load_twiddles(float2 *tw_s, const FftPlan &p) {
    for (int i = threadIdx.x; i < p.T; i += blockDim.x) tw_s[i] = p.tw[i];
}

// Complex-to-complex FFT of `ntraces` rows.  Input row i: in + i*in_stride,
// first in_len bins read, the rest treated as zero (one-sided spectra).
// Output row i: out + i*out_stride, first out_len bins written, times scale.
__global__ void __launch_bounds__(KKB_FFT_THREADS)
k_fft_c2c(const float2 *__restrict__ in, long long in_stride, int in_len,
          float2 *__restrict__ out, long long out_stride, int out_len,
          long long ntraces, int G, int inverse, float scale, FftPlan p) {
    extern __shared__ float2 smem[];
    const int T = p.T;
    float2 *a = smem;
    float2 *b = smem + G * T;
    float2 *tw = smem + 2 * G * T;
    load_twiddles(tw, p);
    const long long t0 = (long long)blockIdx.x * G;
    const float sgn = inverse ? -1.f : 1.f;
    for (int g = 0; g < G; ++g) {
        const long long tr = t0 + g;
        const bool live = tr < ntraces;
        const float2 *row = in + (live ? tr : 0) * in_stride;
        for (int t = threadIdx.x; t < T; t += blockDim.x) {
            float2 v = make_float2(0.f, 0.f);
            if (live && t < in_len) v = row[t];
            a[g * T + fft_sw(t, T)] = make_float2(v.x, sgn * v.y);
        }
    }
    __syncthreads();
    float2 *res = stockham(a, b, G, p, tw);
    const float sy = sgn * scale;
    for (int g = 0; g < G; ++g) {
        const long long tr = t0 + g;
        if (tr >= ntraces) break;
        float2 *row = out + tr * out_stride;
        for (int t = threadIdx.x; t < out_len; t += blockDim.x) {
            const float2 v = res[g * T + fft_sw(t, T)];
            row[t] = make_float2(v.x * scale, v.y * sy);
        }
    }
}

// Real-input FFT of `ntraces` float rows (stride T), two rows packed as one
// complex row per transform.  Writes bins [0, K) of each row's spectrum to
// out + row*out_stride, each multiplied by bin_scale[k] (NULL = 1).
__global__ void __launch_bounds__(KKB_FFT_THREADS)
k_fft_r2c_pairs(const float *__restrict__ in, long long ntraces, float2 *__restrict__ out,
                long long out_stride, int K, const float *__restrict__ bin_scale, int G,
                FftPlan p, int grp) {
    extern __shared__ float2 smem[];
    const int T = p.T;
    float2 *a = smem;
    float2 *b = smem + G * T;
    float2 *tw = smem + 2 * G * T;
    load_twiddles(tw, p);
    const long long pair0 = (long long)blockIdx.x * G;
    const bool vec4 = (T & 3) == 0;
    const long long ppg = (grp + 1) / 2;  // pairs per group (k_r2c's pairing rule)
    for (int g = 0; g < G; ++g) {
        const long long pi = pair0 + g, gi = pi / ppg, q = pi - gi * ppg;
        const long long r0 = gi * grp + 2 * q;
        const bool l0 = r0 < ntraces, l1 = l0 && 2 * q + 1 < grp && r0 + 1 < ntraces;
        const float *x0 = in + (l0 ? r0 : 0) * T;
        const float *x1 = in + (l1 ? r0 + 1 : 0) * T;
        if (vec4) {
            for (int t = 4 * threadIdx.x; t < T; t += 4 * blockDim.x) {
                float4 u = l0 ? __ldg(reinterpret_cast<const float4 *>(x0 + t)) : make_float4(0, 0, 0, 0);
                float4 w = l1 ? __ldg(reinterpret_cast<const float4 *>(x1 + t)) : make_float4(0, 0, 0, 0);
                float2 *d = a + g * T;
                d[fft_sw(t, T)] = make_float2(u.x, w.x);
                d[fft_sw(t + 1, T)] = make_float2(u.y, w.y);
                d[fft_sw(t + 2, T)] = make_float2(u.z, w.z);
                d[fft_sw(t + 3, T)] = make_float2(u.w, w.w);
            }
        } else {
            for (int t = threadIdx.x; t < T; t += blockDim.x)
                a[g * T + fft_sw(t, T)] = make_float2(l0 ? x0[t] : 0.f, l1 ? x1[t] : 0.f);
        }
    }
    __syncthreads();
    float2 *res = stockham(a, b, G, p, tw);
    for (int g = 0; g < G; ++g) {
        const long long pi = pair0 + g, gi = pi / ppg, q = pi - gi * ppg;
        const long long r0 = gi * grp + 2 * q;
        if (r0 >= ntraces) break;
        const bool has1 = 2 * q + 1 < grp && r0 + 1 < ntraces;
        float2 *o0 = out + r0 * out_stride;
        float2 *o1 = out + (r0 + 1) * out_stride;
        for (int k = threadIdx.x; k < K; k += blockDim.x) {
            const float2 zk = res[g * T + fft_sw(k, T)];
            const float2 zn = res[g * T + fft_sw(k == 0 ? 0 : T - k, T)];
            const float s = bin_scale ? bin_scale[k] : 1.0f;
            // X0 = (Z_k + conj(Z_-k)) / 2 ; X1 = (Z_k - conj(Z_-k)) / (2i)
            o0[k] = make_float2(0.5f * s * (zk.x + zn.x), 0.5f * s * (zk.y - zn.y));
            if (has1) o1[k] = make_float2(0.5f * s * (zk.y + zn.y), -0.5f * s * (zk.x - zn.x));
        }
    }
}

// Direct DFT fallback for lengths with a prime factor > 31.
__global__ void k_dft_direct(const float2 *__restrict__ in, long long in_stride, int in_len,
                             float2 *__restrict__ out, long long out_stride, int out_len,
                             long long ntraces, int inverse, float scale, FftPlan p) {
    const int T = p.T;
    long long tr = blockIdx.y;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < out_len; k += gridDim.x * blockDim.x) {
        double ar = 0.0, ai = 0.0;
        for (int t = 0; t < in_len; ++t) {
            float2 v = in[tr * in_stride + t];
            float2 w = p.tw[(long long)k * t % T];
            if (inverse) w.y = -w.y;
            ar += (double)v.x * w.x - (double)v.y * w.y;
            ai += (double)v.x * w.y + (double)v.y * w.x;
        }
        out[tr * out_stride + k] = make_float2((float)ar * scale, (float)ai * scale);
    }
}

__global__ void k_real_to_complex(const float *__restrict__ in, long long n, float2 *__restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = make_float2(in[i], 0.f);
}

// ------------------------------------------------------------- four-step (T > 8192)
// X[k1 + T1 k2] = sum_n2 W_T2^(n2 k2) W_T^(n2 k1) sum_n1 W_T1^(n1 k1) x[n1 T2 + n2]:
// three batched transposes around two batches of single-CTA transforms.
// MODE 0: A[tr][n2][n1] = x[tr][n1 T2 + n2]         (zero past in_len)
// MODE 1: A[tr][k1][n2] = B[tr][n2][k1] * W_T^(+-n2 k1)
// MODE 2: out[tr][k2 T1 + k1] = B[tr][k1][k2] * scale (* bin_scale), k < out_len
template <int MODE>
__global__ void __launch_bounds__(256)
k_fourstep(const float2 *__restrict__ src, long long src_stride, int src_len, float2 *__restrict__ dst,
           long long dst_stride, int dst_len, int R, int C, const float2 *__restrict__ tw, int T,
           int inverse, float scale, const float *__restrict__ bin_scale) {
    // transpose of an R x C matrix (row r, column c) per trace, 32 x 32 tiles
    __shared__ float2 tile[32][33];
    const long long tr = blockIdx.z;
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    const float2 *s = src + tr * src_stride;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        float2 v = make_float2(0.f, 0.f);
        if (r < R && c < C) {
            const long long e = (long long)r * C + c;
            if (MODE != 0 || e < src_len) v = s[e];
            if (MODE == 1) {  // source row r = n2, column c = k1
                float2 w = tw[(long long)r * c % T];
                if (inverse) w.y = -w.y;
                v = make_float2(v.x * w.x - v.y * w.y, v.x * w.y + v.y * w.x);
            }
        }
        tile[i][threadIdx.x] = v;
    }
    __syncthreads();
    float2 *d = dst + tr * dst_stride;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;  // destination row c, column r
        if (r < R && c < C) {
            const long long e = (long long)c * R + r;
            float2 v = tile[threadIdx.x][i];
            if (MODE == 2) {
                if (e >= dst_len) continue;
                const float sc = scale * (bin_scale ? bin_scale[e] : 1.0f);
                v = make_float2(v.x * sc, v.y * sc);
            }
            d[e] = v;
        }
    }
}

int fft_c2c(const float2 *in, long long in_stride, int in_len, float2 *out, long long out_stride,
            int out_len, long long ntraces, int T, bool inverse, float scale, cudaStream_t s);

static int fft_c2c_large(const FftPlan &p, const float2 *in, long long in_stride, int in_len,
                         float2 *out, long long out_stride, int out_len, long long ntraces,
                         bool inverse, float scale, const float *bin_scale, cudaStream_t s) {
    const int T = p.T, T1 = p.T1, T2 = p.T2;
    if (ntraces > 65535) {
        set_error("four-step FFT: %lld traces per call exceed the grid limit", ntraces);
        return KKB_ERR_UNSUPPORTED;
    }
    float2 *A = nullptr, *B = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&A, sizeof(float2) * (size_t)ntraces * T, s), "cudaMallocAsync(4step A)");
    KKB_TRY_CUDA(cudaMallocAsync(&B, sizeof(float2) * (size_t)ntraces * T, s), "cudaMallocAsync(4step B)");
    const dim3 blk(32, 8);
    int st = KKB_OK;
    // x as T1 rows (n1) x T2 columns (n2) -> A rows n2 of length T1
    k_fourstep<0><<<dim3(ceil_div(T2, 32), ceil_div(T1, 32), ntraces), blk, 0, s>>>(
        in, in_stride, in_len, A, T, T, T1, T2, p.tw, T, 0, 1.f, nullptr);
    KKB_CHECK_LAUNCH("k_fourstep<load>");
    if (!st) st = fft_c2c(A, T1, T1, B, T1, T1, ntraces * T2, T1, inverse, 1.0f, s);
    if (!st) {
        // B rows n2 (T2) x columns k1 (T1), twiddled -> A rows k1 of length T2
        k_fourstep<1><<<dim3(ceil_div(T1, 32), ceil_div(T2, 32), ntraces), blk, 0, s>>>(
            B, T, T, A, T, T, T2, T1, p.tw, T, inverse ? 1 : 0, 1.f, nullptr);
        KKB_CHECK_LAUNCH("k_fourstep<twiddle>");
        st = fft_c2c(A, T2, T2, B, T2, T2, ntraces * T1, T2, inverse, 1.0f, s);
    }
    if (!st) {
        // B rows k1 (T1) x columns k2 (T2) -> natural order k = k2 T1 + k1
        k_fourstep<2><<<dim3(ceil_div(T2, 32), ceil_div(T1, 32), ntraces), blk, 0, s>>>(
            B, T, T, out, out_stride, out_len, T1, T2, p.tw, T, 0, scale, bin_scale);
        KKB_CHECK_LAUNCH("k_fourstep<store>");
    }
    cudaFreeAsync(A, s);
    cudaFreeAsync(B, s);
    return st;
}

// ------------------------------------------------------------- host launchers
// Compile-time-specialised kernels (fft_ct.cu) for T in {1024, 1536, 2048, 4096};
// KKB_FFT_GENERIC=1 in the environment forces the runtime-plan kernels (tests).
static const bool g_use_ct = [] {
    const char *e = getenv("KKB_FFT_GENERIC");
    return !(e && e[0] == '1');
}();

static int traces_per_cta(int T) {
    int G = KKB_FFT_TARGET_ELEMS / T;
    return G < 1 ? 1 : G;
}

static int smem_bytes(int T, int G) { return (2 * G + 1) * T * (int)sizeof(float2); }

static int ensure_smem(const void *fn, int bytes) {
    if (bytes > 48 * 1024) {
        KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                     "cudaFuncSetAttribute(fft smem)");
    }
    return KKB_OK;
}

int fft_c2c(const float2 *in, long long in_stride, int in_len, float2 *out, long long out_stride,
            int out_len, long long ntraces, int T, bool inverse, float scale, cudaStream_t s) {
    if (ntraces <= 0) return KKB_OK;
    FftPlan p;
    int st = get_fft_plan(T, &p);
    if (st) return st;
    if (p.large) return fft_c2c_large(p, in, in_stride, in_len, out, out_stride, out_len, ntraces,
                                      inverse, scale, nullptr, s);
    if (p.direct) {
        dim3 grid((unsigned)ceil_div(out_len, 256), (unsigned)ntraces);
        k_dft_direct<<<grid, 256, 0, s>>>(in, in_stride, in_len, out, out_stride, out_len, ntraces,
                                          inverse ? 1 : 0, scale, p);
        KKB_CHECK_LAUNCH("k_dft_direct");
        return KKB_OK;
    }
    if (fft_ct_supported(T) && g_use_ct)
        return fft_c2c_ct(in, in_stride, in_len, out, out_stride, out_len, ntraces, T, inverse, scale,
                          p.tws, s);
    int G = traces_per_cta(T);
    int sm = smem_bytes(T, G);
    st = ensure_smem((const void *)k_fft_c2c, sm);
    if (st) return st;
    k_fft_c2c<<<(unsigned)ceil_div(ntraces, G), KKB_FFT_THREADS, sm, s>>>(
        in, in_stride, in_len, out, out_stride, out_len, ntraces, G, inverse ? 1 : 0, scale, p);
    KKB_CHECK_LAUNCH("k_fft_c2c");
    return KKB_OK;
}

int fft_c2c_scatter(const float2 *in, long long in_stride, int in_len, int out_len,
                    long long ntraces, int T, bool inverse, float scale, const RowScatter &sc,
                    cudaStream_t s) {
    if (ntraces <= 0) return KKB_OK;
    if (sc.ndst < 1 || sc.ndst > KKB_ROW_SCATTER_MAX || sc.rows_per_frame < 1) return KKB_ERR_ARG;
    if (fft_ct_supported(T) && g_use_ct && ntraces <= 0x7fffffffLL) {
        FftPlan p;
        int st = get_fft_plan(T, &p);
        if (st) return st;
        return fft_c2c_ct(in, in_stride, in_len, nullptr, out_len, out_len, ntraces, T, inverse,
                          scale, p.tws, s, &sc);
    }
    // other lengths: transform into scratch, then one strided copy per destination
    float2 *tmp = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&tmp, sizeof(float2) * (size_t)ntraces * out_len, s),
                 "cudaMallocAsync(scatter scratch)");
    int st = fft_c2c(in, in_stride, in_len, tmp, out_len, out_len, ntraces, T, inverse, scale, s);
    const long long frames = ntraces / sc.rows_per_frame;
    const size_t row_bytes = sizeof(float2) * (size_t)sc.rows_per_frame * out_len;
    for (int d = 0; d < sc.ndst && !st; ++d) {
        cudaError_t e = cudaMemcpy2DAsync(sc.dst[d] + sc.off, sizeof(float2) * (size_t)sc.frame_stride,
                                          tmp, row_bytes, row_bytes, (size_t)frames,
                                          cudaMemcpyDeviceToDevice, s);
        if (e != cudaSuccess) st = cuda_status(e, "scatter copy");
    }
    cudaFreeAsync(tmp, s);
    return st;
}

int fft_r2c(const float *in, long long ntraces, int T, float2 *out, long long out_stride, int K,
            const float *bin_scale, cudaStream_t s, float2 *scratch_c2c, long long group_rows) {
    if (ntraces <= 0) return KKB_OK;
    // pairing groups; the whole batch as one group pairs like groups of 2
    const int grp = group_rows > 0 && group_rows <= 0x7fffffffLL ? (int)group_rows : 2;
    FftPlan p;
    int st = get_fft_plan(T, &p);
    if (st) return st;
    if (p.direct || p.large) {
        // promote to complex (scratch holds ntraces*T) then the direct DFT or
        // the four-step transform; scaling by bin_scale is not supported here
        // (callers fold it elsewhere)
        if (!scratch_c2c || bin_scale) {
            set_error("direct-DFT r2c path needs scratch and no bin scale");
            return KKB_ERR_UNSUPPORTED;
        }
        long long n = ntraces * (long long)T;
        k_real_to_complex<<<(unsigned)std::min<long long>(ceil_div(n, 256), 65535), 256, 0, s>>>(
            in, n, scratch_c2c);
        KKB_CHECK_LAUNCH("k_real_to_complex");
        return fft_c2c(scratch_c2c, T, T, out, out_stride, K, ntraces, T, false, 1.0f, s);
    }
    if (fft_ct_supported(T) && g_use_ct)
        return fft_r2c_ct(in, 0, ntraces, T, out, out_stride, K, bin_scale, p.tws, s, grp);
    int G = traces_per_cta(T);
    int sm = smem_bytes(T, G);
    st = ensure_smem((const void *)k_fft_r2c_pairs, sm);
    if (st) return st;
    long long npairs = ceil_div(ntraces, grp) * ((grp + 1) / 2);
    k_fft_r2c_pairs<<<(unsigned)ceil_div(npairs, G), KKB_FFT_THREADS, sm, s>>>(
        in, ntraces, out, out_stride, K, bin_scale, G, p, grp);
    KKB_CHECK_LAUNCH("k_fft_r2c_pairs");
    return KKB_OK;
}

}  // namespace kkb
