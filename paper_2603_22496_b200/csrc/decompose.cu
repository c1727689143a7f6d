// K2: per-frequency-bin element -> virtual-plane-wave contraction (Eq. 3).
//
// Replaces the einsum of compress.shear_and_sum (compress.py:78-81) and of
// the reference's complex64 benchmark stage (bench.py:130-135):
//   Y[b, m, k] = sum_l X[b, l, k] * R[m, l, k]
// with b = (frame, transmit) rows, X the per-element spectra (k fastest, the
// layout the FFT writes), R the cached phase ramps exp(2 pi i f_k tau_lm)
// with the one-sided weight and the 1/T of the inverse FFT folded in.
//
// Ramps are built once per plan in float64 (phase in cycles reduced to
// [-1/2, 1/2] before sincospi) and rounded once to complex64: at config 5
// the phase reaches ~68 cycles and a float32 phase would cost 3-6e-6 of
// relative error.
//
// Contraction: each thread owns one bin k and a register tile of NB rows x
// MC receive angles (complex accumulators), streaming l; X and R loads are
// coalesced along k, every X value feeds MC FMAs and every R value NB.  FP32
// FMA (4 per complex MAC): exact enough for the 1e-6 max-abs reference tests.

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kk.cuh"

namespace kkb {

__global__ void k_build_ramps(const double *__restrict__ tau, int L, int M,
                              const double *__restrict__ freq, const double *__restrict__ scale,
                              int Kb, float2 *ramps) {
    const long long total = (long long)M * L * Kb;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int k = (int)(i % Kb);
        long long ml = i / Kb;
        int l = (int)(ml % L), m = (int)(ml / L);
        double cyc = tau[(long long)l * M + m] * freq[k];  // phase in cycles
        double r = cyc - rint(cyc);
        double sn, cs;
        sincospi(2.0 * r, &sn, &cs);
        double sc = scale[k];
        ramps[i] = make_float2((float)(cs * sc), (float)(sn * sc));
    }
}

int build_ramps(const double *tau_host, int L, int M, const double *freq_host,
                const double *scale_host, int Kb, float2 *ramps, cudaStream_t s) {
    double *d = nullptr;
    size_t n_tau = (size_t)L * M, bytes = sizeof(double) * (n_tau + 2 * (size_t)Kb);
    KKB_TRY_CUDA(cudaMallocAsync(&d, bytes, s), "cudaMallocAsync(ramp inputs)");
    KKB_TRY_CUDA(cudaMemcpyAsync(d, tau_host, sizeof(double) * n_tau, cudaMemcpyHostToDevice, s), "tau");
    KKB_TRY_CUDA(cudaMemcpyAsync(d + n_tau, freq_host, sizeof(double) * Kb, cudaMemcpyHostToDevice, s),
                 "freq");
    KKB_TRY_CUDA(cudaMemcpyAsync(d + n_tau + Kb, scale_host, sizeof(double) * Kb,
                                 cudaMemcpyHostToDevice, s),
                 "scale");
    long long total = (long long)M * L * Kb;
    int blocks = (int)std::min<long long>(ceil_div(total, 256), 148 * 32);
    k_build_ramps<<<blocks, 256, 0, s>>>(d, L, M, d + n_tau, d + n_tau + Kb, Kb, ramps);
    KKB_CHECK_LAUNCH("k_build_ramps");
    // host arrays may be freed by the caller right after return
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync ramps");
    cudaFreeAsync(d, s);
    return KKB_OK;
}

#define KKB_CT_KX 64  // bins per CTA (threads along x)
#define KKB_CT_BY 4   // row groups per CTA (threads along y)

template <int NB, int MC>
__global__ void __launch_bounds__(KKB_CT_KX *KKB_CT_BY)
k_contract(const float2 *__restrict__ X, long long ldx, const float2 *__restrict__ R,
           long long ldr, float2 *__restrict__ Y, long long ldy, long long B, int L, int M, int Kb) {
    const int k = blockIdx.x * KKB_CT_KX + threadIdx.x;
    const long long b0 = ((long long)blockIdx.y * KKB_CT_BY + threadIdx.y) * NB;
    const int m0 = blockIdx.z * MC;
    if (k >= Kb || b0 >= B) return;
    float2 acc[NB][MC];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < MC; ++j) acc[i][j] = make_float2(0.f, 0.f);
    const int nb = (int)min((long long)NB, B - b0);
    const int mc = min(MC, M - m0);
    const float2 *xp = X + b0 * L * ldx + k;
    const float2 *rp = R + (long long)m0 * L * ldr + k;
    for (int l = 0; l < L; ++l) {
        float2 xv[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i)
            xv[i] = (i < nb) ? __ldg(xp + ((long long)i * L + l) * ldx) : make_float2(0.f, 0.f);
#pragma unroll
        for (int j = 0; j < MC; ++j) {
            if (j < mc) {
                const float2 r = __ldg(rp + ((long long)j * L + l) * ldr);
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    acc[i][j].x = fmaf(xv[i].x, r.x, acc[i][j].x);
                    acc[i][j].x = fmaf(-xv[i].y, r.y, acc[i][j].x);
                    acc[i][j].y = fmaf(xv[i].x, r.y, acc[i][j].y);
                    acc[i][j].y = fmaf(xv[i].y, r.x, acc[i][j].y);
                }
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        if (i >= nb) break;
#pragma unroll
        for (int j = 0; j < MC; ++j)
            if (j < mc) Y[((b0 + i) * M + m0 + j) * ldy + k] = acc[i][j];
    }
}

template <int NB, int MC>
static int launch_contract(const float2 *X, long long ldx, const float2 *R, long long ldr, float2 *Y,
                           long long ldy, long long B, int L, int M, int Kb, cudaStream_t s) {
    dim3 block(KKB_CT_KX, KKB_CT_BY);
    dim3 grid((unsigned)ceil_div(Kb, KKB_CT_KX), (unsigned)ceil_div(B, (long long)NB * KKB_CT_BY),
              (unsigned)ceil_div(M, MC));
    if (grid.y > 65535u) {
        set_error("contraction batch too large (%lld rows)", B);
        return KKB_ERR_UNSUPPORTED;
    }
    k_contract<NB, MC><<<grid, block, 0, s>>>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb);
    KKB_CHECK_LAUNCH("k_contract");
    return KKB_OK;
}

int contract(const float2 *X, long long ldx, const float2 *R, long long ldr, float2 *Y,
             long long ldy, long long B, int L, int M, int Kb, cudaStream_t s) {
    if (B <= 0 || Kb <= 0) return KKB_OK;
    if (M <= 4) return launch_contract<8, 4>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
    if (M <= 8) return launch_contract<6, 8>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
    if (M <= 12) return launch_contract<4, 12>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
    return launch_contract<4, 16>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
}

}  // namespace kkb
