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
// Contraction: a CTA owns KT bins x BT rows; element chunks of X and R stream
// through shared memory (cp.async, double-buffered, coalesced along k), and
// each thread keeps an NB x MC register tile of complex accumulators, so each
// shared X value feeds MC FMAs and each R value NB.  FP32 FMA (4 per complex
// MAC): within the 1e-6 max-abs bound of the reference's compress tests.

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
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

// Tile: KT bins x BT rows per CTA, all (<= MC) receive angles; the element
// axis streams through shared memory in chunks of LC with cp.async double
// buffering.  Thread (kx, bg) owns bin k0+kx and rows b0 + bg*NB .. +NB-1.
#define KKB_CT_KT 32
#ifndef KKB_CT_NB
#define KKB_CT_NB 4       // rows per thread (register tile NB x MC)
#endif
#ifndef KKB_CT_MINB
#define KKB_CT_MINB 2     // CTAs per SM requested for MC <= 12
#endif
#define KKB_CT_BT (8 * KKB_CT_NB)  // rows per CTA: 8 row groups of 32 bin-threads
#define KKB_CT_LC 4
#define KKB_CT_THREADS 256
static_assert(KKB_CT_BT == 16 || KKB_CT_BT == 32, "wide staging covers 16 or 32 rows");

__device__ __forceinline__ void cp_async8z(void *smem_dst, const void *gsrc, bool valid) {
    unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz)
                 : "memory");
}

__device__ __forceinline__ void cp_async16z(void *smem_dst, const void *gsrc, bool valid) {
    unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz)
                 : "memory");
}

template <int MC>
__global__ void __launch_bounds__(KKB_CT_THREADS, MC <= 12 ? KKB_CT_MINB : 1)
k_contract(const float2 *__restrict__ X, long long ldx, const float2 *__restrict__ R,
           long long ldr, float2 *__restrict__ Y, long long ldy, long long B, int L, int M, int Kb) {
    constexpr int KT = KKB_CT_KT, BT = KKB_CT_BT, NB = KKB_CT_NB, LC = KKB_CT_LC;
    extern __shared__ __align__(16) float2 csm[];
    float2 *Xs = csm;                       // [2][LC][BT][KT]
    float2 *Rs = csm + 2 * LC * BT * KT;    // [2][LC][MC][KT]
    const int tid = threadIdx.x;
    const int kx = tid % KT, bg = tid / KT;
    const int k0 = blockIdx.x * KT;
    const long long b0 = (long long)blockIdx.y * BT;
    const int m0 = blockIdx.z * MC;
    const int nlc = (L + LC - 1) / LC;

    // 16-byte copies (2 bins) when the row strides are even; otherwise 8-byte
    const bool wide = ((ldx | ldr) & 1) == 0;
    // wide path: thread copies bins (2kc, 2kc+1) of rows bbA = tid/16 and bbA+16 for
    // each of the LC elements, and of R rows (j, ll) = divmod(tid/16 + 16*it, LC)
    constexpr int RROWS = LC * MC;                       // R rows per stage
    constexpr int RIT = (RROWS + 15) / 16;               // R copies per thread
    const int kc = tid & 15, bbA = tid >> 4;
    const int kw = k0 + 2 * kc;
    const bool kok = kw < Kb;
    const float2 *xA = X + ((b0 + bbA) * L) * ldx + kw;
    const float2 *xB = xA + (long long)16 * L * ldx;
    const bool okA = kok && b0 + bbA < B, okB = kok && b0 + bbA + 16 < B;
    auto stage = [&](int c, int buf) {
        const int l0 = c * LC;
        if (wide) {
            float2 *xs = Xs + buf * LC * BT * KT + bbA * KT + 2 * kc;
#pragma unroll
            for (int ll = 0; ll < LC; ++ll) {
                const bool lok = l0 + ll < L;
                const long long off = (long long)(l0 + ll) * ldx;
                cp_async16z(xs + ll * BT * KT, okA && lok ? xA + off : X, okA && lok);
                if (BT > 16)
                    cp_async16z(xs + ll * BT * KT + 16 * KT, okB && lok ? xB + off : X, okB && lok);
            }
#pragma unroll
            for (int it = 0; it < RIT; ++it) {
                const int rr = bbA + 16 * it;
                if (rr < RROWS) {
                    const int ll = rr / MC, j = rr - ll * MC;
                    const int m = m0 + j, l = l0 + ll;
                    const bool ok = kok && m < M && l < L;
                    const float2 *src = ok ? R + ((long long)m * L + l) * ldr + kw : R;
                    cp_async16z(&Rs[((buf * LC + ll) * MC + j) * KT + 2 * kc], src, ok);
                }
            }
        } else {
            for (int i = tid; i < LC * BT * KT; i += KKB_CT_THREADS) {
                const int kk = i % KT, rr = i / KT, bb = rr % BT, ll = rr / BT;
                const long long b = b0 + bb;
                const int l = l0 + ll, k = k0 + kk;
                const bool ok = b < B && l < L && k < Kb;
                const float2 *src = ok ? X + (b * L + l) * ldx + k : X;
                cp_async8z(&Xs[((buf * LC + ll) * BT + bb) * KT + kk], src, ok);
            }
            for (int i = tid; i < LC * MC * KT; i += KKB_CT_THREADS) {
                const int kk = i % KT, rr = i / KT, j = rr % MC, ll = rr / MC;
                const int m = m0 + j, l = l0 + ll, k = k0 + kk;
                const bool ok = m < M && l < L && k < Kb;
                const float2 *src = ok ? R + ((long long)m * L + l) * ldr + k : R;
                cp_async8z(&Rs[((buf * LC + ll) * MC + j) * KT + kk], src, ok);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    float2 acc[NB][MC];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < MC; ++j) acc[i][j] = make_float2(0.f, 0.f);

    stage(0, 0);
    for (int c = 0; c < nlc; ++c) {
        const int buf = c & 1;
        if (c + 1 < nlc) {
            stage(c + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
#pragma unroll
        for (int ll = 0; ll < LC; ++ll) {
            float2 xv[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) xv[i] = Xs[((buf * LC + ll) * BT + bg * NB + i) * KT + kx];
#pragma unroll
            for (int j = 0; j < MC; ++j) {
                const float2 r = Rs[((buf * LC + ll) * MC + j) * KT + kx];
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    acc[i][j].x = fmaf(xv[i].x, r.x, acc[i][j].x);
                    acc[i][j].x = fmaf(-xv[i].y, r.y, acc[i][j].x);
                    acc[i][j].y = fmaf(xv[i].x, r.y, acc[i][j].y);
                    acc[i][j].y = fmaf(xv[i].y, r.x, acc[i][j].y);
                }
            }
        }
        __syncthreads();  // buffer `buf` is refilled by the next iteration's stage()
    }
    const int k = k0 + kx;
    if (k >= Kb) return;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const long long b = b0 + bg * NB + i;
        if (b >= B) break;
#pragma unroll
        for (int j = 0; j < MC; ++j)
            if (m0 + j < M) Y[(b * M + m0 + j) * ldy + k] = acc[i][j];
    }
}

template <int MC>
static int launch_contract(const float2 *X, long long ldx, const float2 *R, long long ldr, float2 *Y,
                           long long ldy, long long B, int L, int M, int Kb, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(Kb, KKB_CT_KT), (unsigned)ceil_div(B, KKB_CT_BT),
              (unsigned)ceil_div(M, MC));
    if (grid.y > 65535u) {
        set_error("contraction batch too large (%lld rows)", B);
        return KKB_ERR_UNSUPPORTED;
    }
    const int sm = (int)sizeof(float2) * 2 * KKB_CT_LC * KKB_CT_KT * (KKB_CT_BT + MC);
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_contract<MC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                 "smem attr contract");
    k_contract<MC><<<grid, KKB_CT_THREADS, sm, s>>>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb);
    KKB_CHECK_LAUNCH("k_contract");
    return KKB_OK;
}

// ------------------------------------------------------------- symmetric form
// The reference's receive sets are symmetric multisets (sampling.py:55-57)
// and element positions are centred (core.py:32-38), so for a (+theta,
// -theta) pair the ramps satisfy R_{L-1-l}(theta) = conj(R_l(theta)) =
// R_l(-theta).  With S_l = X_l + X_{L-1-l}, D_l = X_l - X_{L-1-l} (l < L/2):
//   Y(+theta) = A + iB,  Y(-theta) = A - iB,
//   A = sum_l S_l cos(phi_l),  B = sum_l D_l sin(phi_l)
// (cos/sin carry the one-sided weight and 1/T).  4 real FMAs per l-pair and
// angle pair instead of 16: the contraction drops ~4x in arithmetic.
// Class p = one +theta/-theta pair (or a lone theta = 0); CS[p][j][k] =
// (cos, sin) * scale for j < ceil(L/2) (the middle element of odd L has
// phi = 0 and no mirror).
#ifndef KKB_CS_NB6
#define KKB_CS_NB6 2   // rows per thread of the 6-class instance (config 4: M = 11)
#endif
#ifndef KKB_CS_LC
#define KKB_CS_LC 4    // element pairs per cp.async stage
#endif

struct SymClasses {
    int P;
    short mp[KKB_MAX_CLASSES];  // output receive index of +theta
    short mm[KKB_MAX_CLASSES];  // output receive index of -theta, -1 for theta = 0
};

// One tile: KT bins from k0, BT rows from b0 (X rows counted from X, Y rows
// from Y; rows >= B are not read or written), classes from p0.
template <int PC, int NB>
__device__ __forceinline__ void contract_sym_tile(const float2 *__restrict__ X, long long ldx,
                                                  const float2 *__restrict__ CS, long long ldc,
                                                  float2 *__restrict__ Y, long long ldy, long long B, int L,
                                                  int M, int Kb, const SymClasses &cls, int k0, long long b0,
                                                  int p0, float2 *csm) {
    constexpr int KT = KKB_CT_KT, BT = 8 * NB, LC = KKB_CS_LC;
    static_assert(BT == 16 || BT == 32, "staging covers 16 or 2 x 16 rows");
    float2 *Xl = csm;                     // [2][LC][BT][KT]
    float2 *Xr = Xl + 2 * LC * BT * KT;   // [2][LC][BT][KT] mirrored elements
    float2 *Cs = Xr + 2 * LC * BT * KT;   // [2][LC][PC][KT]
    const int tid = threadIdx.x;
    const int kx = tid % KT, bg = tid / KT;
    const int Lp = (L + 1) / 2;
    const int nlc = (Lp + LC - 1) / LC;
    const int kc = tid & 15, bbA = tid >> 4;
    const int kw = k0 + 2 * kc;
    const bool kok = kw < Kb;
    const float2 *xA = X + ((b0 + bbA) * L) * ldx + kw;
    const float2 *xB = xA + (long long)16 * L * ldx;
    const bool okA = kok && b0 + bbA < B, okB = kok && b0 + bbA + 16 < B;
    constexpr int CROWS = LC * PC;
    constexpr int CIT = (CROWS + 15) / 16;

    auto stage = [&](int c, int buf) {
        const int j0 = c * LC;
#pragma unroll
        for (int ll = 0; ll < LC; ++ll) {
            const int j = j0 + ll, r = L - 1 - j;
            const bool jok = j < Lp, rok = jok && r != j;
            const long long offl = (long long)j * ldx, offr = (long long)r * ldx;
            float2 *xl = Xl + ((buf * LC + ll) * BT + bbA) * KT + 2 * kc;
            float2 *xr = Xr + ((buf * LC + ll) * BT + bbA) * KT + 2 * kc;
            cp_async16z(xl, okA && jok ? xA + offl : X, okA && jok);
            cp_async16z(xr, okA && rok ? xA + offr : X, okA && rok);
            if (BT > 16) {
                cp_async16z(xl + 16 * KT, okB && jok ? xB + offl : X, okB && jok);
                cp_async16z(xr + 16 * KT, okB && rok ? xB + offr : X, okB && rok);
            }
        }
#pragma unroll
        for (int it = 0; it < CIT; ++it) {
            const int rr = bbA + 16 * it;
            if (rr < CROWS) {
                const int ll = rr / PC, q = rr - ll * PC;
                const int p = p0 + q, j = j0 + ll;
                const bool ok = kok && p < cls.P && j < Lp;
                const float2 *src = ok ? CS + ((long long)p * Lp + j) * ldc + kw : CS;
                cp_async16z(&Cs[((buf * LC + ll) * PC + q) * KT + 2 * kc], src, ok);
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };

    float2 A[NB][PC], Bv[NB][PC];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int q = 0; q < PC; ++q) A[i][q] = Bv[i][q] = make_float2(0.f, 0.f);

    stage(0, 0);
    for (int c = 0; c < nlc; ++c) {
        const int buf = c & 1;
        if (c + 1 < nlc) {
            stage(c + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
#pragma unroll
        for (int ll = 0; ll < LC; ++ll) {
            float2 S[NB], D[NB];
#pragma unroll
            for (int i = 0; i < NB; ++i) {
                const int off = ((buf * LC + ll) * BT + bg * NB + i) * KT + kx;
                const float2 xl = Xl[off], xr = Xr[off];
                S[i] = make_float2(xl.x + xr.x, xl.y + xr.y);
                D[i] = make_float2(xl.x - xr.x, xl.y - xr.y);
            }
#pragma unroll
            for (int q = 0; q < PC; ++q) {
                const float2 cs = Cs[((buf * LC + ll) * PC + q) * KT + kx];
#pragma unroll
                for (int i = 0; i < NB; ++i) {
                    A[i][q].x = fmaf(S[i].x, cs.x, A[i][q].x);
                    A[i][q].y = fmaf(S[i].y, cs.x, A[i][q].y);
                    Bv[i][q].x = fmaf(D[i].x, cs.y, Bv[i][q].x);
                    Bv[i][q].y = fmaf(D[i].y, cs.y, Bv[i][q].y);
                }
            }
        }
        __syncthreads();
    }
    const int k = k0 + kx;
    if (k >= Kb) return;
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        const long long b = b0 + bg * NB + i;
        if (b >= B) break;
#pragma unroll
        for (int q = 0; q < PC; ++q) {
            const int p = p0 + q;
            if (p >= cls.P) break;
            const float2 a = A[i][q], bb = Bv[i][q];
            Y[(b * M + cls.mp[p]) * ldy + k] = make_float2(a.x - bb.y, a.y + bb.x);
            if (cls.mm[p] >= 0) Y[(b * M + cls.mm[p]) * ldy + k] = make_float2(a.x + bb.y, a.y - bb.x);
        }
    }
}

template <int PC, int NB>
__global__ void __launch_bounds__(256, 2)
k_contract_sym(const float2 *__restrict__ X, long long ldx, const float2 *__restrict__ CS,
               long long ldc, float2 *__restrict__ Y, long long ldy, long long B, int L, int M,
               int Kb, const SymClasses cls) {
    extern __shared__ __align__(16) float2 csm[];
    // row tiles last to first: K1 wrote the last rows' spectra most recently,
    // so the first tiles scheduled find them in L2
    contract_sym_tile<PC, NB>(X, ldx, CS, ldc, Y, ldy, B, L, M, Kb, cls, blockIdx.x * KKB_CT_KT,
                              (long long)(gridDim.y - 1 - blockIdx.y) * (8 * NB), blockIdx.z * PC, csm);
}

// Persistent consumer of the stage-1 ring (Stage1Ring, fft.cuh): work item
// i = (row-tile t, bin tile) taken from a global queue in order; waits until
// K1 has written all of tile t's spectra into ring slot t % R, contracts them
// (X read from the slot with L2-only cp.async.cg loads), writes Y rows of the
// tile, and releases the slot for K1's tile t + R.  `started` tells the
// launcher this kernel is resident before K1 floods the SMs.
template <int PC, int NB>
__global__ void __launch_bounds__(256, 2)
k_contract_sym_ring(const float2 *__restrict__ ring, long long ldx, const float2 *__restrict__ CS,
                    long long ldc, float2 *__restrict__ Y, long long ldy, long long B, int L, int M,
                    int Kb, const SymClasses cls, const Stage1Ring rs, int *queue, int *started) {
    constexpr int BT = 8 * NB;
    extern __shared__ __align__(16) float2 csm[];
    __shared__ int item_s;
    if (threadIdx.x == 0) atomicAdd(started, 1);
    const int nkt = (Kb + KKB_CT_KT - 1) / KKB_CT_KT;
    const long long ntiles = (B + BT - 1) / BT;
    const long long nitems = ntiles * nkt;
    for (;;) {
        if (threadIdx.x == 0) item_s = atomicAdd(queue, 1);
        __syncthreads();
        const long long item = item_s;
        if (item >= nitems) return;
        const long long t = item / nkt;
        const int kt = (int)(item - t * nkt);
        const long long rows = B - t * BT < BT ? B - t * BT : BT;
        if (threadIdx.x == 0) ring_wait_geq(rs.fft_done + t, (int)(rows * L / 2), rs.err);
        __syncthreads();
        const float2 *Xs = ring + (t % rs.R) * (long long)BT * L * ldx;
        contract_sym_tile<PC, NB>(Xs, ldx, CS, ldc, Y + t * BT * M * ldy, ldy, rows, L, M, Kb, cls,
                                  kt * KKB_CT_KT, 0, 0, csm);
        __syncthreads();  // every read of the slot done (and item_s reusable)
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(rs.con_done + t, 1);
        }
    }
}

template <int PC, int NB>
static int launch_contract_sym(const float2 *X, long long ldx, const float2 *CS, long long ldc,
                               float2 *Y, long long ldy, long long B, int L, int M, int Kb,
                               const SymClasses &cls, cudaStream_t s) {
    constexpr int BT = 8 * NB;
    dim3 grid((unsigned)ceil_div(Kb, KKB_CT_KT), (unsigned)ceil_div(B, BT),
              (unsigned)ceil_div(cls.P, PC));
    if (grid.y > 65535u) {
        set_error("contraction batch too large (%lld rows)", B);
        return KKB_ERR_UNSUPPORTED;
    }
    const int sm = (int)sizeof(float2) * 2 * KKB_CS_LC * KKB_CT_KT * (2 * BT + PC);
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_contract_sym<PC, NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                 "smem attr contract_sym");
    k_contract_sym<PC, NB><<<grid, 256, sm, s>>>(X, ldx, CS, ldc, Y, ldy, B, L, M, Kb, cls);
    KKB_CHECK_LAUNCH("k_contract_sym");
    return KKB_OK;
}

int contract_sym(const float2 *X, long long ldx, const float2 *CS, long long ldc, float2 *Y,
                 long long ldy, long long B, int L, int M, int Kb, int P, const short *mp,
                 const short *mm, cudaStream_t s) {
    if (B <= 0 || Kb <= 0) return KKB_OK;
    if (P < 1 || P > KKB_MAX_CLASSES || ((ldx | ldc) & 1)) {
        set_error("contract_sym: bad class count %d or odd row stride", P);
        return KKB_ERR_ARG;
    }
    SymClasses cls{};
    cls.P = P;
    for (int p = 0; p < P; ++p) {
        cls.mp[p] = mp[p];
        cls.mm[p] = mm[p];
    }
    // register tile NB x PC complex (A, B) pairs: NB = 4 rows for few classes, 2 otherwise
    if (P <= 3) return launch_contract_sym<3, 4>(X, ldx, CS, ldc, Y, ldy, B, L, M, Kb, cls, s);
    if (P <= 6) return launch_contract_sym<6, KKB_CS_NB6>(X, ldx, CS, ldc, Y, ldy, B, L, M, Kb, cls, s);
    return launch_contract_sym<8, 2>(X, ldx, CS, ldc, Y, ldy, B, L, M, Kb, cls, s);
}

int contract_sym_ring(const float2 *ring, long long ldx, const float2 *CS, long long ldc, float2 *Y,
                      long long ldy, long long B, int L, int M, int Kb, int P, const short *mp,
                      const short *mm, const Stage1Ring &rs, int *queue, int *started, int nctas,
                      cudaStream_t s) {
    if (B <= 0 || Kb <= 0) return KKB_OK;
    if (P < 1 || P > 6 || ((ldx | ldc) & 1)) {
        set_error("contract_sym_ring: 1..6 classes and even row strides");
        return KKB_ERR_ARG;
    }
    SymClasses cls{};
    cls.P = P;
    for (int p = 0; p < P; ++p) {
        cls.mp[p] = mp[p];
        cls.mm[p] = mm[p];
    }
    constexpr int BT = 8 * KKB_CS_NB6;
    const int sm = (int)sizeof(float2) * 2 * KKB_CS_LC * KKB_CT_KT * (2 * BT + 6);
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_contract_sym_ring<6, KKB_CS_NB6>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, sm),
                 "smem attr contract_sym_ring");
    k_contract_sym_ring<6, KKB_CS_NB6><<<nctas, 256, sm, s>>>(ring, ldx, CS, ldc, Y, ldy, B, L, M, Kb, cls, rs,
                                                               queue, started);
    KKB_CHECK_LAUNCH("k_contract_sym_ring");
    return KKB_OK;
}

int contract(const float2 *X, long long ldx, const float2 *R, long long ldr, float2 *Y,
             long long ldy, long long B, int L, int M, int Kb, cudaStream_t s) {
    if (B <= 0 || Kb <= 0) return KKB_OK;
    if (M <= 4) return launch_contract<4>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
    if (M <= 8) return launch_contract<8>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
    if (M <= 12) return launch_contract<12>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
    return launch_contract<16>(X, ldx, R, ldr, Y, ldy, B, L, M, Kb, s);
}

}  // namespace kkb
