// Fused stage 1: K1 (real-pair FFT of the element traces) and K2 (symmetric
// +/-theta contraction over elements) in ONE kernel, so the per-element
// spectra never leave the SM (K1 wrote 3.42 GB of spectra
// per 400 config-4 frames and K2 read them back, 7 of stage 1's 11.6 GB).
//
// Replaces, for one (frame, transmit) row b, the reference's
//   X = rfft(rf, axis=-1) * one_sided / T          (spectral.py:84-93)
//   Y[m, k] = sum_l X[l, k] exp(2 pi i f_k tau_lm)  (compress.py:78-81)
// with the three-kernel path's FFT (fft_ct.cuh, elements 2p, 2p+1 as re / im
// of one complex transform, the same real-pair split) and its symmetric
// contraction (k_contract_sym: S_j = X_j + X_{L-1-j}, D_j = X_j - X_{L-1-j},
// Y(+/-theta) = A +/- iB, A = sum S cos phi, B = sum D sin phi).
//
// CTA = one row b, warp-specialised (setmaxnreg):
//   * four FFT warpgroups (4 x 128 threads, 64 registers): round r, group g
//     transforms FFT pair 2r, 2r+1, L/2-1-2r or L/2-2-2r (elements 4r .. 4r+3
//     and their mirrors L-4-4r .. L-1-4r: exactly what contraction indices
//     j = 4r .. 4r+3 need).  The group's next RF pair is bulk-copied
//     (cp.async.bulk, one mbarrier per group) into its slot while it works;
//     stage 2 writes the bins in natural order into Z[r % 2][g];
//   * two contraction warpgroups (256 threads, 112 registers) own the
//     register accumulators of every (bin, class): thread c takes bins c,
//     c + 256, c + 512 with all classes and, for c < 6, class c of the
//     Nyquist bin.  Round r waits for full[r % 2], contracts the four Z
//     buffers and releases them through empty[r % 2], so the FFT of round
//     r + 1 overlaps the contraction of round r.
//
// The phase factors are not read from a table (the class table is 2.4 MB per
// plan: ~10 GB of L2 reads per 400-frame step): for a uniform array the phase
// is linear in the element index, so each round anchors exp(2 pi i phi) at
// j = 4r and steps it three times by the per-element rotation rho.  Both
// phases (in cycles) are gamma * k with gamma from the plan's float64 delays;
// gamma is split into a 13-bit head (gamma_hi * k is exact in fp32, so its
// whole cycles drop out exactly) and a tail, so the reduced phase is exact to
// ~1e-9 cycles before the MUFU sin/cos (~4e-7 absolute).  The one-sided
// weight / T is applied once to the sums.  Only Y (0.74 MB per config-4
// frame) is written; the frame's RF (8.65 MB) is read once.

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "fft_ct.cuh"

#ifndef S1F_EXP
#define S1F_EXP 0  // experiment builds: 1 = FFT only (contraction skipped), 2 = contraction only
#endif

namespace kkb {
namespace ct {

constexpr int S1F_GROUPS = 4;  // FFT warpgroups (transforms side by side)
constexpr int S1F_PC = 6;      // symmetric classes (M <= 12 receive angles)
constexpr int S1F_CON = 256;   // contraction threads (two warpgroups)
// register split (setmaxnreg): the CTA's pool is 768 x 80 (the launch bound);
// 512 x 64 + 256 x 112 uses it exactly (an .inc beyond the pool would block)
constexpr int S1F_FFT_REGS = 64, S1F_CON_REGS = 112;
static_assert(4 * 128 * S1F_FFT_REGS + S1F_CON * S1F_CON_REGS == 768 * 80, "register pool");

struct S1FClasses {
    int P;
    short mp[S1F_PC];  // output receive index of +theta
    short mm[S1F_PC];  // output receive index of -theta, -1 for theta = 0
};

template <int T>
struct S1F {
    static constexpr int NT = Plan<T>::NT;
    static constexpr int NFFT = S1F_GROUPS * NT;
    static constexpr int NTH = NFFT + S1F_CON;
    static constexpr int K = T / 2 + 1;
};

__device__ __forceinline__ void mb_wait(unsigned mb, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n\t}\n" ::"r"(mb),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mb_arrive(unsigned mb) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(mb) : "memory");
}
__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// phase (cycles) of gamma * k reduced to [-1/2, 1/2]: gamma = hi + lo with hi
// carrying 13 significant bits, so hi * k (|k| < 2^10) is exact
__device__ __forceinline__ float2 unit_phasor(float2 g, float kf) {
    const float x = g.x * kf;
    const float ph = fmaf(g.y, kf, x - rintf(x));
    float sn, cs;
    __sincosf(6.28318530717958648f * ph, &sn, &cs);
    return make_float2(cs, sn);
}

template <int T, typename InT>
__global__ void __launch_bounds__(S1F<T>::NTH, 1)
k_stage1_fused(const InT *__restrict__ rf, int L, const float2 *__restrict__ gam, float2 *__restrict__ Y,
               long long ldy, int M, const S1FClasses cls, const float2 *__restrict__ tw) {
    using P = Plan<T>;
    constexpr int NT = P::NT, NFFT = S1F<T>::NFFT, K = S1F<T>::K, PC = S1F_PC;
    static_assert(K - 1 == 3 * S1F_CON && T % 2 == 0, "bin ownership: 3 x 256 bins + the Nyquist bin");
    // shared memory: Z[2][4][T] bins (float2), W[4][T] FFT workspaces, then the
    // groups' RF slots [4][2T] (InT)
    extern __shared__ __align__(16) float2 sm[];
    float2 *Z = sm, *Wk = sm + (size_t)2 * S1F_GROUPS * T;
    InT *slots = reinterpret_cast<InT *>(sm + (size_t)3 * S1F_GROUPS * T);
    __shared__ __align__(8) unsigned long long mb_slot[S1F_GROUPS], mb_full[2], mb_empty[2];
    __shared__ float2 sgam[S1F_PC * 33];  // per class: anchors of rounds 0 .. L/8-1, then rho's gamma
    __shared__ short smp[PC], smm[PC];
    const int tid = threadIdx.x;
    const long long b = blockIdx.x;
    const int Lh = L >> 1, nrounds = L >> 3;
    const InT *row = rf + b * (long long)L * T;

    if (tid == 0) {
        for (int g = 0; g < S1F_GROUPS; ++g)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb_slot[g])) : "memory");
        for (int i = 0; i < 2; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&mb_full[i])), "r"(NFFT) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&mb_empty[i])), "r"(S1F_CON) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < cls.P * (nrounds + 1); i += blockDim.x) sgam[i] = __ldg(gam + i);
#pragma unroll
    for (int q = 0; q < PC; ++q)
        if (tid == q) {
            smp[q] = cls.mp[q];
            smm[q] = cls.mm[q];
        }
    __syncthreads();

    if (tid < NFFT) {
        // ------------------------------------------------------------ FFT
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(S1F_FFT_REGS));
        const int g = tid / NT;
        const bool leader = (tid & (NT - 1)) == 0;
        float2 *W = Wk + (size_t)g * T;
        InT *slot = slots + (size_t)g * 2 * T;
        constexpr unsigned BYTES = 2u * T * sizeof(InT);
        auto fetch = [&](int r) {  // rows 2p, 2p + 1 are adjacent: one bulk copy
            const int p = g < 2 ? 2 * r + g : Lh - 1 - 2 * r - (g - 2);
            const InT *src = row + (long long)(2 * p) * T;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb_slot[g])), "r"(BYTES)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    sa(slot)),
                "l"(src), "r"(BYTES), "r"(sa(&mb_slot[g]))
                : "memory");
        };
        if (leader) fetch(0);
        using S0 = Stage<T, NT, P::R0>;
        using S1 = Stage<T, NT, P::R1>;
#pragma unroll 1
        for (int r = 0; r < nrounds; ++r) {
            mb_wait(sa(&mb_slot[g]), (unsigned)(r & 1));
#if S1F_EXP == 2
            if (r >= 0) {
                xform_sync<NT>(1 + g);
                if (leader && r + 1 < nrounds) fetch(r + 1);
                mb_wait(sa(&mb_empty[r & 1]), (unsigned)(((r >> 1) & 1) ^ 1));
                mb_arrive(sa(&mb_full[r & 1]));
                continue;
            }
#endif
            S0 a;
#pragma unroll
            for (int t = 0; t < S0::ITER; ++t) {
                const int j = S0::lane_j(t);
                if (S0::ok(j)) {
#pragma unroll
                    for (int rr = 0; rr < P::R0; ++rr) {
                        const int e = j + rr * S0::TR;
                        a.v[t][rr] = make_float2(to_f(slot[e]), to_f(slot[T + e]));
                    }
                }
            }
            a.template compute<1, 0>(tw);
            xform_sync<NT>(1 + g);  // the slot is read, the previous round's stage 2 has read W
            if (leader && r + 1 < nrounds) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                fetch(r + 1);
            }
            a.template store<1, true>(W);
            xform_sync<NT>(1 + g);
            {  // stage 1 in place
                S1 c1;
                c1.template load<true>(W);
                xform_sync<NT>(1 + g);
                c1.template compute<P::R0, 0>(tw);
                c1.template store<P::R0, false>(W);
            }
            xform_sync<NT>(1 + g);
            // stage 2 out of place into Z[r % 2][g] once the contraction of
            // round r - 2 released it (Stage::compute's arithmetic)
            mb_wait(sa(&mb_empty[r & 1]), (unsigned)(((r >> 1) & 1) ^ 1));
            float2 *zb = Z + ((size_t)(r & 1) * S1F_GROUPS + g) * T;
            constexpr int R2 = P::R2, TR2 = T / R2, IT2 = (TR2 + NT - 1) / NT;
            constexpr int NS2 = P::R0 * P::R1, OFF2 = (P::R1 - 1) * P::R0;
#pragma unroll
            for (int t = 0; t < IT2; ++t) {
                const int j = (tid & (NT - 1)) + t * NT;
                if (TR2 % NT == 0 || j < TR2) {
                    float2 v[R2];
#pragma unroll
                    for (int rr = 0; rr < R2; ++rr) v[rr] = W[j + rr * TR2];
                    const int kk = j % NS2;
#pragma unroll
                    for (int rr = 1; rr < R2; ++rr) v[rr] = cmul(v[rr], __ldg(tw + OFF2 + (rr - 1) * NS2 + kk));
                    Dft<R2>::run(v);
#pragma unroll
                    for (int rr = 0; rr < R2; ++rr) zb[j + rr * TR2] = v[rr];
                }
            }
            mb_arrive(sa(&mb_full[r & 1]));
        }
        return;
    }

    // ------------------------------------------------------------ contraction
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(S1F_CON_REGS));
    const int c = tid - NFFT;
    const int qn = c < PC ? c : PC;  // Nyquist-bin class of this thread (PC: none)
    float2 A[3][PC], B[3][PC], An = make_float2(0.f, 0.f), Bn = make_float2(0.f, 0.f);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int q = 0; q < PC; ++q) A[i][q] = B[i][q] = make_float2(0.f, 0.f);

    // S / D of j = 4r .. 4r+3 at bin k from the four transforms (k_r2c's split)
    auto sd = [&](const float2 *zr, int k, float2(&S)[4], float2(&D)[4]) {
        const int kn = k == 0 ? 0 : T - k;
        float2 X[S1F_GROUPS][2];  // X[gg][0] = element 2p, X[gg][1] = element 2p + 1 of group gg's pair
#pragma unroll
        for (int gg = 0; gg < S1F_GROUPS; ++gg) {
            const float2 zk = zr[gg * T + k], zn = zr[gg * T + kn];
            X[gg][0] = make_float2(0.5f * (zk.x + zn.x), 0.5f * (zk.y - zn.y));
            X[gg][1] = make_float2(0.5f * (zk.y + zn.y), -0.5f * (zk.x - zn.x));
        }
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const float2 xl = X[d >> 1][d & 1], xr = X[2 + (d >> 1)][1 - (d & 1)];
            S[d] = make_float2(xl.x + xr.x, xl.y + xr.y);
            D[d] = make_float2(xl.x - xr.x, xl.y - xr.y);
        }
    };
    // A += sum_d S_d cos phi_d, B += sum_d D_d sin phi_d over j = 4r .. 4r+3:
    // the anchor stepped by rho.  The theta = 0 class (phi = 0, sin phi = 0)
    // only sums S.
    auto accum = [&](const float2(&S)[4], const float2(&D)[4], bool centre, float2 g0, float2 gr, float kf,
                     float2 &a, float2 &bb) {
        if (centre) {
#pragma unroll
            for (int d = 0; d < 4; ++d) {
                a.x += S[d].x;
                a.y += S[d].y;
            }
            return;
        }
        float2 u = unit_phasor(g0, kf);
        const float2 rho = unit_phasor(gr, kf);
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            a.x = fmaf(S[d].x, u.x, a.x);
            a.y = fmaf(S[d].y, u.x, a.y);
            bb.x = fmaf(D[d].x, u.y, bb.x);
            bb.y = fmaf(D[d].y, u.y, bb.y);
            if (d < 3) u = cmul(u, rho);
        }
    };
    const int nr1 = nrounds + 1;
#pragma unroll 1
    for (int r = 0; r < nrounds; ++r) {
        mb_wait(sa(&mb_full[r & 1]), (unsigned)((r >> 1) & 1));
        const float2 *zr = Z + (size_t)(r & 1) * S1F_GROUPS * T;
#if S1F_EXP == 1
        if (r >= 0) {
            mb_arrive(sa(&mb_empty[r & 1]));
            continue;
        }
#endif
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const int k = c + i * S1F_CON;
            float2 S[4], D[4];
            sd(zr, k, S, D);
            const float kf = (float)k;  // k < T/2: fftfreq's non-negative bins
#pragma unroll
            for (int q = 0; q < PC; ++q) {
                if (q < cls.P)
                    accum(S, D, smm[q] < 0, sgam[q * nr1 + r], sgam[q * nr1 + nrounds], kf, A[i][q], B[i][q]);
            }
        }
        if (qn < cls.P) {  // Nyquist bin: fftfreq places it at -T/2
            float2 S[4], D[4];
            sd(zr, T / 2, S, D);
            const float kf = (float)(-T / 2);
            accum(S, D, smm[qn] < 0, sgam[qn * nr1 + r], sgam[qn * nr1 + nrounds], kf, An, Bn);
        }
        mb_arrive(sa(&mb_empty[r & 1]));
    }
    // Y(+theta) = A + iB, Y(-theta) = A - iB (times the one-sided weight / T)
    auto emit = [&](int k, int q, float2 a, float2 bb) {
        const float sc = (float)((k == 0 || 2 * k == T ? 1.0 : 2.0) / T);
        Y[(b * M + smp[q]) * ldy + k] = make_float2(sc * (a.x - bb.y), sc * (a.y + bb.x));
        if (smm[q] >= 0) Y[(b * M + smm[q]) * ldy + k] = make_float2(sc * (a.x + bb.y), sc * (a.y - bb.x));
    };
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int q = 0; q < PC; ++q)
            if (q < cls.P) emit(c + i * S1F_CON, q, A[i][q], B[i][q]);
    if (qn < cls.P) emit(T / 2, qn, An, Bn);
}

}  // namespace ct

bool stage1_fused_supported(int T, int L, int P) {
    return T == 1536 && L >= 8 && L <= 256 && (L & 7) == 0 && P >= 1 && P <= ct::S1F_PC;
}

// gamma = tau * fsT (cycles per bin index) split into a 13-significant-bit
// head and a float tail
static float2 split_gamma(double g) {
    if (g == 0.0) return make_float2(0.f, 0.f);
    int e;
    std::frexp(g, &e);  // |g| = m 2^e, m in [0.5, 1)
    const double hi = std::ldexp(std::nearbyint(std::ldexp(g, 13 - e)), e - 13);
    return make_float2((float)hi, (float)(g - hi));
}

// per class q: the anchors' gamma at j = 4r (r < L/8), then the per-element
// step's; tau = (P, L/2 + 1) float64 delays tau[q][j] and the step tau[q][L/2]
void stage1_fused_table(const double *tau, int P, int L, double fsT, std::vector<float2> &out) {
    const int Lh = L / 2, nr = L / 8;
    out.assign((size_t)P * (nr + 1), make_float2(0.f, 0.f));
    for (int q = 0; q < P; ++q) {
        for (int r = 0; r < nr; ++r)
            out[(size_t)q * (nr + 1) + r] = split_gamma(tau[(size_t)q * (Lh + 1) + 4 * r] * fsT);
        out[(size_t)q * (nr + 1) + nr] = split_gamma(tau[(size_t)q * (Lh + 1) + Lh] * fsT);
    }
}

template <int T, typename InT>
static int launch_stage1_fused(const InT *rf, long long B, int L, const float2 *gam, float2 *Y, long long ldy,
                               int M, const ct::S1FClasses &cls, const float2 *tws, cudaStream_t s) {
    const int smem = (int)(sizeof(float2) * 3 * ct::S1F_GROUPS * T + sizeof(InT) * ct::S1F_GROUPS * 2 * T);
    auto fn = ct::k_stage1_fused<T, InT>;
    KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem), "smem attr stage1 fused");
    fn<<<(unsigned)B, ct::S1F<T>::NTH, smem, s>>>(rf, L, gam, Y, ldy, M, cls, tws);
    KKB_CHECK_LAUNCH("k_stage1_fused");
    return KKB_OK;
}

int stage1_fused(const void *rf, int in_kind, long long B, int L, int T, const float2 *gam, float2 *Y,
                 long long ldy, int M, int P, const short *mp, const short *mm, const float2 *tws, cudaStream_t s) {
    if (B <= 0) return KKB_OK;
    if (!stage1_fused_supported(T, L, P) || B > 0x7fffffffLL) {
        set_error("stage1_fused: unsupported shape (T=%d, L=%d, P=%d)", T, L, P);
        return KKB_ERR_UNSUPPORTED;
    }
    ct::S1FClasses cls{};
    cls.P = P;
    for (int q = 0; q < ct::S1F_PC; ++q) {
        cls.mp[q] = q < P ? mp[q] : 0;
        cls.mm[q] = q < P ? mm[q] : -1;
    }
    if (in_kind) return launch_stage1_fused<1536, short>((const short *)rf, B, L, gam, Y, ldy, M, cls, tws, s);
    return launch_stage1_fused<1536, float>((const float *)rf, B, L, gam, Y, ldy, M, cls, tws, s);
}

}  // namespace kkb
