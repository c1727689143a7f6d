// K2 on the 5th-generation tensor cores (tcgen05, kind::tf32): the symmetric
// per-bin contraction of decompose.cu (k_contract_sym) as one real GEMM per
// frequency bin, in split precision ("3xTF32") so the traces keep the FP32
// path's accuracy.  This is the north star's "complex fp32 via split real
// GEMM" candidate (compress.py:78-81, bench.py:130-135); the decomposer uses
// it when KKB_CONTRACT=tc, and bench / ncu decide between the two forms.
//
// Per bin k and 64 (frame, transmit) rows b, with S_j = X_j + X_{L-1-j},
// D_j = X_j - X_{L-1-j} (complex, j < ceil(L/2)) and real class tables
// C_jp = cos(phi_jp) * scale_k, S_jp = sin(phi_jp) * scale_k:
//     [ Re S | Re D ]   (64 x 2Lp)       [ C  0 ]            [ Re A | Re B ]
//     [ Im S | Im D ]   (64 x 2Lp)   x   [ 0  S ] (2Lp x 16) = [ Im A | Im B ]
// an M = 128 (rows x {re, im}), N = 2 x 8 or 2 x 16 (classes), K = 2Lp GEMM whose K
// axis interleaves (S_j, D_j); then Y(+theta_p) = A_p + i B_p and
// Y(-theta_p) = A_p - i B_p as in the FMA kernel.  Every operand is split
// x = hi + lo with hi, lo exact tf32 values; the product sums hi*hi + hi*lo +
// lo*hi (lo*lo ~ 2^-44 dropped) with fp32 accumulation in TMEM.
//
// Layout: operands in shared memory in the canonical K-major no-swizzle UMMA
// layout (tc.cuh): A per (bin, hi|lo) = [4 K-chunks of 16 B][128 rows][16 B]
// for a K step of 16 (8 element pairs); B from a table built once per plan in
// the same layout, [stage][bin][hi|lo][4][N][16 B].  Two stage buffers; 8
// producer warps load stage s+1 into registers while they build stage s's A
// operands, and a ninth warp issues the MMAs (one elected thread) and owns
// the TMEM allocation, so the tensor core multiplies stage s while stage s+1
// is being built.

#include <algorithm>

#include "common.cuh"
#include "kk.cuh"
#include "tc.cuh"

namespace kkb {

#define TC_ROWS 64     // (frame, transmit) rows per CTA (x2 for re/im = MMA M of 128)
#define TC_KB 4        // bins per CTA
#define TC_JC 8        // element pairs per stage (K step of 16 = 2 tf32 MMAs)
#define TC_ABYTES (4 * 128 * 16)   // one (bin, hi|lo) A operand: 8 KB
#define TC_PRODUCERS 256           // 8 warps build the A operands; warp 8 issues the MMAs

// B table: [stage c][bin k][hi|lo][chunk c4][n][4 floats], N = 2 NP columns
// (n < NP: cos on S rows = A terms of class n; n >= NP: sin on D rows = B terms
// of class n - NP); stage c covers element pairs j = 8c .. 8c+7, K index
// kk = 2 (j - 8c) + s (s = 0: S row, 1: D row)
__global__ void k_build_tc_table(const float2 *__restrict__ cs, long long ldc, int P, int Lp, int Kb,
                                 int nstage, int NP, float *__restrict__ tab) {
    const int N = 2 * NP, bbytes = 4 * N * 16;
    const long long total = (long long)nstage * Kb * N * 16;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int kk = (int)(i % 16);
        long long r = i / 16;
        const int n = (int)(r % N);
        r /= N;
        const int k = (int)(r % Kb), c = (int)(r / Kb);
        const int j = c * TC_JC + kk / 2, s = kk & 1;
        const int p = n < NP ? n : n - NP;
        float v = 0.f;
        if (j < Lp && p < P && (n < NP) == (s == 0)) {
            const float2 w = cs[((long long)p * Lp + j) * ldc + k];
            v = s == 0 ? w.x : w.y;
        }
        const float hi = tc::to_tf32(v), lo = tc::to_tf32(v - hi);
        float *base = tab + ((long long)c * Kb + k) * 2 * (bbytes / 4);
        const int off = (kk / 4) * N * 4 + n * 4 + (kk & 3);
        base[off] = hi;
        base[bbytes / 4 + off] = lo;
    }
}

static int tc_classes(int P) { return P <= 8 ? 8 : 16; }

int build_tc_table(const float2 *cs, long long ldc, int P, int L, int Kb, float **tab, long long *bytes,
                   cudaStream_t s) {
    const int Lp = (L + 1) / 2, nstage = (Lp + TC_JC - 1) / TC_JC, NP = tc_classes(P);
    const size_t n = (size_t)nstage * Kb * 2 * (4 * 2 * NP * 16 / 4);
    KKB_TRY_CUDA(cudaMalloc(tab, n * sizeof(float)), "cudaMalloc(tc table)");
    *bytes = (long long)(n * sizeof(float));
    const long long total = (long long)nstage * Kb * 2 * NP * 16;
    k_build_tc_table<<<(unsigned)std::min<long long>(ceil_div(total, 256), 148 * 16), 256, 0, s>>>(
        cs, ldc, P, Lp, Kb, nstage, NP, *tab);
    KKB_CHECK_LAUNCH("k_build_tc_table");
    return KKB_OK;
}

struct TcClasses {
    int P;
    short mp[16], mm[16];
};

__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo) {
    hi = tc::to_tf32(x);
    lo = tc::to_tf32(x - hi);
}

// One stage of one producer thread: element pairs (2q, 2q+1) of stage s, its
// row, the CTA's four bins, as (mirror-left, mirror-right) complex values.
struct TcRegs {
    float2 xl[2][TC_KB], xr[2][TC_KB];
};

__device__ __forceinline__ void tc_load(TcRegs &R, const float2 *__restrict__ X, long long ldx, long long row,
                                        bool rok, int L, int Lp, int Kb, int k0, bool wide, int s, int q) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const int j = s * TC_JC + 2 * q + e, jr = L - 1 - j;
#pragma unroll
        for (int kb = 0; kb < TC_KB; ++kb) R.xl[e][kb] = R.xr[e][kb] = make_float2(0.f, 0.f);
        if (rok && j < Lp) {
            const float2 *pl = X + (row * L + j) * ldx + k0;
            const float2 *pr = X + (row * L + jr) * ldx + k0;
            if (wide) {
                const float4 a0 = __ldg(reinterpret_cast<const float4 *>(pl));
                const float4 a1 = __ldg(reinterpret_cast<const float4 *>(pl) + 1);
                R.xl[e][0] = make_float2(a0.x, a0.y);
                R.xl[e][1] = make_float2(a0.z, a0.w);
                R.xl[e][2] = make_float2(a1.x, a1.y);
                R.xl[e][3] = make_float2(a1.z, a1.w);
                if (jr != j) {
                    const float4 c0 = __ldg(reinterpret_cast<const float4 *>(pr));
                    const float4 c1 = __ldg(reinterpret_cast<const float4 *>(pr) + 1);
                    R.xr[e][0] = make_float2(c0.x, c0.y);
                    R.xr[e][1] = make_float2(c0.z, c0.w);
                    R.xr[e][2] = make_float2(c1.x, c1.y);
                    R.xr[e][3] = make_float2(c1.z, c1.w);
                }
            } else {
#pragma unroll
                for (int kb = 0; kb < TC_KB; ++kb)
                    if (k0 + kb < Kb) {
                        R.xl[e][kb] = __ldg(pl + kb);
                        if (jr != j) R.xr[e][kb] = __ldg(pr + kb);
                    }
            }
        }
    }
}

template <int NP>
__global__ void __launch_bounds__(TC_PRODUCERS + 32, 1)
k_contract_tc(const float2 *__restrict__ X, long long ldx, const float *__restrict__ tab,
              float2 *__restrict__ Y, long long ldy, long long B, int L, int M, int Kb, const TcClasses cls) {
    constexpr int N = 2 * NP;
    constexpr int BBYTES = 4 * N * 16;                          // one (bin, hi|lo) B operand
    constexpr int STAGE = TC_KB * 2 * (TC_ABYTES + BBYTES);
    constexpr int TCOLS = TC_KB * N <= 64 ? 64 : 128;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int b = t & (TC_ROWS - 1), q = (t >> 6) & 3;  // producer: tile row, element-pair pair of the stage
    const int k0 = blockIdx.x * TC_KB;
    const long long b0 = (long long)blockIdx.y * TC_ROWS, row = b0 + b;
    const bool rok = row < B;
    const int Lp = (L + 1) / 2, nstage = (Lp + TC_JC - 1) / TC_JC;
    const bool wide = k0 + TC_KB <= ldx;  // all four bins inside the padded row: two 16-byte loads
    const bool producer = t < TC_PRODUCERS;

    if (warp == 8) tc::tmem_alloc<TCOLS>(&tmem_base);
    if (t == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = tc::instr_desc(2, 128, N);

    TcRegs cur, nxt;
    if (producer) tc_load(cur, X, ldx, row, rok, L, Lp, Kb, k0, wide, 0, q);
    for (int s = 0; s < nstage; ++s) {
        const int buf = s & 1;
        unsigned char *Ab = sm + buf * STAGE;
        unsigned char *Bb = Ab + TC_KB * 2 * TC_ABYTES;
        if (producer) {
            if (s + 1 < nstage) tc_load(nxt, X, ldx, row, rok, L, Lp, Kb, k0, wide, s + 1, q);  // in flight
            if (s >= 2) tc::mbar_wait(&bar[buf], ((s - 2) >> 1) & 1);  // MMAs of stage s-2 read this buffer
            // B operands of the stage: contiguous in the table
            const uint4 *src = reinterpret_cast<const uint4 *>(tab + ((long long)s * Kb + k0) * 2 * (BBYTES / 4));
            uint4 *dst = reinterpret_cast<uint4 *>(Bb);
            const int n16 = TC_KB * 2 * BBYTES / 16, valid = min(TC_KB, Kb - k0) * 2 * BBYTES / 16;
            for (int i = t; i < n16; i += TC_PRODUCERS) dst[i] = i < valid ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
            // A: K chunk q holds kk = 4q .. 4q+3 = (S, D) of pairs 2q, 2q+1; rows b (re), 64 + b (im)
#pragma unroll
            for (int kb = 0; kb < TC_KB; ++kb) {
                const float2 l0 = cur.xl[0][kb], r0 = cur.xr[0][kb], l1 = cur.xl[1][kb], r1 = cur.xr[1][kb];
                float h[8], lo[8];
                split_tf32(l0.x + r0.x, h[0], lo[0]);
                split_tf32(l0.x - r0.x, h[1], lo[1]);
                split_tf32(l1.x + r1.x, h[2], lo[2]);
                split_tf32(l1.x - r1.x, h[3], lo[3]);
                split_tf32(l0.y + r0.y, h[4], lo[4]);
                split_tf32(l0.y - r0.y, h[5], lo[5]);
                split_tf32(l1.y + r1.y, h[6], lo[6]);
                split_tf32(l1.y - r1.y, h[7], lo[7]);
                unsigned char *ahi = Ab + (kb * 2) * TC_ABYTES + q * 128 * 16;
                unsigned char *alo = ahi + TC_ABYTES;
                *reinterpret_cast<float4 *>(ahi + b * 16) = make_float4(h[0], h[1], h[2], h[3]);
                *reinterpret_cast<float4 *>(ahi + (64 + b) * 16) = make_float4(h[4], h[5], h[6], h[7]);
                *reinterpret_cast<float4 *>(alo + b * 16) = make_float4(lo[0], lo[1], lo[2], lo[3]);
                *reinterpret_cast<float4 *>(alo + (64 + b) * 16) = make_float4(lo[4], lo[5], lo[6], lo[7]);
            }
            tc::fence_smem_to_async();
        }
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (warp == 8 && lane == 0) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(Ab), sb = (uint32_t)__cvta_generic_to_shared(Bb);
            const uint64_t da = tc::smem_desc(sa, 128 * 16, 128), db = tc::smem_desc(sb, N * 16, 128);
#pragma unroll
            for (int kb = 0; kb < TC_KB; ++kb)
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    // start-address field += byte offset / 16 (no carry: smem < 256 KB)
                    const uint64_t ah = da + (((kb * 2) * TC_ABYTES + ks * 2 * 128 * 16) >> 4);
                    const uint64_t al = ah + (TC_ABYTES >> 4);
                    const uint64_t bh = db + (((kb * 2) * BBYTES + ks * 2 * N * 16) >> 4);
                    const uint64_t bl = bh + (BBYTES >> 4);
                    const uint32_t d = tmem + kb * N;
                    tc::mma_tf32(d, ah, bh, idesc, s > 0 || ks > 0);
                    tc::mma_tf32(d, ah, bl, idesc, true);
                    tc::mma_tf32(d, al, bh, idesc, true);
                }
            tc::commit(&bar[buf]);
        }
        if (producer) cur = nxt;
    }
    tc::mbar_wait(&bar[(nstage - 1) & 1], ((nstage - 1) >> 1) & 1);
    tc::fence_after_sync();
    // epilogue: TMEM -> smem staging E[bin][128 rows][N] -> Y (producer warps)
    float *E = reinterpret_cast<float *>(sm);
    if (producer) {
        const int quarter = warp & 3, kb0 = (warp >> 2) * 2;
        const int r = quarter * 32 + lane;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int kb = kb0 + kk;
#pragma unroll
            for (int c0 = 0; c0 < N; c0 += 8) {
                float v[8];
                tc::tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + kb * N + c0, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int n = 0; n < 8; n += 4)
                    *reinterpret_cast<float4 *>(E + (kb * 128 + r) * N + c0 + n) =
                        make_float4(v[n], v[n + 1], v[n + 2], v[n + 3]);
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 8) tc::tmem_free<TCOLS>(tmem);
    const int k = k0 + q;
    if (!producer || !rok || k >= Kb) return;
    const float *er = E + (q * 128 + b) * N, *ei = E + (q * 128 + 64 + b) * N;
    for (int p = 0; p < cls.P; ++p) {
        const float ar = er[p], ai = ei[p], br = er[NP + p], bi = ei[NP + p];
        Y[(row * M + cls.mp[p]) * ldy + k] = make_float2(ar - bi, ai + br);
        if (cls.mm[p] >= 0) Y[(row * M + cls.mm[p]) * ldy + k] = make_float2(ar + bi, ai - br);
    }
}

template <int NP>
static int launch_contract_tc(const float2 *X, long long ldx, const float *tab, float2 *Y, long long ldy,
                              long long B, int L, int M, int Kb, const TcClasses &cls, cudaStream_t s) {
    dim3 grid((unsigned)ceil_div(Kb, TC_KB), (unsigned)ceil_div(B, TC_ROWS));
    if (grid.y > 65535u) {
        set_error("contraction batch too large (%lld rows)", B);
        return KKB_ERR_UNSUPPORTED;
    }
    const int smem = 2 * TC_KB * 2 * (TC_ABYTES + 4 * 2 * NP * 16);
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_contract_tc<NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                 "smem attr contract_tc");
    k_contract_tc<NP><<<grid, TC_PRODUCERS + 32, smem, s>>>(X, ldx, tab, Y, ldy, B, L, M, Kb, cls);
    KKB_CHECK_LAUNCH("k_contract_tc");
    return KKB_OK;
}

int contract_tc(const float2 *X, long long ldx, const float *tab, float2 *Y, long long ldy, long long B,
                int L, int M, int Kb, int P, const short *mp, const short *mm, cudaStream_t s) {
    if (B <= 0 || Kb <= 0) return KKB_OK;
    if (P < 1 || P > 16 || (ldx & 1)) {
        set_error("contract_tc: needs 1..16 symmetric classes and an even row stride");
        return KKB_ERR_ARG;
    }
    TcClasses cls{};
    cls.P = P;
    for (int p = 0; p < P; ++p) {
        cls.mp[p] = mp[p];
        cls.mm[p] = mm[p];
    }
    if (P <= 8) return launch_contract_tc<8>(X, ldx, tab, Y, ldy, B, L, M, Kb, cls, s);
    return launch_contract_tc<16>(X, ldx, tab, Y, ldy, B, L, M, Kb, cls, s);
}

}  // namespace kkb
