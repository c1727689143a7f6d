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
// an M = 128 (rows x {re, im}), N = 16 (8 + 8 classes), K = 2Lp GEMM whose K
// axis interleaves (S_j, D_j); then Y(+theta_p) = A_p + i B_p and
// Y(-theta_p) = A_p - i B_p as in the FMA kernel.  Every operand is split
// x = hi + lo with hi, lo exact tf32 values; the product sums hi*hi + hi*lo +
// lo*hi (lo*lo ~ 2^-44 dropped) with fp32 accumulation in TMEM.
//
// Layout: operands in shared memory in the canonical K-major no-swizzle UMMA
// layout (tc.cuh): A per (bin, hi|lo) = [4 K-chunks of 16 B][128 rows][16 B]
// for a K step of 16 (8 element pairs); B from a table built once per plan in
// the same layout, [stage][bin][hi|lo][4][16][16 B].  Two stage buffers: the
// 256 threads build stage s+1's A while the tensor core multiplies stage s.

#include <algorithm>

#include "common.cuh"
#include "kk.cuh"
#include "tc.cuh"

namespace kkb {

#define TC_ROWS 64     // (frame, transmit) rows per CTA (x2 for re/im = MMA M of 128)
#define TC_KB 4        // bins per CTA
#define TC_JC 8        // element pairs per stage (K step of 16 = 2 tf32 MMAs)
#define TC_N 16        // MMA N: classes p < 8 (A terms) | 8 + p (B terms)
#define TC_ABYTES (4 * 128 * 16)   // one (bin, hi|lo) A operand: 8 KB
#define TC_BBYTES (4 * TC_N * 16)  // one (bin, hi|lo) B operand: 1 KB
#define TC_STAGE_BYTES (TC_KB * 2 * (TC_ABYTES + TC_BBYTES))

// B table: [stage c][bin k][hi|lo][chunk c4][n][4 floats]; stage c covers
// element pairs j = 8c .. 8c+7, K index kk = 2 (j - 8c) + s (s = 0: S row, 1: D row)
__global__ void k_build_tc_table(const float2 *__restrict__ cs, long long ldc, int P, int Lp, int Kb,
                                 int nstage, float *__restrict__ tab) {
    const long long total = (long long)nstage * Kb * TC_N * 16;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int kk = (int)(i % 16);
        long long r = i / 16;
        const int n = (int)(r % TC_N);
        r /= TC_N;
        const int k = (int)(r % Kb), c = (int)(r / Kb);
        const int j = c * TC_JC + kk / 2, s = kk & 1;
        const int p = n < 8 ? n : n - 8;
        float v = 0.f;
        if (j < Lp && p < P && (n < 8) == (s == 0)) {
            const float2 w = cs[((long long)p * Lp + j) * ldc + k];
            v = s == 0 ? w.x : w.y;
        }
        const float hi = tc::to_tf32(v), lo = tc::to_tf32(v - hi);
        float *base = tab + ((long long)c * Kb + k) * 2 * (TC_BBYTES / 4);
        const int off = (kk / 4) * TC_N * 4 + n * 4 + (kk & 3);
        base[off] = hi;
        base[TC_BBYTES / 4 + off] = lo;
    }
}

int build_tc_table(const float2 *cs, long long ldc, int P, int L, int Kb, float **tab, long long *bytes,
                   cudaStream_t s) {
    const int Lp = (L + 1) / 2, nstage = (Lp + TC_JC - 1) / TC_JC;
    const size_t n = (size_t)nstage * Kb * 2 * (TC_BBYTES / 4);
    KKB_TRY_CUDA(cudaMalloc(tab, n * sizeof(float)), "cudaMalloc(tc table)");
    *bytes = (long long)(n * sizeof(float));
    const long long total = (long long)nstage * Kb * TC_N * 16;
    k_build_tc_table<<<(unsigned)std::min<long long>(ceil_div(total, 256), 148 * 16), 256, 0, s>>>(
        cs, ldc, P, Lp, Kb, nstage, *tab);
    KKB_CHECK_LAUNCH("k_build_tc_table");
    return KKB_OK;
}

struct TcClasses {
    int P;
    short mp[8], mm[8];
};

__device__ __forceinline__ void split_tf32(float x, float &hi, float &lo) {
    hi = tc::to_tf32(x);
    lo = tc::to_tf32(x - hi);
}

__global__ void __launch_bounds__(256, 1)
k_contract_tc(const float2 *__restrict__ X, long long ldx, const float *__restrict__ tab,
              float2 *__restrict__ Y, long long ldy, long long B, int L, int M, int Kb, const TcClasses cls) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t bar[2];
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int b = t & (TC_ROWS - 1), q = t >> 6;  // row of the tile; element-pair pair q of the stage
    const int k0 = blockIdx.x * TC_KB;
    const long long b0 = (long long)blockIdx.y * TC_ROWS, row = b0 + b;
    const bool rok = row < B;
    const int Lp = (L + 1) / 2, nstage = (Lp + TC_JC - 1) / TC_JC;
    const bool wide = k0 + TC_KB <= ldx;  // all four bins inside the padded row: two 16-byte loads

    if (warp == 0) tc::tmem_alloc<64>(&tmem_base);
    if (t == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;
    const uint32_t idesc = tc::instr_desc(2, 128, TC_N);

    for (int s = 0; s < nstage; ++s) {
        const int buf = s & 1;
        unsigned char *Ab = sm + buf * TC_STAGE_BYTES;
        unsigned char *Bb = Ab + TC_KB * 2 * TC_ABYTES;
        if (s >= 2) tc::mbar_wait(&bar[buf], ((s - 2) >> 1) & 1);  // MMAs of stage s-2 read this buffer
        // B operands of the stage: 8 KB contiguous in the table
        {
            const uint4 *src = reinterpret_cast<const uint4 *>(tab + ((long long)s * Kb + k0) * 2 * (TC_BBYTES / 4));
            uint4 *dst = reinterpret_cast<uint4 *>(Bb);
            const int n16 = TC_KB * 2 * TC_BBYTES / 16, valid = std::min(TC_KB, Kb - k0) * 2 * TC_BBYTES / 16;
            for (int i = t; i < n16; i += 256) dst[i] = i < valid ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
        }
        // A operands: this thread's row, element pairs j = 8s + 2q, 8s + 2q + 1, four bins
        float sr[2][TC_KB], si[2][TC_KB], dr[2][TC_KB], di[2][TC_KB];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int j = s * TC_JC + 2 * q + e, jr = L - 1 - j;
            float2 xl[TC_KB], xr[TC_KB];
#pragma unroll
            for (int kb = 0; kb < TC_KB; ++kb) xl[kb] = xr[kb] = make_float2(0.f, 0.f);
            if (rok && j < Lp) {
                const float2 *pl = X + (row * L + j) * ldx + k0;
                const float2 *pr = X + (row * L + jr) * ldx + k0;
                if (wide) {
                    const float4 a0 = __ldg(reinterpret_cast<const float4 *>(pl));
                    const float4 a1 = __ldg(reinterpret_cast<const float4 *>(pl) + 1);
                    xl[0] = make_float2(a0.x, a0.y);
                    xl[1] = make_float2(a0.z, a0.w);
                    xl[2] = make_float2(a1.x, a1.y);
                    xl[3] = make_float2(a1.z, a1.w);
                    if (jr != j) {
                        const float4 c0 = __ldg(reinterpret_cast<const float4 *>(pr));
                        const float4 c1 = __ldg(reinterpret_cast<const float4 *>(pr) + 1);
                        xr[0] = make_float2(c0.x, c0.y);
                        xr[1] = make_float2(c0.z, c0.w);
                        xr[2] = make_float2(c1.x, c1.y);
                        xr[3] = make_float2(c1.z, c1.w);
                    }
                } else {
#pragma unroll
                    for (int kb = 0; kb < TC_KB; ++kb)
                        if (k0 + kb < Kb) {
                            xl[kb] = __ldg(pl + kb);
                            if (jr != j) xr[kb] = __ldg(pr + kb);
                        }
                }
            }
#pragma unroll
            for (int kb = 0; kb < TC_KB; ++kb) {
                sr[e][kb] = xl[kb].x + xr[kb].x;
                si[e][kb] = xl[kb].y + xr[kb].y;
                dr[e][kb] = xl[kb].x - xr[kb].x;
                di[e][kb] = xl[kb].y - xr[kb].y;
            }
        }
        // K chunk q holds kk = 4q .. 4q+3 = (S, D) of pairs 2q, 2q+1; rows b (re), 64 + b (im)
#pragma unroll
        for (int kb = 0; kb < TC_KB; ++kb) {
            float h[8], l[8];
            split_tf32(sr[0][kb], h[0], l[0]);
            split_tf32(dr[0][kb], h[1], l[1]);
            split_tf32(sr[1][kb], h[2], l[2]);
            split_tf32(dr[1][kb], h[3], l[3]);
            split_tf32(si[0][kb], h[4], l[4]);
            split_tf32(di[0][kb], h[5], l[5]);
            split_tf32(si[1][kb], h[6], l[6]);
            split_tf32(di[1][kb], h[7], l[7]);
            unsigned char *ahi = Ab + (kb * 2) * TC_ABYTES + q * 128 * 16;
            unsigned char *alo = ahi + TC_ABYTES;
            *reinterpret_cast<float4 *>(ahi + b * 16) = make_float4(h[0], h[1], h[2], h[3]);
            *reinterpret_cast<float4 *>(ahi + (64 + b) * 16) = make_float4(h[4], h[5], h[6], h[7]);
            *reinterpret_cast<float4 *>(alo + b * 16) = make_float4(l[0], l[1], l[2], l[3]);
            *reinterpret_cast<float4 *>(alo + (64 + b) * 16) = make_float4(l[4], l[5], l[6], l[7]);
        }
        tc::fence_smem_to_async();
        tc::fence_before_sync();
        __syncthreads();
        tc::fence_after_sync();
        if (t == 0) {
            const uint32_t sa = (uint32_t)__cvta_generic_to_shared(Ab), sb = (uint32_t)__cvta_generic_to_shared(Bb);
#pragma unroll
            for (int kb = 0; kb < TC_KB; ++kb)
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t a_hi = sa + (kb * 2) * TC_ABYTES + ks * 2 * 128 * 16;
                    const uint32_t b_hi = sb + (kb * 2) * TC_BBYTES + ks * 2 * TC_N * 16;
                    const uint64_t ah = tc::smem_desc(a_hi, 128 * 16, 128);
                    const uint64_t al = tc::smem_desc(a_hi + TC_ABYTES, 128 * 16, 128);
                    const uint64_t bh = tc::smem_desc(b_hi, TC_N * 16, 128);
                    const uint64_t bl = tc::smem_desc(b_hi + TC_BBYTES, TC_N * 16, 128);
                    const uint32_t d = tmem + kb * TC_N;
                    tc::mma_tf32(d, ah, bh, idesc, s > 0 || ks > 0);
                    tc::mma_tf32(d, ah, bl, idesc, true);
                    tc::mma_tf32(d, al, bh, idesc, true);
                }
            tc::commit(&bar[buf]);
        }
    }
    tc::mbar_wait(&bar[(nstage - 1) & 1], ((nstage - 1) >> 1) & 1);
    tc::fence_after_sync();
    // epilogue: TMEM -> smem staging E[bin][128 rows][16] -> Y
    float *E = reinterpret_cast<float *>(sm);
    {
        const int quarter = warp & 3, kb0 = (warp >> 2) * 2;
        const int r = quarter * 32 + lane;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
            const int kb = kb0 + kk;
            float v[16];
            tc::tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + kb * TC_N, *reinterpret_cast<float(*)[8]>(v));
            tc::tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + kb * TC_N + 8,
                         *reinterpret_cast<float(*)[8]>(v + 8));
            tc::tmem_ld_wait();
#pragma unroll
            for (int n = 0; n < 16; n += 4)
                *reinterpret_cast<float4 *>(E + (kb * 128 + r) * 16 + n) = make_float4(v[n], v[n + 1], v[n + 2], v[n + 3]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<64>(tmem);
    const int k = k0 + q;
    if (!rok || k >= Kb) return;
    const float *er = E + (q * 128 + b) * 16, *ei = E + (q * 128 + 64 + b) * 16;
    for (int p = 0; p < cls.P; ++p) {
        const float ar = er[p], ai = ei[p], br = er[8 + p], bi = ei[8 + p];
        Y[(row * M + cls.mp[p]) * ldy + k] = make_float2(ar - bi, ai + br);
        if (cls.mm[p] >= 0) Y[(row * M + cls.mm[p]) * ldy + k] = make_float2(ar + bi, ai - br);
    }
}

int contract_tc(const float2 *X, long long ldx, const float *tab, float2 *Y, long long ldy, long long B,
                int L, int M, int Kb, int P, const short *mp, const short *mm, cudaStream_t s) {
    if (B <= 0 || Kb <= 0) return KKB_OK;
    if (P < 1 || P > 8 || (ldx & 1)) {
        set_error("contract_tc: needs 1..8 symmetric classes and an even row stride");
        return KKB_ERR_ARG;
    }
    TcClasses cls{};
    cls.P = P;
    for (int p = 0; p < P; ++p) {
        cls.mp[p] = mp[p];
        cls.mm[p] = mm[p];
    }
    dim3 grid((unsigned)ceil_div(Kb, TC_KB), (unsigned)ceil_div(B, TC_ROWS));
    if (grid.y > 65535u) {
        set_error("contraction batch too large (%lld rows)", B);
        return KKB_ERR_UNSUPPORTED;
    }
    const int smem = 2 * TC_STAGE_BYTES;
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_contract_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                 "smem attr contract_tc");
    k_contract_tc<<<grid, 256, smem, s>>>(X, ldx, tab, Y, ldy, B, L, M, Kb, cls);
    KKB_CHECK_LAUNCH("k_contract_tc");
    return KKB_OK;
}

}  // namespace kkb
