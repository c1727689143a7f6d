// tcgen05 probe: validates the descriptor / layout / TMEM helpers of
// paper_2603_22496_b200/csrc/tc.cuh against a host GEMM (kind::tf32 and
// kind::f16, M = 128, several N) and times back-to-back MMAs.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <vector>

#include "../../paper_2603_22496_b200/csrc/tc.cuh"

using namespace kkb;

// C[128 x N] = A[128 x K] * B[N x K]^T, K = 32 elements, one CTA of 128 threads
template <bool F16>
__global__ void k_probe(const float *A, const float *B, int N, float *C, int reps, long long *cyc, int nacc) {
    constexpr int K = 32;
    constexpr int ESZ = F16 ? 2 : 4;
    constexpr int CHUNKS = K * ESZ / 16;  // 16-byte K chunks per row
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *As = sm;                       // [CHUNKS][128][16 B]
    unsigned char *Bs = sm + CHUNKS * 128 * 16;   // [CHUNKS][N][16 B]
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5;
    // operands into the canonical layout (tf32: pre-rounded, cvt.rna)
    for (int c = 0; c < CHUNKS; ++c) {
        const int e0 = c * 16 / ESZ;
        if (F16) {
            __half h[8];
            for (int i = 0; i < 8; ++i) h[i] = __float2half_rn(A[t * K + e0 + i]);
            *reinterpret_cast<uint4 *>(As + (c * 128 + t) * 16) = *reinterpret_cast<uint4 *>(h);
            for (int r = t; r < N; r += 128) {
                for (int i = 0; i < 8; ++i) h[i] = __float2half_rn(B[r * K + e0 + i]);
                *reinterpret_cast<uint4 *>(Bs + (c * N + r) * 16) = *reinterpret_cast<uint4 *>(h);
            }
        } else {
            float4 v = make_float4(tc::to_tf32(A[t * K + e0]), tc::to_tf32(A[t * K + e0 + 1]),
                                   tc::to_tf32(A[t * K + e0 + 2]), tc::to_tf32(A[t * K + e0 + 3]));
            *reinterpret_cast<float4 *>(As + (c * 128 + t) * 16) = v;
            for (int r = t; r < N; r += 128) {
                v = make_float4(tc::to_tf32(B[r * K + e0]), tc::to_tf32(B[r * K + e0 + 1]),
                                tc::to_tf32(B[r * K + e0 + 2]), tc::to_tf32(B[r * K + e0 + 3]));
                *reinterpret_cast<float4 *>(Bs + (c * N + r) * 16) = v;
            }
        }
    }
    if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t d = tmem_base;
    const uint32_t idesc = tc::instr_desc(F16 ? 0 : 2, 128, N);
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(As), sb = (uint32_t)__cvta_generic_to_shared(Bs);
    if (t == 0) {
        long long c0 = clock64();
        for (int r = 0; r < reps; ++r)
            for (int s = 0; s < CHUNKS / 2; ++s) {
                const uint64_t a = tc::smem_desc(sa + s * 2 * 128 * 16, 128 * 16, 128);
                const uint64_t b = tc::smem_desc(sb + s * 2 * N * 16, N * 16, 128);
                // r > 0: round-robin over nacc independent accumulators (pipelining probe)
                const uint32_t dd = d + (uint32_t)((r % nacc) * N) * (r > 0);
                if (F16)
                    tc::mma_f16(dd, a, b, idesc, s > 0 || r > 0);
                else
                    tc::mma_tf32(dd, a, b, idesc, s > 0 || r > 0);
            }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        *cyc = clock64() - c0;
    }
    __syncthreads();
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    for (int c0 = 0; c0 < N; c0 += 8) {
        float v[8];
        tc::tmem_ld8(d + ((uint32_t)(warp * 32) << 16) + c0, v);
        tc::tmem_ld_wait();
        for (int i = 0; i < 8; ++i) C[t * N + c0 + i] = v[i];
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<256>(d);
}

static float tf32r(float x) {  // host emulation of cvt.rna.tf32 (ties away)
    unsigned u;
    memcpy(&u, &x, 4);
    u = (u + 0x1000u) & ~0x1FFFu;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

int main() {
    const int K = 32;
    int fails = 0;
    for (int f16 = 0; f16 < 2; ++f16)
        for (int N : {16, 32, 64, 256}) {
            std::vector<float> A(128 * K), B(N * K), C(128 * N);
            srand(7 + N);
            for (auto &x : A) x = (rand() % 2001 - 1000) / 1000.0f;
            for (auto &x : B) x = (rand() % 2001 - 1000) / 1000.0f;
            float *dA, *dB, *dC;
            long long *dcyc;
            cudaMalloc(&dA, A.size() * 4);
            cudaMalloc(&dB, B.size() * 4);
            cudaMalloc(&dC, C.size() * 4);
            cudaMalloc(&dcyc, 8);
            cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
            const int chunks = K * (f16 ? 2 : 4) / 16;
            size_t smem = chunks * (128 + N) * 16;
            auto fn = f16 ? k_probe<true> : k_probe<false>;
            cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            fn<<<1, 128, smem>>>(dA, dB, N, dC, 1, dcyc, 1);
            cudaError_t e = cudaDeviceSynchronize();
            cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
            double maxerr = 0;
            for (int i = 0; i < 128; ++i)
                for (int j = 0; j < N; ++j) {
                    double ref = 0;
                    for (int k = 0; k < K; ++k) {
                        float a = A[i * K + k], b = B[j * K + k];
                        if (f16) {
                            a = __half2float(__float2half_rn(a));
                            b = __half2float(__float2half_rn(b));
                        } else {  // inputs pre-rounded with cvt.rna.tf32
                            a = tf32r(a);
                            b = tf32r(b);  // == cvt.rna.tf32
                        }
                        ref += (double)a * b;
                    }
                    maxerr = fmax(maxerr, fabs(ref - C[i * N + j]));
                }
            // timing: many back-to-back MMAs on the same operands
            const int reps = 2000;
            double per[3];
            const int naccs[3] = {1, 2, 4};
            for (int q = 0; q < 3; ++q) {
                const int nacc = N * naccs[q] <= 256 ? naccs[q] : 1;
                fn<<<1, 128, smem>>>(dA, dB, N, dC, reps, dcyc, nacc);
                cudaDeviceSynchronize();
                long long cyc = 0;
                cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
                per[q] = (double)cyc / (reps * (chunks / 2));
            }
            printf("{\"kind\": \"%s\", \"M\": 128, \"N\": %d, \"max_abs_err\": %.3g, \"ok\": %d, "
                   "\"cycles_per_mma_1acc\": %.1f, \"2acc\": %.1f, \"4acc\": %.1f, \"err\": \"%s\"}\n",
                   f16 ? "f16" : "tf32", N, maxerr, maxerr < 1e-4, per[0], per[1], per[2],
                   cudaGetErrorString(e));
            fails += !(maxerr < 1e-4) || e != cudaSuccess;
            cudaFree(dA);
            cudaFree(dB);
            cudaFree(dC);
            cudaFree(dcyc);
        }
    return fails;
}
