// How does a long chain of tcgen05 f16 MMAs accumulate into one fp32 TMEM
// accumulator?  D = sum over R repetitions of A * B^T (A, B fixed random fp16,
// K = 16 per MMA), compared with the exact float64 sum: relative error vs R
// tells whether the accumulator adds round to nearest (error ~ sqrt(R) ulp)
// or truncate (error ~ R ulp, biased).
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp16.h>
#include <vector>

#include "../../paper_2603_22496_b200/csrc/tc.cuh"

using namespace kkb;

__global__ void k_accum(const float *A, const float *B, int N, int reps, float *C) {
    __shared__ __align__(1024) unsigned char As[2 * 128 * 16];
    __shared__ __align__(1024) unsigned char Bs[2 * 256 * 16];
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5;
    for (int c = 0; c < 2; ++c) {
        __half h[8];
        for (int i = 0; i < 8; ++i) h[i] = __float2half_rn(A[t * 16 + c * 8 + i]);
        *reinterpret_cast<uint4 *>(As + (c * 128 + t) * 16) = *reinterpret_cast<uint4 *>(h);
        for (int r = t; r < N; r += 128) {
            for (int i = 0; i < 8; ++i) h[i] = __float2half_rn(B[r * 16 + c * 8 + i]);
            *reinterpret_cast<uint4 *>(Bs + (c * N + r) * 16) = *reinterpret_cast<uint4 *>(h);
        }
    }
    if (warp == 0) tc::tmem_alloc<256>(&tmem_base);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t d = tmem_base, idesc = tc::instr_desc(0, 128, N);
    if (t == 0) {
        const uint64_t a = tc::smem_desc((uint32_t)__cvta_generic_to_shared(As), 128 * 16, 128);
        const uint64_t b = tc::smem_desc((uint32_t)__cvta_generic_to_shared(Bs), N * 16, 128);
        for (int r = 0; r < reps; ++r) tc::mma_f16(d, a, b, idesc, r > 0);
        tc::commit(&bar);
    }
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

int main() {
    const int N = 64;
    std::vector<float> A(128 * 16), B(N * 16), C(128 * N);
    srand(3);
    for (auto &x : A) x = __half2float(__float2half_rn((rand() % 20001 - 10000) / 10000.0f));
    for (auto &x : B) x = __half2float(__float2half_rn((rand() % 20001 - 10000) / 10000.0f * 100.0f));
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    for (int reps : {1, 4, 16, 64, 256, 1024, 4096}) {
        k_accum<<<1, 128>>>(dA, dB, N, reps, dC);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
        double num = 0, den = 0, bias = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < N; ++j) {
                double s = 0;
                for (int k = 0; k < 16; ++k) s += (double)A[i * 16 + k] * B[j * 16 + k];
                // fp32 round-to-nearest sequential accumulation, the FMA kernels' model
                float acc = 0.f;
                for (int r = 0; r < reps; ++r) acc += (float)s;
                const double ref = s * reps;
                num += (C[i * N + j] - ref) * (C[i * N + j] - ref);
                den += ref * ref;
                bias += (C[i * N + j] - ref) / (fabs(ref) + 1e-30) * (ref >= 0 ? 1 : -1);
                (void)acc;
            }
        double rn = 0, rd = 0;
        for (int i = 0; i < 128; ++i)
            for (int j = 0; j < N; ++j) {
                double s = 0;
                for (int k = 0; k < 16; ++k) s += (double)A[i * 16 + k] * B[j * 16 + k];
                float acc = 0.f;
                for (int r = 0; r < reps; ++r) acc += (float)s;
                rn += ((double)acc - s * reps) * ((double)acc - s * reps);
                rd += s * reps * s * reps;
            }
        printf("{\"reps\": %d, \"tc_rel_l2\": %.3g, \"tc_mean_signed_rel\": %.3g, \"fp32_rn_rel_l2\": %.3g, \"err\": \"%s\"}\n",
               reps, sqrt(num / den), bias / (128.0 * N), sqrt(rn / rd), cudaGetErrorString(e));
    }
    return 0;
}
