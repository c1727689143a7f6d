// Probe: kind::f16 MMA (M = 128, N = 128, K = 32 as two K = 16 steps) with
// A K-major no-swizzle and B K-major in the 64-byte (or 32-byte) swizzled
// layout, written by hand with the swizzle XOR; checked against a host GEMM.
// Validates tc::smem_desc_sw before the tensor-core gather uses it.
#include <cmath>
#include <cstdio>
#include <cuda_fp16.h>
#include <vector>

#include "../../paper_2603_22496_b200/csrc/tc.cuh"

using namespace kkb;

// byte offset of (row r, half k) in a K-major swizzled tile with rows of RB bytes
__device__ __forceinline__ int swz(int r, int k, int RB) {
    const int byte = r * RB + 2 * k;
    if (RB == 64) return byte ^ (((byte >> 7) & 3) << 4);
    return byte ^ (((byte >> 7) & 1) << 4);  // RB == 32
}

template <int RB>
__global__ void k_probe(const float *A, const float *B, float *C, int ksteps) {
    constexpr int K = RB / 2, N = 128;
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *As = sm;              // [K/8 chunks][128 rows][16 B]
    unsigned char *Bs = sm + 16384;      // [N rows][RB] swizzled
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5;
    for (int c = 0; c < K / 8; ++c) {
        __half h[8];
        for (int i = 0; i < 8; ++i) h[i] = __float2half_rn(A[t * K + 8 * c + i]);
        *reinterpret_cast<uint4 *>(As + (c * 128 + t) * 16) = *reinterpret_cast<uint4 *>(h);
    }
    for (int k = 0; k < K; ++k) *reinterpret_cast<__half *>(Bs + swz(t, k, RB)) = __float2half_rn(B[t * K + k]);
    if (warp == 0) tc::tmem_alloc<128>(&tmem_base);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t d = tmem_base;
    const uint32_t idesc = tc::instr_desc(0, 128, N, 0);
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(As), sb = (uint32_t)__cvta_generic_to_shared(Bs);
    if (t == 0) {
        for (int s = 0; s < ksteps; ++s) {
            const uint64_t da = tc::smem_desc(sa + s * 2 * 128 * 16, 128 * 16, 128);
            const uint64_t db = tc::smem_desc_sw(sb + s * 32, 8 * RB, RB == 64 ? 4 : 6);
            tc::mma_f16(d, da, db, idesc, s > 0);
        }
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
    if (warp == 0) tc::tmem_free<128>(d);
}

template <int RB>
static int run() {
    constexpr int K = RB / 2, N = 128;
    std::vector<float> A(128 * K), B(N * K), C(128 * N), R(128 * N);
    for (size_t i = 0; i < A.size(); ++i) A[i] = (float)__half2float(__float2half_rn(sinf(0.37f * i) * 2));
    for (size_t i = 0; i < B.size(); ++i) B[i] = (float)__half2float(__float2half_rn(cosf(0.11f * i + 1)));
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)A[m * K + k] * B[n * K + k];
            R[m * N + n] = (float)s;
        }
    float *dA, *dB, *dC;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dC, C.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(k_probe<RB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    k_probe<RB><<<1, 128, 40000>>>(dA, dB, dC, K / 16);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
    double err = 0, ref = 0;
    for (size_t i = 0; i < C.size(); ++i) {
        err = fmax(err, fabs(C[i] - R[i]));
        ref = fmax(ref, fabs(R[i]));
    }
    printf("swizzle %dB K-major B: %s, max abs err %.3g (max |ref| %.3g)\n", RB, cudaGetErrorString(e), err, ref);
    return e != cudaSuccess || err > 1e-3 * ref;
}

int main() {
    int bad = run<64>();
    bad |= run<32>();
    return bad;
}
