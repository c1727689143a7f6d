// tcgen05 kind::f16 M = 128, K = 16 MMA issue rate by B operand layout:
// K-major (the probe's canonical layout) vs MN-major no-swizzle (the
// tensor-core gather's trace windows: core matrices of 8 K-rows x 16 B of
// consecutive N values, LBO = 128 B between 8-deep K groups, SBO = 256 B
// between 16-byte N groups), one accumulator (a dependent chain, as the
// gather's groups of 16 pairs) or several; accumulators = 0 issues the
// gather's split3 asm blocks.  Timing only (operands are zero).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tc_layout_probe tc_layout_probe.cu
#include <cstdio>

#include "../../paper_2603_22496_b200/csrc/tc.cuh"

using namespace kkb;

__global__ void k_layout(int N, int mn_major, int nacc, int reps, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned char *As = sm, *Bs = sm + 8192;
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < (8192 + 2 * 256 * 16 * 2) / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tc::tmem_alloc<512>(&tmem_base);
    if (t == 0) tc::mbar_init(&bar, 1);
    tc::fence_smem_to_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t d = tmem_base;
    const uint32_t idesc = tc::instr_desc(0, 128, N, mn_major);
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(As), sb = (uint32_t)__cvta_generic_to_shared(Bs);
    const uint64_t a = tc::smem_desc(sa, 128 * 16, 128);
    const uint64_t b = mn_major ? tc::smem_desc(sb, 128, 256) : tc::smem_desc(sb, N * 16, 128);
    if (t == 0) {
        long long c0 = clock64();
        if (nacc == 0) {  // the gather's issue form: split3 asm blocks (3 MMAs each), one accumulator
            for (int r = 0; r < reps / 3; ++r) tc::mma_f16_split3(d, a, a, b, b, idesc, r > 0);
        } else {
#pragma unroll 1
            for (int r = 0; r < reps; r += 8) {
#pragma unroll
                for (int u = 0; u < 8; ++u) tc::mma_f16(d + (uint32_t)((u % nacc) * N), a, b, idesc, r + u >= nacc);
            }
        }
        tc::commit(&bar);
        tc::mbar_wait(&bar, 0);
        *cyc = clock64() - c0;
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_free<512>(d);
}

int main() {
    long long *dc;
    cudaMalloc(&dc, 8);
    cudaFuncSetAttribute(k_layout, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192 + 2 * 256 * 16 * 2);
    const int reps = 4000;
    for (int N : {64, 128, 256})
        for (int mn = 0; mn < 2; ++mn)
            for (int nacc : {0, 1, 2, 4}) {
                if (nacc * N > 512) continue;
                k_layout<<<1, 128, 8192 + 2 * 256 * 16 * 2>>>(N, mn, nacc, reps, dc);
                cudaError_t e = cudaDeviceSynchronize();
                long long c = 0;
                cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost);
                printf("{\"M\": 128, \"N\": %d, \"K\": 16, \"b_layout\": \"%s\", \"accumulators\": %d, "
                       "\"cycles_per_mma\": %.1f, \"err\": \"%s\"}\n",
                       N, mn ? "mn_major" : "k_major", nacc, (double)c / (nacc ? reps : reps / 3 * 3),
                       cudaGetErrorString(e));
            }
    return 0;
}
