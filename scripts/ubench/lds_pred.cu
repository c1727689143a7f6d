// Microbenchmark: shared-memory cost of a PREDICATED 128-bit warp load as a
// function of which lanes are active (does a predicated-off lane save
// wavefronts?).  Distinct 16 B addresses per lane.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ bool act(int p, int lane) {
    switch (p) {
        case 0: return true;                              // all 32
        case 1: return false;                             // none
        case 2: return (lane * 7 + 3) % 4 == 0;           // 8 lanes spread over the warp
        case 3: return lane < 8;                          // one quarter
        case 4: return (lane & 1) == 0;                   // 16 alternate lanes
        case 5: return lane < 16;                         // one half
        case 6: return ((lane * 13) % 32) < 6;            // 6 scattered lanes
        case 7: return lane == 5;                         // 1 lane
    }
    return true;
}

__global__ void k(int p, int iters, float *out) {
    __shared__ __align__(16) float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a = (unsigned)__cvta_generic_to_shared(s) + ((lane + warp * 32) & 127) * 16;
    const unsigned pr = act(p, lane) ? 1u : 0u;
    float x = 0.f, y = 0.f, z = 0.f, w = 0.f, acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        const unsigned ai = a ^ ((i & 7) << 11);
        asm volatile("{ .reg .pred q; setp.ne.u32 q, %4, 0; @q ld.shared.v4.f32 {%0,%1,%2,%3}, [%5]; }"
                     : "+f"(x), "+f"(y), "+f"(z), "+f"(w) : "r"(pr), "r"(ai) : "memory");
        acc += (x + y) * (z + w);
        asm volatile("{ .reg .pred q; setp.ne.u32 q, %4, 0; @q ld.shared.v4.f32 {%0,%1,%2,%3}, [%5+16]; }"
                     : "+f"(x), "+f"(y), "+f"(z), "+f"(w) : "r"(pr), "r"(ai) : "memory");
        acc += (x + z) * (y + w);
    }
    if (acc == -1.f) out[0] = acc;
}

int main() {
    float *out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    const char *names[] = {"all 32", "none", "8 spread", "quarter 0", "16 alternate", "half 0", "6 scattered", "1 lane"};
    for (int p = 0; p < 8; ++p) {
        k<<<blocks, threads>>>(p, iters, out);
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(p, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double warp_loads = (double)blocks * threads / 32 * iters * 2;
        double cyc = ms * 1e-3 * clk * 1e3 * sms;
        printf("predicated LDS.128 %-13s %.3f SM-cycles per warp load\n", names[p], cyc / warp_loads);
    }
    return 0;
}
