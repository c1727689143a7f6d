// Microbenchmark: shared-memory wavefront cost of a 128-bit warp load as a
// function of the lane -> address pattern (informs the K5 lane layout).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int pat(int p, int lane) {
    switch (p) {
        case 0: return lane;              // 32 distinct, consecutive
        case 1: return 0;                 // broadcast
        case 2: return lane & 3;          // 4 distinct, cycling
        case 3: return lane >> 2;         // 8 distinct, groups of 4
        case 4: return lane >> 3;         // 4 distinct, groups of 8
        case 5: return lane & 7;          // 8 distinct, cycling
        case 6: return lane >> 1;         // 16 distinct, pairs
        case 7: return lane & 15;         // 16 distinct, cycling
        case 8: return (lane * 7) & 15;   // 16 distinct, shuffled
        case 9: return (lane >> 2) + 8 * (lane & 1);  // mixed
        case 10: return lane >> 4;        // 2 distinct, halves
        case 11: return (lane & 1) * 8;   // 2 distinct, 128 B apart
        case 12: return (lane >> 2) * 2;  // 8 distinct, stride 32 B
        case 13: return lane * 2;         // 32 distinct, stride 32 B
        case 14: return lane < 16 ? (lane >> 1) : 8 + lane;          // half-warp 0 pair-uniform
        case 15: return lane < 8 ? (lane >> 1) : 8 + lane;           // quarter 0 pair-uniform
        case 16: return lane < 4 ? (lane >> 1) : 8 + lane;           // 2 pairs uniform
        case 17: return lane < 2 ? 0 : 8 + lane;                     // 1 pair uniform
        case 18: return lane < 30 ? (lane >> 1) : 16 + lane;         // all but the last pair
        case 19: return (lane & 8) ? 16 + lane : (lane >> 1);        // quarters 0, 2 pair-uniform
        case 20: return (lane & 16) ? (lane >> 1) : 8 + lane;        // half-warp 1 pair-uniform
    }
    return 0;
}

template <int WB>
__global__ void k(int p, int iters, float *out) {
    __shared__ __align__(16) float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a = (unsigned)__cvta_generic_to_shared(s) + ((pat(p, lane) + warp * 32) & 127) * WB;
    float acc = 0.f;
    for (int i = 0; i < iters; ++i) {
        float x, y, z, w;
        const unsigned ai = a ^ ((i & 7) << 11);
        if (WB == 16) {
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(ai) : "memory");
        } else if (WB == 8) {
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(x), "=f"(y) : "r"(ai) : "memory");
            z = x; w = y;
        } else {
            asm volatile("ld.shared.f32 %0, [%1];" : "=f"(x) : "r"(ai) : "memory");
            y = z = w = x;
        }
        acc += (x + y) * (z + w);
        if (WB == 16) {
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4+16];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(ai) : "memory");
        } else if (WB == 8) {
            asm volatile("ld.shared.v2.f32 {%0,%1}, [%2+16];" : "=f"(x), "=f"(y) : "r"(ai) : "memory");
            z = x; w = y;
        } else {
            asm volatile("ld.shared.f32 %0, [%1+16];" : "=f"(x) : "r"(ai) : "memory");
            y = z = w = x;
        }
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
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    const char *names[] = {"lane", "bcast", "lane&3", "lane>>2", "lane>>3", "lane&7", "lane>>1",
                           "lane&15", "(lane*7)&15", "mixed", "lane>>4", "(lane&1)*8", "(lane>>2)*2", "lane*2", "hw0 pairs", "q0 pairs", "2 pairs", "1 pair",
                           "all-but-1", "q0,q2 pairs", "hw1 pairs"};
    for (int wb = 16; wb >= 4; wb /= 2)
    for (int p = 0; p < 21; ++p) {
        auto fn = wb == 16 ? k<16> : (wb == 8 ? k<8> : k<4>);
        fn<<<blocks, threads>>>(p, iters, out);
        cudaEventRecord(e0);
        fn<<<blocks, threads>>>(p, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double warp_loads = (double)blocks * threads / 32 * iters * 2;
        int clk;
        cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        double cyc = ms * 1e-3 * clk * 1e3 * sms;  // SM-cycles (at the nominal clock)
        printf("LDS%-3d %-14s %.3f SM-cycles per warp load (%.3f ms, %s)\n", wb * 8, names[p], cyc / warp_loads, ms,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
