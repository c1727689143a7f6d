// Microbenchmark: can texture fetches (TEX pipe, L1-resident data) add
// bandwidth on top of 128-bit shared loads (LSU pipe)?  Each thread issues
// independent float4 reads at lane-distinct addresses: (a) LDS.128 only,
// (b) tex1Dfetch<float4> only (L1-resident 16 KB buffer), (c) both interleaved.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(cudaTextureObject_t tex, int iters, float *out) {
    __shared__ __align__(16) float4 s[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float4(i, i, i, i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned idx = (lane * 33 + (threadIdx.x >> 5) * 7) & 1023;
    float4 acc = make_float4(0, 0, 0, 0);
    for (int i = 0; i < iters; ++i) {
        const unsigned a = (idx + i * 37) & 1023, b = (idx + i * 53 + 512) & 1023;
        if (MODE == 0 || MODE == 2) {
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(&s[a])) : "memory");
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        if (MODE == 1 || MODE == 2) {
            const float4 v = tex1Dfetch<float4>(tex, (int)b);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        if (MODE == 0) {  // same count of loads as mode 2
            float4 v;
            asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                         : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                         : "r"((unsigned)__cvta_generic_to_shared(&s[b])) : "memory");
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        if (MODE == 1) {
            const float4 v = tex1Dfetch<float4>(tex, (int)a);
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
    }
    if (acc.x + acc.y + acc.z + acc.w == -1.f) out[0] = acc.x;
}

int main() {
    float4 *buf;
    cudaMalloc(&buf, 1024 * sizeof(float4));
    cudaMemset(buf, 0, 1024 * sizeof(float4));
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = buf;
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = 1024 * sizeof(float4);
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex;
    cudaCreateTextureObject(&tex, &rd, &td, nullptr);
    float *out;
    cudaMalloc(&out, 4);
    int sms, clk;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    const char *names[] = {"LDS.128 x2", "TEX float4 x2", "LDS.128 + TEX"};
    for (int m = 0; m < 3; ++m) {
        auto fn = m == 0 ? k<0> : (m == 1 ? k<1> : k<2>);
        fn<<<blocks, threads>>>(tex, iters, out);
        cudaEventRecord(e0);
        fn<<<blocks, threads>>>(tex, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double loads = (double)blocks * threads / 32 * iters * 2;  // warp-level float4 loads
        const double cyc = ms * 1e-3 * clk * 1e3 * sms;
        printf("%-16s %.3f SM-cycles per warp float4 load  (%s)\n", names[m], cyc / loads,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
