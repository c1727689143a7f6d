// Microbenchmark: L2 read bandwidth of this B200 (the SURVEY §8(d) gather
// roofline denominator) -- a working set that stays L2-resident, read with
// 128-bit loads by every SM, many passes; bytes delivered / time.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_read(const float4 *__restrict__ p, long long n4, int passes, float *out) {
    float acc = 0.f;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (int r = 0; r < passes; ++r) {
        // rotate the start so consecutive passes do not hit the same lines per SM
        const long long off = ((long long)r * 4099 * 32) % n4;
        for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4; i += stride) {
            long long j = i + off;
            if (j >= n4) j -= n4;
            const float4 v = __ldcg(p + j);  // cache-global: L2, not L1
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == -1.f) out[0] = acc;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *out;
    cudaMalloc(&out, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const long long sizes_mb[] = {8, 16, 32, 48, 64, 96};
    for (long long mb : sizes_mb) {
        const long long bytes = mb << 20, n4 = bytes / 16;
        float4 *p;
        cudaMalloc(&p, bytes);
        cudaMemset(p, 0, bytes);
        const int passes = (int)(8192 / mb);
        for (int blocks_per_sm : {4, 8}) {
            const int grid = sms * blocks_per_sm, block = 256;
            k_read<<<grid, block>>>(p, n4, 2, out);  // warm L2
            cudaEventRecord(e0);
            k_read<<<grid, block>>>(p, n4, passes, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("{\"working_set_MB\": %lld, \"ctas_per_sm\": %d, \"L2_read_GBps\": %.1f, \"err\": \"%s\"}\n", mb,
                   blocks_per_sm, (double)bytes * passes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
        }
        cudaFree(p);
    }
    return 0;
}
