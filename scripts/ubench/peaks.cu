// Measured on-chip peaks for the rooflines MEASURED_PEAKS.json lacks:
//   * shared-memory load bandwidth with conflict-free 128-bit warp loads
//     (LDS.128, lane-consecutive: 4 wavefronts of 128 B per warp load) — the
//     K5 gather's binding resource (16 B of taps per pixel-pair from SMEM);
//   * FP32 FMA throughput (K2 contraction, FFT butterflies);
//   * FP64 add/mul throughput (K5's per-tap delay math: 4 DADD/DMUL + 1 DADD.RD).
// Every SM runs many resident warps of independent chains; best of 5 runs
// timed with CUDA events.  Prints one JSON object.  (Shared loads are
// ld.volatile: plain ld.shared of a period-2 address pattern gets hoisted
// out of the loop by ptxas.)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_lds128(int iters, float *out) {
    __shared__ __align__(16) float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned a = (unsigned)__cvta_generic_to_shared(s) + ((warp * 32 + lane) & 511) * 16;
    float acc0 = 0.f, acc1 = 0.f;
    for (int i = 0; i < iters; ++i) {
        const unsigned ai = a ^ ((i & 1) << 13);
        float x, y, z, w, x1, y1, z1, w1;
        asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(x), "=f"(y), "=f"(z), "=f"(w) : "r"(ai) : "memory");
        asm volatile("ld.volatile.shared.v4.f32 {%0,%1,%2,%3}, [%4+16384];" : "=f"(x1), "=f"(y1), "=f"(z1), "=f"(w1) : "r"(ai) : "memory");
        acc0 += (x + y) + (z + w);
        acc1 += (x1 + y1) + (z1 + w1);
    }
    if (acc0 + acc1 == -1.f) out[0] = acc0;
}

template <int CH>
__global__ void k_ffma(int iters, float *out) {
    float a[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) a[j] = threadIdx.x * 1e-7f + j;
    const float b = 0.999999f, c = 1e-7f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = fmaf(a[j], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += a[j];
    if (s == -1.f) out[0] = s;
}

template <int CH>
__global__ void k_dadd(int iters, double *out) {
    double a[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) a[j] = threadIdx.x * 1e-7 + j;
    const double b = 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < CH; ++j) a[j] = __dadd_rn(a[j], b);
    }
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < CH; ++j) s += a[j];
    if (s == -1.0) out[0] = s;
}

template <class F>
static float timed(F launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();  // warm-up
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess || (le = cudaDeviceSynchronize()) != cudaSuccess) {
        fprintf(stderr, "launch failed: %s\n", cudaGetErrorString(le));
        return -1.f;
    }
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float *outf;
    double *outd;
    cudaMalloc(&outf, 16);
    cudaMalloc(&outd, 16);
    printf("{\n \"tool\": \"scripts/ubench/peaks.cu\",\n \"sm_count\": %d,\n", sms);

    {   // LDS.128: 4 CTAs x 512 threads per SM, 2 loads of 16 B per thread per iteration
        const int threads = 512, blocks = sms * 4, iters = 1 << 13;
        float ms = timed([&] { k_lds128<<<blocks, threads>>>(iters, outf); });
        double bytes = (double)blocks * threads * iters * 2 * 16;
        printf(" \"smem_lds128\": {\"GBps\": %.1f, \"ms\": %.3f, \"what\": \"conflict-free LDS.128, 2048 threads/SM\", "
               "\"err\": \"%s\"},\n", bytes / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
    }
    {   // FFMA: 8 independent chains, 4 x 512 threads per SM
        const int threads = 512, blocks = sms * 4, iters = 1 << 14;
        float ms = timed([&] { k_ffma<8><<<blocks, threads>>>(iters, outf); });
        double flops = 2.0 * blocks * threads * (double)iters * 8;
        printf(" \"fp32_fma\": {\"TFLOPs\": %.2f, \"ms\": %.3f, \"err\": \"%s\"},\n",
               flops / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
    }
    {   // DADD: 8 independent chains
        const int threads = 512, blocks = sms * 4, iters = 1 << 12;
        float ms = timed([&] { k_dadd<8><<<blocks, threads>>>(iters, outd); });
        double ops = (double)blocks * threads * iters * 8;
        printf(" \"fp64_add\": {\"Gops\": %.1f, \"ms\": %.3f, \"err\": \"%s\"}\n",
               ops / (ms * 1e-3) / 1e9, ms, cudaGetErrorString(cudaGetLastError()));
    }
    printf("}\n");
    return 0;
}
