// Display and budgeting epilogues on the device.
//
// * gamma_match (metrics.py:175-202): normalise an intensity image by its
//   maximum and find the exponent g in [lo, hi] whose mean (I/max)^g matches
//   the mean of the reference image's (R/maxR)^0.5, by golden-section search
//   (metrics.py:156-172) -- the search's comparisons run on the host, every
//   evaluation of the objective is a device reduction in float64:
//     k_max_reduce   per-CTA maxima            -> k_finish_max (fixed order)
//     k_pow_sum      per-CTA sums of (x/m)^g   -> k_finish_sum (fixed order)
//   so the result is deterministic (run to run and across launches), and
//   differs from numpy's pairwise mean only in the last bits of each sum.
// * last_read_sample (cli.py:110-128): the largest sample the kk gather can
//   read on a grid, max over pixels of max_n(x sin + z cos) + max_m(z cos -
//   x sin); the max is exact in any order, so the result is bit-identical.

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"

namespace kkb {

#define KKB_RED_THREADS 256
#define KKB_RED_BLOCKS 296  // 2 x 148 SMs

__device__ __forceinline__ double block_sum(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = 0.0;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += sh[i];
    __syncthreads();
    return t;
}

__device__ __forceinline__ double block_max(double v, double *sh) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double t = -INFINITY;
    if (threadIdx.x == 0)
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = fmax(t, sh[i]);
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(KKB_RED_THREADS)
k_max_reduce(const double *__restrict__ x, long long n, double *part) {
    __shared__ double sh[32];
    double m = -INFINITY;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        m = fmax(m, x[i]);
    m = block_max(m, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = m;
}

// sum over i of (x[i] * inv_max) ^ g, with inv_max = 1 / max read on device
__global__ void __launch_bounds__(KKB_RED_THREADS)
k_pow_sum(const double *__restrict__ x, long long n, const double *__restrict__ maxv, double g,
          double *part) {
    __shared__ double sh[32];
    const double m = *maxv;
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        s += g == 0.5 ? sqrt(x[i] / m) : pow(x[i] / m, g);  // numpy's ** 0.5 is sqrt
    s = block_sum(s, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
}

// one CTA: fold the per-CTA partials in index order (deterministic)
__global__ void k_finish(const double *__restrict__ part, int nb, int op, double *out) {
    if (threadIdx.x != 0) return;
    double t = op ? -INFINITY : 0.0;
    for (int i = 0; i < nb; ++i) t = op ? fmax(t, part[i]) : t + part[i];
    *out = t;
}

__global__ void k_pow_map(const double *__restrict__ x, long long n, const double *__restrict__ maxv,
                          double g, double *out) {
    const double m = *maxv;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = pow(x[i] / m, g);
}

namespace {
int blocks_for(long long n) {
    return (int)std::max<long long>(1, std::min<long long>(KKB_RED_BLOCKS, ceil_div(n, KKB_RED_THREADS)));
}
}  // namespace

// scratch: >= KKB_RED_BLOCKS + 4 doubles of device memory
int device_max(const double *x, long long n, double *scratch, double *out, cudaStream_t s) {
    const int nb = blocks_for(n);
    k_max_reduce<<<nb, KKB_RED_THREADS, 0, s>>>(x, n, scratch);
    KKB_CHECK_LAUNCH("k_max_reduce");
    k_finish<<<1, 32, 0, s>>>(scratch, nb, 1, out);
    KKB_CHECK_LAUNCH("k_finish");
    return KKB_OK;
}

int device_pow_mean(const double *x, long long n, const double *maxv, double g, double *scratch,
                    double *out_dev, double *out_host, cudaStream_t s) {
    const int nb = blocks_for(n);
    k_pow_sum<<<nb, KKB_RED_THREADS, 0, s>>>(x, n, maxv, g, scratch);
    KKB_CHECK_LAUNCH("k_pow_sum");
    k_finish<<<1, 32, 0, s>>>(scratch, nb, 0, out_dev);
    KKB_CHECK_LAUNCH("k_finish");
    double sum = 0.0;
    KKB_TRY_CUDA(cudaMemcpyAsync(&sum, out_dev, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H pow sum");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync pow sum");
    *out_host = sum / (double)n;
    return KKB_OK;
}

int pow_map(const double *x, long long n, const double *maxv, double g, double *out, cudaStream_t s) {
    const int nb = (int)std::max<long long>(1, std::min<long long>(148 * 8, ceil_div(n, 256)));
    k_pow_map<<<nb, 256, 0, s>>>(x, n, maxv, g, out);
    KKB_CHECK_LAUNCH("k_pow_map");
    return KKB_OK;
}

// ------------------------------------------------------------- last read sample
// per pixel: tin = max_n(x sin_n + z cos_n), tout = max_m(z cos_m - x sin_m)
// (each product IEEE-rounded, then the sum: numpy's order in cli.py:118-124)
__global__ void __launch_bounds__(KKB_RED_THREADS)
k_last_read(const double *__restrict__ x, int nx, const double *__restrict__ z, int nz,
            const double *__restrict__ sin_t, const double *__restrict__ cos_t, int n_tx,
            const double *__restrict__ sin_r, const double *__restrict__ cos_r, int n_rx, double *part) {
    __shared__ double sh[32];
    double best = -INFINITY;
    const long long P = (long long)nx * nz;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P;
         p += (long long)gridDim.x * blockDim.x) {
        const double xv = x[p / nz], zv = z[p % nz];
        double tin = -INFINITY, tout = -INFINITY;
        for (int n = 0; n < n_tx; ++n)
            tin = fmax(tin, __dadd_rn(__dmul_rn(xv, sin_t[n]), __dmul_rn(zv, cos_t[n])));
        for (int m = 0; m < n_rx; ++m)
            tout = fmax(tout, __dadd_rn(__dmul_rn(zv, cos_r[m]), -__dmul_rn(xv, sin_r[m])));
        best = fmax(best, __dadd_rn(tin, tout));
    }
    best = block_max(best, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = best;
}

int last_read_max(const double *x, int nx, const double *z, int nz, const double *sin_t,
                  const double *cos_t, int n_tx, const double *sin_r, const double *cos_r, int n_rx,
                  double *scratch, double *out, cudaStream_t s) {
    const int nb = blocks_for((long long)nx * nz);
    k_last_read<<<nb, KKB_RED_THREADS, 0, s>>>(x, nx, z, nz, sin_t, cos_t, n_tx, sin_r, cos_r, n_rx,
                                               scratch);
    KKB_CHECK_LAUNCH("k_last_read");
    k_finish<<<1, 32, 0, s>>>(scratch, nb, 1, out);
    KKB_CHECK_LAUNCH("k_finish");
    return KKB_OK;
}

}  // namespace kkb
