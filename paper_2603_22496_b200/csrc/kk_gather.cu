// K4 delay tables, K5 kk pixel gather, K6 detection / log-compression epilogue.
//
// K5 replaces _kk_kernel (beamform.py:212-236).  Work decomposition:
//   * CTA = one TZ x TX pixel tile of one frame (TZ = 32*WZ rows along depth,
//     lanes along z so a warp reads neighbouring samples; TX = WX*PX columns,
//     each thread owns PX pixels of one row).
//   * The (transmit n, receive-chunk) stages are pipelined: while stage s is
//     summed, the per-pair trace windows of stage s+1 stream from L2/HBM into
//     the other shared-memory buffer with cp.async (LDGSTS, zero-fill outside
//     [0, T)).  A window covers every tap the tile can read for that pair
//     (tile-corner delays +-1 sample: the delay is affine in (ix, iz)).
//   * Per pixel-pair: fi = ((ltx+ltz)+lrz-lrx)*fs+shift in float64 with
//     explicit _rn intrinsics (no FMA contraction: the exact IEEE sequence
//     of beamform.py:223,225), floor via RD(fi + 1.5*2^52) (no F2I), the
//     in-window predicate on the integer, the lerp weight from the mantissa
//     of fi - (floor(fi) - 1).  Taps and partial sums over receive angles
//     are float32; each transmit's partial is folded into a float64 total,
//     in fixed order (deterministic; no atomics).
// Output complex64 or complex128, plus optional fused |IQ|^2 and per-frame
// max for the dB epilogue (K6).

#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kk.cuh"

namespace kkb {

__device__ int g_device_error = 0;

int take_device_error(int *out) {
    int h = 0;
    KKB_TRY_CUDA(cudaMemcpyFromSymbol(&h, g_device_error, sizeof(int)), "read device error");
    int z = 0;
    KKB_TRY_CUDA(cudaMemcpyToSymbol(g_device_error, &z, sizeof(int)), "clear device error");
    *out = h;
    return KKB_OK;
}

// ------------------------------------------------------------- K4: LUTs
// x = x0 + dx*i (core.py:133-138): mul then add;  v = (x*s)/c (beamform.py:124-125)
__global__ void k_build_luts(double x0, double dx, int nx, double z0, double dz, int nz,
                             const double *__restrict__ sin_tx, const double *__restrict__ cos_tx,
                             int n_tx, const double *__restrict__ sin_rx,
                             const double *__restrict__ cos_rx, int n_rx, double c,
                             double *ltx, double *ltz, double *lrx, double *lrz) {
    const long long total = (long long)(nx + nz) * (n_tx + n_rx);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        long long r = i;
        if (r < (long long)nx * n_tx) {
            int ix = (int)(r / n_tx), n = (int)(r % n_tx);
            double x = __dadd_rn(x0, __dmul_rn(dx, (double)ix));
            ltx[r] = __ddiv_rn(__dmul_rn(x, sin_tx[n]), c);
            continue;
        }
        r -= (long long)nx * n_tx;
        if (r < (long long)nz * n_tx) {
            int iz = (int)(r / n_tx), n = (int)(r % n_tx);
            double z = __dadd_rn(z0, __dmul_rn(dz, (double)iz));
            ltz[r] = __ddiv_rn(__dmul_rn(z, cos_tx[n]), c);
            continue;
        }
        r -= (long long)nz * n_tx;
        if (r < (long long)nx * n_rx) {
            int ix = (int)(r / n_rx), m = (int)(r % n_rx);
            double x = __dadd_rn(x0, __dmul_rn(dx, (double)ix));
            lrx[r] = __ddiv_rn(__dmul_rn(x, sin_rx[m]), c);
            continue;
        }
        r -= (long long)nx * n_rx;
        {
            int iz = (int)(r / n_rx), m = (int)(r % n_rx);
            double z = __dadd_rn(z0, __dmul_rn(dz, (double)iz));
            lrz[r] = __ddiv_rn(__dmul_rn(z, cos_rx[m]), c);
        }
    }
}

int build_kk_luts(double x0, double dx, int nx, double z0, double dz, int nz, const double *sin_tx,
                  const double *cos_tx, int n_tx, const double *sin_rx, const double *cos_rx,
                  int n_rx, double c, double *ltx, double *ltz, double *lrx, double *lrz,
                  cudaStream_t s) {
    long long total = (long long)(nx + nz) * (n_tx + n_rx);
    int blocks = (int)std::min<long long>(ceil_div(total, 256), 4096);
    k_build_luts<<<blocks, 256, 0, s>>>(x0, dx, nx, z0, dz, nz, sin_tx, cos_tx, n_tx, sin_rx,
                                        cos_rx, n_rx, c, ltx, ltz, lrx, lrz);
    KKB_CHECK_LAUNCH("k_build_luts");
    return KKB_OK;
}

// (rows, cols) -> (cols, rows)
__global__ void k_transpose_f64(const double *__restrict__ in, int rows, int cols, double *out) {
    long long total = (long long)rows * cols;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int r = (int)(i / cols), c = (int)(i % cols);
        out[(long long)c * rows + r] = in[i];
    }
}

int transpose_f64(const double *in, int rows, int cols, double *out, cudaStream_t s) {
    long long total = (long long)rows * cols;
    int blocks = (int)std::min<long long>(ceil_div(total, 256), 4096);
    k_transpose_f64<<<blocks, 256, 0, s>>>(in, rows, cols, out);
    KKB_CHECK_LAUNCH("k_transpose_f64");
    return KKB_OK;
}

// ------------------------------------------------------------- delay helper
__device__ __forceinline__ double kk_delay(double t1, double lz, double lx, double fs, double shift) {
    // ((ltx + ltz) + lrz - lrx) * fs + shift, IEEE round-to-nearest at every step
    return __dadd_rn(__dmul_rn(__dsub_rn(__dadd_rn(t1, lz), lx), fs), shift);
}

// Tap index of one (pixel, pair): linear i0 = floor(fi) valid iff 0 <= i0 <= T-2,
// nearest j = floor(fi + 0.5) valid iff 0 <= j <= T-1 (beamform.py:226-235).
// y = RD(arg + 1.5*2^52) is returned for the lerp weight.
template <bool LINEAR>
__device__ __forceinline__ bool tap_index(double fi, int T, int &F, double &y) {
    y = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC);
    F = __double2loint(y);
    return (__double2hiint(y) == KKB_MAGIC_HI) &&
           ((unsigned)F <= (unsigned)(LINEAR ? T - 2 : T - 1));
}

// Diagnostic twin of the gather's index math: idx[ix, iz, n, m] = tap index or -1.
template <bool LINEAR>
__global__ void k_kk_taps(const double *__restrict__ ltx, const double *__restrict__ ltz,
                          const double *__restrict__ lrx, const double *__restrict__ lrz, int N,
                          int M, int T, int nx, int nz, double fs, double shift, int *idx) {
    const long long total = (long long)nx * nz * N * M;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int m = (int)(i % M);
        long long r = i / M;
        int n = (int)(r % N);
        r /= N;
        int iz = (int)(r % nz), ix = (int)(r / nz);
        double t1 = __dadd_rn(ltx[(long long)ix * N + n], ltz[(long long)iz * N + n]);
        double fi = kk_delay(t1, lrz[(long long)iz * M + m], lrx[(long long)ix * M + m], fs, shift);
        int F;
        double y;
        idx[i] = tap_index<LINEAR>(fi, T, F, y) ? F : -1;
    }
}

int kk_taps(const double *ltx, const double *ltz, const double *lrx, const double *lrz, int N, int M,
            int T, int nx, int nz, double fs, double shift, int linear, int *idx, cudaStream_t s) {
    long long total = (long long)nx * nz * N * M;
    int blocks = (int)std::min<long long>(ceil_div(total, 256), 148 * 32);
    if (linear)
        k_kk_taps<true><<<blocks, 256, 0, s>>>(ltx, ltz, lrx, lrz, N, M, T, nx, nz, fs, shift, idx);
    else
        k_kk_taps<false><<<blocks, 256, 0, s>>>(ltx, ltz, lrx, lrz, N, M, T, nx, nz, fs, shift, idx);
    KKB_CHECK_LAUNCH("k_kk_taps");
    return KKB_OK;
}

// ------------------------------------------------------------- window size pre-pass
// One thread per (tile, n, m): taps the tile can touch span
// [floor(min corner fi) - 1, floor(max corner fi) + 2]; record the maximum length.
__global__ void k_kk_window(const double *__restrict__ ltx, const double *__restrict__ ltz,
                            const double *__restrict__ lrx, const double *__restrict__ lrz, int N,
                            int M, int nx, int nz, int TX, int TZ, double fs, double shift,
                            int *wmax) {
    const int tiles_z = (nz + TZ - 1) / TZ, tiles_x = (nx + TX - 1) / TX;
    const long long total = (long long)tiles_z * tiles_x * N * M;
    int best = 0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int m = (int)(i % M);
        long long r = i / M;
        int n = (int)(r % N);
        r /= N;
        int tx = (int)(r % tiles_x), tz = (int)(r / tiles_x);
        int ixs[2] = {tx * TX, min(tx * TX + TX - 1, nx - 1)};
        int izs[2] = {tz * TZ, min(tz * TZ + TZ - 1, nz - 1)};
        double lo = 1e300, hi = -1e300;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) {
                int ix = ixs[a], iz = izs[b];
                double t1 = __dadd_rn(ltx[(long long)ix * N + n], ltz[(long long)iz * N + n]);
                double fi = kk_delay(t1, lrz[(long long)iz * M + m], lrx[(long long)ix * M + m], fs,
                                     shift);
                lo = fmin(lo, fi);
                hi = fmax(hi, fi);
            }
        double span = floor(hi) - floor(lo) + 4.0;
        int w = span > 1e9 ? 1000000000 : (int)span;
        best = max(best, w);
    }
    atomicMax(wmax, best);
}

int kk_window(const double *ltx, const double *ltz, const double *lrx, const double *lrz, int N,
              int M, int nx, int nz, double fs, double shift, int *window_out, cudaStream_t s) {
    int *d = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&d, sizeof(int), s), "cudaMallocAsync(window)");
    KKB_TRY_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s), "memset(window)");
    k_kk_window<<<512, 256, 0, s>>>(ltx, ltz, lrx, lrz, N, M, nx, nz, KKB_KK_TX, KKB_KK_TZ, fs, shift,
                                    d);
    KKB_CHECK_LAUNCH("k_kk_window");
    int h = 0;
    KKB_TRY_CUDA(cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s), "copy window");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync window");
    cudaFreeAsync(d, s);
    // round up to a multiple of 2 samples (16 B) for tidy cp.async rows
    *window_out = (h + 1) & ~1;
    return KKB_OK;
}

// ------------------------------------------------------------- K5 kernel
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc, bool valid) {
    unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
    int sz = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int Nw>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(Nw) : "memory");
}

struct KKArgs {
    const float2 *data;
    long long data_fs;  // frame stride, complex elements
    int N, M, T;
    const double *ltx;   // (X, N)
    const double *ltzT;  // (N, Z)
    const double *lrx;   // (X, M)
    const double *lrzT;  // (M, Z)
    const double *w;     // (M,) or null
    double fs, shift;
    int nx, nz;
    int W;    // window length (samples)
    int MCH;  // receive angles per pipeline stage
    void *out;
    int out_kind;
    long long out_fs;
    float *inten;
    unsigned *fmax;
};

template <int WZ, int WX, int PX, bool LINEAR>
__global__ void __launch_bounds__(WZ *WX * 32)
k_kk_gather(const KKArgs a) {
    constexpr int TZ = 32 * WZ;
    constexpr int TX = WX * PX;
    constexpr int NT = WZ * WX * 32;
    const int N = a.N, M = a.M, T = a.T, W = a.W, MCH = a.MCH, nx = a.nx, nz = a.nz;
    const int nchunk = (M + MCH - 1) / MCH;
    const int nstage = N * nchunk;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2 *win = reinterpret_cast<float2 *>(smem_raw);              // [2][MCH][W]
    double *lrz_s = reinterpret_cast<double *>(win + 2 * MCH * W);    // [M][TZ]
    double *lrx_s = lrz_s + M * TZ;                                   // [M][TX]
    double *ltx_s = lrx_s + M * TX;                                   // [N][TX]
    float *w_s = reinterpret_cast<float *>(ltx_s + N * TX);           // [M]
    int *lo_s = reinterpret_cast<int *>(w_s + M);                     // [3][MCH] (slot s % 3)

    const int tid = threadIdx.x;
    const int f = blockIdx.z;
    const int ix0 = blockIdx.y * TX, iz0 = blockIdx.x * TZ;
    const int lane = tid & 31, warp = tid >> 5;
    const int wz = warp % WZ, wx = warp / WZ;
    const int rz = wz * 32 + lane;
    const int iz = iz0 + rz;
    const int izc = min(iz, nz - 1);
    const int cx = wx * PX;
    const int cxb = min(TX - 1, nx - 1 - ix0);   // last valid local column
    const int rzb = min(TZ - 1, nz - 1 - iz0);   // last valid local row

    for (int i = tid; i < M * TZ; i += NT) {
        int m = i / TZ, r = i - m * TZ;
        lrz_s[i] = a.lrzT[(long long)m * nz + min(iz0 + r, nz - 1)];
    }
    for (int i = tid; i < M * TX; i += NT) {
        int m = i / TX, c = i - m * TX;
        lrx_s[i] = a.lrx[(long long)min(ix0 + c, nx - 1) * M + m];
    }
    for (int i = tid; i < N * TX; i += NT) {
        int n = i / TX, c = i - n * TX;
        ltx_s[i] = a.ltx[(long long)min(ix0 + c, nx - 1) * N + n];
    }
    for (int i = tid; i < M; i += NT) w_s[i] = a.w ? (float)a.w[i] : 1.0f;
    __syncthreads();

    const float2 *dframe = a.data + (long long)f * a.data_fs;
    const double fs = a.fs, shift = a.shift;

    // window start of stage s for its chunk-local receive index q (thread q computes)
    auto stage_lo = [&](int s, int q) -> int {
        int n = s / nchunk, m = (s - n * nchunk) * MCH + q;
        double lo = 1e300;
        double tza = a.ltzT[(long long)n * nz + iz0];
        double tzb = a.ltzT[(long long)n * nz + iz0 + rzb];
        double t1[4] = {__dadd_rn(ltx_s[n * TX], tza), __dadd_rn(ltx_s[n * TX], tzb),
                        __dadd_rn(ltx_s[n * TX + cxb], tza), __dadd_rn(ltx_s[n * TX + cxb], tzb)};
        double lz[4] = {lrz_s[m * TZ], lrz_s[m * TZ + rzb], lrz_s[m * TZ], lrz_s[m * TZ + rzb]};
        double lx[4] = {lrx_s[m * TX], lrx_s[m * TX], lrx_s[m * TX + cxb], lrx_s[m * TX + cxb]};
#pragma unroll
        for (int c = 0; c < 4; ++c) lo = fmin(lo, kk_delay(t1[c], lz[c], lx[c], fs, shift));
        lo = floor(lo) - 1.0;
        lo = fmax(fmin(lo, 1.0e9), -1.0e9);
        return (int)lo;
    };
    auto issue = [&](int s, int buf) {
        int n = s / nchunk, m0 = (s - n * nchunk) * MCH;
        int mc = min(MCH, M - m0);
        const int *lo_q = lo_s + (s % 3) * MCH;
        for (int i = tid; i < mc * W; i += NT) {
            int q = i / W, e = i - q * W;
            int smp = lo_q[q] + e;
            bool ok = (unsigned)smp < (unsigned)T;
            const float2 *src = dframe + ((long long)n * M + m0 + q) * T + (ok ? smp : 0);
            cp_async8(&win[(buf * MCH + q) * W + e], src, ok);
        }
        cp_async_commit();
    };

    if (tid < min(MCH, M)) lo_s[tid] = stage_lo(0, tid);
    __syncthreads();
    issue(0, 0);

    double accd_r[PX], accd_i[PX];
    float accr[PX], acci[PX];
    double t1[PX];
#pragma unroll
    for (int j = 0; j < PX; ++j) {
        accd_r[j] = accd_i[j] = 0.0;
        accr[j] = acci[j] = 0.f;
    }

    for (int s = 0; s < nstage; ++s) {
        const int buf = s & 1;
        const int n = s / nchunk, ch = s - n * nchunk, m0 = ch * MCH;
        const int mc = min(MCH, M - m0);
        // window starts of stage s+1 go to slot (s+1)%3: slot (s-2)%3 was last read
        // before the previous iteration's first barrier, so no reader remains
        if (s + 1 < nstage) {
            int n1 = (s + 1) / nchunk, m1 = ((s + 1) - n1 * nchunk) * MCH;
            if (tid < min(MCH, M - m1)) lo_s[((s + 1) % 3) * MCH + tid] = stage_lo(s + 1, tid);
        }
        __syncthreads();
        if (s + 1 < nstage) {
            issue(s + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();

        if (ch == 0) {
            double tz = a.ltzT[(long long)n * nz + izc];
#pragma unroll
            for (int j = 0; j < PX; ++j) t1[j] = __dadd_rn(ltx_s[n * TX + min(cx + j, cxb)], tz);
        }
        const float2 *wb = win + buf * MCH * W;
        for (int q = 0; q < mc; ++q) {
            const int m = m0 + q;
            const double lz = lrz_s[m * TZ + min(rz, rzb)];
            const float wm = w_s[m];
            const int lo = lo_s[(s % 3) * MCH + q];
            const float2 *wv = wb + q * W;
#pragma unroll
            for (int j = 0; j < PX; ++j) {
                const double lx = lrx_s[m * TX + min(cx + j, cxb)];
                const double fi = kk_delay(t1[j], lz, lx, fs, shift);
                int F;
                double y;
                if (tap_index<LINEAR>(fi, T, F, y)) {
                    if (LINEAR) {
                        const int e = min(max(F - lo, 0), W - 2);
                        const float2 d0 = wv[e], d1 = wv[e + 1];
                        const float fr = frac_from_floor(fi, y);
                        const float vr = fmaf(fr, d1.x - d0.x, d0.x);
                        const float vi = fmaf(fr, d1.y - d0.y, d0.y);
                        accr[j] = fmaf(wm, vr, accr[j]);
                        acci[j] = fmaf(wm, vi, acci[j]);
                    } else {
                        const float2 d = wv[min(max(F - lo, 0), W - 1)];
                        accr[j] = fmaf(wm, d.x, accr[j]);
                        acci[j] = fmaf(wm, d.y, acci[j]);
                    }
                }
            }
        }
        if (ch == nchunk - 1) {
#pragma unroll
            for (int j = 0; j < PX; ++j) {
                accd_r[j] += (double)accr[j];
                accd_i[j] += (double)acci[j];
                accr[j] = acci[j] = 0.f;
            }
        }
    }

    // epilogue: IQ (+ fused intensity and frame max)
    float fmx = 0.f;
    if (iz < nz) {
#pragma unroll
        for (int j = 0; j < PX; ++j) {
            const int ix = ix0 + cx + j;
            if (ix < nx) {
                const long long p = (long long)f * a.out_fs + (long long)ix * nz + iz;
                if (a.out_kind == KKB_OUT_C128) {
                    reinterpret_cast<double2 *>(a.out)[p] = make_double2(accd_r[j], accd_i[j]);
                } else {
                    reinterpret_cast<float2 *>(a.out)[p] =
                        make_float2((float)accd_r[j], (float)accd_i[j]);
                }
                if (a.inten) {
                    float I = (float)(accd_r[j] * accd_r[j] + accd_i[j] * accd_i[j]);
                    a.inten[p] = I;
                    fmx = fmaxf(fmx, I);
                }
            }
        }
    }
    if (a.fmax) {
        // warp max, then one atomic per warp (non-negative floats order as uints)
        for (int o = 16; o > 0; o >>= 1) fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
        if (lane == 0) atomicMax(a.fmax + f, __float_as_uint(fmx));
    }
}

static size_t kk_smem_bytes(int N, int M, int W, int MCH) {
    return sizeof(float2) * 2 * MCH * W + sizeof(double) * ((size_t)M * KKB_KK_TZ + (size_t)M * KKB_KK_TX +
                                                            (size_t)N * KKB_KK_TX) +
           sizeof(float) * M + sizeof(int) * 3 * MCH;
}

int kk_gather(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
              const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
              double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
              long long out_fs, float *inten, unsigned *fmax, int W, cudaStream_t s) {
    if (n_frames <= 0 || nx <= 0 || nz <= 0) return KKB_OK;
    if (W < 2) W = 2;
    // receive angles per stage: as many as fit a ~96 KB double buffer
    const size_t budget = 200 * 1024;
    int MCH = M;
    while (MCH > 1 && kk_smem_bytes(N, M, W, MCH) > budget) MCH = (MCH + 1) / 2;
    size_t sm = kk_smem_bytes(N, M, W, MCH);
    if (sm > 227 * 1024) {
        set_error("kk tile needs %zu B of shared memory (N=%d M=%d window=%d)", sm, N, M, W);
        return KKB_ERR_UNSUPPORTED;
    }
    KKArgs a{data, data_fs, N, M, T, ltx, ltzT, lrx, lrzT, w, fs, shift, nx, nz, W, MCH,
             out, out_kind, out_fs, inten, fmax};
    dim3 grid((unsigned)ceil_div(nz, KKB_KK_TZ), (unsigned)ceil_div(nx, KKB_KK_TX), (unsigned)n_frames);
    dim3 block(KKB_KK_WZ * KKB_KK_WX * 32);
    if (linear) {
        auto fn = k_kk_gather<KKB_KK_WZ, KKB_KK_WX, KKB_KK_PX, true>;
        KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                     "smem attr kk");
        fn<<<grid, block, sm, s>>>(a);
    } else {
        auto fn = k_kk_gather<KKB_KK_WZ, KKB_KK_WX, KKB_KK_PX, false>;
        KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                     "smem attr kk");
        fn<<<grid, block, sm, s>>>(a);
    }
    KKB_CHECK_LAUNCH("k_kk_gather");
    return KKB_OK;
}

// ------------------------------------------------------------- K6 epilogues
__global__ void k_log_compress(const float *__restrict__ inten, const unsigned *__restrict__ fmax,
                               int n_frames, long long P, float floor_db, float *db) {
    const long long total = (long long)n_frames * P;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        int f = (int)(i / P);
        float mx = __uint_as_float(fmax[f]);
        float v = inten[i];
        float d = (mx > 0.f && v > 0.f) ? 10.0f * log10f(v / mx) : floor_db;
        db[i] = fmaxf(d, floor_db);
    }
}

int log_compress(const float *inten, const unsigned *fmax, int n_frames, long long P, float floor_db,
                 float *db, cudaStream_t s) {
    long long total = (long long)n_frames * P;
    if (total <= 0) return KKB_OK;
    int blocks = (int)std::min<long long>(ceil_div(total, 256), 148 * 16);
    k_log_compress<<<blocks, 256, 0, s>>>(inten, fmax, n_frames, P, floor_db, db);
    KKB_CHECK_LAUNCH("k_log_compress");
    return KKB_OK;
}

// coherent |sum_j B_j|^2 / incoherent sum_j |B_j|^2 (beamform.py:396-411), float64
__global__ void k_compound(const double2 *__restrict__ im, int J, long long P, int mode, double *out) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < P;
         p += (long long)gridDim.x * blockDim.x) {
        double ar = 0.0, ai = 0.0, acc = 0.0;
        for (int j = 0; j < J; ++j) {
            double2 v = im[(long long)j * P + p];
            if (mode == 0) {
                ar += v.x;
                ai += v.y;
            } else {
                acc += v.x * v.x + v.y * v.y;
            }
        }
        out[p] = mode == 0 ? ar * ar + ai * ai : acc;
    }
}

int compound(const void *images, int J, long long P, int mode, double *out, cudaStream_t s) {
    if (P <= 0) return KKB_OK;
    int blocks = (int)std::min<long long>(ceil_div(P, 256), 148 * 16);
    k_compound<<<blocks, 256, 0, s>>>(reinterpret_cast<const double2 *>(images), J, P, mode, out);
    KKB_CHECK_LAUNCH("k_compound");
    return KKB_OK;
}

}  // namespace kkb
