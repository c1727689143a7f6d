// K4 delay tables, K5 kk pixel gather, K6 detection / log-compression epilogue.
//
// K5 replaces _kk_kernel (beamform.py:212-236).  Work decomposition:
//   * CTA = one TZ x TX = 32 x 64 pixel tile of one frame (8 warps); a warp
//     covers 8 depth rows x 32 columns and lane (zt, xt) = (lane % 4, lane / 4)
//     owns the 2 x 4 pixels rows zt + {0, 4}, columns xt + {0, 8, 16, 24}, so
//     the per-receive table reads (row delays, column delays, window start +
//     weight) are shared by 8 taps.
//   * The (transmit n, receive-chunk) stages are pipelined: while stage s is
//     summed, the trace windows of stage s+1 are loaded into registers and
//     written to the other shared-memory buffer as (2 d0 - d1, d1 - d0)
//     float4 entries (one 16 B read per linear tap pair).  A window covers
//     every tap the tile can read for that pair (tile-corner delays +-1
//     sample: the delay is affine in (ix, iz)); window starts for all pairs
//     are computed once per CTA.
//   * Per pixel-pair: fi = ((ltx+ltz)+lrz-lrx)*fs+shift in float64 with
//     explicit _rn intrinsics (no FMA contraction: the exact IEEE sequence
//     of beamform.py:223,225), then ONE round-down add of 1.5*2^20 whose high
//     word minus 0x41380000 is floor(fi) and whose low word is frac*2^32 —
//     the in-window predicate is folded into the staged window (entries of
//     out-of-trace samples are zero), the lerp weight is (low >> 9) | 1.0f.
//     Taps and the per-pixel sum are float32, accumulated in fixed order
//     (deterministic, no atomics).  A batch runs KKB_KK_FR frames per CTA: the
//     tables and every tap's index math are shared, only the window reads
//     and the accumulators are per frame.
//   * Geometries whose window or pair tables do not fit shared memory run the
//     per-pixel kernel k_kk_direct (same index math, lerp and epilogue).
// Output complex64 or complex128, plus optional fused |IQ|^2 (optionally
// accumulated across receive sets) and per-frame max for the dB epilogue
// (K6), and optional P2P stores of every pixel into peers' image buffers
// (fused row-block all-gather, kkb_kk_plan_run_scatter).

#include <algorithm>
#include <atomic>
#include <cstring>
#include <cstdlib>
#include <type_traits>
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
// sv = RD(arg + 1.5*2^20) (arg = fi, or RN(fi + 0.5) for nearest): for
// |arg| < 2^19 its high word minus 0x41380000 is floor(arg) exactly (the
// round-down never crosses an integer) and its low word is frac(arg)*2^32;
// any larger |arg| gives F >= 2^19 or F < 0, i.e. out of window.  This one
// function is the index math of the K5 gather and of kkb_kk_taps.
#define KKB_FLOOR_MAGIC2 1572864.0   // 1.5 * 2^20: ulp 2^-32
#define KKB_MAGIC2_HI 0x41380000     // high word of 1.5*2^20 + 0
template <bool LINEAR>
__device__ __forceinline__ bool tap_index(double fi, int T, int &F, double &sv) {
    sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC2);
    F = __double2hiint(sv) - KKB_MAGIC2_HI;
    return (unsigned)F <= (unsigned)(LINEAR ? T - 2 : T - 1);
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
// One thread per (tile, n, m) of each tile size: taps the tile can touch span
// [floor(min corner fi) - 1, floor(max corner fi) + 2]; wmax[s] = the largest
// length over the tiles of size s (big, mid, small) — one launch, one sync.
struct KKTileSizes {
    int tx[4], tz[4];
};

__global__ void k_kk_window(const double *__restrict__ ltx, const double *__restrict__ ltz,
                            const double *__restrict__ lrx, const double *__restrict__ lrz, int N,
                            int M, int nx, int nz, KKTileSizes ts, double fs, double shift,
                            int *wmax) {
    long long cum[5] = {0, 0, 0, 0, 0};
    for (int s = 0; s < 4; ++s)
        cum[s + 1] = cum[s] + (long long)((nz + ts.tz[s] - 1) / ts.tz[s]) *
                                  ((nx + ts.tx[s] - 1) / ts.tx[s]) * N * M;
    int best[4] = {0, 0, 0, 0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < cum[4];
         i += (long long)gridDim.x * blockDim.x) {
        const int sz = i < cum[1] ? 0 : (i < cum[2] ? 1 : (i < cum[3] ? 2 : 3));
        const int TX = ts.tx[sz], TZ = ts.tz[sz];
        const int tiles_x = (nx + TX - 1) / TX;
        long long r = i - cum[sz];
        int m = (int)(r % M);
        r /= M;
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
        best[sz] = max(best[sz], w);
    }
    for (int s = 0; s < 4; ++s)
        if (best[s]) atomicMax(wmax + s, best[s]);
}

int kk_window(const double *ltx, const double *ltz, const double *lrx, const double *lrz, int N,
              int M, int nx, int nz, double fs, double shift, KKWindows *win, cudaStream_t s) {
    int *d = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&d, 4 * sizeof(int), s), "cudaMallocAsync(window)");
    KKB_TRY_CUDA(cudaMemsetAsync(d, 0, 4 * sizeof(int), s), "memset(window)");
    KKTileSizes ts{{KKB_KK_TX, KKB_KK_M_TX, KKB_KK_S_TX, KKB_KK_TC_TX},
                   {KKB_KK_TZ, KKB_KK_M_TZ, KKB_KK_S_TZ, KKB_KK_TC_TZ}};
    k_kk_window<<<512, 256, 0, s>>>(ltx, ltz, lrx, lrz, N, M, nx, nz, ts, fs, shift, d);
    KKB_CHECK_LAUNCH("k_kk_window");
    int h[4] = {0, 0, 0, 0};
    KKB_TRY_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, s), "copy window");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync window");
    cudaFreeAsync(d, s);
    // round up to a multiple of 2 samples (16 B) for tidy cp.async rows
    win->big = (h[0] + 1) & ~1;
    win->mid = (h[1] + 1) & ~1;
    win->small = (h[2] + 1) & ~1;
    win->tc = (h[3] + 1) & ~1;
    win->bad = 0;
    if (const char *k = getenv("KKB_KK_WINDOW_SHRINK")) {  // fault injection (tests): undersized windows
        const int d = atoi(k);
        win->big = std::max(2, win->big - d);
        win->mid = std::max(2, win->mid - d);
        win->small = std::max(2, win->small - d);
        win->tc = std::max(2, win->tc - d);
    }
    return KKB_OK;
}

// ------------------------------------------------------------- K5 kernel
// Tile: TZ = 8*WZ depth rows x TX = 8*CX*WX lateral columns.  A warp covers an
// 8 x 8CX patch; lane (zt, xt) = (lane % 4, lane / 4) owns the 2 x CX pixels
// rows zt + {0, 4}, columns xt + 8j (j < CX) of it.  For a fixed (a, b) the 32
// lanes form a 4 x 8 block whose delays span only ~3*dfi/dz + 7*dfi/dx
// samples, so their tap reads hit a few shared-memory words (broadcast).
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
    int accum;  // 1: intensity += |IQ|^2 (incoherent multi-set compounding)
    // fused row-block all-gather: when ndst > 0 every IQ pixel is also stored
    // at dst[d] + dst_off + ix*nz + iz for d < ndst (peers' image buffers
    // mapped over NVLink with CUDA IPC; the stores are the collective)
    int ndst;
    long long dst_off;
    void *dst[KKB_MAX_DST];
    int n_frames;  // frames in the batch (the multi-frame instance skips the tail)
    // incoherent multi-set compounding (KKSets; the MS kernel instances only)
    int nsets;
    int set_m0[KKB_MAX_SETS + 1];
    long long out_set_stride;
    // when set, the launch is the tensor-core gather's standby: every CTA
    // returns at once unless *run_if != 0 (kk_gather_tc.cu, non-finite batch)
    const unsigned *run_if;
};

// packed LUT index: tile row r -> (r/8)*4 + r%4 pair slot, a = (r/4)&1
__device__ __forceinline__ int prow(int r) { return ((r >> 3) << 3) + ((r & 3) << 1) + ((r >> 2) & 1); }
// tile column c -> warp block c/(8CX), lane slot c%8, column j = (c/8)%CX: the
// CX columns of one lane are contiguous (CX/2 16-byte reads)
template <int CX>
__device__ __forceinline__ int pcol(int c) {
    return (c / (8 * CX)) * (8 * CX) + (c & 7) * CX + ((c >> 3) % CX);
}

// |IQ|^2 as one explicit float sequence (no contraction choice left to the
// compiler), shared by the tiled and per-pixel kernels
__device__ __forceinline__ float mag2(float vr, float vi) { return __fmaf_rn(vr, vr, __fmul_rn(vi, vi)); }

// IQ pixel store (complex64 or complex128)
__device__ __forceinline__ void store_iq(void *out, int kind, long long px, float vr, float vi) {
    if (kind == KKB_OUT_C128)
        reinterpret_cast<double2 *>(out)[px] = make_double2(vr, vi);
    else
        reinterpret_cast<float2 *>(out)[px] = make_float2(vr, vi);
}

// MS: the stage sequence runs set by set (set j: transmits n asc, receive
// chunks of [set_m0[j], set_m0[j+1]) asc); at the end of each set its image is
// stored, |B_j|^2 added to a per-pixel running intensity and the sums reset.
template <int WZ, int WX, int CX, bool LINEAR, int FR, bool MS = false>
__global__ void __launch_bounds__(WZ *WX * 32, KKB_KK_MIN_CTAS * KKB_KK_WZ * KKB_KK_WX / (WZ * WX))
k_kk_gather(const KKArgs a) {
    if (a.run_if && *a.run_if == 0) return;
    constexpr int TZ = 8 * WZ;
    constexpr int TX = 8 * CX * WX;
    constexpr int NT = WZ * WX * 32;
    // staged window entries per thread (the big instance stages KKB_KK_STAGE_ELEMS)
    constexpr int EPT = KKB_KK_STAGE_ELEMS / (32 * KKB_KK_WZ * KKB_KK_WX);
    using Entry = typename std::conditional<LINEAR, float4, float2>::type;
    const int N = a.N, M = a.M, T = a.T, W = a.W, MCH = a.MCH, nx = a.nx, nz = a.nz;
    int nchunk = (M + MCH - 1) / MCH;
    int nstage = N * nchunk;
    int set = 0, set_end = M;  // MS: current set and its receive range end
    if constexpr (MS) {
        nstage = 0;
        for (int j = 0; j < a.nsets; ++j) nstage += N * ((a.set_m0[j + 1] - a.set_m0[j] + MCH - 1) / MCH);
        set_end = a.set_m0[1];
        nchunk = (set_end + MCH - 1) / MCH;
    }

    extern __shared__ __align__(16) unsigned char smem_raw[];
    Entry *win = reinterpret_cast<Entry *>(smem_raw);                  // [2][FR][MCH][W]
    double *lrz_p = reinterpret_cast<double *>(win + 2 * FR * MCH * W);  // [M][TZ] packed rows
    double *lrx_p = lrz_p + M * TZ;                                    // [M][TX] packed cols
    double *ltz_p = lrx_p + M * TX;                                    // [N][TZ]
    double *ltx_p = ltz_p + N * TZ;                                    // [N][TX]
    // per (n, m): window start lo and weight w[m] (bits), one 8 B read per receive
    int2 *lw_s = reinterpret_cast<int2 *>(ltx_p + N * TX);             // [N][M]

    const int tid = threadIdx.x;
    // FR frames per CTA share the tables and every tap's index math; the
    // taps of frame fr come from its own window block
    const int f0 = blockIdx.z * FR;
    const int ix0 = blockIdx.y * TX, iz0 = blockIdx.x * TZ;
    const int lane = tid & 31, warp = tid >> 5;
    const int wz = warp % WZ, wx = warp / WZ;
    const int zt = lane & 3, xt = lane >> 2;
    const int zq = wz * 4 + zt;   // packed row-pair slot (rows zq-> r, r+4)
    const int xq = wx * 8 + xt;   // packed column slot (cols c + 8j, j < CX)
    const int rzb = min(TZ - 1, nz - 1 - iz0);
    const int cxb = min(TX - 1, nx - 1 - ix0);

    for (int i = tid; i < M * TZ; i += NT) {
        int m = i / TZ, r = i - m * TZ;
        lrz_p[m * TZ + prow(r)] = a.lrzT[(long long)m * nz + min(iz0 + r, nz - 1)];
    }
    for (int i = tid; i < N * TZ; i += NT) {
        int n = i / TZ, r = i - n * TZ;
        ltz_p[n * TZ + prow(r)] = a.ltzT[(long long)n * nz + min(iz0 + r, nz - 1)];
    }
    for (int i = tid; i < M * TX; i += NT) {
        int m = i / TX, c = i - m * TX;
        lrx_p[m * TX + pcol<CX>(c)] = a.lrx[(long long)min(ix0 + c, nx - 1) * M + m];
    }
    for (int i = tid; i < N * TX; i += NT) {
        int n = i / TX, c = i - n * TX;
        ltx_p[n * TX + pcol<CX>(c)] = a.ltx[(long long)min(ix0 + c, nx - 1) * N + n];
    }
    __syncthreads();

    const double fs = a.fs, shift = a.shift;
    // window start of every (n, m): floor of the smallest corner delay, minus 1
    for (int i = tid; i < N * M; i += NT) {
        const int n = i / M, m = i - n * M;
        double lo = 1e300;
#pragma unroll
        for (int cr = 0; cr < 2; ++cr)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int r = cr ? rzb : 0, c = cc ? cxb : 0;
                const double t1 = __dadd_rn(ltx_p[n * TX + pcol<CX>(c)], ltz_p[n * TZ + prow(r)]);
                lo = fmin(lo, kk_delay(t1, lrz_p[m * TZ + prow(r)], lrx_p[m * TX + pcol<CX>(c)], fs, shift));
            }
        lo = fmax(fmin(floor(lo) - 1.0, 1.0e9), -1.0e9);
        lw_s[i] = make_int2((int)lo, __float_as_int(a.w ? (float)a.w[m] : 1.0f));
    }
    __syncthreads();

    // register-staged window entries of one stage; entry tid + i*NT of a stage
    // is (frame fr, receive q, sample e) of the [FR][MCH][W] window block,
    // the same every stage
    float2 s0[EPT], s1[EPT];
    int qe[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int idx = tid + i * NT, fr = idx / (MCH * W), rem = idx - fr * MCH * W, q = rem / W;
        qe[i] = (fr << 26) | (q << 16) | (rem - q * W);
    }
    // stage (n, m0): receive angles m0 .. m0+mc-1 of transmit n, all FR frames
    auto load_stage = [&](int n, int m0, int mend) {
        const int mc = min(MCH, mend - m0);
        const int2 *lo_q = lw_s + n * M + m0;
        const float2 *base0 = a.data + (long long)f0 * a.data_fs + (long long)(n * M + m0) * T;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            s0[i] = s1[i] = make_float2(0.f, 0.f);
            const int fr = qe[i] >> 26, q = (qe[i] >> 16) & 1023, e = qe[i] & 0xFFFF;
            if (tid + i * NT < FR * MCH * W && q < mc) {
                const float2 *base = base0;
                if constexpr (FR > 1) {
                    // frames past the batch re-read the first frame (results discarded)
                    const int fe = f0 + fr < a.n_frames ? f0 + fr : f0;
                    base = a.data + (long long)fe * a.data_fs + (long long)(n * M + m0) * T;
                }
                const int smp = lo_q[q].x + e;
                const float2 *tr = base + q * T;
                // entry smp stays zero unless a tap at smp is in the reference's
                // window: linear 0 <= i0 <= T-2 (both d0, d1 exist), nearest 0 <= j <= T-1
                if ((unsigned)smp <= (unsigned)(LINEAR ? T - 2 : T - 1)) {
                    s0[i] = __ldg(tr + smp);
                    if (LINEAR) s1[i] = __ldg(tr + smp + 1);
                }
            }
        }
    };
    auto store_stage = [&](int m0, int mend, int buf) {
        const int mc = min(MCH, mend - m0);
        Entry *wb = win + buf * FR * MCH * W;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int idx = tid + i * NT;
            if (idx < FR * MCH * W && ((qe[i] >> 16) & 1023) < mc) {
                if constexpr (LINEAR) {
                    // (2 d0 - d1, d1 - d0): the lerp becomes e0 + (1 + frac) * diff
                    wb[idx] = make_float4(fmaf(2.f, s0[i].x, -s1[i].x), fmaf(2.f, s0[i].y, -s1[i].y),
                                          s1[i].x - s0[i].x, s1[i].y - s0[i].y);
                } else {
                    wb[idx] = s0[i];
                }
            }
        }
    };

    float accr[FR][2][CX], acci[FR][2][CX];  // float32 per-pixel sums, fixed order
    double t1[2][CX];
#if KKB_KK_CHECK
    unsigned emax = 0;  // largest raw window index over live pairs (must stay in the window)
#endif
#pragma unroll
    for (int fr = 0; fr < FR; ++fr)
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int q = 0; q < CX; ++q) accr[fr][p][q] = acci[fr][p][q] = 0.f;
    load_stage(0, 0, set_end);
    store_stage(0, set_end, 0);
    __syncthreads();
    int n = 0, ch = 0;           // current stage
    int n1 = 0, ch1 = 0;         // next stage
    int mb = 0, mb1 = 0;         // MS: first receive angle of the current / next stage's set
    int set_end1 = set_end, nchunk1 = nchunk;
    for (int s = 0; s < nstage; ++s) {
        const int buf = s & 1;
        int m0, mc;
        bool set_done = false;
        n1 = n;
        ch1 = ch + 1;
        if constexpr (MS) {
            m0 = mb + ch * MCH;
            mc = min(MCH, set_end - m0);
            mb1 = mb;
            set_end1 = set_end;
            nchunk1 = nchunk;
            if (ch1 == nchunk) {
                ch1 = 0;
                ++n1;
                if (n1 == N) {  // next set
                    set_done = true;
                    n1 = 0;
                    if (set + 1 < a.nsets) {
                        mb1 = set_end;
                        set_end1 = a.set_m0[set + 2];
                        nchunk1 = (set_end1 - mb1 + MCH - 1) / MCH;
                    }
                }
            }
            if (s + 1 < nstage) load_stage(n1, mb1 + ch1 * MCH, set_end1);  // in flight during this stage's sums
        } else {
            m0 = ch * MCH;
            mc = min(MCH, M - m0);
            if (ch1 == nchunk) {
                ch1 = 0;
                ++n1;
            }
            if (s + 1 < nstage) load_stage(n1, ch1 * MCH, M);  // in flight during this stage's sums
        }
        if (ch == 0) {
            const double2 tz = reinterpret_cast<const double2 *>(ltz_p + n * TZ)[zq];
            double txv[CX];
#pragma unroll
            for (int j = 0; j < CX / 2; ++j) {
                const double2 tx = reinterpret_cast<const double2 *>(ltx_p + n * TX + xq * CX)[j];
                txv[2 * j] = tx.x;
                txv[2 * j + 1] = tx.y;
            }
#pragma unroll
            for (int j = 0; j < CX; ++j) {
                t1[0][j] = __dadd_rn(txv[j], tz.x);
                t1[1][j] = __dadd_rn(txv[j], tz.y);
            }
        }
        const Entry *wb = win + buf * FR * MCH * W;
        const int2 *lw_n = lw_s + n * M + m0;
        constexpr int kQUnroll = KKB_KK_QUNROLL;
#pragma unroll kQUnroll
        for (int q = 0; q < mc; ++q) {
            const int m = m0 + q;
#if KKB_KK_CHECK
            unsigned eq = 0;  // largest raw window index of this pair's taps (clamp check)
#endif
            const double2 lz = reinterpret_cast<const double2 *>(lrz_p + m * TZ)[zq];
            double lxv[CX];
#pragma unroll
            for (int j = 0; j < CX / 2; ++j) {
                const double2 lx = reinterpret_cast<const double2 *>(lrx_p + m * TX + xq * CX)[j];
                lxv[2 * j] = lx.x;
                lxv[2 * j + 1] = lx.y;
            }
            const int2 lw = lw_n[q];
            const float wm = __int_as_float(lw.y);
            // window index e = floor(arg) - lo = hi(sv) - (0x41380000 + lo); the
            // in-window predicate of tap_index() is folded into the staged window
            // (entries whose tap would be invalid are zero), so no per-tap test
            const int loC = lw.x + KKB_MAGIC2_HI;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
#pragma unroll
                for (int r = 0; r < CX; ++r) {
                    const double fi = kk_delay(t1[p][r], p ? lz.y : lz.x, lxv[r], fs, shift);
                    const double sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC2);
                    const unsigned raw = (unsigned)(__double2hiint(sv) - loC);
#if KKB_KK_CHECK
                    eq = max(eq, raw);
#endif
                    const unsigned e = min(raw, (unsigned)(LINEAR ? W - 2 : W - 1));
                    const float f1 = __uint_as_float(((unsigned)__double2loint(sv) >> 9) + 0x3F800000u);
#pragma unroll
                    for (int fr = 0; fr < FR; ++fr) {
                        const Entry *wv = wb + (fr * MCH + q) * W;
                        if constexpr (LINEAR) {
                            const float4 v = wv[e];
                            accr[fr][p][r] = fmaf(wm, fmaf(f1, v.z, v.x), accr[fr][p][r]);
                            acci[fr][p][r] = fmaf(wm, fmaf(f1, v.w, v.y), acci[fr][p][r]);
                        } else {
                            const float2 v = wv[e];
                            accr[fr][p][r] = fmaf(wm, v.x, accr[fr][p][r]);
                            acci[fr][p][r] = fmaf(wm, v.y, acci[fr][p][r]);
                        }
                    }
                }
            }
            // a clamped index reads a wrong entry unless the pair's whole window
            // lies outside the trace (every entry zero, e.g. |fi| >= 2^19)
#if KKB_KK_CHECK
            if (lw.x <= (LINEAR ? T - 2 : T - 1) && lw.x + W > 0) emax = max(emax, eq);
#endif
        }
        if constexpr (MS) {
            if (set_done) {
                // image of this set; |B|^2 added to the intensity in global memory
                // (the same float op order as one accumulating launch per set);
                // after the last set, the frame max
                const bool last = set + 1 == a.nsets;
#pragma unroll
                for (int fr = 0; fr < FR; ++fr) {
                    const int f = f0 + fr;
                    float fmx = 0.f;
                    if (f < a.n_frames) {
#pragma unroll
                        for (int p = 0; p < 2; ++p) {
                            const int iz = iz0 + wz * 8 + p * 4 + zt;
#pragma unroll
                            for (int r = 0; r < CX; ++r) {
                                const int ix = ix0 + wx * 8 * CX + r * 8 + xt;
                                if (iz < nz && ix < nx) {
                                    const float vr = accr[fr][p][r], vi = acci[fr][p][r];
                                    const long long px = (long long)f * a.out_fs + (long long)ix * nz + iz;
                                    if (a.out) store_iq(a.out, a.out_kind, set * a.out_set_stride + px, vr, vi);
                                    float I = mag2(vr, vi);
                                    if (set > 0 || a.accum) I = __fadd_rn(I, a.inten[px]);
                                    a.inten[px] = I;
                                    fmx = fmaxf(fmx, I);
                                }
                            }
                        }
                    }
                    if (last && a.fmax && f0 + fr < a.n_frames) {
                        for (int o = 16; o > 0; o >>= 1) fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
                        if (lane == 0) atomicMax(a.fmax + f, __float_as_uint(fmx));
                    }
#pragma unroll
                    for (int p = 0; p < 2; ++p)
#pragma unroll
                        for (int r = 0; r < CX; ++r) accr[fr][p][r] = acci[fr][p][r] = 0.f;
                }
                ++set;
            }
        }
        // buffer buf^1 was last read in stage s-1, which every thread finished
        // before the barrier that ended it
        if constexpr (MS) {
            if (s + 1 < nstage) store_stage(mb1 + ch1 * MCH, set_end1, buf ^ 1);
            mb = mb1;
            set_end = set_end1;
            nchunk = nchunk1;
        } else {
            if (s + 1 < nstage) store_stage(ch1 * MCH, M, buf ^ 1);
        }
        __syncthreads();
        n = n1;
        ch = ch1;
    }

#if KKB_KK_CHECK
    if (emax > (unsigned)(LINEAR ? W - 2 : W - 1)) atomicOr(&g_device_error, KKB_DEVERR_KK_WINDOW);
#endif
    if constexpr (MS) return;  // every set's epilogue ran inside the loop

    // epilogue: IQ (+ fused intensity and frame max), per frame
#pragma unroll
    for (int fr = 0; fr < FR; ++fr) {
        const int f = f0 + fr;
        if (f >= a.n_frames) break;
        float fmx = 0.f;
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int iz = iz0 + wz * 8 + p * 4 + zt;
#pragma unroll
            for (int r = 0; r < CX; ++r) {
                const int ix = ix0 + wx * 8 * CX + r * 8 + xt;
                if (iz < nz && ix < nx) {
                    const float vr = accr[fr][p][r], vi = acci[fr][p][r];
                    const long long px = (long long)f * a.out_fs + (long long)ix * nz + iz;
                    if (a.out) store_iq(a.out, a.out_kind, px, vr, vi);
                    for (int d = 0; d < a.ndst; ++d) store_iq(a.dst[d], a.out_kind, a.dst_off + px, vr, vi);
                    if (a.inten) {
                        float I = mag2(vr, vi);
                        if (a.accum) I = __fadd_rn(I, a.inten[px]);  // sets compounded in call order
                        a.inten[px] = I;
                        fmx = fmaxf(fmx, I);
                    }
                }
            }
        }
        if (a.fmax) {
            for (int o = 16; o > 0; o >>= 1) fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
            if (lane == 0) atomicMax(a.fmax + f, __float_as_uint(fmx));
        }
    }
}

// Per-pixel fallback of K5 for geometries whose per-tile trace window does not
// fit the staging buffer (very coarse grids / steep delays): one thread per
// (frame, pixel), taps read through L1.  Every float operation is the tiled
// kernel's: the same index math (kk_delay + tap_index), the lerp as
// (2 d0 - d1) + (1 + frac) (d1 - d0), one float32 accumulator over the pairs
// in (n, m) order, and the same intensity / accumulation expressions — so the
// two kernels give bit-identical images (tested), whichever one a plan, a
// row block of it or a batch size dispatches to.
template <bool LINEAR, bool MS = false>
__global__ void __launch_bounds__(256)
k_kk_direct(const KKArgs a) {
    if (a.run_if && *a.run_if == 0) return;
    const long long P = (long long)a.nx * a.nz;
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const int f = blockIdx.y;
    float fmx = 0.f;
    if (i < P) {
        const int ix = (int)(i / a.nz), iz = (int)(i % a.nz);
        const float2 *dframe = a.data + (long long)f * a.data_fs;
        const long long px = (long long)f * a.out_fs + i;
        const int nsets = MS ? a.nsets : 1;
        for (int j = 0; j < nsets; ++j) {
            const int mb = MS ? a.set_m0[j] : 0, me = MS ? a.set_m0[j + 1] : a.M;
            float ar = 0.f, ai = 0.f;
            for (int n = 0; n < a.N; ++n) {
                const double t1 = __dadd_rn(a.ltx[(long long)ix * a.N + n], a.ltzT[(long long)n * a.nz + iz]);
                for (int m = mb; m < me; ++m) {
                    const double fi = kk_delay(t1, a.lrzT[(long long)m * a.nz + iz], a.lrx[(long long)ix * a.M + m],
                                               a.fs, a.shift);
                    int F;
                    double sv;
                    if (!tap_index<LINEAR>(fi, a.T, F, sv)) continue;
                    const float wm = a.w ? (float)a.w[m] : 1.0f;
                    const float2 *tr = dframe + (long long)(n * a.M + m) * a.T;
                    const float2 d0 = __ldg(tr + F);
                    if (LINEAR) {
                        const float2 d1 = __ldg(tr + F + 1);
                        const float f1 = __uint_as_float(((unsigned)__double2loint(sv) >> 9) + 0x3F800000u);
                        const float vx = fmaf(f1, d1.x - d0.x, fmaf(2.f, d0.x, -d1.x));
                        const float vy = fmaf(f1, d1.y - d0.y, fmaf(2.f, d0.y, -d1.y));
                        ar = fmaf(wm, vx, ar);
                        ai = fmaf(wm, vy, ai);
                    } else {
                        ar = fmaf(wm, d0.x, ar);
                        ai = fmaf(wm, d0.y, ai);
                    }
                }
            }
            if (a.out) store_iq(a.out, a.out_kind, (MS ? j * a.out_set_stride : 0) + px, ar, ai);
            if (!MS)
                for (int d = 0; d < a.ndst; ++d) store_iq(a.dst[d], a.out_kind, a.dst_off + px, ar, ai);
            if (a.inten) {
                float I = mag2(ar, ai);
                if ((MS && j > 0) || a.accum) I = __fadd_rn(I, a.inten[px]);
                a.inten[px] = I;
                fmx = I;
            }
        }
    }
    if (a.fmax) {
        for (int o = 16; o > 0; o >>= 1) fmx = fmaxf(fmx, __shfl_xor_sync(0xffffffffu, fmx, o));
        if ((threadIdx.x & 31) == 0) atomicMax(a.fmax + f, __float_as_uint(fmx));
    }
}

static size_t kk_smem_bytes(int N, int M, int W, int MCH, bool linear, int tz = KKB_KK_TZ,
                            int tx = KKB_KK_TX, int fr = 1) {
    size_t entry = linear ? sizeof(float4) : sizeof(float2);
    return entry * 2 * fr * MCH * W + sizeof(double) * ((size_t)(M + N) * tz + (size_t)(M + N) * tx) +
           sizeof(int2) * (size_t)N * M;
}

template <int WZ, int WX, int CX, int FR, bool MS = false>
static int launch_tiled(const KKArgs &a, int n_frames, size_t sm, bool linear, cudaStream_t s) {
    constexpr int TZ = 8 * WZ, TX = 8 * CX * WX;
    dim3 grid((unsigned)ceil_div(a.nz, TZ), (unsigned)ceil_div(a.nx, TX),
              (unsigned)ceil_div(n_frames, FR));
    dim3 block(WZ * WX * 32);
    if (linear) {
        auto fn = k_kk_gather<WZ, WX, CX, true, FR, MS>;
        KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                     "smem attr kk");
        fn<<<grid, block, sm, s>>>(a);
    } else {
        auto fn = k_kk_gather<WZ, WX, CX, false, FR, MS>;
        KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                     "smem attr kk");
        fn<<<grid, block, sm, s>>>(a);
    }
    KKB_CHECK_LAUNCH("k_kk_gather");
    return KKB_OK;
}

// ------------------------------------------------------------- instance selection
static std::atomic<int> g_last_instance{-1};
int kk_last_instance() { return g_last_instance.load(); }

// window entries each instance stages per pipeline stage: EPT per thread
constexpr int kKKEPT = KKB_KK_STAGE_ELEMS / (32 * KKB_KK_WZ * KKB_KK_WX);

struct InstanceShape {
    int tz, tx, stage, W, resident, warps;  // resident: CTAs per SM the launch bounds aim for
};

static InstanceShape instance_shape(int inst, const KKWindows &win) {
    switch (inst) {
        case KKB_KK_INST_SMALL:
            return {KKB_KK_S_TZ, KKB_KK_S_TX, kKKEPT * 32 * KKB_KK_S_WZ * KKB_KK_S_WX,
                    std::max(2, win.small), KKB_KK_MIN_CTAS * KKB_KK_WZ * KKB_KK_WX / (KKB_KK_S_WZ * KKB_KK_S_WX),
                    KKB_KK_S_WZ * KKB_KK_S_WX};
        case KKB_KK_INST_MID:
            return {KKB_KK_M_TZ, KKB_KK_M_TX, kKKEPT * 32 * KKB_KK_M_WZ * KKB_KK_M_WX,
                    std::max(2, win.mid), KKB_KK_MIN_CTAS * KKB_KK_WZ * KKB_KK_WX / (KKB_KK_M_WZ * KKB_KK_M_WX),
                    KKB_KK_M_WZ * KKB_KK_M_WX};
        default:
            return {KKB_KK_TZ, KKB_KK_TX, KKB_KK_STAGE_ELEMS, std::max(2, win.big), KKB_KK_MIN_CTAS,
                    KKB_KK_WZ * KKB_KK_WX};
    }
}

static bool instance_fits(int inst, int N, int M, bool linear, const KKWindows &win, int n_frames) {
    if (inst == KKB_KK_INST_DIRECT) return true;
    if (win.bad & (1 << inst)) return false;  // kk_check_windows found a tap outside its window
    const InstanceShape sh = instance_shape(inst, win);
    const int fr = inst == KKB_KK_INST_BIG_FR ? KKB_KK_FR : 1;
    if (inst == KKB_KK_INST_BIG_FR && (n_frames < 2 || KKB_KK_FR < 2)) return false;
    return sh.W <= sh.stage && fr * sh.W <= sh.stage &&
           kk_smem_bytes(N, M, sh.W, 1, linear, sh.tz, sh.tx, fr) <= 200 * 1024;
}

// Wave model of one launch (profiles/r02a_instance_sweep.jsonl: config-5 row
// blocks at 1-8 ranks, config-4 batches of 1-400 frames, configs 1-3): the
// busiest SM runs ceil(CTAs / SMs) CTAs; with k of them resident at once it
// sustains eff(k x warps) of its full-occupancy rate (a lone 8-warp CTA
// reaches ~0.88: the shared-memory pipe is the limiter, not latency); the
// full-occupancy cost per pixel-pair differs by instance (measured at 400
// frames: two frames per CTA 1.00, one 1.02, 32 x 32 tiles 1.07, 16 x 16
// tiles 1.42 — smaller tiles stage the same windows and tables for fewer
// pixels).  The dispatch takes the instance with the smallest modelled time.
static double instance_cost(int inst, long long ctas, long long sms) {
    static const double rel[5] = {0.0, 1.42, 1.07, 1.02, 1.00};
    const InstanceShape sh = instance_shape(inst, KKWindows{2, 2, 2, 0, 2});
    const int fr = inst == KKB_KK_INST_BIG_FR ? KKB_KK_FR : 1;
    const long long per_sm = ceil_div(ctas, sms);
    const double resident = (double)std::min<long long>(per_sm, sh.resident);
    const double eff = std::min(1.0, 0.75 + resident * sh.warps / 64.0);
    return (double)per_sm * sh.tz * sh.tx * fr * rel[inst] / eff;
}

// ------------------------------------------------------------- plan-time window proof
// Every (pixel, pair) of one tile size, evaluated with the gather's own index
// arithmetic (kk_delay, the round-down magic add, the window start from the
// tile's corner delays): flags the tile size in *bad (and the device error
// word) if any tap's window index would leave [0, W-2] (linear) / [0, W-1]
// (nearest) while the pair's window overlaps the trace.  The tables are fixed
// per plan and the index math is frame-independent, so one pass at plan
// creation proves the clamp in k_kk_gather (e = min(raw, W-2)) never changes
// a tap for any launch of the plan; an instance that fails is not dispatched.
template <bool LINEAR>
__global__ void __launch_bounds__(256)
k_kk_window_check(const double *__restrict__ ltx, const double *__restrict__ ltz,
                  const double *__restrict__ lrx, const double *__restrict__ lrz, int N, int M,
                  int T, int nx, int nz, int TX, int TZ, int W, double fs, double shift, int bit,
                  int *bad) {
    extern __shared__ int lo_s[];  // [M]
    const int tiles_z = (nz + TZ - 1) / TZ;
    const int tz = blockIdx.x % tiles_z, tx = blockIdx.x / tiles_z, n = blockIdx.y;
    const int iz0 = tz * TZ, ix0 = tx * TX;
    const int rzb = min(TZ - 1, nz - 1 - iz0), cxb = min(TX - 1, nx - 1 - ix0);
    for (int m = threadIdx.x; m < M; m += blockDim.x) {
        double lo = 1e300;
        for (int cr = 0; cr < 2; ++cr)
            for (int cc = 0; cc < 2; ++cc) {
                const int iz = iz0 + (cr ? rzb : 0), ix = ix0 + (cc ? cxb : 0);
                const double t1 = __dadd_rn(ltx[(long long)ix * N + n], ltz[(long long)iz * N + n]);
                lo = fmin(lo, kk_delay(t1, lrz[(long long)iz * M + m], lrx[(long long)ix * M + m], fs, shift));
            }
        lo_s[m] = (int)fmax(fmin(floor(lo) - 1.0, 1.0e9), -1.0e9);
    }
    __syncthreads();
    const unsigned lim = (unsigned)(LINEAR ? W - 2 : W - 1);
    const int rows = rzb + 1, total = rows * (cxb + 1) * M;
    bool badf = false;
    for (int i = threadIdx.x; i < total; i += blockDim.x) {
        const int m = i % M, px = i / M, r = px % rows, c = px / rows;
        const int iz = iz0 + r, ix = ix0 + c, lo = lo_s[m];
        const double t1 = __dadd_rn(ltx[(long long)ix * N + n], ltz[(long long)iz * N + n]);
        const double fi = kk_delay(t1, lrz[(long long)iz * M + m], lrx[(long long)ix * M + m], fs, shift);
        const double sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC2);
        const unsigned raw = (unsigned)(__double2hiint(sv) - (lo + KKB_MAGIC2_HI));
        const bool live = lo <= (LINEAR ? T - 2 : T - 1) && lo + W > 0;
        badf |= live && raw > lim;
    }
    if (__syncthreads_or(badf) && threadIdx.x == 0) {
        atomicOr(bad, bit);
        atomicOr(&g_device_error, KKB_DEVERR_KK_WINDOW);
    }
}

// Tensor-core gather windows, per (tile, pair) of its 4 x 32 tile: the
// smallest and largest live tap index over the tile's pixels, with the
// gather's own index arithmetic (exact: every pixel is evaluated).  The
// window starts at the smallest; it takes one K = 16 MMA step when the taps
// span <= 16 samples (linear: F + 1 included), else two; a span beyond 32
// makes the plan ineligible (the table is dropped, the FMA gather runs).
template <bool LINEAR>
__global__ void __launch_bounds__(256)
k_kk_tc_windows(const double *__restrict__ ltx, const double *__restrict__ ltz, const double *__restrict__ lrx,
                const double *__restrict__ lrz, int N, int M, int T, int nx, int nz, double fs, double shift,
                int *__restrict__ tc_lo, int *over_flag) {
    const int TZ = KKB_KK_TC_TZ, TX = KKB_KK_TC_TX;
    const int tiles_z = (nz + TZ - 1) / TZ;
    const long long NM = (long long)N * M, total = (long long)tiles_z * ((nx + TX - 1) / TX) * NM;
    bool over = false;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const long long tile = i / NM;
        const int pr = (int)(i % NM), n = pr / M, m = pr % M;
        const int iz0 = (int)(tile % tiles_z) * TZ, ix0 = (int)(tile / tiles_z) * TX;
        const int rzb = min(TZ - 1, nz - 1 - iz0), cxb = min(TX - 1, nx - 1 - ix0);
        int fmin_ = 0x7fffffff, fmax_ = -1;
        for (int c = 0; c <= cxb; ++c)
            for (int r = 0; r <= rzb; ++r) {
                const int iz = iz0 + r, ix = ix0 + c;
                const double t1 = __dadd_rn(ltx[(long long)ix * N + n], ltz[(long long)iz * N + n]);
                const double fi = kk_delay(t1, lrz[(long long)iz * M + m], lrx[(long long)ix * M + m], fs, shift);
                const double sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC2);
                const int F = __double2hiint(sv) - KKB_MAGIC2_HI;
                if ((unsigned)F <= (unsigned)(LINEAR ? T - 2 : T - 1)) {
                    fmin_ = min(fmin_, F);
                    fmax_ = max(fmax_, F);
                }
            }
        const int lo = fmax_ < 0 ? 0 : fmin_;                          // no live tap: any window
        const int span = fmax_ < 0 ? 1 : fmax_ - fmin_ + 1 + (LINEAR ? 1 : 0);  // samples touched
        over |= span > KKB_KK_TC_W;
        tc_lo[i] = lo * 2 + (span <= 16 ? 1 : 0);
    }
    if (__syncthreads_or(over) && threadIdx.x == 0) atomicOr(over_flag, 1);
}

int kk_check_windows(const double *ltx, const double *ltz, const double *lrx, const double *lrz,
                     int N, int M, int T, int nx, int nz, double fs, double shift, int linear,
                     KKWindows *win, cudaStream_t s) {
    win->bad = 0;
    win->tc_lo = nullptr;
    win->tc_ksteps = -1;
    if ((size_t)M * sizeof(int) > 48 * 1024) return KKB_OK;  // huge pair tables: no tile fits anyway
    int *d = nullptr;
    // d[0]: failed tile sizes; d[1]: the tensor-core windows exceed 32 samples
    KKB_TRY_CUDA(cudaMallocAsync(&d, 2 * sizeof(int), s), "cudaMallocAsync(window check)");
    KKB_TRY_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(int), s), "memset(window check)");
    const int insts[3] = {KKB_KK_INST_BIG, KKB_KK_INST_MID, KKB_KK_INST_SMALL};
    for (int k = 0; k < 3; ++k) {
        const InstanceShape sh = instance_shape(insts[k], *win);
        if (sh.W > sh.stage) continue;  // this tile size never runs (per-pixel kernel instead)
        const long long tiles = ceil_div(nz, sh.tz) * ceil_div(nx, sh.tx);
        if (tiles > 0x7fffffffLL || N > 65535) continue;
        dim3 grid((unsigned)tiles, (unsigned)N);
        const size_t smem = sizeof(int) * (size_t)M;
        if (linear)
            k_kk_window_check<true><<<grid, 256, smem, s>>>(ltx, ltz, lrx, lrz, N, M, T, nx, nz, sh.tx,
                                                            sh.tz, sh.W, fs, shift, 1 << insts[k], d);
        else
            k_kk_window_check<false><<<grid, 256, smem, s>>>(ltx, ltz, lrx, lrz, N, M, T, nx, nz, sh.tx,
                                                             sh.tz, sh.W, fs, shift, 1 << insts[k], d);
        KKB_CHECK_LAUNCH("k_kk_window_check");
    }
    {  // the tensor-core gather's exact per (tile, pair) windows
        const long long ntc = ceil_div(nz, KKB_KK_TC_TZ) * ceil_div(nx, KKB_KK_TC_TX) * (long long)N * M;
        if (cudaMalloc(&win->tc_lo, sizeof(int) * (size_t)ntc) == cudaSuccess) {
            const int blocks = (int)std::min<long long>(ceil_div(ntc, 256), 148LL * 16);
            if (linear)
                k_kk_tc_windows<true><<<blocks, 256, 0, s>>>(ltx, ltz, lrx, lrz, N, M, T, nx, nz, fs, shift,
                                                             win->tc_lo, d + 1);
            else
                k_kk_tc_windows<false><<<blocks, 256, 0, s>>>(ltx, ltz, lrx, lrz, N, M, T, nx, nz, fs, shift,
                                                              win->tc_lo, d + 1);
            KKB_CHECK_LAUNCH("k_kk_tc_windows");
        } else {
            cudaGetLastError();  // no table: the tensor-core gather is not dispatched
            win->tc_lo = nullptr;
        }
    }
    int hh[2] = {0, 0};
    KKB_TRY_CUDA(cudaMemcpyAsync(hh, d, sizeof(hh), cudaMemcpyDeviceToHost, s), "copy window check");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync window check");
    cudaFreeAsync(d, s);
    // a tile size that failed disables its instances (big covers both frame counts)
    const int h = hh[0];
    win->bad = h | ((h & (1 << KKB_KK_INST_BIG)) ? (1 << KKB_KK_INST_BIG_FR) : 0);
    win->tc_ksteps = -1;
    if (hh[1] && win->tc_lo) {  // too steep for the tensor-core tile: not eligible (not an error)
        cudaFree(win->tc_lo);
        win->tc_lo = nullptr;
    }
    if (win->tc_lo) {  // the K-step count (bench's tensor roofline, kkb_kk_plan_tc_ksteps)
        const size_t ntc = (size_t)(ceil_div(nz, KKB_KK_TC_TZ) * ceil_div(nx, KKB_KK_TC_TX)) * N * M;
        std::vector<int> h(ntc);
        if (cudaMemcpy(h.data(), win->tc_lo, sizeof(int) * ntc, cudaMemcpyDeviceToHost) == cudaSuccess) {
            long long k = 0;
            for (int v : h) k += (v & 1) ? 1 : 2;
            win->tc_ksteps = k;
        }
    }
    return KKB_OK;
}

// KKB_KK_INST forces an instance when it fits (KKB_KK_DIRECT=1 /
// KKB_KK_SMALL=1 / KKB_KK_FR1=1: older test hooks); the per-pixel kernel
// runs when no tile's window fits its stage.
static int select_instance(int N, int M, int nx, int nz, int n_frames, bool linear, const KKWindows &win) {
    static const int order[4] = {KKB_KK_INST_BIG_FR, KKB_KK_INST_BIG, KKB_KK_INST_MID, KKB_KK_INST_SMALL};
    auto fits = [&](int i) { return instance_fits(i, N, M, linear, win, n_frames); };
    auto env1 = [](const char *k) {
        const char *v = getenv(k);
        return v && v[0] == '1';
    };
    if (const char *f = getenv("KKB_KK_INST")) {
        const char *names[5] = {"direct", "small", "mid", "big", "big_fr"};
        for (int i = 0; i < 5; ++i)
            if (!strcmp(f, names[i]) && fits(i)) return i;
    }
    if (env1("KKB_KK_DIRECT")) return KKB_KK_INST_DIRECT;
    if (env1("KKB_KK_SMALL") && fits(KKB_KK_INST_SMALL)) return KKB_KK_INST_SMALL;
    const bool no_fr = env1("KKB_KK_FR1");
    const long long sms = sm_count();
    int best = KKB_KK_INST_DIRECT;
    double best_cost = 0.0;
    for (int inst : order) {
        if ((inst == KKB_KK_INST_BIG_FR && no_fr) || !fits(inst)) continue;
        const InstanceShape sh = instance_shape(inst, win);
        const int fr = inst == KKB_KK_INST_BIG_FR ? KKB_KK_FR : 1;
        const long long ctas = ceil_div(nz, sh.tz) * ceil_div(nx, sh.tx) * ceil_div(n_frames, fr);
        const double c = instance_cost(inst, ctas, sms);
        if (best == KKB_KK_INST_DIRECT || c < best_cost) {
            best = inst;
            best_cost = c;
        }
    }
    return best;
}

int kk_gather(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
              const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
              double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
              long long out_fs, float *inten, unsigned *fmax, const KKWindows &win, cudaStream_t s,
              int accum, const KKScatter *sc, long long data_ns, const KKSets *sets, const TcPlanes *tcp) {
    if (n_frames <= 0 || nx <= 0 || nz <= 0) return KKB_OK;
    const bool ms = sets != nullptr;
    // a receive subset of a larger trace array (transmit stride data_ns > M*T):
    // gathered into dense (F, N, M, T) scratch first, so the kernels keep the
    // dense row arithmetic (a runtime transmit stride costs K5 0.5-8%)
    float2 *dense = nullptr;
    if (data_ns > 0 && data_ns != (long long)M * T) {
        if (data_ns < (long long)M * T) return KKB_ERR_ARG;
        const size_t row = sizeof(float2) * (size_t)M * T;
        KKB_TRY_CUDA(cudaMallocAsync(&dense, row * (size_t)n_frames * N, s), "cudaMallocAsync(dense traces)");
        for (int f = 0; f < n_frames; ++f) {
            cudaError_t e = cudaMemcpy2DAsync(dense + (size_t)f * N * M * T, row, data + f * data_fs,
                                              sizeof(float2) * (size_t)data_ns, row, (size_t)N,
                                              cudaMemcpyDeviceToDevice, s);
            if (e != cudaSuccess) {
                cudaFreeAsync(dense, s);
                return cuda_status(e, "copy trace subset");
            }
        }
        data = dense;
        data_fs = (long long)N * M * T;
    }
    struct FreeDense {
        float2 *p;
        cudaStream_t s;
        ~FreeDense() {
            if (p) cudaFreeAsync(p, s);
        }
    } free_dense{dense, s};
    KKArgs a{data, data_fs, N, M, T, ltx, ltzT, lrx,
             lrzT, w, fs, shift, nx, nz, 2, 0,
             out, out_kind, out_fs, inten, fmax, accum, 0, 0, {}, n_frames};
    if (sc) {
        a.ndst = sc->ndst;
        a.dst_off = sc->dst_off;
        for (int d = 0; d < sc->ndst; ++d) a.dst[d] = sc->dst[d];
    }
    if (ms) {
        if (sc || sets->nsets < 1 || sets->nsets > KKB_MAX_SETS) return KKB_ERR_ARG;
        a.nsets = sets->nsets;
        for (int j = 0; j <= sets->nsets; ++j) a.set_m0[j] = sets->m0[j];
        a.out_set_stride = sets->out_set_stride;
    }
    const int inst = select_instance(N, M, nx, nz, n_frames, linear != 0, win);
    auto launch_fma = [&](KKArgs a) -> int {
        if (inst == KKB_KK_INST_DIRECT) {
            // steep geometry or huge pair tables: per-pixel kernel
            dim3 grid((unsigned)ceil_div((long long)nx * nz, 256), (unsigned)n_frames);
            if (ms) {
                if (linear)
                    k_kk_direct<true, true><<<grid, 256, 0, s>>>(a);
                else
                    k_kk_direct<false, true><<<grid, 256, 0, s>>>(a);
            } else if (linear)
                k_kk_direct<true><<<grid, 256, 0, s>>>(a);
            else
                k_kk_direct<false><<<grid, 256, 0, s>>>(a);
            KKB_CHECK_LAUNCH("k_kk_direct");
            return KKB_OK;
        }
        const InstanceShape sh = instance_shape(inst, win);
        const int FR = inst == KKB_KK_INST_BIG_FR ? KKB_KK_FR : 1;
        // receive angles per stage: bounded by the register staging and shared memory
        int MCH = std::max(1, std::min(M, sh.stage / (FR * sh.W)));
        while (MCH > 1 && kk_smem_bytes(N, M, sh.W, MCH, linear, sh.tz, sh.tx, FR) > 200 * 1024) MCH = (MCH + 1) / 2;
        if (const char *fm = getenv("KKB_KK_MCH"))  // test hook: fewer receive angles per stage
            MCH = std::max(1, std::min(MCH, atoi(fm)));
        const size_t sm = kk_smem_bytes(N, M, sh.W, MCH, linear, sh.tz, sh.tx, FR);
        a.W = sh.W;
        a.MCH = MCH;
        const bool lin = linear != 0;
        switch (inst) {
            case KKB_KK_INST_SMALL:
                return ms ? launch_tiled<KKB_KK_S_WZ, KKB_KK_S_WX, KKB_KK_S_CX, 1, true>(a, n_frames, sm, lin, s)
                          : launch_tiled<KKB_KK_S_WZ, KKB_KK_S_WX, KKB_KK_S_CX, 1>(a, n_frames, sm, lin, s);
            case KKB_KK_INST_MID:
                return ms ? launch_tiled<KKB_KK_M_WZ, KKB_KK_M_WX, KKB_KK_M_CX, 1, true>(a, n_frames, sm, lin, s)
                          : launch_tiled<KKB_KK_M_WZ, KKB_KK_M_WX, KKB_KK_M_CX, 1>(a, n_frames, sm, lin, s);
            case KKB_KK_INST_BIG_FR:
                return ms ? launch_tiled<KKB_KK_WZ, KKB_KK_WX, KKB_KK_CX, KKB_KK_FR, true>(a, n_frames, sm, lin, s)
                          : launch_tiled<KKB_KK_WZ, KKB_KK_WX, KKB_KK_CX, KKB_KK_FR>(a, n_frames, sm, lin, s);
            default:
                return ms ? launch_tiled<KKB_KK_WZ, KKB_KK_WX, KKB_KK_CX, 1, true>(a, n_frames, sm, lin, s)
                          : launch_tiled<KKB_KK_WZ, KKB_KK_WX, KKB_KK_CX, 1>(a, n_frames, sm, lin, s);
        }
    };
    // tensor-core gather (kk_gather_tc.cu): single-set launches without peer
    // scatter whose plan holds exact tile windows of <= KKB_KK_TC_W samples.
    // The FMA instance is launched behind it as a standby that only runs when
    // the batch holds a NaN / Inf sample (the reference propagates those per
    // tap; a tensor-core product would spread them over the window).
    {
        // default: batches of >= KKB_KK_TC_MIN_FRAMES frames with linear taps,
        // >= KKB_KK_TC_MIN_FRAMES_NEAREST with nearest taps (the FMA gather's
        // cheaper taps hold out longer) — the measured crossovers,
        // profiles/r02_gather_tc_sweep.jsonl: below them the per-pair weight
        // rows do not amortise; KKB_KK_INST forces an instance either way,
        // KKB_KK_TC=0 disables it
        const char *fi = getenv("KKB_KK_INST");
        const char *tcv = getenv("KKB_KK_TC");
        const int min_frames = linear ? KKB_KK_TC_MIN_FRAMES : KKB_KK_TC_MIN_FRAMES_NEAREST;
        const bool want = fi ? !strcmp(fi, "tc") : !(tcv && tcv[0] == '0') && n_frames >= min_frames;
        const bool tc_ok = !ms && !sc && win.tc_lo && !(win.bad & (1 << KKB_KK_INST_TC));
        if (tcp) {  // traces split by K3: the tensor-core gather or nothing
            if (!tc_ok || ms || sc) {
                set_error("kk: split-plane traces need the tensor-core gather, which this plan cannot run");
                return KKB_ERR_UNSUPPORTED;
            }
            const int rc = kk_gather_tc_planes(tcp->planes, tcp->fbound, tcp->nonfinite, N, M, T, ltx, ltzT, lrx,
                                               lrzT, nx, nz, w, fs, shift, linear, out, out_kind, n_frames, out_fs,
                                               inten, fmax, win.tc_lo, accum, s, [&](const unsigned *run_if) {
                                                   KKArgs b = a;
                                                   b.run_if = run_if;
                                                   return launch_fma(b);
                                               });
            if (rc == KKB_OK) g_last_instance.store(KKB_KK_INST_TC);
            return rc;
        }
        if (want && tc_ok) {
            const int rc = kk_gather_tc(data, N, M, T, ltx, ltzT, lrx, lrzT, nx, nz, w, fs, shift, linear, out,
                                        out_kind, n_frames, data_fs, out_fs, inten, fmax, win.tc_lo, accum, s,
                                        [&](const unsigned *run_if) {
                                            KKArgs b = a;
                                            b.run_if = run_if;
                                            return launch_fma(b);
                                        });
            if (rc != KKB_ERR_UNSUPPORTED) {
                g_last_instance.store(KKB_KK_INST_TC);
                return rc;
            }
        }
    }
    g_last_instance.store(inst | (ms ? KKB_KK_INST_SETS : 0));
    return launch_fma(a);
}

// ------------------------------------------------------------- K6 epilogues
// one CTA row per frame (blockIdx.y); float4 body when P % 4 == 0 and both
// buffers are 16 B aligned
__device__ __forceinline__ float db_of(float v, float mx, float floor_db) {
    const float d = (mx > 0.f && v > 0.f) ? 10.0f * log10f(v / mx) : floor_db;
    return fmaxf(d, floor_db);
}

// 10 log10(v / mx) = 10 log10(2) (log2 v - log2 mx) with the MUFU log2 (abs
// error ~2^-22 in log2, ~1e-6 dB); the same approximation on both terms keeps
// the frame maximum at exactly 0 dB.  Frames whose max is not a normal float
// take db_of.
__device__ __forceinline__ float db_fast(float v, float l2mx, float floor_db) {
    const float d = v > 0.f ? 3.01029995663981195f * (__log2f(v) - l2mx) : floor_db;
    return fmaxf(d, floor_db);
}

__global__ void __launch_bounds__(256)
k_log_compress(const float *__restrict__ inten, const unsigned *__restrict__ fmax, long long P,
               float floor_db, float *db, bool vec) {
    const int f = gridDim.y - 1 - blockIdx.y;  // last frames first: the gather wrote them last (L2)
    const float mx = __uint_as_float(fmax[f]);
    const float *src = inten + (long long)f * P;
    float *dst = db + (long long)f * P;
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (vec && mx >= 1.17549435e-38f) {
        const float l2mx = __log2f(mx);
        const float4 *s4 = reinterpret_cast<const float4 *>(src);
        float4 *d4 = reinterpret_cast<float4 *>(dst);
        for (long long i = t0; i < P / 4; i += stride) {
            const float4 v = __ldcs(s4 + i);  // read once: stream past L2
            __stcs(d4 + i, make_float4(db_fast(v.x, l2mx, floor_db), db_fast(v.y, l2mx, floor_db),
                                       db_fast(v.z, l2mx, floor_db), db_fast(v.w, l2mx, floor_db)));
        }
    } else {
        for (long long i = t0; i < P; i += stride) dst[i] = db_of(src[i], mx, floor_db);
    }
}

int log_compress(const float *inten, const unsigned *fmax, int n_frames, long long P, float floor_db,
                 float *db, cudaStream_t s) {
    if ((long long)n_frames * P <= 0) return KKB_OK;
    if (n_frames > 65535) return KKB_ERR_UNSUPPORTED;
    const bool vec = (P & 3) == 0 && (((uintptr_t)inten | (uintptr_t)db) & 15) == 0;
    const long long per = vec ? P / 4 : P;
    const int bx = (int)std::max<long long>(1, std::min<long long>(ceil_div(per, 256),
                                                                   std::max(1, 148 * 8 / n_frames)));
    k_log_compress<<<dim3(bx, n_frames), 256, 0, s>>>(inten, fmax, P, floor_db, db, vec);
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
