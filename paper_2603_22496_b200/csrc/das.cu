// K7: conventional CPWC delay-and-sum over element data (comparison kernel).
//
// Replaces _das_kernel (beamform.py:178-209).  Same sampling rules as K5:
// per (pixel, transmit n, element l)
//   skip if |x - u_l| > z * tan_max                       (beamform.py:191)
//   h  = hyp[ix + base_l, iz] (+ frac_l * (hyp[.. + 1, iz] - h) if frac_l > 0)
//   fi = ((ltx + ltz) + h) * fs + shift                   (beamform.py:189,198)
// all in float64 with explicit IEEE round-to-nearest steps, so tap indices
// and gating are bit-identical to the reference; taps are float32 lerps,
// element partials float32, transmit totals float64 (per-pixel kernel; the
// tiled kernel below sums per-element float32 partials into float64).
//
// One thread per pixel, consecutive threads along depth (the reference's
// flattened p = ix*nz + iz order), hyp rows and traces read through L1
// (a warp's 32 depth neighbours touch one or two 128 B lines per element).

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"
#include "kk.cuh"

namespace kkb {

#define KKB_FLOOR_MAGIC2_DAS 1572864.0  // 1.5 * 2^20 (see tap_index, kk_gather.cu)
#define KKB_MAGIC2_HI_DAS 0x41380000

template <bool LINEAR>
__global__ void __launch_bounds__(256)
k_das_gather(const float2 *__restrict__ data, int N, int L, int T, const double *__restrict__ ltx,
             const double *__restrict__ ltz, const double *__restrict__ hyp,
             const long long *__restrict__ base, const double *__restrict__ frac,
             const double *__restrict__ xcoord, const double *__restrict__ zcoord,
             const double *__restrict__ upos, double tan_max, const double *__restrict__ weights,
             double fs, double shift, int nx, int nz, void *out, int out_kind) {
    const long long P = (long long)nx * nz;
    const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (p >= P) return;
    const int ix = (int)(p / nz), iz = (int)(p % nz);
    const double x = xcoord[ix], z = zcoord[iz];
    const double zt = __dmul_rn(z, tan_max);
    double ar = 0.0, ai = 0.0;
    for (int n = 0; n < N; ++n) {
        const double tx = __dadd_rn(ltx[(long long)ix * N + n], ltz[(long long)iz * N + n]);
        const float2 *dn = data + (long long)n * L * T;
        float pr = 0.f, pi = 0.f;
        for (int l = 0; l < L; ++l) {
            if (fabs(__dsub_rn(x, __ldg(upos + l))) > zt) continue;
            const long long r0 = ix + __ldg(base + l);
            double h = hyp[r0 * nz + iz];
            const double fr = __ldg(frac + l);
            if (fr > 0.0) h = __dadd_rn(h, __dmul_rn(fr, __dsub_rn(hyp[(r0 + 1) * nz + iz], h)));
            const double fi = __dadd_rn(__dmul_rn(__dadd_rn(tx, h), fs), shift);
            const float w = weights ? (float)__ldg(weights + l) : 1.0f;
            const float2 *tr = dn + (long long)l * T;
            if (LINEAR) {
                const double y = __dadd_rd(fi, KKB_FLOOR_MAGIC);
                const int F = __double2loint(y);
                if (__double2hiint(y) == KKB_MAGIC_HI && (unsigned)F <= (unsigned)(T - 2)) {
                    const float2 d0 = __ldg(tr + F), d1 = __ldg(tr + F + 1);
                    const float f = frac_from_floor(fi, y);
                    pr = fmaf(w, fmaf(f, d1.x - d0.x, d0.x), pr);
                    pi = fmaf(w, fmaf(f, d1.y - d0.y, d0.y), pi);
                }
            } else {
                const double y = __dadd_rd(__dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC);
                const int F = __double2loint(y);
                if (__double2hiint(y) == KKB_MAGIC_HI && (unsigned)F <= (unsigned)(T - 1)) {
                    const float2 d = __ldg(tr + F);
                    pr = fmaf(w, d.x, pr);
                    pi = fmaf(w, d.y, pi);
                }
            }
        }
        ar += (double)pr;
        ai += (double)pi;
    }
    if (out_kind == KKB_OUT_C128)
        reinterpret_cast<double2 *>(out)[p] = make_double2(ar, ai);
    else
        reinterpret_cast<float2 *>(out)[p] = make_float2((float)ar, (float)ai);
}

static int das_gather_direct(const float2 *data, int n_tx, int n_el, int n_t, const double *ltx,
                             const double *ltz, const double *hyp, const long long *base,
                             const double *frac, const double *xcoord, const double *zcoord,
                             const double *upos, double tan_max, const double *weights, double fs,
                             double shift, int linear, int nx, int nz, void *out, int out_kind,
                             cudaStream_t s) {
    long long P = (long long)nx * nz;
    if (P <= 0) return KKB_OK;
    unsigned blocks = (unsigned)ceil_div(P, 256);
    if (linear)
        k_das_gather<true><<<blocks, 256, 0, s>>>(data, n_tx, n_el, n_t, ltx, ltz, hyp, base, frac,
                                                  xcoord, zcoord, upos, tan_max, weights, fs, shift,
                                                  nx, nz, out, out_kind);
    else
        k_das_gather<false><<<blocks, 256, 0, s>>>(data, n_tx, n_el, n_t, ltx, ltz, hyp, base, frac,
                                                   xcoord, zcoord, upos, tan_max, weights, fs, shift,
                                                   nx, nz, out, out_kind);
    KKB_CHECK_LAUNCH("k_das_gather");
    return KKB_OK;
}

// ===================================================================== tiled K7
// The same sums with K5's structure: a CTA owns a 32 x 32 pixel tile, stages
// per (element l, chunk of transmits) the trace windows its pixels can touch
// into shared memory as (2 d0 - d1, d1 - d0) float4 entries, and reads one
// 16 B entry per tap.  Loop order is element-outer: the receive path h(l,
// pixel) -- hyp lookup, frac interpolation, the receive gate -- is evaluated
// once per (pixel, element) and reused for every transmit; per tap the float64
// work is fi = ((ltx + ltz) + h) fs + shift (beamform.py:189,198, same IEEE
// order) and the floor add.  Taps are float32, per-element partials over the
// transmits float32, the pixel total float64.
//
// Window bounds per (tile, n, l): tx = RN(ltx + ltz) is monotone in x and z,
// so its extremes are tile corners; the hyp table is monotone in z for every
// row, so over the tile's rows [ix0 + base_l, ix1 + base_l (+1 if frac_l > 0)]
// its minimum
// is at the tile's first depth and its maximum at the last; every later step
// (+, * fs, + shift, floor) is monotone.  lo = floor(fi_min) - 1 and the
// window is sized for floor(fi_max) + 2.  Entries of out-of-trace samples are
// zero, so the reference's in-window test needs no per-tap predicate.
#define KKB_DAS_TZ 32
#ifndef KKB_DAS_CX
#define KKB_DAS_CX 2  // pixel columns per lane
#endif
#define KKB_DAS_TX (16 * KKB_DAS_CX)
#if KKB_DAS_CX > 2 || defined(KKB_DAS_FLOAT_TOTAL)
typedef float das_total_t;  // 8 pixels per lane: float totals keep registers < 128
#else
typedef double das_total_t;
#endif
#define KKB_DAS_NT 256
#define KKB_DAS_STAGE 1024
#ifndef KKB_DAS_QUNROLL
#define KKB_DAS_QUNROLL 1  // transmits per unrolled step of the tap loop
#endif
#ifndef KKB_DAS_MINB
#define KKB_DAS_MINB 2  // CTAs per SM (register cap 128)
#endif

__device__ __forceinline__ int das_prow(int r) { return ((r >> 3) << 3) + ((r & 3) << 1) + ((r >> 2) & 1); }
// tile column c -> warp block c/(8CX), lane slot c%8, column j = (c/8)%CX (a lane's CX
// columns contiguous)
__device__ __forceinline__ int das_pcol(int c) {
    constexpr int CX = KKB_DAS_CX;
    return (c / (8 * CX)) * (8 * CX) + (c & 7) * CX + ((c >> 3) % CX);
}

struct DasArgs {
    const float2 *data;
    int N, L, T;
    const double *ltx, *ltz, *hyp;
    const long long *base;
    const double *frac, *xcoord, *zcoord, *upos;
    double tan_max;
    const double *w;
    double fs, shift;
    int nx, nz, W, NCH;
    void *out;
    int out_kind;
    int groups;       // element groups per tile (grid = tiles x groups)
    double2 *part;    // [groups][nx*nz] partial sums when groups > 1
};

__device__ __forceinline__ double das_fi(double tx, double h, double fs, double shift) {
    return __dadd_rn(__dmul_rn(__dadd_rn(tx, h), fs), shift);
}

// hyp extremes over rows [r0, r1] at depths iz_lo (min) and iz_hi (max)
__device__ __forceinline__ void hyp_range(const double *hyp, int nz, long long r0, long long r1,
                                          int iz_lo, int iz_hi, double &hmin, double &hmax) {
    hmin = 1e300;
    hmax = -1e300;
    for (long long r = r0; r <= r1; ++r) {
        hmin = fmin(hmin, hyp[r * nz + iz_lo]);
        hmax = fmax(hmax, hyp[r * nz + iz_hi]);
    }
}

// pre-pass: one CTA per tile, the largest window any (n, l) needs
__global__ void __launch_bounds__(256)
k_das_window(const DasArgs a, int *wmax) {
    extern __shared__ double dsm[];
    double *tmin = dsm, *tmax = tmin + a.N, *hmin = tmax + a.N, *hmax = hmin + a.L;
    const int tiles_z = (a.nz + KKB_DAS_TZ - 1) / KKB_DAS_TZ;
    const int ix0 = (blockIdx.x / tiles_z) * KKB_DAS_TX, iz0 = (blockIdx.x % tiles_z) * KKB_DAS_TZ;
    const int ix1 = min(ix0 + KKB_DAS_TX, a.nx) - 1, iz1 = min(iz0 + KKB_DAS_TZ, a.nz) - 1;
    for (int n = threadIdx.x; n < a.N; n += blockDim.x) {
        double lo = 1e300, hi = -1e300;
        for (int c = 0; c < 4; ++c) {
            const int ix = (c & 1) ? ix1 : ix0, iz = (c & 2) ? iz1 : iz0;
            const double t = __dadd_rn(a.ltx[(long long)ix * a.N + n], a.ltz[(long long)iz * a.N + n]);
            lo = fmin(lo, t);
            hi = fmax(hi, t);
        }
        tmin[n] = lo;
        tmax[n] = hi;
    }
    for (int l = threadIdx.x; l < a.L; l += blockDim.x)
        hyp_range(a.hyp, a.nz, ix0 + a.base[l], ix1 + a.base[l] + (a.frac[l] > 0.0), iz0, iz1,
                  hmin[l], hmax[l]);
    __syncthreads();
    int best = 0;
    for (int i = threadIdx.x; i < a.N * a.L; i += blockDim.x) {
        const int n = i / a.L, l = i - n * a.L;
        const double lo = das_fi(tmin[n], hmin[l], a.fs, a.shift);
        const double hi = das_fi(tmax[n], hmax[l], a.fs, a.shift);
        const double span = floor(hi) - floor(lo) + 4.0;
        best = max(best, span > 1e9 ? 1000000000 : (int)span);
    }
    atomicMax(wmax, best);
}

template <bool LINEAR>
__global__ void __launch_bounds__(KKB_DAS_NT, KKB_DAS_MINB)
k_das_tile(const DasArgs a) {
    constexpr int TZ = KKB_DAS_TZ, TX = KKB_DAS_TX, NT = KKB_DAS_NT;
    constexpr int EPT = KKB_DAS_STAGE / NT;
    using Entry = typename std::conditional<LINEAR, float4, float2>::type;
    const int N = a.N, L = a.L, T = a.T, W = a.W, NCH = a.NCH, nx = a.nx, nz = a.nz;
    const int nchunk = (N + NCH - 1) / NCH;
    // this CTA's elements [lbeg, lend): tiles are split over element groups so
    // a one-frame image still fills every SM
    const int grp = blockIdx.x % a.groups;
    const int lbeg = (int)((long long)L * grp / a.groups), lend = (int)((long long)L * (grp + 1) / a.groups);

    extern __shared__ __align__(16) unsigned char smem_raw[];
    Entry *win = reinterpret_cast<Entry *>(smem_raw);                    // [2][NCH][W]
    double *ltz_p = reinterpret_cast<double *>(win + 2 * NCH * W);       // [N][TZ] packed rows
    double *ltx_p = ltz_p + N * TZ;                                      // [N][TX] packed cols
    double *tmin = ltx_p + N * TX;                                       // [N]
    double *hmin = tmin + N;                                             // [L]
    int *lo_s = reinterpret_cast<int *>(hmin + L);                       // [2][NCH]
    int *elist = lo_s + 2 * NCH;                                         // [L] live elements
    __shared__ int n_live;

    const int tid = threadIdx.x;
    const int tiles_z = (nz + TZ - 1) / TZ;
    const int tile = blockIdx.x / a.groups;
    const int ix0 = (tile / tiles_z) * TX, iz0 = (tile % tiles_z) * TZ;
    const int ix1 = min(ix0 + TX, nx) - 1, iz1 = min(iz0 + TZ, nz) - 1;
    const int lane = tid & 31, warp = tid >> 5;
    const int wz = warp % 4, wx = warp / 4;
    const int zt = lane & 3, xt = lane >> 2;
    const int zq = wz * 4 + zt, xq = wx * 8 + xt;

    for (int i = tid; i < N * TZ; i += NT) {
        const int n = i / TZ, r = i - n * TZ;
        ltz_p[n * TZ + das_prow(r)] = a.ltz[(long long)min(iz0 + r, nz - 1) * N + n];
    }
    for (int i = tid; i < N * TX; i += NT) {
        const int n = i / TX, c = i - n * TX;
        ltx_p[n * TX + das_pcol(c)] = a.ltx[(long long)min(ix0 + c, nx - 1) * N + n];
    }
    for (int n = tid; n < N; n += NT) {
        double lo = 1e300;
        for (int c = 0; c < 4; ++c) {
            const int ix = (c & 1) ? ix1 : ix0, iz = (c & 2) ? iz1 : iz0;
            lo = fmin(lo, __dadd_rn(a.ltx[(long long)ix * N + n], a.ltz[(long long)iz * N + n]));
        }
        tmin[n] = lo;
    }
    if (tid == 0) {
        // elements whose receive gate closes for EVERY pixel of the tile contribute
        // nothing (beamform.py:191): min |x - u| > z_max * tan_max, same rounding
        int k = 0;
        const double xl = a.xcoord[ix0], xh = a.xcoord[ix1];
        const double zt = __dmul_rn(a.zcoord[iz1], a.tan_max);
        for (int l = lbeg; l < lend; ++l) {
            const double u = a.upos[l];
            const double dmin = u < xl ? __dsub_rn(xl, u) : (u > xh ? __dsub_rn(u, xh) : 0.0);
            if (!(fabs(dmin) > zt)) elist[k++] = l;
        }
        n_live = k;
    }
    for (int l = tid; l < L; l += NT) {
        double hmx;
        hyp_range(a.hyp, nz, ix0 + a.base[l], ix1 + a.base[l] + (a.frac[l] > 0.0), iz0, iz1, hmin[l],
                  hmx);
    }
    __syncthreads();

    const int nstage = n_live * nchunk;
    const double fs = a.fs, shift = a.shift;
    // window start of (transmit n, element l)
    auto lo_of = [&](int n, int l) -> int {
        const double v = floor(das_fi(tmin[n], hmin[l], fs, shift)) - 1.0;
        return (int)fmax(fmin(v, 1.0e9), -1.0e9);
    };
    float2 s0[EPT], s1[EPT];
    int qe[EPT];
#pragma unroll
    for (int i = 0; i < EPT; ++i) {
        const int idx = tid + i * NT, q = idx / W;
        qe[i] = (q << 16) | (idx - q * W);
    }
    auto load_stage = [&](int l, int n0) {
        const int cnt = min(NCH, N - n0) * W;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int idx = tid + i * NT;
            s0[i] = s1[i] = make_float2(0.f, 0.f);
            if (idx < cnt) {
                const int q = qe[i] >> 16, e = qe[i] & 0xFFFF;
                const int smp = lo_of(n0 + q, l) + e;
                const float2 *tr = a.data + ((long long)(n0 + q) * L + l) * T;
                if ((unsigned)smp <= (unsigned)(LINEAR ? T - 2 : T - 1)) {
                    s0[i] = __ldg(tr + smp);
                    if (LINEAR) s1[i] = __ldg(tr + smp + 1);
                }
            }
        }
    };
    auto store_stage = [&](int l, int n0, int buf) {
        const int cnt = min(NCH, N - n0) * W;
        Entry *wb = win + buf * NCH * W;
#pragma unroll
        for (int i = 0; i < EPT; ++i) {
            const int idx = tid + i * NT;
            if (idx < cnt) {
                if constexpr (LINEAR) {
                    wb[idx] = make_float4(fmaf(2.f, s0[i].x, -s1[i].x), fmaf(2.f, s0[i].y, -s1[i].y),
                                          s1[i].x - s0[i].x, s1[i].y - s0[i].y);
                } else {
                    wb[idx] = s0[i];
                }
            }
        }
        if (tid < min(NCH, N - n0)) lo_s[buf * NCH + tid] = lo_of(n0 + tid, l) + KKB_MAGIC2_HI_DAS;
    };

    // this lane's pixels: rows zq -> r, r + 4 of the packed slot, cols c + 8j
    constexpr int CX = KKB_DAS_CX;
    int ixp[CX], izp[2];
#pragma unroll
    for (int j = 0; j < CX; ++j) ixp[j] = min(ix0 + wx * 8 * CX + j * 8 + xt, nx - 1);
#pragma unroll
    for (int j = 0; j < 2; ++j) izp[j] = min(iz0 + wz * 8 + j * 4 + zt, nz - 1);
    das_total_t accr[2][CX], acci[2][CX];
    double h[2][CX], hn[2][CX];
    float pr[2][CX], pi[2][CX];
    unsigned gate = 0, gaten = 0;  // bit (p * CX + r): pixel skips this element
    float wl = 1.f, wln = 1.f;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int r = 0; r < CX; ++r) {
            accr[p][r] = acci[p][r] = 0.0;
            pr[p][r] = pi[p][r] = 0.f;
            h[p][r] = hn[p][r] = 0.0;
        }
    // receive path of element l for the lane's 4 pixels (beamform.py:190-197):
    // issued one stage ahead so the hyp loads overlap the previous stage
    auto receive_path = [&](int l) {
        const long long bl = a.base[l];
        const double fr = a.frac[l], ul = a.upos[l];
        wln = a.w ? (float)a.w[l] : 1.f;
        gaten = 0;
#pragma unroll
        for (int p = 0; p < 2; ++p)
#pragma unroll
            for (int r = 0; r < CX; ++r) {
                const long long row = ixp[r] + bl;
                double hv = a.hyp[row * nz + izp[p]];
                if (fr > 0.0) hv = __dadd_rn(hv, __dmul_rn(fr, __dsub_rn(a.hyp[(row + 1) * nz + izp[p]], hv)));
                hn[p][r] = hv;
                if (fabs(__dsub_rn(a.xcoord[ixp[r]], ul)) > __dmul_rn(a.zcoord[izp[p]], a.tan_max))
                    gaten |= 1u << (p * CX + r);
            }
    };

    if (nstage > 0) {
        load_stage(elist[0], 0);
        store_stage(elist[0], 0, 0);
        receive_path(elist[0]);
    }
    __syncthreads();
    int li = 0, ch = 0;  // position in the live-element list, transmit chunk
    for (int s = 0; s < nstage; ++s) {
        const int buf = s & 1;
        int li1 = li, ch1 = ch + 1;
        if (ch1 == nchunk) {
            ch1 = 0;
            ++li1;
        }
        const int l1 = elist[min(li1, n_live - 1)];
        if (ch == 0) {
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int r = 0; r < CX; ++r) h[p][r] = hn[p][r];
            gate = gaten;
            wl = wln;
        }
        if (s + 1 < nstage) {
            load_stage(l1, ch1 * NCH);  // in flight during this stage's sums
            if (ch1 == 0) receive_path(l1);
        }
        const int n0 = ch * NCH;
        const int nc = min(NCH, N - n0);
        const Entry *wb = win + buf * NCH * W;
        const int *lo_b = lo_s + buf * NCH;
        constexpr int kQU = KKB_DAS_QUNROLL;
#pragma unroll kQU
        for (int q = 0; q < nc; ++q) {
            const int n = n0 + q;
            const double2 tz = reinterpret_cast<const double2 *>(ltz_p + n * TZ)[zq];
            double txv[CX];
#pragma unroll
            for (int j = 0; j < CX / 2; ++j) {
                const double2 tx = reinterpret_cast<const double2 *>(ltx_p + n * TX + xq * CX)[j];
                txv[2 * j] = tx.x;
                txv[2 * j + 1] = tx.y;
            }
            const int loC = lo_b[q];
            const Entry *wv = wb + q * W;
#pragma unroll
            for (int p = 0; p < 2; ++p) {
#pragma unroll
                for (int r = 0; r < CX; ++r) {
                    const double t = __dadd_rn(txv[r], p ? tz.y : tz.x);
                    const double fi = das_fi(t, h[p][r], fs, shift);
                    const double sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), KKB_FLOOR_MAGIC2_DAS);
                    const unsigned e = min((unsigned)(__double2hiint(sv) - loC),
                                           (unsigned)(LINEAR ? W - 2 : W - 1));
                    // gated pixels weigh 0 (the reference skips them, beamform.py:191)
                    const float m = ((gate >> (p * CX + r)) & 1u) ? 0.f : wl;
                    if constexpr (LINEAR) {
                        const float4 v = wv[e];
                        const float f1 = __uint_as_float(((unsigned)__double2loint(sv) >> 9) + 0x3F800000u);
                        pr[p][r] = fmaf(m, fmaf(f1, v.z, v.x), pr[p][r]);
                        pi[p][r] = fmaf(m, fmaf(f1, v.w, v.y), pi[p][r]);
                    } else {
                        const float2 v = wv[e];
                        pr[p][r] = fmaf(m, v.x, pr[p][r]);
                        pi[p][r] = fmaf(m, v.y, pi[p][r]);
                    }
                }
            }
        }
        if (ch == nchunk - 1) {  // element l done: fold its weighted partial
#pragma unroll
            for (int p = 0; p < 2; ++p)
#pragma unroll
                for (int r = 0; r < CX; ++r) {
                    accr[p][r] += (das_total_t)pr[p][r];
                    acci[p][r] += (das_total_t)pi[p][r];
                    pr[p][r] = pi[p][r] = 0.f;
                }
        }
        if (s + 1 < nstage) store_stage(l1, ch1 * NCH, buf ^ 1);
        __syncthreads();
        li = li1;
        ch = ch1;
    }
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int iz = iz0 + wz * 8 + p * 4 + zt;
#pragma unroll
        for (int r = 0; r < CX; ++r) {
            const int ix = ix0 + wx * 8 * CX + r * 8 + xt;
            if (iz < nz && ix < nx) {
                const long long px = (long long)ix * nz + iz;
                if (a.groups > 1)
                    a.part[(long long)grp * nx * nz + px] = make_double2(accr[p][r], acci[p][r]);
                else if (a.out_kind == KKB_OUT_C128)
                    reinterpret_cast<double2 *>(a.out)[px] = make_double2(accr[p][r], acci[p][r]);
                else
                    reinterpret_cast<float2 *>(a.out)[px] = make_float2((float)accr[p][r], (float)acci[p][r]);
            }
        }
    }
}

// element-group partials -> image, summed in group order (deterministic)
__global__ void k_das_reduce(const double2 *__restrict__ part, int groups, long long P, void *out,
                             int out_kind) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P;
         i += (long long)gridDim.x * blockDim.x) {
        double r = 0.0, im = 0.0;
        for (int g = 0; g < groups; ++g) {
            const double2 v = part[(long long)g * P + i];
            r += v.x;
            im += v.y;
        }
        if (out_kind == KKB_OUT_C128)
            reinterpret_cast<double2 *>(out)[i] = make_double2(r, im);
        else
            reinterpret_cast<float2 *>(out)[i] = make_float2((float)r, (float)im);
    }
}

static size_t das_smem(int N, int L, int W, int NCH, bool linear) {
    return (linear ? sizeof(float4) : sizeof(float2)) * 2 * (size_t)NCH * W +
           sizeof(double) * ((size_t)N * (KKB_DAS_TZ + KKB_DAS_TX) + N + L) +
           sizeof(int) * (2 * (size_t)NCH + L);
}

int das_gather(const float2 *data, int n_tx, int n_el, int n_t, const double *ltx, const double *ltz,
               const double *hyp, int n_hyp_rows, const long long *base, const double *frac,
               const double *xcoord, const double *zcoord, const double *upos, double tan_max,
               const double *weights, double fs, double shift, int linear, int nx, int nz,
               void *out, int out_kind, cudaStream_t s) {
    (void)n_hyp_rows;
    if ((long long)nx * nz <= 0) return KKB_OK;
    const char *force = getenv("KKB_DAS_DIRECT");  // test hook: the per-pixel fallback kernel
    // the tiled kernel's floor add resolves |fi| < 2^19; longer traces use the
    // per-pixel kernel (1.5*2^52 magic)
    if ((force && force[0] == '1') || n_t > (1 << 19))
        return das_gather_direct(data, n_tx, n_el, n_t, ltx, ltz, hyp, base, frac, xcoord, zcoord,
                                 upos, tan_max, weights, fs, shift, linear, nx, nz, out, out_kind, s);
    DasArgs a{data, n_tx, n_el, n_t, ltx, ltz, hyp, base, frac, xcoord, zcoord, upos, tan_max,
              weights, fs, shift, nx, nz, 0, 0, out, out_kind, 1, nullptr};
    const int tiles = (int)(ceil_div(nx, KKB_DAS_TX) * ceil_div(nz, KKB_DAS_TZ));
    // window pre-pass (synchronous: the launch shape depends on it)
    int *d = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&d, sizeof(int), s), "cudaMallocAsync(das window)");
    KKB_TRY_CUDA(cudaMemsetAsync(d, 0, sizeof(int), s), "memset(das window)");
    const size_t wsm = sizeof(double) * 2 * ((size_t)n_tx + n_el);
    if (wsm > 200 * 1024) {
        cudaFreeAsync(d, s);
        return das_gather_direct(data, n_tx, n_el, n_t, ltx, ltz, hyp, base, frac, xcoord, zcoord,
                                 upos, tan_max, weights, fs, shift, linear, nx, nz, out, out_kind, s);
    }
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_das_window, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)wsm),
                 "smem attr das window");
    k_das_window<<<tiles, 256, wsm, s>>>(a, d);
    KKB_CHECK_LAUNCH("k_das_window");
    int W = 0;
    KKB_TRY_CUDA(cudaMemcpyAsync(&W, d, sizeof(int), cudaMemcpyDeviceToHost, s), "copy das window");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync das window");
    cudaFreeAsync(d, s);
    W = (W + 1) & ~1;
    int NCH = std::max(1, std::min(n_tx, KKB_DAS_STAGE / std::max(W, 2)));
    const size_t sm = das_smem(n_tx, n_el, W, NCH, linear != 0);
    if (W > KKB_DAS_STAGE || W < 2 || sm > 200 * 1024)  // steep geometry: per-pixel kernel
        return das_gather_direct(data, n_tx, n_el, n_t, ltx, ltz, hyp, base, frac, xcoord, zcoord,
                                 upos, tan_max, weights, fs, shift, linear, nx, nz, out, out_kind, s);
    a.W = W;
    a.NCH = NCH;
    // element groups: enough CTAs for ~4 per SM (a single frame has few tiles)
    const int want = 4 * sm_count();
    a.groups = std::max(1, std::min(std::max(1, n_el / 8), (want + tiles - 1) / tiles));
    double2 *part = nullptr;
    const long long P = (long long)nx * nz;
    if (a.groups > 1) {
        KKB_TRY_CUDA(cudaMallocAsync(&part, sizeof(double2) * P * a.groups, s), "cudaMallocAsync(das partials)");
        a.part = part;
    }
    const unsigned grid = (unsigned)((long long)tiles * a.groups);
    if (linear) {
        KKB_TRY_CUDA(cudaFuncSetAttribute(k_das_tile<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                     "smem attr das");
        k_das_tile<true><<<grid, KKB_DAS_NT, sm, s>>>(a);
    } else {
        KKB_TRY_CUDA(cudaFuncSetAttribute(k_das_tile<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                     "smem attr das");
        k_das_tile<false><<<grid, KKB_DAS_NT, sm, s>>>(a);
    }
    KKB_CHECK_LAUNCH("k_das_tile");
    if (a.groups > 1) {
        k_das_reduce<<<(unsigned)std::min<long long>(ceil_div(P, 256), 148 * 8), 256, 0, s>>>(
            part, a.groups, P, out, out_kind);
        KKB_CHECK_LAUNCH("k_das_reduce");
        cudaFreeAsync(part, s);
    }
    return KKB_OK;
}

}  // namespace kkb
