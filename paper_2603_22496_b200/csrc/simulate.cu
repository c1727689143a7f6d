// K8: forward RF simulator (harness input generation).
//
// Replaces _render_traces (simulate.py:187-220), the numba kernel behind
// simulate_rf (simulate.py:223-296): for every (transmit n, element l) trace
// and every scatterer s IN INPUT ORDER,
//   dist = sqrt((sx - u_l)^2 + sz^2)
//   tau  = (sx sin_n + sz cos_n) / c + dist / c      (written as * inv_c)
//   tc   = (tau - t0) fs,   j in [ceil(tc - half), floor(tc + half)] ∩ [0, T-1]
//   q = j - tc + half, i0 = floor(q), v = lerp(wave, q)
//   out[n, l, j] = float32(out[n, l, j] + amp * v)        (amp = refl [/ sqrt(dist)])
// Every operation is an explicit _rn intrinsic in the reference's order (no
// FMA contraction) and each sample's float32 read-add-round follows the
// scatterer order, so the traces are BIT-IDENTICAL to the reference.
//
// Layout: a warp owns one SEGMENT (KKB_SIM_SEG samples, in shared memory) of
// one trace; a CTA holds 8 such (trace, segment) units, so a T = 4096 volume
// keeps ~48 warps per SM in flight.  Scatterers stream through shared memory
// in chunks of 256 (coalesced loads shared by the CTA); each lane derives the
// echo (tc, amplitude, sample range) of one scatterer in float64 into a
// per-warp table, then every lane walks the 32 echoes IN ORDER and updates the
// samples it owns (j = lane mod 32).  A sample is only ever touched by one
// lane, so the scatterer order per sample holds without warp barriers.
// Work is N·L·S·(pulse length) sample updates (config 5 speckle: 7936 traces
// x 3.3 M scatterers x 21 samples).

#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace kkb {

#define KKB_SIM_CHUNK 256
#define KKB_SIM_WARPS 4

__global__ void __launch_bounds__(32 * KKB_SIM_WARPS, 3)
k_render_traces(float *__restrict__ out, int n_tx, int n_el, int n_t, const double *__restrict__ sx,
                const double *__restrict__ sz, const double *__restrict__ refl, long long n_sc,
                const double *__restrict__ upos, const double *__restrict__ sin_t,
                const double *__restrict__ cos_t, double inv_c, double fs, double t0,
                const double *__restrict__ wave, int n_w, double half, int spread, int nseg,
                int seg_len) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double *c_sx = reinterpret_cast<double *>(smem_raw);          // [CHUNK]
    double *c_sz = c_sx + KKB_SIM_CHUNK;                           // [CHUNK]
    double *c_rf = c_sz + KKB_SIM_CHUNK;                           // [CHUNK]
    double *e_tc = c_rf + KKB_SIM_CHUNK;                           // [WARPS][32] echo centre tc
    double2 *e_fa = reinterpret_cast<double2 *>(e_tc + 32 * KKB_SIM_WARPS);  // [WARPS][32] (frac, amp)
    int4 *e_rng = reinterpret_cast<int4 *>(e_fa + 32 * KKB_SIM_WARPS);       // [WARPS][32] (j0, j1, b, -)
    double2 *w_s = reinterpret_cast<double2 *>(e_rng + 32 * KKB_SIM_WARPS);  // [n_w] (w[i], w[i+1])
    float *segs = reinterpret_cast<float *>(w_s + n_w);           // [WARPS][seg_len]

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long unit = (long long)blockIdx.x * KKB_SIM_WARPS + warp;  // (trace, segment)
    const long long p = unit / nseg;                                       // trace n * n_el + l
    const int seg0 = (int)(unit % nseg) * seg_len;
    const int seg1 = min(seg0 + seg_len, n_t) - 1;
    const bool active = p < (long long)n_tx * n_el;
    float *seg = segs + (size_t)warp * seg_len;
    double *my_tc = e_tc + 32 * warp;
    double2 *my_fa = e_fa + 32 * warp;
    int4 *my_rng = e_rng + 32 * warp;
    for (int i = threadIdx.x; i < n_w; i += blockDim.x)
        w_s[i] = make_double2(wave[i], i + 1 < n_w ? wave[i + 1] : 0.0);
    // accumulate onto the caller's traces, as _render_traces adds into `out`
    if (active)
        for (int j = seg0 + lane; j <= seg1; j += 32) seg[j - seg0] = out[p * n_t + j];
    const int n = active ? (int)(p / n_el) : 0, l = active ? (int)(p % n_el) : 0;
    const double u = upos[l], sn = sin_t[n], cs = cos_t[n];

    for (long long s0 = 0; s0 < n_sc; s0 += KKB_SIM_CHUNK) {
        const int cnt = (int)min((long long)KKB_SIM_CHUNK, n_sc - s0);
        __syncthreads();  // previous chunk consumed
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            c_sx[i] = sx[s0 + i];
            c_sz[i] = sz[s0 + i];
            c_rf[i] = refl[s0 + i];
        }
        __syncthreads();
        if (!active) continue;
        for (int b = 0; b < cnt; b += 32) {
            // lane k derives the echo of scatterer b + k
            int j0 = 1, j1 = 0;
            bool fast = true;
            if (b + lane < cnt) {
                const double x = c_sx[b + lane], z = c_sz[b + lane];
                const double ddx = __dadd_rn(x, -u);
                const double dist = __dsqrt_rn(__dadd_rn(__dmul_rn(ddx, ddx), __dmul_rn(z, z)));
                const double tau = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(x, sn), __dmul_rn(z, cs)), inv_c),
                                             __dmul_rn(dist, inv_c));
                double amp = c_rf[b + lane];
                if (spread) amp = __ddiv_rn(amp, __dsqrt_rn(dist));
                const double tc = __dmul_rn(__dadd_rn(tau, -t0), fs);
                const double lo = ceil(__dadd_rn(tc, -half)), hi = floor(__dadd_rn(tc, half));
                // the reference's window clip [0, T-1], then this warp's segment
                j0 = (int)fmin(fmax(lo, (double)seg0), (double)(seg1 + 1));
                j1 = (int)fmax(fmin(hi, (double)seg1), (double)(seg0 - 1));
                // For tc >= 128 (and half <= 127) the reference's q = (j - tc) + half
                // is exact: both sums are multiples of ulp(tc) below 2^8, so
                // floor(q) = j + floor(half - tc) and q - floor(q) = frac(half - tc)
                // for every sample of the echo -- computed once here.
                const double hm = __dadd_rn(half, -tc);
                const double bfl = floor(hm);
                fast = tc >= 128.0 && j0 <= j1;
                my_tc[lane] = tc;
                my_fa[lane] = make_double2(__dadd_rn(hm, -bfl), amp);
                my_rng[lane] = make_int4(j0, j1, fast ? (int)bfl : 0, 0);
            } else {
                my_rng[lane] = make_int4(j0, j1, 0, 0);
            }
            const bool all_fast = __all_sync(0xffffffffu, fast || j0 > j1) && n_w <= 32;
            __syncwarp();
            const int kmax = min(32, cnt - b);
            if (all_fast) {
                // pulse <= 32 samples: each lane owns at most one sample of an echo
                // (j = lane mod 32).  Derive 8 echoes' (sample, amp * v) branch-free,
                // then apply the 8 read-add-round-writes in scatterer order.
                for (int k0 = 0; k0 < kmax; k0 += 8) {
                    int jj[8];
                    double vv[8];
#pragma unroll
                    for (int v8 = 0; v8 < 8; ++v8) {
                        const int k = (k0 + v8) & 31;
                        const int4 r = my_rng[k];
                        const int j = r.x + ((lane - r.x) & 31);
                        const bool ok = k0 + v8 < kmax && j <= r.y;
                        const double2 fa = my_fa[k];
                        const int i0 = ok ? j + r.z : 0;  // in [0, n_w - 1] by construction
                        const double2 w = w_s[i0];
                        const double lerp = __dadd_rn(w.x, __dmul_rn(fa.x, __dadd_rn(w.y, -w.x)));
                        const double v = (fa.x > 0.0 && i0 + 1 < n_w) ? lerp : w.x;
                        vv[v8] = __dmul_rn(fa.y, v);
                        jj[v8] = ok ? j - seg0 : -1;
                    }
#pragma unroll
                    for (int v8 = 0; v8 < 8; ++v8)
                        if (jj[v8] >= 0) seg[jj[v8]] = (float)__dadd_rn((double)seg[jj[v8]], vv[v8]);
                }
            } else {
                // general path: the reference's per-sample arithmetic verbatim
                for (int k = 0; k < kmax; ++k) {
                    const int4 r = my_rng[k];
                    int j = r.x + ((lane - r.x) & 31);
                    if (j > r.y) continue;
                    const double tck = my_tc[k], ak = my_fa[k].y;
                    for (; j <= r.y; j += 32) {
                        const double q = __dadd_rn(__dadd_rn((double)j, -tck), half);
                        const double fl = floor(q);
                        if (fl < 0.0 || fl > (double)(n_w - 1)) continue;
                        const int i0 = (int)fl;
                        const double2 w = w_s[i0];
                        double v = w.x;
                        const double fr = __dadd_rn(q, -fl);
                        if (fr > 0.0 && i0 + 1 < n_w) v = __dadd_rn(v, __dmul_rn(fr, __dadd_rn(w.y, -v)));
                        seg[j - seg0] = (float)__dadd_rn((double)seg[j - seg0], __dmul_rn(ak, v));
                    }
                }
            }
            __syncwarp();  // the echo table is rewritten by the next 32 scatterers
        }
    }
    if (active) {
        float *dst = out + p * n_t;
        for (int j = seg0 + lane; j <= seg1; j += 32) dst[j] = seg[j - seg0];
    }
}

int render_traces(float *out, int n_tx, int n_el, int n_t, const double *sx, const double *sz,
                  const double *refl, long long n_sc, const double *upos, const double *sin_t,
                  const double *cos_t, double inv_c, double fs, double t0, const double *wave,
                  int n_w, double half, int spread, cudaStream_t s) {
    const long long rows = (long long)n_tx * n_el;
    if (rows <= 0 || n_t <= 0) return KKB_OK;
    // segment length: whole traces when shared memory still holds >= 12 warps
    // per SM, else halves / quarters (a warp walks every scatterer of its
    // trace, so shorter segments trade occupancy for repeated echo walks)
    int seg_len = (int)ceil_div(n_t, 32) * 32;
    const char *env = getenv("KKB_SIM_SEG");
    if (env) seg_len = std::max(32, atoi(env) / 32 * 32);
    else
        while (seg_len > 1024 && (size_t)seg_len * 4 * 12 > 200 * 1024) seg_len = (int)ceil_div(seg_len / 2, 32) * 32;
    const int nseg = (int)ceil_div(n_t, seg_len);
    const size_t fixed = sizeof(double) * 3 * KKB_SIM_CHUNK + sizeof(double2) * (size_t)n_w;
    const size_t per_warp = (sizeof(double) + sizeof(double2) + sizeof(int4)) * 32 + sizeof(float) * (size_t)seg_len;
    const size_t sm = fixed + per_warp * KKB_SIM_WARPS;
    if (sm > 227 * 1024) {
        set_error("render_traces: %d-sample segments exceed shared memory", seg_len);
        return KKB_ERR_UNSUPPORTED;
    }
    KKB_TRY_CUDA(cudaFuncSetAttribute(k_render_traces, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm),
                 "smem attr render");
    k_render_traces<<<(unsigned)ceil_div(rows * nseg, KKB_SIM_WARPS), 32 * KKB_SIM_WARPS, sm, s>>>(
        out, n_tx, n_el, n_t, sx, sz, refl, n_sc, upos, sin_t, cos_t, inv_c, fs, t0, wave, n_w, half,
        spread, nseg, seg_len);
    KKB_CHECK_LAUNCH("k_render_traces");
    return KKB_OK;
}

}  // namespace kkb
