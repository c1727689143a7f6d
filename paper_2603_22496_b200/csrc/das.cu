// K7: conventional CPWC delay-and-sum over element data (comparison kernel).
//
// Replaces _das_kernel (beamform.py:178-209).  Same sampling rules as K5:
// per (pixel, transmit n, element l)
//   skip if |x - u_l| > z * tan_max                       (beamform.py:191)
//   h  = hyp[ix + base_l, iz] (+ frac_l * (hyp[.. + 1, iz] - h) if frac_l > 0)
//   fi = ((ltx + ltz) + h) * fs + shift                   (beamform.py:189,198)
// all in float64 with explicit IEEE round-to-nearest steps, so tap indices
// and gating are bit-identical to the reference; taps are float32 lerps,
// element partials float32, transmit totals float64.
//
// One thread per pixel, consecutive threads along depth (the reference's
// flattened p = ix*nz + iz order), hyp rows and traces read through L1
// (a warp's 32 depth neighbours touch one or two 128 B lines per element).

#include <algorithm>

#include "common.cuh"
#include "kk.cuh"

namespace kkb {

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

int das_gather(const float2 *data, int n_tx, int n_el, int n_t, const double *ltx, const double *ltz,
               const double *hyp, int n_hyp_rows, const long long *base, const double *frac,
               const double *xcoord, const double *zcoord, const double *upos, double tan_max,
               const double *weights, double fs, double shift, int linear, int nx, int nz,
               void *out, int out_kind, cudaStream_t s) {
    (void)n_hyp_rows;
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

}  // namespace kkb
