/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Not part of the product.  Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline / reference arm may load
 * this library, and only as the checker or the timed CPU baseline.
 *
 * Plain-C restatement of the numba-compiled loops of the reference package
 * `kkbeam` (arXiv 2603.22496, /root/reference/pkg/src/kkbeam):
 *
 *   oracle_kk_kernel      <- beamform.py:212-236  (_kk_kernel)
 *   oracle_das_kernel     <- beamform.py:178-209  (_das_kernel)
 *   oracle_render_traces  <- simulate.py:187-220  (_render_traces)
 *
 * Arithmetic follows numba's typing of those loops exactly (numba without
 * fastmath emits plain IEEE ops, no FMA contraction; compile this file with
 * -ffp-contract=off):
 *   - delay index math in float64 in the source order
 *       fi = ((ltx + ltz) + lrz - lrx) * fs + shift      (beamform.py:223,225)
 *   - tap difference d1 - d0 in complex64 (float32 per component)
 *   - (fi - i0) * (d1 - d0) promotes to complex128 (naive complex multiply)
 *   - accumulation in complex128, transmit ascending then channel ascending.
 * Pixels are split over OpenMP threads; each pixel's sum is owned by one
 * thread so the result is bit-identical for any thread count (criterion 10,
 * test_acceptance.py:334-362).
 *
 * Every pixel range entry point takes [p_begin, p_end) in flattened
 * (ix * nz + iz) order so that large configurations can be checked on a
 * sample of pixels.
 */
#include <math.h>
#include <stdint.h>
#include <omp.h>

typedef struct { float re, im; } c64_t;

/* numba complex128 multiply a*b (a real promoted to complex with 0 imag). */
static inline void cmul_real(double a, double br, double bi, double *outr, double *outi)
{
    /* (a + 0i)(br + bi i) = (a*br - 0*bi) + (a*bi + 0*br) i */
    double zr = 0.0 * bi;
    double zi = 0.0 * br;
    *outr = a * br - zr;
    *outi = a * bi + zi;
}

void oracle_kk_kernel(const c64_t *data, int64_t n_tx, int64_t n_rx, int64_t n_t,
                      const double *ltx, const double *ltz,
                      const double *lrx, const double *lrz,
                      const double *weights, double fs, double shift, int linear,
                      int64_t nx, int64_t nz, int64_t p_begin, int64_t p_end,
                      double *out /* complex128 interleaved, indexed p - p_begin */,
                      int num_threads)
{
    if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(static)
    for (int64_t p = p_begin; p < p_end; ++p) {
        int64_t ix = p / nz;
        int64_t iz = p % nz;
        double accr = 0.0, acci = 0.0;
        for (int64_t n = 0; n < n_tx; ++n) {
            double tx = ltx[ix * n_tx + n] + ltz[iz * n_tx + n];
            for (int64_t m = 0; m < n_rx; ++m) {
                double fi = (tx + lrz[iz * n_rx + m] - lrx[ix * n_rx + m]) * fs + shift;
                const c64_t *tr = data + (n * n_rx + m) * n_t;
                if (linear) {
                    int64_t i0 = (int64_t)floor(fi);
                    if (0 <= i0 && i0 + 1 <= n_t - 1) {
                        c64_t d0 = tr[i0], d1 = tr[i0 + 1];
                        float dr = d1.re - d0.re, di = d1.im - d0.im; /* complex64 */
                        double f = fi - (double)i0;
                        double pr, pi;
                        cmul_real(f, (double)dr, (double)di, &pr, &pi);
                        double vr = (double)d0.re + pr, vi = (double)d0.im + pi;
                        double wr, wi;
                        cmul_real(weights[m], vr, vi, &wr, &wi);
                        accr += wr;
                        acci += wi;
                    }
                } else {
                    int64_t j = (int64_t)floor(fi + 0.5);
                    if (0 <= j && j <= n_t - 1) {
                        double wr, wi;
                        cmul_real(weights[m], (double)tr[j].re, (double)tr[j].im, &wr, &wi);
                        accr += wr;
                        acci += wi;
                    }
                }
            }
        }
        out[2 * (p - p_begin)] = accr;
        out[2 * (p - p_begin) + 1] = acci;
    }
}

void oracle_das_kernel(const c64_t *data, int64_t n_tx, int64_t n_el, int64_t n_t,
                       const double *ltx, const double *ltz, const double *hyp,
                       const int64_t *base, const double *frac,
                       const double *xcoord, const double *zcoord, const double *upos,
                       double tan_max, const double *weights, double fs, double shift,
                       int linear, int64_t nx, int64_t nz, int64_t p_begin, int64_t p_end,
                       double *out, int num_threads)
{
    if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(static)
    for (int64_t p = p_begin; p < p_end; ++p) {
        int64_t ix = p / nz;
        int64_t iz = p % nz;
        double accr = 0.0, acci = 0.0;
        for (int64_t n = 0; n < n_tx; ++n) {
            double tx = ltx[ix * n_tx + n] + ltz[iz * n_tx + n];
            for (int64_t l = 0; l < n_el; ++l) {
                if (fabs(xcoord[ix] - upos[l]) > zcoord[iz] * tan_max) continue;
                int64_t r0 = ix + base[l];
                double h = hyp[r0 * nz + iz];
                double fr = frac[l];
                if (fr > 0.0) h += fr * (hyp[(r0 + 1) * nz + iz] - h);
                double fi = (tx + h) * fs + shift;
                const c64_t *tr = data + (n * n_el + l) * n_t;
                if (linear) {
                    int64_t i0 = (int64_t)floor(fi);
                    if (0 <= i0 && i0 + 1 <= n_t - 1) {
                        c64_t d0 = tr[i0], d1 = tr[i0 + 1];
                        float dr = d1.re - d0.re, di = d1.im - d0.im;
                        double f = fi - (double)i0;
                        double pr, pi;
                        cmul_real(f, (double)dr, (double)di, &pr, &pi);
                        double vr = (double)d0.re + pr, vi = (double)d0.im + pi;
                        double wr, wi;
                        cmul_real(weights[l], vr, vi, &wr, &wi);
                        accr += wr;
                        acci += wi;
                    }
                } else {
                    int64_t j = (int64_t)floor(fi + 0.5);
                    if (0 <= j && j <= n_t - 1) {
                        double wr, wi;
                        cmul_real(weights[l], (double)tr[j].re, (double)tr[j].im, &wr, &wi);
                        accr += wr;
                        acci += wi;
                    }
                }
            }
        }
        out[2 * (p - p_begin)] = accr;
        out[2 * (p - p_begin) + 1] = acci;
    }
}

void oracle_render_traces(float *out, int64_t n_tx, int64_t n_el, int64_t n_t,
                          const double *sx, const double *sz, const double *refl, int64_t n_sc,
                          const double *upos, const double *sin_t, const double *cos_t,
                          double inv_c, double fs, double t0,
                          const double *wave, int64_t n_w, double half, int spread,
                          int num_threads)
{
    if (num_threads > 0) omp_set_num_threads(num_threads);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n_tx * n_el; ++p) {
        int64_t n = p / n_el;
        int64_t l = p % n_el;
        float *tr = out + p * n_t;
        for (int64_t s = 0; s < n_sc; ++s) {
            double ddx = sx[s] - upos[l];
            double dist = sqrt(ddx * ddx + sz[s] * sz[s]);
            double tau = (sx[s] * sin_t[n] + sz[s] * cos_t[n]) * inv_c + dist * inv_c;
            double amp = refl[s];
            if (spread) amp /= sqrt(dist);
            double tc = (tau - t0) * fs;
            int64_t j0 = (int64_t)ceil(tc - half);
            int64_t j1 = (int64_t)floor(tc + half);
            if (j0 < 0) j0 = 0;
            if (j1 > n_t - 1) j1 = n_t - 1;
            for (int64_t j = j0; j <= j1; ++j) {
                double q = (double)j - tc + half;
                int64_t i0 = (int64_t)floor(q);
                if (i0 < 0 || i0 > n_w - 1) continue;
                double v = wave[i0];
                double fr = q - (double)i0;
                if (fr > 0.0 && i0 + 1 < n_w) v += fr * (wave[i0 + 1] - v);
                tr[j] = (float)((double)tr[j] + amp * v);
            }
        }
    }
}
