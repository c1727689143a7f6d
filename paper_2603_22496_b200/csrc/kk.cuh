// Internal declarations of the gather / LUT / epilogue / decomposition kernels.
#pragma once

#include <vector>

#include <functional>

#include <cuda_fp16.h>
#include <cuda_runtime.h>

// kk gather tile: TZ = 8*WZ depth rows x TX = 8*CX*WX lateral columns per CTA
// (a warp covers 8 x 8CX pixels, 2 x CX per lane)
#ifndef KKB_KK_WZ
#define KKB_KK_WZ 4   // warps along depth
#endif
#ifndef KKB_KK_WX
#define KKB_KK_WX 2   // warps along x
#endif
#ifndef KKB_KK_CX
#define KKB_KK_CX 4   // pixel columns per lane (measured r1: 4 beats 2 by 14%, 8 spills)
#endif
#define KKB_KK_TZ (8 * KKB_KK_WZ)
#define KKB_KK_TX (8 * KKB_KK_CX * KKB_KK_WX)
// small-tile instance for batches whose big-tile grid cannot fill the SMs (a
// single small frame): 16 x 16 pixels, 2 warps; the per-pixel sums run in the
// same (n, m) order, so both instances give bit-identical images
#define KKB_KK_S_WZ 2
#define KKB_KK_S_WX 1
#define KKB_KK_S_CX 2
#define KKB_KK_S_TZ (8 * KKB_KK_S_WZ)
#define KKB_KK_S_TX (8 * KKB_KK_S_CX * KKB_KK_S_WX)
// mid-size instance: 32 x 32 pixels, 4 warps (2 x 4 pixels per lane like the
// big one) for grids between the two, e.g. config-5 row blocks at 4-8 ranks
#define KKB_KK_M_WZ 4
#define KKB_KK_M_WX 1
#define KKB_KK_M_CX 4
#define KKB_KK_M_TZ (8 * KKB_KK_M_WZ)
#define KKB_KK_M_TX (8 * KKB_KK_M_CX * KKB_KK_M_WX)
#ifndef KKB_KK_STAGE_ELEMS
#define KKB_KK_STAGE_ELEMS 1024  // window entries staged per pipeline stage
#endif
#ifndef KKB_KK_MIN_CTAS
#define KKB_KK_MIN_CTAS 2        // occupancy target (caps registers at 128)
#endif
#ifndef KKB_KK_FR
#define KKB_KK_FR 2              // frames per CTA of the batched (big-tile) gather
#endif
#ifndef KKB_KK_CHECK
#define KKB_KK_CHECK 0           // 1: K5 also checks every tap's window index in the loop (debug;
                                 // +11% K5 time; kk_check_windows proves it per plan instead)
#endif
#ifndef KKB_KK_QUNROLL
#define KKB_KK_QUNROLL 1         // receive-loop unroll of the gather
#endif

namespace kkb {

int take_device_error(int *out);

int build_kk_luts(double x0, double dx, int nx, double z0, double dz, int nz, const double *sin_tx,
                  const double *cos_tx, int n_tx, const double *sin_rx, const double *cos_rx,
                  int n_rx, double c, double *ltx, double *ltz, double *lrx, double *lrz,
                  cudaStream_t s);

int transpose_f64(const double *in, int rows, int cols, double *out, cudaStream_t s);

// shared-memory trace window (samples) one tile of each instance needs
struct KKWindows {
    int big, mid, small;
    int bad;  // bit (1 << KKB_KK_INST_*): instance whose window failed kk_check_windows
    int tc;   // window of the tensor-core gather's tile (KKB_KK_TC_TZ x KKB_KK_TC_TX)
    // per (tensor-core tile, pair): the exact window start (the smallest live
    // tap index of the tile's pixels) * 2 + 1 when every live tap sits in its
    // first 16 samples (one K = 16 step); device, owned by the plan; null when
    // the tensor-core gather cannot take the plan
    int *tc_lo;
    // sum over (tile, pair) of the K = 16 steps one frame group takes (1 or 2
    // each): the tensor-core work of a launch (-1: not eligible)
    long long tc_ksteps;
};
// Synchronises `s` (one launch for the three tile sizes).
int kk_window(const double *ltx, const double *ltz, const double *lrx, const double *lrz, int N,
              int M, int nx, int nz, double fs, double shift, KKWindows *win, cudaStream_t s);

#define KKB_MAX_DST 8
// fused row-block all-gather targets of the gather epilogue (device pointers)
struct KKScatter {
    int ndst;
    long long dst_off;
    void *dst[KKB_MAX_DST];
};

#define KKB_MAX_SETS 8
// incoherent multi-set compounding in one launch: receive angles
// [m0[j], m0[j+1]) form set j (m0[0] = 0, m0[nsets] = M); each set's image B_j
// is summed separately (pairs n asc, m asc within the set, as a launch over
// that set alone), stored at out + j * out_set_stride when out is set, and
// intensity = sum_j |B_j|^2 in set order
struct KKSets {
    int nsets;
    int m0[KKB_MAX_SETS + 1];
    long long out_set_stride;
};

int kk_gather(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
              const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
              double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
              long long out_fs, float *inten, unsigned *fmax, const KKWindows &win, cudaStream_t s,
              int accum = 0, const KKScatter *sc = nullptr,
              long long data_ns = 0,  // 0: M*T (dense (N, M, T) traces)
              const KKSets *sets = nullptr, const struct TcPlanes *tcp = nullptr);

// Plan-time proof that no tap of these tables leaves its tile's staged window
// (every tile size whose window fits; synchronises `s`): sets win->bad, and
// the device error word on a failure.
int kk_check_windows(const double *ltx, const double *ltz, const double *lrx, const double *lrz,
                     int N, int M, int T, int nx, int nz, double fs, double shift, int linear,
                     KKWindows *win, cudaStream_t s);

// tensor-core (tcgen05) form of K5 (kk_gather_tc.cu): 4 x 32-pixel tiles,
// 64 frames per work item, persistent CTAs; tc_lo = KKWindows::tc_lo.  fma_fallback(run_if) launches the FMA instance as a standby
// that runs only when *run_if != 0 (a non-finite sample in the batch).
// KKB_ERR_UNSUPPORTED (nothing launched) when the shape does not fit.
int kk_gather_tc(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
                 const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
                 double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
                 long long out_fs, float *inten, unsigned *fmax, const int *tc_lo, int accum,
                 cudaStream_t s, const std::function<int(const unsigned *)> &fma_fallback);
// Traces already split into the tensor-core gather's planes (tcplanes.cuh) by
// K3 (fft_c2c_planes), with their per-frame bounds and non-finite flag; the
// complex64 traces passed beside them are read only by the FMA standby (when
// the flag is set).  kk_gather then runs the tensor-core gather or fails with
// KKB_ERR_UNSUPPORTED: no FMA instance can read planes.
struct TcPlanes {
    const __half *planes;
    const unsigned *fbound;
    const unsigned *nonfinite;
};
int kk_gather_tc_planes(const __half *planes, const unsigned *fbound, const unsigned *nonfinite, int N, int M,
                        int T, const double *ltx, const double *ltzT, const double *lrx, const double *lrzT, int nx,
                        int nz, const double *w, double fs, double shift, int linear, void *out, int out_kind,
                        int n_frames, long long out_fs, float *inten, unsigned *fmax, const int *tc_lo, int accum,
                        cudaStream_t s, const std::function<int(const unsigned *)> &fma_fallback);
#define KKB_KK_TC_TZ 4   // tensor-core tile: 4 depth rows x 32 columns (128 pixels = M)
#define KKB_KK_TC_TX 32
#define KKB_KK_TC_W 32    // window samples per (tile, pair)
#define KKB_KK_TC_MIN_FRAMES 48          // default dispatch: linear batches of at least this many frames
#define KKB_KK_TC_MIN_FRAMES_NEAREST 128 // ... and nearest-tap batches of at least this many

// instance the last kk_gather dispatch launched (KKB_KK_INST_*, include/kkb.h)
int kk_last_instance();

int kk_taps(const double *ltx, const double *ltz, const double *lrx, const double *lrz, int N, int M,
            int T, int nx, int nz, double fs, double shift, int linear, int *idx, cudaStream_t s);

int log_compress(const float *inten, const unsigned *fmax, int n_frames, long long P, float floor_db,
                 float *db, cudaStream_t s);

int compound(const void *images, int J, long long P, int mode, double *out, cudaStream_t s);

int das_gather(const float2 *data, int n_tx, int n_el, int n_t, const double *ltx, const double *ltz,
               const double *hyp, int n_hyp_rows, const long long *base, const double *frac,
               const double *xcoord, const double *zcoord, const double *upos, double tan_max,
               const double *weights, double fs, double shift, int linear, int nx, int nz,
               void *out, int out_kind, cudaStream_t s);

// decomposition (ramps + per-bin contraction)
int build_ramps(const double *tau_host, int L, int M, const double *freq_host,
                const double *scale_host, int Kb, float2 *ramps, cudaStream_t s);
#define KKB_MAX_CLASSES 64  // symmetric angle classes per contraction launch
int contract_sym(const float2 *X, long long ldx, const float2 *CS, long long ldc, float2 *Y,
                 long long ldy, long long B, int L, int M, int Kb, int P, const short *mp,
                 const short *mm, cudaStream_t s);
int contract(const float2 *X, long long ldx, const float2 *R, long long ldr, float2 *Y,
             long long ldy, long long B, int L, int M, int Kb, cudaStream_t s);
struct Stage1Ring;
// persistent ring consumer of contract_sym (decomposer ring mode), nctas CTAs
int contract_sym_ring(const float2 *ring, long long ldx, const float2 *CS, long long ldc, float2 *Y,
                      long long ldy, long long B, int L, int M, int Kb, int P, const short *mp,
                      const short *mm, const Stage1Ring &rs, int *queue, int *started, int nctas,
                      cudaStream_t s);
// fused stage 1 (stage1_fused.cu): K1 + K2 in one kernel for uniform
// symmetric arrays.  stage1_fused_table turns the float64 class delays tau
// (P, L/2 + 1: tau[q][j] for j < L/2, the per-element step at tau[q][L/2])
// and the bin spacing fsT into the kernel's split phase slopes gam
// (P, L/8 + 1 float2)
bool stage1_fused_supported(int T, int L, int P);
void stage1_fused_table(const double *tau, int P, int L, double fsT, std::vector<float2> &out);
int stage1_fused(const void *rf, int in_kind, long long B, int L, int T, const float2 *gam, float2 *Y,
                 long long ldy, int M, int P, const short *mp, const short *mm, const float2 *tws, cudaStream_t s);
// tensor-core (tcgen05, 3xTF32) form of contract_sym (contract_tc.cu)
int build_tc_table(const float2 *cs, long long ldc, int P, int L, int Kb, float **tab, long long *bytes,
                   cudaStream_t s);
int contract_tc(const float2 *X, long long ldx, const float *tab, float2 *Y, long long ldy, long long B,
                int L, int M, int Kb, int P, const short *mp, const short *mm, cudaStream_t s);

// K8 forward simulator (simulate.cu)
int render_traces(float *out, int n_tx, int n_el, int n_t, const double *sx, const double *sz,
                  const double *refl, long long n_sc, const double *upos, const double *sin_t,
                  const double *cos_t, double inv_c, double fs, double t0, const double *wave,
                  int n_w, double half, int spread, cudaStream_t s);

// display / budgeting epilogues (display.cu); scratch >= 300 doubles (device)
int device_max(const double *x, long long n, double *scratch, double *out, cudaStream_t s);
int device_pow_mean(const double *x, long long n, const double *maxv, double g, double *scratch,
                    double *out_dev, double *out_host, cudaStream_t s);
int pow_map(const double *x, long long n, const double *maxv, double g, double *out, cudaStream_t s);
int last_read_max(const double *x, int nx, const double *z, int nz, const double *sin_t,
                  const double *cos_t, int n_tx, const double *sin_r, const double *cos_r, int n_rx,
                  double *scratch, double *out, cudaStream_t s);

}  // namespace kkb
