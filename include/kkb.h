/*
 * kkb.h — C ABI of the B200-native KK beamforming hot path (libkkb.so).
 *
 * Drop-in boundary for the reference package `kkbeam` (arXiv 2603.22496).
 * The reference has no FFI: its operator boundary is the flat-array numba
 * kernels its Python wrappers look up at call time, plus the Python
 * signatures around them.  Each entry point below names the reference
 * interface it replaces (paths relative to /root/reference/pkg/src/kkbeam).
 *
 * Conventions (all entry points):
 *   - Array pointers are DEVICE pointers unless the parameter name ends in
 *     `_host`.  Layouts are C row-major, the reference's own (core.py:28-29,
 *     beamform.py:83-93): RF float32 (N, L, T); analytic / decomposed data
 *     complex64 interleaved (re, im) float pairs; LUTs float64 (X, N) etc.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Every call is asynchronous on that stream.
 *   - Return 0 (KKB_OK) or a negative KKB_ERR_* code; kkb_last_error() gives
 *     the message.  Kernels never raise: shape/geometry validation belongs
 *     to the caller (the reference validates in Python before its kernels,
 *     beamform.py:239-254,356-359; compress.py:110-119).
 *   - Output buffers are caller-allocated and fully overwritten
 *     (beamform.py:280,362 allocate `out` and the kernel writes every pixel).
 */
#ifndef KKB_H
#define KKB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KKB_OK 0
#define KKB_ERR_ARG (-1)          /* bad argument value          -> ConfigError   */
#define KKB_ERR_SHAPE (-2)        /* inconsistent shapes/geometry -> GeometryError */
#define KKB_ERR_CUDA (-3)         /* CUDA runtime failure                          */
#define KKB_ERR_NOMEM (-4)        /* device allocation failed                      */
#define KKB_ERR_UNSUPPORTED (-5)  /* size outside what the kernels support         */
#define KKB_ERR_FORMAT (-6)       /* malformed KKRF container     -> FileFormatError */
#define KKB_ERR_IO (-7)           /* operating-system I/O failure -> OSError         */

/* image output element type */
#define KKB_OUT_C64 0   /* complex64  (throughput path, BASELINE config 5 "fp32 complex IQ") */
#define KKB_OUT_C128 1  /* complex128 (ComplexImage dtype, core.py:232)                      */

/* ------------------------------------------------------------ library */
const char *kkb_version(void);
const char *kkb_last_error(void);
/* SM count and compute capability of the current device. */
int kkb_device_info(int *sm_count, int *cc_major, int *cc_minor);
/* Number of kernel launches this library issued since load (all threads). */
long long kkb_launch_count(void);
/* Reads and clears the device-side error word (synchronous): a bit mask of
 * KKB_DEVERR_* raised by kernels since the last call (0 = none). */
int kkb_take_device_error(int *flag);
/* K5: a tap's window index fell outside the trace window staged for its tile
 * (the index is clamped to the last staged entry; the image is then wrong).
 * The window sizing makes this impossible; the flag proves it at run time. */
#define KKB_DEVERR_KK_WINDOW 1

/* ------------------------------------------------------------ K4: delay tables
 * Replaces build_kk_luts / _tx_tables (beamform.py:121-126,159-175):
 *   ltx[ix,n] = x[ix]*sin_tx[n]/c   ltz[iz,n] = z[iz]*cos_tx[n]/c
 *   lrx[ix,m] = x[ix]*sin_rx[m]/c   lrz[iz,m] = z[iz]*cos_rx[m]/c
 * with x = x0 + dx*ix, z = z0 + dz*iz (core.py:133-138), every product and
 * quotient IEEE-rounded in that order -> bit-identical to the reference.
 * sin/cos arrays are device copies of numpy's np.sin/np.cos values. */
int kkb_build_kk_luts(double x0, double dx, int nx, double z0, double dz, int nz,
                      const double *sin_tx, const double *cos_tx, int n_tx,
                      const double *sin_rx, const double *cos_rx, int n_rx, double c,
                      double *ltx, double *ltz, double *lrx, double *lrz, void *stream);

/* ------------------------------------------------------------ K5: kk pixel gather
 * Replaces _kk_kernel (beamform.py:212-236), called by kk (beamform.py:363-374):
 *   out[f,ix,iz] = sum_n sum_m w[m] * lerp(data[f,n,m,:], fi)
 *   fi = ((ltx[ix,n] + ltz[iz,n]) + lrz[iz,m] - lrx[ix,m]) * fs + shift
 * linear (linear != 0): i0 = floor(fi), read iff 0 <= i0 && i0+1 <= T-1;
 * nearest: j = floor(fi + 0.5), read iff 0 <= j <= T-1; else adds 0.
 * fi is evaluated in float64 in exactly that order (tap indices and the
 * in-window predicate are bit-identical to the reference); taps and the
 * per-pixel sum are float32 in a fixed order (the reference's c64 pixel
 * accumulation differs from its c128 image by ~2e-7).
 * `weights` may be NULL (all ones, beamform.py:239-241).
 * n_frames frames share the tables: data frame f at data + f*data_frame_stride
 * (complex elements), out frame f at out + f*out_frame_stride (elements).
 * `intensity` (may be NULL): also writes |out|^2 as float32, frame stride
 * out_frame_stride (the detection of beamform.py:378-380, fused).
 * `frame_max` (may be NULL, n_frames uint32, zeroed by the call): receives the bit
 * pattern of max |out|^2 per frame for the dB epilogue. */
int kkb_kk(const void *data, int n_tx, int n_rx, int n_t,
           const double *ltx, const double *ltz, const double *lrx, const double *lrz,
           int nx, int nz, const double *weights, double fs, double shift, int linear,
           void *out, int out_kind, int n_frames, long long data_frame_stride,
           long long out_frame_stride, float *intensity, unsigned int *frame_max,
           void *stream);

/* Plan form of K5 for repeated launches on fixed tables (the device-resident
 * throughput path): copies the tables, builds depth-major copies of ltz/lrz,
 * and sizes the shared-memory trace window once (synchronises `stream`). */
typedef struct kkb_kk_plan kkb_kk_plan;
int kkb_kk_plan_create(const double *ltx, const double *ltz, const double *lrx, const double *lrz,
                       int n_tx, int n_rx, int n_t, int nx, int nz, const double *weights,
                       double fs, double shift, int linear, void *stream, kkb_kk_plan **out);
int kkb_kk_plan_run(kkb_kk_plan *p, const void *data, int n_frames, long long data_frame_stride,
                    void *out, int out_kind, long long out_frame_stride, float *intensity,
                    unsigned int *frame_max, void *stream);
/* kkb_kk_plan_run with flags: KKB_RUN_ACCUMULATE_INTENSITY adds |IQ|^2 to
 * `intensity` instead of overwriting it -- incoherent compounding of receive
 * sets (compound_incoherent, beamform.py:405-411; cli.py:257-266), one call
 * per set; frame_max (zeroed by each call) then holds the max of the sum. */
#define KKB_RUN_ACCUMULATE_INTENSITY 1
int kkb_kk_plan_run_ex(kkb_kk_plan *p, const void *data, int n_frames, long long data_frame_stride,
                       void *out, int out_kind, long long out_frame_stride, float *intensity,
                       unsigned int *frame_max, int flags, void *stream);
/* Incoherent multi-set compounding in ONE launch (the
 * reference's hybrid / multi-j acquisitions, cli.py:100-107,257-266, with
 * compound_incoherent, beamform.py:405-411): the plan is built over the
 * concatenated receive angles of n_sets (<= 8) sets, set j being angles
 * [set_begin_host[j], set_begin_host[j+1]) (0 = first < ... < last = M).
 * Each set's image B_j is summed in the order a plan over that set alone
 * uses (bit-identical to it when both run the tiled kernel), stored at out + j*out_set_stride (+ f*out_frame_stride,
 * complex elements; out may be NULL), and intensity (required) = sum_j |B_j|^2 in set
 * order (+ the existing intensity with KKB_RUN_ACCUMULATE_INTENSITY);
 * frame_max (zeroed) gets its per-frame max.  The tables are staged once
 * for all sets. */
int kkb_kk_plan_run_sets(kkb_kk_plan *p, const void *data, int n_frames,
                         long long data_frame_stride, int n_sets, const int *set_begin_host,
                         void *out, int out_kind, long long out_frame_stride,
                         long long out_set_stride, float *intensity, unsigned int *frame_max,
                         int flags, void *stream);
/* Fused row-block all-gather: run the plan (whose
 * tables are this rank's lateral rows) and store every IQ pixel straight into
 * each of the n_dst (<= 8) full-image buffers dst_host[d] (device pointers:
 * this rank's own buffer and the peers' buffers mapped with CUDA IPC over
 * NVLink) at dst_offset + ix*nz + iz (+ f*out_frame_stride).  The P2P stores
 * from the gather epilogue replace the NCCL all-gather; the caller orders
 * completion (stream sync + a barrier) before reading its image. */
int kkb_kk_plan_run_scatter(kkb_kk_plan *p, const void *data, int n_frames,
                            long long data_frame_stride, void *const *dst_host, int n_dst,
                            long long dst_offset, int out_kind, long long out_frame_stride,
                            void *stream);
/* kkb_kk_plan_run_ex on a receive subset of a larger trace array: transmit n's
 * traces start at data + n*data_tx_stride (complex elements, a multiple of T;
 * 0 = M*T), so a
 * plan over M receive angles can read M consecutive rows of (N, M_total, T)
 * traces decomposed once for several receive sets.  The subset rows are
 * copied into dense stream-ordered scratch before the gather (the kernels
 * keep dense row arithmetic); kkb_kk_plan_run_sets is the one-launch form of
 * multi-set compounding. */
int kkb_kk_plan_run_strided(kkb_kk_plan *p, const void *data, int n_frames,
                            long long data_frame_stride, long long data_tx_stride, void *out,
                            int out_kind, long long out_frame_stride, float *intensity,
                            unsigned int *frame_max, int flags, void *stream);
/* trace window (samples per pair) the plan stages in shared memory */
int kkb_kk_plan_window(const kkb_kk_plan *p);
/* Plan-time proof of the window sizing: at creation the plan evaluates every
 * (pixel, pair) tap index with the gather's own arithmetic against each tile
 * size's staged window; bit (1 << KKB_KK_INST_*) is set for an instance that
 * would clamp a tap (the dispatch then never uses it, and
 * KKB_DEVERR_KK_WINDOW is raised).  0 = every tiled instance proven. */
int kkb_kk_plan_window_check(const kkb_kk_plan *p);
/* kkb_kk_plan_run_ex on traces already split by kkb_decomposer_run_planes:
 * the tensor-core gather reads the planes and frame bounds; traces (dense
 * (F, N, M, T) complex64) are read only by the FMA standby when *nonfinite is
 * set.  KKB_ERR_UNSUPPORTED when the plan cannot run the tensor-core gather
 * (kkb_kk_plan_tc_ksteps < 0): no other instance reads planes. */
int kkb_kk_plan_run_planes(kkb_kk_plan *p, const void *planes, const unsigned *frame_bound,
                           const unsigned *nonfinite, const void *traces, int n_frames, void *out, int out_kind,
                           long long out_frame_stride, float *intensity, unsigned int *frame_max, int flags,
                           void *stream);
/* Tensor-core gather work of the plan: the number of K = 16 MMA steps (1 or 2
 * per tile and pair, from the plan's exact per-tile windows) one group of 8
 * frames takes; -1 when the plan is not eligible for the tensor-core gather
 * (tile windows beyond 32 samples).  A launch of F frames issues
 * ksteps x ceil(F/8) x 3 MMAs of 128 x 16 x 16 (M x N x K) per group. */
long long kkb_kk_plan_tc_ksteps(const kkb_kk_plan *p);
/* K5 instance the last kk launch of this process dispatched to (any plan,
 * any thread): the per-pixel kernel, or the tiled kernel with 16x16 / 32x32
 * / 32x64 pixel tiles, the last one with one or KKB_KK_FR (2) frames per CTA;
 * KKB_KK_INST_SETS is or-ed in for the multi-set form.  -1 before any launch.
 * Selection: a wave model over the tiled FMA instances; environment override
 * KKB_KK_INST=direct|small|mid|big|big_fr|tc (tests, measurements). */
#define KKB_KK_INST_DIRECT 0
#define KKB_KK_INST_SMALL 1
#define KKB_KK_INST_MID 2
#define KKB_KK_INST_BIG 3
#define KKB_KK_INST_BIG_FR 4
#define KKB_KK_INST_TC 5     /* tensor-core gather (tcgen05, split fp16): 8 x 16 tiles, <= 128 frames per
                                per CTA, <= 128 pairs; an experiment, only when forced (slower, see DESIGN) */
#define KKB_KK_INST_SETS 16
int kkb_kk_last_instance(void);
int kkb_kk_plan_destroy(kkb_kk_plan *p);

/* Diagnostic twin of K5's index math (same device function): writes the tap
 * index of every (pixel, pair) as int32 idx[ix, iz, n, m], -1 when the read
 * falls outside the window.  Used to prove the indices bit-identical to the
 * reference's floor((((ltx+ltz)+lrz)-lrx)*fs+shift) (beamform.py:225-233). */
int kkb_kk_taps(const double *ltx, const double *ltz, const double *lrx, const double *lrz,
                int n_tx, int n_rx, int n_t, int nx, int nz, double fs, double shift, int linear,
                int *idx, void *stream);

/* ------------------------------------------------------------ K7: DAS comparison gather
 * Replaces _das_kernel (beamform.py:178-209), called by das (beamform.py:281-297).
 * hyp is (nx + l_eff, nz); base int64 (L,); frac (L,); xcoord (X,), zcoord
 * (Z,), upos (L,); tan_max = +inf disables the receive gate (beamform.py:48). */
int kkb_das(const void *data, int n_tx, int n_el, int n_t,
            const double *ltx, const double *ltz, const double *hyp, int n_hyp_rows,
            const long long *base, const double *frac, const double *xcoord,
            const double *zcoord, const double *upos, double tan_max,
            const double *weights, double fs, double shift, int linear,
            int nx, int nz, void *out, int out_kind, void *stream);

/* ------------------------------------------------------------ K1/K3: spectral
 * Replaces analytic_signal (spectral.py:84-93): length-T FFT of each float32
 * trace, one-sided weights (spectral.py:65-81), inverse FFT -> complex64.
 * Any T >= 1 up to 2^20: one transform per CTA for T <= 8192 (mixed radix
 * 2/3/4/5/8 plus direct odd radices <= 31, direct DFT for larger prime
 * factors), a four-step T = T1 x T2 transform above 8192 (direct DFT when T
 * has no such split). */
int kkb_analytic_signal(const float *rf, long long n_traces, int n_t, void *out, void *stream);

/* ------------------------------------------------------------ K1-K3: decomposition
 * Replaces shear_and_sum (compress.py:54-82), the data path of compress
 * (compress.py:120): complex (N, L, T) -> complex64 (N, M, T),
 *   out[n,m] = IFFT( sum_l FFT(data[n,l]) * exp(2 pi i f tau_lm) ),
 *   tau_lm = positions[l] * (sin(angles[m]) / c),  f = fftfreq(T, 1/fs).
 * positions_host / angles_host are host arrays. */
int kkb_shear_and_sum(const void *data, int n_tx, int n_el, int n_t,
                      const double *positions_host, const double *angles_host, int n_rx,
                      double fs, double c, void *out, void *stream);
/* Plan form of kkb_shear_and_sum for repeated calls on one geometry (the
 * reference's compress per frame): the phase ramps are built once.
 * kkb_shear_plan_run is asynchronous on `stream`; same arithmetic as
 * kkb_shear_and_sum (which is create + run + destroy). */
typedef struct kkb_shear_plan kkb_shear_plan;
int kkb_shear_plan_create(const double *positions_host, const double *angles_host, int n_el, int n_rx,
                          int n_t, double fs, double c, kkb_shear_plan **out);
int kkb_shear_plan_run(kkb_shear_plan *p, const void *data, int n_tx, void *out, void *stream);
int kkb_shear_plan_destroy(kkb_shear_plan *p);

/* ------------------------------------------------------------ fused stage 1 plan
 * Device-resident, batched form of analytic_signal + compress — the data
 * flow of the reference's complex64 benchmark stages (bench.py:113-153):
 * real FFT of the RF -> one-sided weights x cached ramps, contracted over
 * elements per bin -> inverse FFT, for F frames at once.  Ramps (the
 * reference caches them too, bench.py:124-125) and scratch live in the plan. */
typedef struct kkb_decomposer kkb_decomposer;

int kkb_decomposer_create(int n_tx, int n_el, int n_t, const double *positions_host,
                          const double *angles_host, int n_rx, double fs, double c,
                          int max_frames, kkb_decomposer **out);
/* rf: (F, N, L, T) float32; traces: (F, N, M, T) complex64. */
int kkb_decomposer_run(kkb_decomposer *p, const float *rf, int n_frames, void *traces,
                       void *stream);
/* int16-quantised RF ingest: rf is
 * (F, N, L, T) int16; each sample is converted exactly to float32 (inside the
 * FFT load for T in {1024, 1536, 2048, 4096}, by a widening pass otherwise),
 * identical to running the float32 path on rf.astype(float32). */
int kkb_decomposer_run_i16(kkb_decomposer *p, const short *rf, int n_frames, void *traces,
                           void *stream);
/* Pipelined mode: process chunk_frames per pass, rotating passes over `slots`
 * (1..4) internal streams (forked from / joined back into the caller's
 * stream), so one pass's FFT overlaps the previous pass's contraction and the
 * spectra are consumed while L2-resident.  Reallocates scratch (synchronous). */
int kkb_decomposer_set_pipeline(kkb_decomposer *p, int chunk_frames, int slots);
/* Transmit-sharded stage 1 with a fused trace all-gather (SURVEY §8(e),
 * config 5 alternative): a plan created for this rank's n_tx transmits
 * decomposes rf ((F, n_tx, L, T), float32, or int16 if rf_is_i16) and the
 * inverse FFT's epilogue stores trace (f, n, m) into each of the ndst (<= 8)
 * buffers dsts_host[d] (device pointers: this rank's full (F, N, M, T) trace
 * buffer and the peers' buffers mapped with CUDA IPC over NVLink) at complex64
 * element dst_offset + f*frame_stride + (n*M + m)*T — dst_offset = n0*M*T for
 * a rank holding transmits [n0, n0 + n_tx), frame_stride = N*M*T.  Per-row
 * arithmetic is independent of the transmit split, so the assembled traces
 * equal a single plan's bit for bit.  The caller orders completion (stream
 * sync + a barrier) before any rank reads its traces. */
int kkb_decomposer_run_scatter(kkb_decomposer *p, const void *rf, int rf_is_i16, int n_frames,
                               void *const *dsts_host, int ndst, long long dst_offset,
                               long long frame_stride, void *stream);
/* Number of +/- receive-angle classes of the symmetric contraction the plan
 * uses (0: general contraction).  The reference guarantees the symmetry
 * (ReceiveAngleSet, sampling.py:55-57; centred positions, core.py:32-38). */
int kkb_decomposer_symmetric_classes(const kkb_decomposer *p);
/* Contraction form of the plan's K2 (north star: "complex fp32 via split real
 * GEMM or fp32 FMA, whichever ncu shows faster"): KKB_CONTRACT_FMA, the
 * symmetric FP32-FMA kernel (default), or KKB_CONTRACT_TENSOR, the same
 * symmetric contraction as one real GEMM per bin on the tcgen05 tensor cores
 * in split precision (3xTF32: hi*hi + hi*lo + lo*hi, fp32 accumulation in
 * TMEM).  The tensor form needs the symmetric geometry with <= 16 angle
 * classes (KKB_ERR_UNSUPPORTED otherwise).  Environment KKB_CONTRACT=tc
 * selects it at creation. */
#define KKB_CONTRACT_FMA 0
#define KKB_CONTRACT_TENSOR 1
int kkb_decomposer_set_contraction(kkb_decomposer *p, int form);
int kkb_decomposer_contraction(const kkb_decomposer *p);
/* Fused stage 1 (opt-in): the real FFT (K1) and the symmetric FMA
 * contraction (K2) as ONE warp-specialised kernel per (frame, transmit) row,
 * the per-element spectra kept in shared memory instead of round-tripping
 * through HBM (replaces rfft * one_sided / T and the compress einsum,
 * spectral.py:84-93, compress.py:78-81): 3.8 instead of 11.6 GB of DRAM
 * traffic per 400 config-4 frames, but measured slower than K1 -> K2 on the
 * B200 (issue- and latency-bound), so plans default to K1 -> K2.
 * Its phase factors come from float64 phases anchored every four element
 * pairs and stepped by the per-element rotation, so it needs a uniform array
 * (the reference's TransducerArray, core.py:32-38); eligible plans: T = 1536,
 * L a multiple of 8 up to 256, symmetric receive set with <= 6 classes
 * (M <= 12).  Traces differ from the unfused path by ~1e-7 relative (both
 * within the 1e-5 bound).  set_fused(p, 1) selects it (environment
 * KKB_S1_FUSED=1 at creation); set_fused(p, 1) on an ineligible plan is
 * KKB_ERR_UNSUPPORTED.  fused() reports whether the plan's stage 1 runs
 * fused. */
int kkb_decomposer_set_fused(kkb_decomposer *p, int on);
int kkb_decomposer_fused(const kkb_decomposer *p);
/* Stage-1 ring mode: K1 (real FFT) and a persistent K2 (contraction, FMA
 * form) run concurrently, the spectra handed over through `slots` row-tile
 * slots of an L2-resident ring (16 (frame, transmit) rows each) instead of a
 * full spectra array in HBM; `consumer_ctas` persistent K2 CTAs (0: half the
 * SMs).  Used for float32 / int16 RF with a compile-time FFT length, an even
 * element count and <= 6 symmetric classes; otherwise the three-kernel path
 * runs.  slots = 0 turns it off.  Environment KKB_S1_RING=slots[,ctas] sets
 * it at creation.  kkb_decomposer_ring_error (synchronous) reports a bounded
 * spin that timed out (1), which would mean a scheduling failure. */
int kkb_decomposer_set_ring(kkb_decomposer *p, int slots, int consumer_ctas);
int kkb_decomposer_ring_error(kkb_decomposer *p, int *flag);
/* One stage of stage 1 at a time, for the reference's staged benchmark
 * (kkbeam.bench._kk_stage_fns, bench.py:113-153): stage 0 the real FFT of rf
 * ((F, N, L, T) float32) into the plan's spectra ("reorg_fft"), 1 the
 * contraction with the one-sided weights folded into the cached ramps
 * ("hilbert_compress"), 2 the inverse FFT into traces ((F, N, M, T)
 * complex64, "ifft").  Same launches and results as kkb_decomposer_run;
 * F <= the plan's max_frames, stages in order 0, 1, 2 on one stream. */
int kkb_decomposer_run_stage(kkb_decomposer *p, int stage, const float *rf, int n_frames, void *traces,
                             void *stream);
/* analytic_signal one stage at a time (the staged DAS benchmark,
 * kkbeam.bench._das_stage_fns, bench.py:91-110): stage 0 real FFT of rf
 * ((n_traces, T) float32) into spec ((n_traces, T/2 + 1) complex64, caller
 * scratch), 1 one-sided weights / T applied to spec in place, 2 inverse FFT
 * into out ((n_traces, T) complex64).  0 + 1 + 2 == kkb_analytic_signal. */
int kkb_analytic_signal_stage(int stage, const float *rf, long long n_traces, int n_t, void *spec, void *out,
                              void *stream);
/* Stage 1 emitting the tensor-core gather's split trace planes instead of
 * complex64 traces (the fused bench path; kkb_kk_plan_run_planes consumes
 * them): K1, K2, a per-frame bound (max over the frame's traces of the L1
 * norm of their bins, >= every |sample|) into frame_bound[F], then K3
 * writes each trace scaled by its frame's power of two and split into fp16
 * halves (hi + lo) as planes (kkb_tc_planes_bytes(F, N*M, T) bytes, layout
 * in the library's tcplanes.cuh).  A NaN / Inf bin sets *nonfinite, and only
 * then are the complex64 traces ((F, N, M, T)) written too — for the FMA
 * gather, which then runs instead.  T in {1024, 1536, 2048}; F <= the plan's
 * max_frames. */
int kkb_decomposer_run_planes(kkb_decomposer *p, const float *rf, int n_frames, void *planes,
                              unsigned *frame_bound, unsigned *nonfinite, void *traces, void *stream);
/* bytes of the split planes of F frames of `pairs` traces of T samples */
long long kkb_tc_planes_bytes(int n_frames, int pairs, int n_t);
/* bytes of device scratch held by the plan */
long long kkb_decomposer_workspace_bytes(const kkb_decomposer *p);
int kkb_decomposer_destroy(kkb_decomposer *p);

/* ------------------------------------------------------------ K6: log-compression epilogue
 * dB display map (new; the reference has no log compression):
 * db[f,p] = max(10*log10(intensity[f,p] / max_f), floor_db), max_f from the
 * frame_max array filled by kkb_kk. */
int kkb_log_compress(const float *intensity, const unsigned int *frame_max, int n_frames,
                     long long pixels_per_frame, float floor_db, float *db, void *stream);

/* Element-wise compounding over J images (beamform.py:396-411):
 * mode 0 coherent |sum_j B_j|^2, mode 1 incoherent sum_j |B_j|^2.
 * images: J x P complex128; out: P float64. */
int kkb_compound(const void *images, int n_images, long long n_pixels, int mode,
                 double *out, void *stream);

/* ------------------------------------------------------------ K8: forward RF simulator
 * Replaces _render_traces (simulate.py:187-220), the kernel of simulate_rf
 * (simulate.py:223-296): adds the pulse echo of every scatterer (input order)
 * to out (n_tx, n_el, n_t) float32 (accumulates: simulate_rf passes zeros).
 * sx, sz, refl: (n_sc,) float64; upos (n_el,); sin_t, cos_t (n_tx,) numpy's
 * np.sin/np.cos of the transmit angles; wave (n_w,) the pulse waveform; half =
 * its peak index; spread != 0 divides by sqrt(distance).  All arrays device
 * pointers.  Bit-identical to the reference (float64 in its operation order,
 * float32 accumulation in scatterer order).  The caller performs the
 * window-overflow check (simulate.py:246-264). */
int kkb_render_traces(float *out, int n_tx, int n_el, int n_t, const double *sx, const double *sz,
                      const double *refl, long long n_sc, const double *upos, const double *sin_t,
                      const double *cos_t, double inv_c, double fs, double t0, const double *wave,
                      int n_w, double half, int spread, void *stream);

/* ------------------------------------------------------------ KKRF container I/O
 * The reference's binary RF container (rffile.py:1-26): 59-byte little-endian
 * head "<4sHB3I5d", N f64 transmit angles, M f64 receive angles (kind 2), then
 * the C-order payload (float32 kind 0, complex64 kinds 1/2).  These calls move
 * bytes; the reference's validation rules and messages (read_container,
 * rffile.py:116-178) live in the Python mirror.  Payload transfers to/from
 * DEVICE memory stream through two pinned 16 MiB buffers so disk and PCIe
 * overlap; they return with the copies complete. */
typedef struct kkb_kkrf_header {
    char magic[4];
    uint16_t version;
    uint8_t kind;                /* 0 real RF, 1 analytic RF, 2 compressed RF */
    uint32_t num_transmits;
    uint32_t num_channels;       /* elements L (kinds 0/1) or receive angles M (kind 2) */
    uint32_t num_samples;
    double sampling_frequency, center_frequency, sound_speed, pitch, start_time;
    long long head_bytes;        /* 59 */
    long long file_bytes;        /* file size (filled by kkb_kkrf_read_header) */
} kkb_kkrf_header;

/* Parses the fixed head (no validation beyond its length: KKB_ERR_FORMAT). */
int kkb_kkrf_read_header(const char *path, kkb_kkrf_header *header);
/* Reads `bytes` at `offset` into dst (host, or device when dst_is_device). */
int kkb_kkrf_read_bytes(const char *path, long long offset, long long bytes, void *dst,
                        int dst_is_device, void *stream);
/* Ensemble ingest (cli.py:110-128 reads one container per frame): frame f's
 * frame_bytes payload at offsets_host[f] of paths_host[f] lands in device
 * memory at dst + f*frame_bytes.  `threads` (1..64) reader threads, each with
 * its own pinned double-buffered staging and stream, overlap the file reads
 * with the H2D copies; the copies wait for work already queued on `stream`
 * and are complete on return (synchronous). */
int kkb_kkrf_read_ensemble(const char *const *paths_host, const long long *offsets_host,
                           int n_files, long long frame_bytes, void *dst, int threads,
                           void *stream);
/* Writes head, angle tables (rx_host only for kind 2) and the payload
 * (host, or device when payload_is_device), replacing `path`. */
int kkb_kkrf_write(const char *path, const kkb_kkrf_header *header, const double *tx_host,
                   const double *rx_host, const void *payload, long long payload_bytes,
                   int payload_is_device, void *stream);

/* ------------------------------------------------------------ display / budgeting
 * Max of a float64 device array (synchronous; result on the host). */
int kkb_max_f64(const double *x, long long n, double *max_host, void *stream);
/* Replaces gamma_match (metrics.py:175-202): normalise `image` (n float64,
 * device) by its max and golden-section search (metrics.py:156-172, same
 * steps) the exponent g in [lo, hi] (tolerance tol) whose mean (I/max)^g
 * matches mean((R/maxR)^0.5) of `reference`.  Every objective evaluation is
 * a deterministic device reduction.  gamma -> *gamma_host; `mapped` (device,
 * may be NULL) receives (I/max)^gamma.  KKB_ERR_SHAPE if either max <= 0. */
int kkb_gamma_match(const double *image, const double *reference, long long n, double lo,
                    double hi, double tol, double *gamma_host, double *mapped, void *stream);
/* The maximum over the (nx, nz) grid of max_n(x sin_n + z cos_n) +
 * max_m(z cos_m - x sin_m): the delay numerator of the last sample the kk
 * gather reads (cli.py:110-128, the compress guard-band budget).  Arrays are
 * device float64 (x: nx, z: nz, sin/cos of the transmit and receive angles);
 * bit-identical to the reference's numpy expression. */
int kkb_last_read_sample_max(const double *x, int nx, const double *z, int nz,
                             const double *sin_t, const double *cos_t, int n_tx,
                             const double *sin_r, const double *cos_r, int n_rx,
                             double *max_host, void *stream);

/* ------------------------------------------------------------ CUDA IPC for row-block P2P
 * A plain cudaMalloc buffer (IPC handles need allocation base pointers), its
 * 64-byte handle, and mapping / unmapping a peer process's handle. */
int kkb_ipc_alloc(long long bytes, void **ptr);
int kkb_ipc_free(void *ptr);
int kkb_ipc_get_handle(const void *ptr, void *handle64);
int kkb_ipc_open_handle(const void *handle64, void **ptr);
int kkb_ipc_close_handle(void *ptr);

#ifdef __cplusplus
}
#endif
#endif /* KKB_H */
