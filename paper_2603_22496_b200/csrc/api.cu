// C ABI of libkkb (include/kkb.h): validation, temporaries, plans.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>
#include <map>

#include "common.cuh"
#include "fft.cuh"
#include "kk.cuh"

#define KKB_VERSION_STR "kkb-b200 0.1.0 (sm_100a)"

namespace kkb {

static thread_local std::string t_last_error;
static std::atomic<long long> g_launches{0};

void set_error(const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    t_last_error = buf;
}

int cuda_status(cudaError_t e, const char *what) {
    set_error("%s: %s", what, cudaGetErrorString(e));
    return e == cudaErrorMemoryAllocation ? KKB_ERR_NOMEM : KKB_ERR_CUDA;
}

void count_launch(int n) { g_launches += n; }

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

// numpy.fft.fftfreq(T, 1/fs)[k]: integer bin times 1/(T*d), d = 1/fs
static double fftfreq(int k, int T, double fs) {
    double d = 1.0 / fs;
    double val = 1.0 / (T * d);
    int half = (T - 1) / 2 + 1;  // count of non-negative bins
    int kk = k < half ? k : k - T;
    return kk * val;
}

// one_sided_weights (spectral.py:65-81)
static double one_sided(int k, int T) {
    if (k == 0) return 1.0;
    if (T % 2 == 0) {
        if (k < T / 2) return 2.0;
        if (k == T / 2) return 1.0;
        return 0.0;
    }
    return k <= (T - 1) / 2 ? 2.0 : 0.0;
}

__global__ void k_scale_bins(float2 *X, long long ntr, long long ld, int K, const float *scale) {
    const long long total = ntr * K;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        long long r = i / K;
        int k = (int)(i - r * K);
        float2 v = X[r * ld + k];
        float s = scale[k];
        X[r * ld + k] = make_float2(v.x * s, v.y * s);
    }
}

// RAII device scratch on a stream (stream-ordered allocator)
struct Scratch {
    void *p = nullptr;
    cudaStream_t s;
    explicit Scratch(cudaStream_t st) : s(st) {}
    int alloc(size_t bytes) {
        if (bytes == 0) bytes = 16;
        cudaError_t e = cudaMallocAsync(&p, bytes, s);
        if (e != cudaSuccess) return cuda_status(e, "cudaMallocAsync");
        return KKB_OK;
    }
    ~Scratch() {
        if (p) cudaFreeAsync(p, s);
    }
};

}  // namespace kkb

using namespace kkb;

// =====================================================================
// library
extern "C" const char *kkb_version(void) { return KKB_VERSION_STR; }
extern "C" const char *kkb_last_error(void) { return t_last_error.c_str(); }
extern "C" long long kkb_launch_count(void) { return g_launches.load(); }

extern "C" int kkb_device_info(int *sms, int *major, int *minor) {
    int dev = 0;
    KKB_TRY_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    cudaDeviceProp prop;
    KKB_TRY_CUDA(cudaGetDeviceProperties(&prop, dev), "cudaGetDeviceProperties");
    if (sms) *sms = prop.multiProcessorCount;
    if (major) *major = prop.major;
    if (minor) *minor = prop.minor;
    return KKB_OK;
}

extern "C" int kkb_take_device_error(int *flag) { return take_device_error(flag); }

// =====================================================================
// K4
extern "C" int kkb_build_kk_luts(double x0, double dx, int nx, double z0, double dz, int nz,
                                 const double *sin_tx, const double *cos_tx, int n_tx,
                                 const double *sin_rx, const double *cos_rx, int n_rx, double c,
                                 double *ltx, double *ltz, double *lrx, double *lrz, void *stream) {
    if (nx < 1 || nz < 1 || n_tx < 1 || n_rx < 1 || !(c > 0)) {
        set_error("build_kk_luts: bad sizes");
        return KKB_ERR_ARG;
    }
    return build_kk_luts(x0, dx, nx, z0, dz, nz, sin_tx, cos_tx, n_tx, sin_rx, cos_rx, n_rx, c, ltx,
                         ltz, lrx, lrz, as_stream(stream));
}

// =====================================================================
// K5 (stateless): transposes the z tables, sizes the window, gathers
static int check_kk_args(int n_tx, int n_rx, int n_t, int nx, int nz, int out_kind) {
    if (n_tx < 1 || n_rx < 1 || n_t < 2 || nx < 1 || nz < 1) {
        set_error("kk: bad sizes N=%d M=%d T=%d X=%d Z=%d", n_tx, n_rx, n_t, nx, nz);
        return KKB_ERR_ARG;
    }
    if (out_kind != KKB_OUT_C64 && out_kind != KKB_OUT_C128) {
        set_error("kk: unknown out_kind %d", out_kind);
        return KKB_ERR_ARG;
    }
    if (n_t > (1 << 19)) {  // tap_index: RD(fi + 1.5*2^20) resolves |fi| < 2^19
        set_error("kk: %d samples per trace exceed the 2^19 tap-index range", n_t);
        return KKB_ERR_UNSUPPORTED;
    }
    return KKB_OK;
}

struct kkb_kk_plan {
    int N, M, T, nx, nz, linear;
    KKWindows win;  // trace windows of the big / mid / small tiles
    double fs, shift;
    double *ltx, *ltzT, *lrx, *lrzT, *w;  // one allocation
};

extern "C" int kkb_kk_plan_create(const double *ltx, const double *ltz, const double *lrx,
                                  const double *lrz, int n_tx, int n_rx, int n_t, int nx, int nz,
                                  const double *weights, double fs, double shift, int linear,
                                  void *stream, kkb_kk_plan **out) {
    int st = check_kk_args(n_tx, n_rx, n_t, nx, nz, KKB_OUT_C64);
    if (st) return st;
    cudaStream_t s = as_stream(stream);
    kkb_kk_plan *p = new (std::nothrow) kkb_kk_plan();
    if (!p) return KKB_ERR_NOMEM;
    p->N = n_tx;
    p->M = n_rx;
    p->T = n_t;
    p->nx = nx;
    p->nz = nz;
    p->linear = linear;
    p->fs = fs;
    p->shift = shift;
    size_t n_ltx = (size_t)nx * n_tx, n_ltz = (size_t)nz * n_tx, n_lrx = (size_t)nx * n_rx,
           n_lrz = (size_t)nz * n_rx;
    double *buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, sizeof(double) * (n_ltx + n_ltz + n_lrx + n_lrz + n_rx));
    if (e != cudaSuccess) {
        delete p;
        return cuda_status(e, "cudaMalloc(kk plan)");
    }
    p->ltx = buf;
    p->ltzT = buf + n_ltx;
    p->lrx = p->ltzT + n_ltz;
    p->lrzT = p->lrx + n_lrx;
    p->w = weights ? p->lrzT + n_lrz : nullptr;
    auto fail = [&](int code) {
        cudaFree(buf);
        if (p->win.tc_lo) cudaFree(p->win.tc_lo);
        delete p;
        return code;
    };
    if ((e = cudaMemcpyAsync(p->ltx, ltx, sizeof(double) * n_ltx, cudaMemcpyDeviceToDevice, s)))
        return fail(cuda_status(e, "copy ltx"));
    if ((e = cudaMemcpyAsync(p->lrx, lrx, sizeof(double) * n_lrx, cudaMemcpyDeviceToDevice, s)))
        return fail(cuda_status(e, "copy lrx"));
    if (weights &&
        (e = cudaMemcpyAsync(p->w, weights, sizeof(double) * n_rx, cudaMemcpyDeviceToDevice, s)))
        return fail(cuda_status(e, "copy weights"));
    if ((st = transpose_f64(ltz, nz, n_tx, p->ltzT, s))) return fail(st);
    if ((st = transpose_f64(lrz, nz, n_rx, p->lrzT, s))) return fail(st);
    if ((st = kk_window(ltx, ltz, lrx, lrz, n_tx, n_rx, nx, nz, fs, shift, &p->win, s))) return fail(st);
    if ((st = kk_check_windows(ltx, ltz, lrx, lrz, n_tx, n_rx, n_t, nx, nz, fs, shift, linear, &p->win, s)))
        return fail(st);
    *out = p;
    return KKB_OK;
}

extern "C" int kkb_kk_plan_window(const kkb_kk_plan *p) { return p ? p->win.big : -1; }

extern "C" int kkb_kk_plan_window_check(const kkb_kk_plan *p) { return p ? p->win.bad : -1; }

extern "C" long long kkb_kk_plan_tc_ksteps(const kkb_kk_plan *p) { return p ? p->win.tc_ksteps : -1; }

extern "C" int kkb_kk_last_instance(void) { return kk_last_instance(); }

extern "C" int kkb_kk_plan_run_strided(kkb_kk_plan *p, const void *data, int n_frames,
                                       long long data_frame_stride, long long data_tx_stride,
                                       void *out, int out_kind, long long out_frame_stride,
                                       float *intensity, unsigned int *frame_max, int flags,
                                       void *stream) {
    if (!p || (flags & ~KKB_RUN_ACCUMULATE_INTENSITY) ||
        (data_tx_stride != 0 && (data_tx_stride < (long long)p->M * p->T || data_tx_stride % p->T))) {
        set_error("kk_plan_run: bad flags or transmit stride (a multiple of T, >= M*T)");
        return KKB_ERR_ARG;
    }
    int st = check_kk_args(p->N, p->M, p->T, p->nx, p->nz, out_kind);
    if (st) return st;
    if (frame_max)
        KKB_TRY_CUDA(cudaMemsetAsync(frame_max, 0, sizeof(unsigned) * (size_t)n_frames, as_stream(stream)),
                     "zero frame_max");
    return kk_gather(reinterpret_cast<const float2 *>(data), p->N, p->M, p->T, p->ltx, p->ltzT,
                     p->lrx, p->lrzT, p->nx, p->nz, p->w, p->fs, p->shift, p->linear, out,
                     out_kind, n_frames, data_frame_stride, out_frame_stride, intensity, frame_max,
                     p->win, as_stream(stream), (flags & KKB_RUN_ACCUMULATE_INTENSITY) ? 1 : 0,
                     nullptr, data_tx_stride);
}

extern "C" int kkb_kk_plan_run_ex(kkb_kk_plan *p, const void *data, int n_frames,
                                  long long data_frame_stride, void *out, int out_kind,
                                  long long out_frame_stride, float *intensity,
                                  unsigned int *frame_max, int flags, void *stream) {
    return kkb_kk_plan_run_strided(p, data, n_frames, data_frame_stride, 0, out, out_kind,
                                   out_frame_stride, intensity, frame_max, flags, stream);
}

extern "C" int kkb_kk_plan_run_planes(kkb_kk_plan *p, const void *planes, const unsigned *frame_bound,
                                      const unsigned *nonfinite, const void *traces, int n_frames, void *out,
                                      int out_kind, long long out_frame_stride, float *intensity,
                                      unsigned int *frame_max, int flags, void *stream) {
    if (!p || !planes || !frame_bound || !nonfinite || !traces || (flags & ~KKB_RUN_ACCUMULATE_INTENSITY)) {
        set_error("kk_plan_run_planes: planes, bounds, flag and traces are required");
        return KKB_ERR_ARG;
    }
    int st = check_kk_args(p->N, p->M, p->T, p->nx, p->nz, out_kind);
    if (st) return st;
    if (frame_max)
        KKB_TRY_CUDA(cudaMemsetAsync(frame_max, 0, sizeof(unsigned) * (size_t)n_frames, as_stream(stream)),
                     "zero frame_max");
    const TcPlanes tcp{reinterpret_cast<const __half *>(planes), frame_bound, nonfinite};
    return kk_gather(reinterpret_cast<const float2 *>(traces), p->N, p->M, p->T, p->ltx, p->ltzT, p->lrx, p->lrzT,
                     p->nx, p->nz, p->w, p->fs, p->shift, p->linear, out, out_kind, n_frames,
                     (long long)p->N * p->M * p->T, out_frame_stride, intensity, frame_max, p->win, as_stream(stream),
                     (flags & KKB_RUN_ACCUMULATE_INTENSITY) ? 1 : 0, nullptr, 0, nullptr, &tcp);
}

extern "C" int kkb_kk_plan_run_sets(kkb_kk_plan *p, const void *data, int n_frames,
                                    long long data_frame_stride, int n_sets,
                                    const int *set_begin_host, void *out, int out_kind,
                                    long long out_frame_stride, long long out_set_stride,
                                    float *intensity, unsigned int *frame_max, int flags,
                                    void *stream) {
    if (!p || !set_begin_host || !intensity || n_sets < 1 || n_sets > KKB_MAX_SETS ||
        (flags & ~KKB_RUN_ACCUMULATE_INTENSITY)) {
        set_error("kk_plan_run_sets: intensity buffer, 1 <= n_sets <= %d, known flags", KKB_MAX_SETS);
        return KKB_ERR_ARG;
    }
    KKSets sets{};
    sets.nsets = n_sets;
    sets.out_set_stride = out_set_stride;
    for (int j = 0; j <= n_sets; ++j) sets.m0[j] = set_begin_host[j];
    bool ok = sets.m0[0] == 0 && sets.m0[n_sets] == p->M;
    for (int j = 0; j < n_sets; ++j) ok = ok && sets.m0[j + 1] > sets.m0[j];
    if (!ok) {
        set_error("kk_plan_run_sets: set bounds must rise strictly from 0 to M=%d", p->M);
        return KKB_ERR_ARG;
    }
    int st = check_kk_args(p->N, p->M, p->T, p->nx, p->nz, out_kind);
    if (st) return st;
    if (frame_max)
        KKB_TRY_CUDA(cudaMemsetAsync(frame_max, 0, sizeof(unsigned) * (size_t)n_frames, as_stream(stream)),
                     "zero frame_max");
    return kk_gather(reinterpret_cast<const float2 *>(data), p->N, p->M, p->T, p->ltx, p->ltzT,
                     p->lrx, p->lrzT, p->nx, p->nz, p->w, p->fs, p->shift, p->linear, out,
                     out_kind, n_frames, data_frame_stride, out_frame_stride, intensity, frame_max,
                     p->win, as_stream(stream), (flags & KKB_RUN_ACCUMULATE_INTENSITY) ? 1 : 0,
                     nullptr, 0, &sets);
}

extern "C" int kkb_kk_plan_run_scatter(kkb_kk_plan *p, const void *data, int n_frames,
                                       long long data_frame_stride, void *const *dst_host,
                                       int n_dst, long long dst_offset, int out_kind,
                                       long long out_frame_stride, void *stream) {
    if (!p || n_dst < 1 || n_dst > KKB_MAX_DST || !dst_host || dst_offset < 0) {
        set_error("kk_plan_run_scatter: 1 <= n_dst <= %d destinations, offset >= 0", KKB_MAX_DST);
        return KKB_ERR_ARG;
    }
    int st = check_kk_args(p->N, p->M, p->T, p->nx, p->nz, out_kind);
    if (st) return st;
    KKScatter sc{};
    sc.ndst = n_dst;
    sc.dst_off = dst_offset;
    for (int d = 0; d < n_dst; ++d) {
        if (!dst_host[d]) {
            set_error("kk_plan_run_scatter: null destination %d", d);
            return KKB_ERR_ARG;
        }
        sc.dst[d] = dst_host[d];
    }
    return kk_gather(reinterpret_cast<const float2 *>(data), p->N, p->M, p->T, p->ltx, p->ltzT,
                     p->lrx, p->lrzT, p->nx, p->nz, p->w, p->fs, p->shift, p->linear, nullptr,
                     out_kind, n_frames, data_frame_stride, out_frame_stride, nullptr, nullptr,
                     p->win, as_stream(stream), 0, &sc);
}

// ------------------------------------------------------------- CUDA IPC (row-block P2P)
extern "C" int kkb_ipc_alloc(long long bytes, void **ptr) {
    if (bytes <= 0 || !ptr) {
        set_error("ipc_alloc: bad size");
        return KKB_ERR_ARG;
    }
    *ptr = nullptr;
    KKB_TRY_CUDA(cudaMalloc(ptr, (size_t)bytes), "cudaMalloc(ipc buffer)");
    return KKB_OK;
}

extern "C" int kkb_ipc_free(void *ptr) {
    if (ptr) KKB_TRY_CUDA(cudaFree(ptr), "cudaFree(ipc buffer)");
    return KKB_OK;
}

extern "C" int kkb_ipc_get_handle(const void *ptr, void *handle64) {
    if (!ptr || !handle64) return KKB_ERR_ARG;
    cudaIpcMemHandle_t h;
    KKB_TRY_CUDA(cudaIpcGetMemHandle(&h, const_cast<void *>(ptr)), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "CUDA IPC handles are 64 bytes");
    memcpy(handle64, &h, sizeof(h));
    return KKB_OK;
}

extern "C" int kkb_ipc_open_handle(const void *handle64, void **ptr) {
    if (!handle64 || !ptr) return KKB_ERR_ARG;
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    *ptr = nullptr;
    KKB_TRY_CUDA(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return KKB_OK;
}

extern "C" int kkb_ipc_close_handle(void *ptr) {
    if (ptr) KKB_TRY_CUDA(cudaIpcCloseMemHandle(ptr), "cudaIpcCloseMemHandle");
    return KKB_OK;
}

extern "C" int kkb_kk_plan_run(kkb_kk_plan *p, const void *data, int n_frames,
                               long long data_frame_stride, void *out, int out_kind,
                               long long out_frame_stride, float *intensity,
                               unsigned int *frame_max, void *stream) {
    return kkb_kk_plan_run_ex(p, data, n_frames, data_frame_stride, out, out_kind, out_frame_stride,
                              intensity, frame_max, 0, stream);
}

extern "C" int kkb_kk_plan_destroy(kkb_kk_plan *p) {
    if (!p) return KKB_OK;
    cudaFree(p->ltx);
    if (p->win.tc_lo) cudaFree(p->win.tc_lo);
    delete p;
    return KKB_OK;
}

extern "C" int kkb_kk(const void *data, int n_tx, int n_rx, int n_t, const double *ltx,
                      const double *ltz, const double *lrx, const double *lrz, int nx, int nz,
                      const double *weights, double fs, double shift, int linear, void *out,
                      int out_kind, int n_frames, long long data_frame_stride,
                      long long out_frame_stride, float *intensity, unsigned int *frame_max,
                      void *stream) {
    int st = check_kk_args(n_tx, n_rx, n_t, nx, nz, out_kind);
    if (st) return st;
    kkb_kk_plan *p = nullptr;
    st = kkb_kk_plan_create(ltx, ltz, lrx, lrz, n_tx, n_rx, n_t, nx, nz, weights, fs, shift, linear,
                            stream, &p);
    if (st) return st;
    st = kkb_kk_plan_run(p, data, n_frames, data_frame_stride, out, out_kind, out_frame_stride,
                         intensity, frame_max, stream);
    cudaStreamSynchronize(as_stream(stream));
    kkb_kk_plan_destroy(p);
    return st;
}

extern "C" int kkb_kk_taps(const double *ltx, const double *ltz, const double *lrx,
                           const double *lrz, int n_tx, int n_rx, int n_t, int nx, int nz,
                           double fs, double shift, int linear, int *idx, void *stream) {
    int st = check_kk_args(n_tx, n_rx, n_t, nx, nz, KKB_OUT_C64);
    if (st) return st;
    return kk_taps(ltx, ltz, lrx, lrz, n_tx, n_rx, n_t, nx, nz, fs, shift, linear, idx,
                   as_stream(stream));
}

// =====================================================================
// K7
extern "C" int kkb_das(const void *data, int n_tx, int n_el, int n_t, const double *ltx,
                       const double *ltz, const double *hyp, int n_hyp_rows, const long long *base,
                       const double *frac, const double *xcoord, const double *zcoord,
                       const double *upos, double tan_max, const double *weights, double fs,
                       double shift, int linear, int nx, int nz, void *out, int out_kind,
                       void *stream) {
    if (n_tx < 1 || n_el < 1 || n_t < 2 || nx < 1 || nz < 1 || n_hyp_rows < nx) {
        set_error("das: bad sizes");
        return KKB_ERR_ARG;
    }
    if (out_kind != KKB_OUT_C64 && out_kind != KKB_OUT_C128) {
        set_error("das: unknown out_kind %d", out_kind);
        return KKB_ERR_ARG;
    }
    return das_gather(reinterpret_cast<const float2 *>(data), n_tx, n_el, n_t, ltx, ltz, hyp,
                      n_hyp_rows, base, frac, xcoord, zcoord, upos, tan_max, weights, fs, shift,
                      linear, nx, nz, out, out_kind, as_stream(stream));
}

// =====================================================================
// K1/K3: analytic_signal
extern "C" int kkb_analytic_signal(const float *rf, long long n_traces, int n_t, void *out,
                                   void *stream) {
    if (n_traces < 0 || n_t < 1 || n_t > KKB_FFT_MAX_T_TOTAL) {
        set_error("analytic_signal: unsupported T=%d", n_t);
        return n_t > KKB_FFT_MAX_T_TOTAL ? KKB_ERR_UNSUPPORTED : KKB_ERR_ARG;
    }
    if (n_traces == 0) return KKB_OK;
    cudaStream_t s = as_stream(stream);
    const int T = n_t, K = T / 2 + 1;
    std::vector<float> sc(K);
    for (int k = 0; k < K; ++k) sc[k] = (float)(one_sided(k, T) / T);
    FftPlan plan;
    int st = get_fft_plan(T, &plan);
    if (st) return st;
    Scratch spec(s), scale(s), promo(s);
    if ((st = spec.alloc(sizeof(float2) * (size_t)n_traces * K))) return st;
    if ((st = scale.alloc(sizeof(float) * K))) return st;
    KKB_TRY_CUDA(cudaMemcpyAsync(scale.p, sc.data(), sizeof(float) * K, cudaMemcpyHostToDevice, s),
                 "copy weights");
    float2 *X = (float2 *)spec.p;
    if (plan.direct || plan.large) {
        if ((st = promo.alloc(sizeof(float2) * (size_t)n_traces * T))) return st;
        if ((st = fft_r2c(rf, n_traces, T, X, K, K, nullptr, s, (float2 *)promo.p))) return st;
        long long total = n_traces * K;
        k_scale_bins<<<(unsigned)std::min<long long>(ceil_div(total, 256), 4096), 256, 0, s>>>(
            X, n_traces, K, K, (const float *)scale.p);
        KKB_CHECK_LAUNCH("k_scale_bins");
    } else {
        if ((st = fft_r2c(rf, n_traces, T, X, K, K, (const float *)scale.p, s, nullptr))) return st;
    }
    st = fft_c2c(X, K, K, (float2 *)out, T, T, n_traces, T, true, 1.0f, s);
    cudaStreamSynchronize(s);  // host weights vector dies here
    return st;
}

// =====================================================================
// K1-K3: shear_and_sum on complex input, all T bins
struct kkb_shear_plan {
    int L, M, T;
    float2 *ramps;  // (M, L, T): exp(2 pi i f_k u_l sin(theta_m) / c) / T, float64-built
};

extern "C" int kkb_shear_plan_create(const double *positions_host, const double *angles_host, int n_el,
                                     int n_rx, int n_t, double fs, double c, kkb_shear_plan **out) {
    if (!out || n_el < 1 || n_rx < 1 || n_t < 1 || n_t > KKB_FFT_MAX_T_TOTAL || !(c > 0)) {
        set_error("shear_plan: bad sizes");
        return KKB_ERR_ARG;
    }
    const int T = n_t;
    std::vector<double> tau((size_t)n_el * n_rx), freq(T), scale(T, 1.0 / T);
    for (int m = 0; m < n_rx; ++m) {
        double q = sin(angles_host[m]) / c;  // compress.py:79  positions * (sin(theta) / c)
        for (int l = 0; l < n_el; ++l) tau[(size_t)l * n_rx + m] = positions_host[l] * q;
    }
    for (int k = 0; k < T; ++k) freq[k] = fftfreq(k, T, fs);
    kkb_shear_plan *p = new (std::nothrow) kkb_shear_plan();
    if (!p) return KKB_ERR_NOMEM;
    p->L = n_el;
    p->M = n_rx;
    p->T = T;
    cudaError_t e = cudaMalloc(&p->ramps, sizeof(float2) * (size_t)n_rx * n_el * T);
    if (e != cudaSuccess) {
        delete p;
        return cuda_status(e, "cudaMalloc(shear ramps)");
    }
    int st = build_ramps(tau.data(), n_el, n_rx, freq.data(), scale.data(), T, p->ramps, 0);
    if (st) {
        cudaFree(p->ramps);
        delete p;
        return st;
    }
    *out = p;
    return KKB_OK;
}

extern "C" int kkb_shear_plan_run(kkb_shear_plan *p, const void *data, int n_tx, void *out, void *stream) {
    if (!p || n_tx < 1) {
        set_error("shear_plan_run: bad plan or transmit count");
        return KKB_ERR_ARG;
    }
    cudaStream_t s = as_stream(stream);
    const int T = p->T, L = p->L, M = p->M;
    const long long ntr = (long long)n_tx * L;
    Scratch xs(s), ys(s);
    int st;
    if ((st = xs.alloc(sizeof(float2) * (size_t)ntr * T))) return st;
    if ((st = ys.alloc(sizeof(float2) * (size_t)n_tx * M * T))) return st;
    float2 *X = (float2 *)xs.p, *Y = (float2 *)ys.p;
    if ((st = fft_c2c((const float2 *)data, T, T, X, T, T, ntr, T, false, 1.0f, s))) return st;
    if ((st = contract(X, T, p->ramps, T, Y, T, n_tx, L, M, T, s))) return st;
    return fft_c2c(Y, T, T, (float2 *)out, T, T, (long long)n_tx * M, T, true, 1.0f, s);
}

extern "C" int kkb_shear_plan_destroy(kkb_shear_plan *p) {
    if (!p) return KKB_OK;
    cudaFree(p->ramps);
    delete p;
    return KKB_OK;
}

extern "C" int kkb_shear_and_sum(const void *data, int n_tx, int n_el, int n_t,
                                 const double *positions_host, const double *angles_host, int n_rx,
                                 double fs, double c, void *out, void *stream) {
    if (n_tx < 1 || n_el < 1 || n_rx < 1 || n_t < 1 || n_t > KKB_FFT_MAX_T_TOTAL || !(c > 0)) {
        set_error("shear_and_sum: bad sizes");
        return KKB_ERR_ARG;
    }
    kkb_shear_plan *p = nullptr;
    int st = kkb_shear_plan_create(positions_host, angles_host, n_el, n_rx, n_t, fs, c, &p);
    if (st) return st;
    st = kkb_shear_plan_run(p, data, n_tx, out, stream);
    cudaStreamSynchronize(as_stream(stream));
    kkb_shear_plan_destroy(p);
    return st;
}

#define KKB_RING_TILE_ROWS 16  // rows of one contraction tile (k_contract_sym<6, 2>)

// =====================================================================
// fused stage-1 plan
struct kkb_decomposer {
    int N, L, T, M, K, ldk, chunk;  // ldk: spectral row stride (K rounded up to even)
    double fs = 0.0;
    float2 *ramps = nullptr;
    float2 *X = nullptr;            // slots x chunk frames of spectra
    float2 *Y = nullptr;            // slots x chunk frames of contracted bins
    long long bytes = 0;
    // pipelined mode (kkb_decomposer_set_pipeline): chunks rotate over `slots`
    // streams so one chunk's FFT overlaps the previous chunk's contraction and
    // its spectra are consumed while still L2-resident
    int slots = 1;
    cudaStream_t st[4] = {};
    cudaEvent_t ev[5] = {};
    // symmetric contraction (k_contract_sym): P > 0 classes when the element
    // positions are centred (pos[L-1-l] == -pos[l]) and every receive angle has
    // an exact negative partner (or is 0) — always true for the reference's
    // TransducerArray / ReceiveAngleSet.  cs = (P, ceil(L/2), ldk) cos/sin table.
    int P = 0;
    float2 *cs = nullptr;
    std::vector<short> mp, mm;
    // tensor-core contraction (k_contract_tc, kkb_decomposer_set_contraction):
    // 3xTF32 class tables in the UMMA operand layout, built on first use
    int form = KKB_CONTRACT_FMA;
    float *tctab = nullptr;
    // fused stage 1 (stage1_fused.cu, kkb_decomposer_set_fused): K1 + K2 in one
    // kernel for a uniform symmetric array
    int s1f_ok = 0, s1f_on = 0;
    float2 *s1f_gam = nullptr;  // (P, L/8 + 1) split phase slopes (stage1_fused_table)
    // stage-1 ring mode (kkb_decomposer_set_ring): K1 and a persistent K2 run
    // concurrently, the spectra passing through R L2-resident row-tile slots
    int ring_R = 0, ring_ctas = 0;
    float2 *ring = nullptr;
    int *ring_cnt = nullptr;  // fft_done[tiles] | con_done[tiles] | queue | started | err
    long long ring_tiles = 0;
    cudaStream_t ring_side = nullptr;
    cudaEvent_t ring_ev[2] = {};
};

// Pair receive angles into +/- classes and build the cos/sin table; P = 0
// (general contraction) when the geometry is not symmetric or KKB_NO_SYM=1.
static int build_symmetric_classes(kkb_decomposer *p, const double *pos, const double *ang,
                                   double c, const std::vector<double> &freq,
                                   const std::vector<double> &scale) {
    const char *env = getenv("KKB_NO_SYM");
    if (env && env[0] == '1') return KKB_OK;
    const int L = p->L, M = p->M;
    for (int l = 0; l < L; ++l)
        if (pos[L - 1 - l] != -pos[l]) return KKB_OK;
    std::vector<int> used(M, 0);
    std::vector<short> mp, mm;
    for (int m = 0; m < M; ++m) {
        if (used[m] || ang[m] < 0) continue;
        used[m] = 1;
        if (ang[m] == 0.0) {
            mp.push_back((short)m);
            mm.push_back(-1);
            continue;
        }
        int partner = -1;
        for (int q = 0; q < M && partner < 0; ++q)
            if (!used[q] && ang[q] == -ang[m]) partner = q;
        if (partner < 0) return KKB_OK;
        used[partner] = 1;
        mp.push_back((short)m);
        mm.push_back((short)partner);
    }
    for (int m = 0; m < M; ++m)
        if (!used[m]) return KKB_OK;
    const int P = (int)mp.size(), Lp = (L + 1) / 2;
    if (P > KKB_MAX_CLASSES) return KKB_OK;
    std::vector<double> tau((size_t)Lp * P);
    for (int q = 0; q < P; ++q) {
        const double s = sin(ang[mp[q]]) / c;  // compress.py:79 order: positions * (sin/c)
        for (int j = 0; j < Lp; ++j) tau[(size_t)j * P + q] = pos[j] * s;
    }
    KKB_TRY_CUDA(cudaMalloc(&p->cs, sizeof(float2) * (size_t)P * Lp * p->ldk), "cudaMalloc(cs)");
    int st = build_ramps(tau.data(), Lp, P, freq.data(), scale.data(), p->ldk, p->cs, 0);
    if (st) return st;
    p->P = P;
    p->mp = mp;
    p->mm = mm;
    p->bytes += (long long)(sizeof(float2) * (size_t)P * Lp * p->ldk);
    // fused stage 1: needs a uniform array (the phase is linear in the element
    // index) and a length / class count the kernel is built for
    if (stage1_fused_supported(p->T, L, P)) {
        const double step = (pos[L - 1] - pos[0]) / (L - 1);
        bool uniform = step > 0;
        for (int l = 0; l + 1 < L && uniform; ++l)
            uniform = fabs((pos[l + 1] - pos[l]) - step) <= 1e-9 * step;
        if (uniform) {
            const int Lh = L / 2;
            std::vector<double> t((size_t)P * (Lh + 1));
            for (int q = 0; q < P; ++q) {
                for (int j = 0; j < Lh; ++j) t[(size_t)q * (Lh + 1) + j] = tau[(size_t)j * P + q];
                t[(size_t)q * (Lh + 1) + Lh] = step * (sin(ang[mp[q]]) / c);
            }
            std::vector<float2> gam;
            stage1_fused_table(t.data(), P, L, 1.0 / (p->T * (1.0 / p->fs)), gam);  // fftfreq's bin spacing
            KKB_TRY_CUDA(cudaMalloc(&p->s1f_gam, sizeof(float2) * gam.size()), "cudaMalloc(s1f table)");
            KKB_TRY_CUDA(cudaMemcpy(p->s1f_gam, gam.data(), sizeof(float2) * gam.size(), cudaMemcpyHostToDevice),
                         "copy s1f table");
            p->bytes += (long long)(sizeof(float2) * gam.size());
            p->s1f_ok = 1;
            // opt-in: measured slower than K1 -> K2 at config 4
            const char *e = getenv("KKB_S1_FUSED");
            p->s1f_on = e && e[0] == '1';
        }
    }
    return KKB_OK;
}

extern "C" int kkb_decomposer_create(int n_tx, int n_el, int n_t, const double *positions_host,
                                     const double *angles_host, int n_rx, double fs, double c,
                                     int max_frames, kkb_decomposer **out) {
    if (n_tx < 1 || n_el < 1 || n_rx < 1 || n_t < 2 || n_t > KKB_FFT_MAX_T_TOTAL || max_frames < 1 ||
        !(c > 0)) {
        set_error("decomposer: bad sizes");
        return KKB_ERR_ARG;
    }
    FftPlan plan;
    int st = get_fft_plan(n_t, &plan);
    if (st) return st;
    (void)plan;  // lengths without a single-CTA plan are promoted to complex per pass (run)
    kkb_decomposer *p = new (std::nothrow) kkb_decomposer();
    if (!p) return KKB_ERR_NOMEM;
    p->N = n_tx;
    p->L = n_el;
    p->T = n_t;
    p->M = n_rx;
    p->K = n_t / 2 + 1;
    p->ldk = p->K + (p->K & 1);
    p->chunk = max_frames;
    p->fs = fs;
    const int K = p->K, ldk = p->ldk;
    std::vector<double> tau((size_t)n_el * n_rx), freq(K), scale(K);
    for (int m = 0; m < n_rx; ++m) {
        double q = sin(angles_host[m]) / c;
        for (int l = 0; l < n_el; ++l) tau[(size_t)l * n_rx + m] = positions_host[l] * q;
    }
    for (int k = 0; k < K; ++k) {
        freq[k] = fftfreq(k, n_t, fs);
        scale[k] = one_sided(k, n_t) / n_t;
    }
    size_t rb = sizeof(float2) * (size_t)n_rx * n_el * ldk;
    size_t xb = sizeof(float2) * (size_t)max_frames * n_tx * n_el * ldk;
    size_t yb = sizeof(float2) * (size_t)max_frames * n_tx * n_rx * ldk;
    cudaError_t e;
    if ((e = cudaMalloc(&p->ramps, rb)) || (e = cudaMalloc(&p->X, xb)) || (e = cudaMalloc(&p->Y, yb))) {
        cudaFree(p->ramps);
        cudaFree(p->X);
        cudaFree(p->Y);
        delete p;
        return cuda_status(e, "cudaMalloc(decomposer)");
    }
    p->bytes = (long long)(rb + xb + yb);
    // ramps at row stride ldk: build K bins (+1 zero pad bin when K is odd)
    freq.resize(ldk, 0.0);
    scale.resize(ldk, 0.0);
    st = build_ramps(tau.data(), n_el, n_rx, freq.data(), scale.data(), ldk, p->ramps, 0);
    if (!st) st = build_symmetric_classes(p, positions_host, angles_host, c, freq, scale);
    if (!st) {  // KKB_CONTRACT=tc: tensor-core contraction by default (falls back if unsupported)
        const char *f = getenv("KKB_CONTRACT");
        if (f && !strcmp(f, "tc") && p->P >= 1 && p->P <= 16)
            st = kkb_decomposer_set_contraction(p, KKB_CONTRACT_TENSOR);
    }
    if (!st) {  // KKB_S1_RING=R[,ctas]: stage-1 ring mode by default
        if (const char *r = getenv("KKB_S1_RING")) {
            int R = atoi(r), ctas = 0;
            if (const char *c2 = strchr(r, ',')) ctas = atoi(c2 + 1);
            if (R >= 2) st = kkb_decomposer_set_ring(p, R, ctas);
        }
    }
    if (st) {
        cudaFree(p->ramps);
        cudaFree(p->X);
        cudaFree(p->Y);
        cudaFree(p->cs);
        cudaFree(p->s1f_gam);
        delete p;
        return st;
    }
    *out = p;
    return KKB_OK;
}

extern "C" int kkb_decomposer_symmetric_classes(const kkb_decomposer *p) { return p ? p->P : -1; }

extern "C" int kkb_decomposer_set_contraction(kkb_decomposer *p, int form) {
    if (!p || (form != KKB_CONTRACT_FMA && form != KKB_CONTRACT_TENSOR)) {
        set_error("set_contraction: form must be KKB_CONTRACT_FMA or KKB_CONTRACT_TENSOR");
        return KKB_ERR_ARG;
    }
    if (form == KKB_CONTRACT_TENSOR) {
        if (p->P < 1 || p->P > 16) {
            set_error("tensor-core contraction needs a symmetric geometry with 1..16 angle classes (P=%d)", p->P);
            return KKB_ERR_UNSUPPORTED;
        }
        if (!p->tctab) {
            long long bytes = 0;
            int st = build_tc_table(p->cs, p->ldk, p->P, p->L, p->K, &p->tctab, &bytes, 0);
            if (st) return st;
            KKB_TRY_CUDA(cudaStreamSynchronize(0), "sync tc table");
            p->bytes += bytes;
        }
    }
    p->form = form;
    return KKB_OK;
}

extern "C" int kkb_decomposer_contraction(const kkb_decomposer *p) { return p ? p->form : -1; }

extern "C" int kkb_decomposer_set_fused(kkb_decomposer *p, int on) {
    if (!p || (on != 0 && on != 1)) return KKB_ERR_ARG;
    if (on && !p->s1f_ok) {
        set_error("fused stage 1 needs T = 1536, L a multiple of 8, a uniform symmetric array and <= 6 angle classes");
        return KKB_ERR_UNSUPPORTED;
    }
    p->s1f_on = on;
    return KKB_OK;
}

extern "C" int kkb_decomposer_fused(const kkb_decomposer *p) { return p ? (p->s1f_ok && p->s1f_on) : -1; }

// the fused stage-1 kernel runs instead of K1 -> K2 (FMA form, no ring)
static bool use_s1f(const kkb_decomposer *p) { return p->s1f_ok && p->s1f_on && p->form == KKB_CONTRACT_FMA; }

extern "C" int kkb_decomposer_set_ring(kkb_decomposer *p, int slots, int consumer_ctas) {
    if (!p || slots < 0 || slots == 1 || consumer_ctas < 0) {
        set_error("set_ring: slots 0 (off) or >= 2, consumer_ctas >= 0");
        return KKB_ERR_ARG;
    }
    KKB_TRY_CUDA(cudaDeviceSynchronize(), "sync before ring realloc");
    cudaFree(p->ring);
    p->ring = nullptr;
    p->ring_R = 0;
    if (slots == 0) return KKB_OK;
    const size_t bytes = sizeof(float2) * (size_t)slots * KKB_RING_TILE_ROWS * p->L * p->ldk;
    KKB_TRY_CUDA(cudaMalloc(&p->ring, bytes), "cudaMalloc(ring)");
    if (!p->ring_side) {
        KKB_TRY_CUDA(cudaStreamCreateWithFlags(&p->ring_side, cudaStreamNonBlocking), "ring stream");
        for (int i = 0; i < 2; ++i)
            KKB_TRY_CUDA(cudaEventCreateWithFlags(&p->ring_ev[i], cudaEventDisableTiming), "ring event");
    }
    p->ring_R = slots;
    // consumers must leave every SM room for K1 (a consumer CTA takes half an
    // SM's registers): at most one per SM
    p->ring_ctas = std::min(consumer_ctas > 0 ? consumer_ctas : sm_count() / 2, sm_count());
    return KKB_OK;
}

extern "C" int kkb_decomposer_ring_error(kkb_decomposer *p, int *flag) {
    if (!p || !flag) return KKB_ERR_ARG;
    *flag = 0;
    if (!p->ring_cnt) return KKB_OK;
    KKB_TRY_CUDA(cudaDeviceSynchronize(), "sync ring error");
    unsigned e = 0;
    KKB_TRY_CUDA(cudaMemcpy(&e, p->ring_cnt + 2 * p->ring_tiles + 2, sizeof(e), cudaMemcpyDeviceToHost), "read ring error");
    *flag = (int)e;
    return KKB_OK;
}

extern "C" long long kkb_decomposer_workspace_bytes(const kkb_decomposer *p) { return p ? p->bytes : 0; }

// exact int16 -> float32 widening (the reference consumes q.astype(float32))
__global__ void k_i16_to_f32(const short *__restrict__ in, long long n, float *__restrict__ out) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        out[i] = (float)in[i];
}

__global__ void k_wait_started(const int *started, unsigned *err) {
    if (threadIdx.x == 0) ring_wait_geq(started, 1, err);
}

// K1 -> K2 through the L2 ring for F frames (one pass), then K3 on `s`.
static int decomposer_run_ring(kkb_decomposer *p, const void *rf_c, int in_kind, int F, float2 *tr_c,
                               cudaStream_t s) {
    const int N = p->N, L = p->L, T = p->T, M = p->M, K = p->K, ldk = p->ldk;
    const long long B = (long long)F * N;
    const long long tiles = (B + KKB_RING_TILE_ROWS - 1) / KKB_RING_TILE_ROWS;
    if (tiles > p->ring_tiles) {
        cudaFree(p->ring_cnt);
        p->ring_cnt = nullptr;
        KKB_TRY_CUDA(cudaMalloc(&p->ring_cnt, sizeof(int) * (size_t)(2 * tiles + 3)), "cudaMalloc(ring counters)");
        p->ring_tiles = tiles;
    }
    int *fft_done = p->ring_cnt, *con_done = p->ring_cnt + tiles, *queue = con_done + tiles, *started = queue + 1;
    unsigned *err = reinterpret_cast<unsigned *>(started + 1);
    KKB_TRY_CUDA(cudaMemsetAsync(p->ring_cnt, 0, sizeof(int) * (size_t)(2 * tiles + 3), s), "zero ring counters");
    Stage1Ring rs;
    rs.fft_done = fft_done;
    rs.con_done = con_done;
    rs.R = p->ring_R;
    rs.con_per_tile = (K + 31) / 32;
    rs.traces_per_tile = (long long)KKB_RING_TILE_ROWS * L;
    rs.err = err;
    FftPlan plan;
    int st = get_fft_plan(T, &plan);
    if (st) return st;
    float2 *Y = p->Y;
    // the persistent consumer first (side stream), K1 once it is resident
    KKB_TRY_CUDA(cudaEventRecord(p->ring_ev[0], s), "record ring fork");
    KKB_TRY_CUDA(cudaStreamWaitEvent(p->ring_side, p->ring_ev[0], 0), "wait ring fork");
    st = contract_sym_ring(p->ring, ldk, p->cs, ldk, Y, ldk, B, L, M, K, p->P, p->mp.data(), p->mm.data(), rs,
                           queue, started, p->ring_ctas, p->ring_side);
    if (st) return st;
    k_wait_started<<<1, 32, 0, s>>>(started, err);
    KKB_CHECK_LAUNCH("k_wait_started");
    st = fft_r2c_ct_ring(rf_c, in_kind, B * L, T, p->ring, ldk, K, nullptr, plan.tws, s, rs);
    if (st) return st;
    KKB_TRY_CUDA(cudaEventRecord(p->ring_ev[1], p->ring_side), "record ring join");
    KKB_TRY_CUDA(cudaStreamWaitEvent(s, p->ring_ev[1], 0), "wait ring join");
    return fft_c2c(Y, ldk, K, tr_c, T, T, B * M, T, true, 1.0f, s);
}

static int decomposer_run(kkb_decomposer *p, const void *rf, int in_kind, int n_frames,
                          void *traces, void *stream, const RowScatter *scatter = nullptr) {
    if (!p || n_frames < 0) return KKB_ERR_ARG;
    cudaStream_t s = as_stream(stream);
    const int N = p->N, L = p->L, T = p->T, M = p->M, K = p->K, ldk = p->ldk;
    // int16 RF: converted exactly inside the compile-time real FFT's load; other
    // lengths convert each chunk to float32 first (k_i16_to_f32)
    const bool i16_direct = in_kind && fft_ct_supported(T);
    const size_t esz = in_kind ? sizeof(short) : sizeof(float);
    FftPlan plan;
    int st = get_fft_plan(T, &plan);
    if (st) return st;
    const bool piped = p->slots > 1 && n_frames > p->chunk;
    if (piped) {  // fork: slot streams wait for work already queued on the caller stream
        KKB_TRY_CUDA(cudaEventRecord(p->ev[4], s), "record fork");
        for (int i = 0; i < p->slots; ++i)
            KKB_TRY_CUDA(cudaStreamWaitEvent(p->st[i], p->ev[4], 0), "wait fork");
    }
    const size_t xslot = (size_t)p->chunk * N * L * ldk, yslot = (size_t)p->chunk * N * M * ldk;
    int ci = 0;
    for (int f0 = 0; f0 < n_frames; f0 += p->chunk, ++ci) {
        const int slot = piped ? ci % p->slots : 0;
        cudaStream_t cs = piped ? p->st[slot] : s;
        float2 *X = p->X + slot * xslot, *Y = p->Y + slot * yslot;
        int F = std::min(p->chunk, n_frames - f0);
        const char *rf_c = (const char *)rf + (size_t)f0 * N * L * T * esz;
        float2 *tr_c = (float2 *)traces + (size_t)f0 * N * M * T;
        float *conv = nullptr;
        if (in_kind && !i16_direct) {
            const long long n = (long long)F * N * L * T;
            KKB_TRY_CUDA(cudaMallocAsync(&conv, sizeof(float) * (size_t)n, cs), "cudaMallocAsync(i16 convert)");
            k_i16_to_f32<<<(unsigned)std::min<long long>(ceil_div(n, 256), 148 * 32), 256, 0, cs>>>(
                (const short *)rf_c, n, conv);
            KKB_CHECK_LAUNCH("k_i16_to_f32");
            rf_c = (const char *)conv;
        }
        if (p->ring_R > 0 && !scatter && !piped && !(in_kind && !i16_direct) && fft_ct_supported(T) &&
            !(L & 1) && p->P >= 1 && p->P <= 6 && p->form == KKB_CONTRACT_FMA) {
            if ((st = decomposer_run_ring(p, rf_c, in_kind, F, tr_c, cs))) return st;
            continue;
        }
        if (use_s1f(p) && (in_kind == 0 || i16_direct)) {
            st = stage1_fused(rf_c, in_kind, (long long)F * N, L, T, p->s1f_gam, Y, ldk, M, p->P,
                              p->mp.data(), p->mm.data(), plan.tws, cs);
        } else if (i16_direct) {
            st = fft_r2c_ct(rf_c, 1, (long long)F * N * L, T, X, ldk, K, nullptr, plan.tws, cs, L);
        } else if (plan.direct || plan.large) {
            // lengths without a single-CTA real plan: promote to complex first
            float2 *promo = nullptr;
            KKB_TRY_CUDA(cudaMallocAsync(&promo, sizeof(float2) * (size_t)F * N * L * T, cs),
                         "cudaMallocAsync(promote)");
            st = fft_r2c((const float *)rf_c, (long long)F * N * L, T, X, ldk, K, nullptr, cs, promo, L);
            cudaFreeAsync(promo, cs);
        } else {
            st = fft_r2c((const float *)rf_c, (long long)F * N * L, T, X, ldk, K, nullptr, cs,
                         nullptr, L);
        }
        if (conv) cudaFreeAsync(conv, cs);
        if (st) return st;
        if (use_s1f(p) && (in_kind == 0 || i16_direct))
            st = KKB_OK;  // Y written by the fused kernel
        else if (p->form == KKB_CONTRACT_TENSOR)
            st = contract_tc(X, ldk, p->tctab, Y, ldk, (long long)F * N, L, M, K, p->P, p->mp.data(),
                             p->mm.data(), cs);
        else if (p->P > 0)
            st = contract_sym(X, ldk, p->cs, ldk, Y, ldk, (long long)F * N, L, M, K, p->P,
                              p->mp.data(), p->mm.data(), cs);
        else
            st = contract(X, ldk, p->ramps, ldk, Y, ldk, (long long)F * N, L, M, K, cs);
        if (st) return st;
        if (scatter) {  // fused all-gather: rows land in every rank's full trace buffer
            RowScatter sc = *scatter;
            sc.off += (long long)f0 * sc.frame_stride;
            sc.rows_per_frame = N * M;
            st = fft_c2c_scatter(Y, ldk, K, T, (long long)F * N * M, T, true, 1.0f, sc, cs);
        } else {
            st = fft_c2c(Y, ldk, K, tr_c, T, T, (long long)F * N * M, T, true, 1.0f, cs);
        }
        if (st) return st;
    }
    if (piped) {  // join
        for (int i = 0; i < p->slots; ++i) {
            KKB_TRY_CUDA(cudaEventRecord(p->ev[i], p->st[i]), "record join");
            KKB_TRY_CUDA(cudaStreamWaitEvent(s, p->ev[i], 0), "wait join");
        }
    }
    return KKB_OK;
}

// One stage of the plan's stage 1 at a time, for the reference's staged
// benchmark (bench.py:113-153 reorg_fft / hilbert_compress / ifft): stage 0
// real FFT of rf into the plan's spectra, 1 contraction (one-sided weights
// folded into the ramps) into its contracted bins, 2 inverse FFT to traces.
// The stages are the three-kernel path's own launches (same results as
// kkb_decomposer_run); n_frames <= the plan's frames per pass.
extern "C" int kkb_decomposer_run_stage(kkb_decomposer *p, int stage, const float *rf, int n_frames,
                                        void *traces, void *stream) {
    if (!p || n_frames < 0 || stage < 0 || stage > 2) return KKB_ERR_ARG;
    if (n_frames > p->chunk) {
        set_error("decomposer stage: %d frames exceed the plan's %d per pass", n_frames, p->chunk);
        return KKB_ERR_ARG;
    }
    if (n_frames == 0) return KKB_OK;
    cudaStream_t s = as_stream(stream);
    const int N = p->N, L = p->L, T = p->T, M = p->M, K = p->K, ldk = p->ldk;
    FftPlan plan;
    int st = get_fft_plan(T, &plan);
    if (st) return st;
    const long long F = n_frames;
    if (stage == 0) {
        if (!rf) return KKB_ERR_ARG;
        if (plan.direct || plan.large) {
            float2 *promo = nullptr;
            KKB_TRY_CUDA(cudaMallocAsync(&promo, sizeof(float2) * (size_t)F * N * L * T, s), "cudaMallocAsync(promote)");
            st = fft_r2c(rf, F * N * L, T, p->X, ldk, K, nullptr, s, promo, L);
            cudaFreeAsync(promo, s);
            return st;
        }
        return fft_r2c(rf, F * N * L, T, p->X, ldk, K, nullptr, s, nullptr, L);
    }
    if (stage == 1) {
        if (p->form == KKB_CONTRACT_TENSOR)
            return contract_tc(p->X, ldk, p->tctab, p->Y, ldk, F * N, L, M, K, p->P, p->mp.data(), p->mm.data(), s);
        if (p->P > 0)
            return contract_sym(p->X, ldk, p->cs, ldk, p->Y, ldk, F * N, L, M, K, p->P, p->mp.data(),
                                p->mm.data(), s);
        return contract(p->X, ldk, p->ramps, ldk, p->Y, ldk, F * N, L, M, K, s);
    }
    if (!traces) return KKB_ERR_ARG;
    return fft_c2c(p->Y, ldk, K, (float2 *)traces, T, T, F * N * M, T, true, 1.0f, s);
}

// One stage of analytic_signal (spectral.py:84-93) at a time, for the
// reference's staged DAS benchmark (bench.py:91-110): stage 0 real FFT of the
// rows into spec ((n_traces, T/2 + 1) complex64, caller scratch), 1 the
// one-sided weights / T on spec in place, 2 inverse FFT of spec into out
// ((n_traces, T) complex64).  Stages 0 + 1 + 2 equal kkb_analytic_signal.
extern "C" int kkb_analytic_signal_stage(int stage, const float *rf, long long n_traces, int n_t, void *spec,
                                         void *out, void *stream) {
    if (n_traces < 0 || n_t < 1 || n_t > KKB_FFT_MAX_T_TOTAL || stage < 0 || stage > 2 || !spec) {
        set_error("analytic_signal_stage: bad arguments (stage %d, T=%d)", stage, n_t);
        return n_t > KKB_FFT_MAX_T_TOTAL ? KKB_ERR_UNSUPPORTED : KKB_ERR_ARG;
    }
    if (n_traces == 0) return KKB_OK;
    cudaStream_t s = as_stream(stream);
    const int T = n_t, K = T / 2 + 1;
    FftPlan plan;
    int st = get_fft_plan(T, &plan);
    if (st) return st;
    float2 *X = (float2 *)spec;
    if (stage == 0) {
        if (!rf) return KKB_ERR_ARG;
        if (plan.direct || plan.large) {
            Scratch promo(s);
            if ((st = promo.alloc(sizeof(float2) * (size_t)n_traces * T))) return st;
            return fft_r2c(rf, n_traces, T, X, K, K, nullptr, s, (float2 *)promo.p);
        }
        return fft_r2c(rf, n_traces, T, X, K, K, nullptr, s, nullptr);
    }
    if (stage == 1) {
        // one-sided weights / T per length, built once per process (device
        // tables, kept for the process lifetime: a staged benchmark calls this
        // per repetition)
        static std::mutex mu;
        static std::map<std::pair<int, int>, float *> tables;  // (device, T) -> weights
        int devid = 0;
        KKB_TRY_CUDA(cudaGetDevice(&devid), "get device");
        float *w = nullptr;
        {
            std::lock_guard<std::mutex> lock(mu);
            auto it = tables.find({devid, T});
            if (it != tables.end()) {
                w = it->second;
            } else {
                std::vector<float> sc(K);
                for (int k = 0; k < K; ++k) sc[k] = (float)(one_sided(k, T) / T);
                KKB_TRY_CUDA(cudaMalloc(&w, sizeof(float) * K), "cudaMalloc(one-sided weights)");
                KKB_TRY_CUDA(cudaMemcpy(w, sc.data(), sizeof(float) * K, cudaMemcpyHostToDevice), "copy weights");
                tables[{devid, T}] = w;
            }
        }
        const long long total = n_traces * K;
        k_scale_bins<<<(unsigned)std::min<long long>(ceil_div(total, 256), 4096), 256, 0, s>>>(X, n_traces, K, K, w);
        KKB_CHECK_LAUNCH("k_scale_bins");
        return KKB_OK;
    }
    if (!out) return KKB_ERR_ARG;
    return fft_c2c(X, K, K, (float2 *)out, T, T, n_traces, T, true, 1.0f, s);
}

extern "C" long long kkb_tc_planes_bytes(int n_frames, int pairs, int n_t) {
    if (n_frames < 0 || pairs < 0 || n_t < 0) return -1;
    return 4LL * 2 * ((n_frames + 7) / 8) * 8 * (long long)pairs * n_t;
}

// Stage 1 emitting the tensor-core gather's split planes (K1, K2, the frame
// bounds, K3 into planes; traces written only for a batch with a non-finite
// bin).  One pass: n_frames <= the plan's frames per pass.
extern "C" int kkb_decomposer_run_planes(kkb_decomposer *p, const float *rf, int n_frames, void *planes,
                                         unsigned *fbound, unsigned *nonfinite, void *traces, void *stream) {
    if (!p || !rf || !planes || !fbound || !nonfinite || !traces || n_frames < 0) return KKB_ERR_ARG;
    if (n_frames > p->chunk) {
        set_error("decomposer planes: %d frames exceed the plan's %d per pass", n_frames, p->chunk);
        return KKB_ERR_ARG;
    }
    if (!(p->T == 1024 || p->T == 1536 || p->T == 2048)) {
        set_error("decomposer planes: T = %d (1024, 1536 or 2048)", p->T);
        return KKB_ERR_UNSUPPORTED;
    }
    cudaStream_t s = as_stream(stream);
    KKB_TRY_CUDA(cudaMemsetAsync(fbound, 0, sizeof(unsigned) * (size_t)n_frames, s), "zero frame bounds");
    KKB_TRY_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(unsigned), s), "zero flag");
    if (n_frames == 0) return KKB_OK;
    int st;
    FftPlan plan;
    if ((st = get_fft_plan(p->T, &plan))) return st;
    if (use_s1f(p)) {
        if ((st = stage1_fused(rf, 0, (long long)n_frames * p->N, p->L, p->T, p->s1f_gam, p->Y, p->ldk,
                               p->M, p->P, p->mp.data(), p->mm.data(), plan.tws, s)))
            return st;
    } else {
        if ((st = kkb_decomposer_run_stage(p, 0, rf, n_frames, nullptr, stream))) return st;
        if ((st = kkb_decomposer_run_stage(p, 1, rf, n_frames, nullptr, stream))) return st;
    }
    const long long rows = (long long)n_frames * p->N * p->M;
    if ((st = frame_bound(p->Y, p->ldk, p->K, rows, p->N * p->M, 1.0f, fbound, nonfinite, s))) return st;
    return fft_c2c_planes(p->Y, p->ldk, p->K, p->T, n_frames, p->N * p->M, 1.0f, plan.tws, fbound, nonfinite,
                          (float2 *)traces, (__half *)planes, s);
}

// Pipelined mode: `chunk_frames` per pass, passes rotated over `slots` (1..4)
// streams; reallocates the plan's scratch (slots x chunk frames).
extern "C" int kkb_decomposer_set_pipeline(kkb_decomposer *p, int chunk_frames, int slots) {
    if (!p || chunk_frames < 1 || slots < 1 || slots > 4) {
        set_error("set_pipeline: chunk >= 1, 1 <= slots <= 4");
        return KKB_ERR_ARG;
    }
    KKB_TRY_CUDA(cudaDeviceSynchronize(), "sync before realloc");
    const size_t xb = sizeof(float2) * (size_t)slots * chunk_frames * p->N * p->L * p->ldk;
    const size_t yb = sizeof(float2) * (size_t)slots * chunk_frames * p->N * p->M * p->ldk;
    float2 *X = nullptr, *Y = nullptr;
    cudaError_t e;
    if ((e = cudaMalloc(&X, xb)) || (e = cudaMalloc(&Y, yb))) {
        cudaFree(X);
        return cuda_status(e, "cudaMalloc(decomposer pipeline)");
    }
    cudaFree(p->X);
    cudaFree(p->Y);
    p->X = X;
    p->Y = Y;
    p->bytes = (long long)(sizeof(float2) * (size_t)p->M * p->L * p->ldk + xb + yb);
    for (int i = p->slots; i < slots; ++i) {
        if (i == 0) continue;
        KKB_TRY_CUDA(cudaStreamCreateWithFlags(&p->st[i], cudaStreamNonBlocking), "stream create");
    }
    if (slots > 1 && !p->st[0]) {
        KKB_TRY_CUDA(cudaStreamCreateWithFlags(&p->st[0], cudaStreamNonBlocking), "stream create");
        for (int i = 0; i < 5; ++i)
            KKB_TRY_CUDA(cudaEventCreateWithFlags(&p->ev[i], cudaEventDisableTiming), "event create");
    }
    p->chunk = chunk_frames;
    p->slots = slots;
    return KKB_OK;
}

extern "C" int kkb_decomposer_run(kkb_decomposer *p, const float *rf, int n_frames, void *traces,
                                  void *stream) {
    return decomposer_run(p, rf, 0, n_frames, traces, stream);
}

extern "C" int kkb_decomposer_run_i16(kkb_decomposer *p, const short *rf, int n_frames,
                                      void *traces, void *stream) {
    return decomposer_run(p, rf, 1, n_frames, traces, stream);
}

extern "C" int kkb_decomposer_run_scatter(kkb_decomposer *p, const void *rf, int rf_is_i16,
                                          int n_frames, void *const *dsts, int ndst,
                                          long long dst_offset, long long frame_stride,
                                          void *stream) {
    if (!p || !dsts || ndst < 1 || ndst > KKB_ROW_SCATTER_MAX || n_frames < 0 || dst_offset < 0 ||
        frame_stride < (long long)p->N * p->M * p->T) {
        set_error("decomposer_run_scatter: 1 <= ndst <= %d, frame_stride >= n_tx*M*T",
                  KKB_ROW_SCATTER_MAX);
        return KKB_ERR_ARG;
    }
    RowScatter sc;
    sc.ndst = ndst;
    sc.frame_stride = frame_stride;
    sc.off = dst_offset;
    for (int d = 0; d < ndst; ++d) {
        if (!dsts[d]) {
            set_error("decomposer_run_scatter: null destination %d", d);
            return KKB_ERR_ARG;
        }
        sc.dst[d] = (float2 *)dsts[d];
    }
    return decomposer_run(p, rf, rf_is_i16 ? 1 : 0, n_frames, nullptr, stream, &sc);
}

extern "C" int kkb_decomposer_destroy(kkb_decomposer *p) {
    if (!p) return KKB_OK;
    for (int i = 0; i < 4; ++i)
        if (p->st[i]) cudaStreamDestroy(p->st[i]);
    for (int i = 0; i < 5; ++i)
        if (p->ev[i]) cudaEventDestroy(p->ev[i]);
    cudaFree(p->ramps);
    cudaFree(p->X);
    cudaFree(p->Y);
    cudaFree(p->cs);
    cudaFree(p->s1f_gam);
    cudaFree(p->tctab);
    cudaFree(p->ring);
    cudaFree(p->ring_cnt);
    if (p->ring_side) cudaStreamDestroy(p->ring_side);
    for (int i = 0; i < 2; ++i)
        if (p->ring_ev[i]) cudaEventDestroy(p->ring_ev[i]);
    delete p;
    return KKB_OK;
}

// =====================================================================
// K6
extern "C" int kkb_log_compress(const float *intensity, const unsigned int *frame_max, int n_frames,
                                long long pixels_per_frame, float floor_db, float *db, void *stream) {
    return log_compress(intensity, frame_max, n_frames, pixels_per_frame, floor_db, db,
                        as_stream(stream));
}

extern "C" int kkb_compound(const void *images, int n_images, long long n_pixels, int mode,
                            double *out, void *stream) {
    if (n_images < 1 || (mode != 0 && mode != 1)) {
        set_error("compound: need >= 1 image and mode 0/1");
        return KKB_ERR_ARG;
    }
    return compound(images, n_images, n_pixels, mode, out, as_stream(stream));
}

extern "C" int kkb_render_traces(float *out, int n_tx, int n_el, int n_t, const double *sx,
                                 const double *sz, const double *refl, long long n_sc,
                                 const double *upos, const double *sin_t, const double *cos_t,
                                 double inv_c, double fs, double t0, const double *wave, int n_w,
                                 double half, int spread, void *stream) {
    if (n_tx < 0 || n_el < 0 || n_t < 0 || n_sc < 0 || n_w < 1 || !(fs > 0.0) || !(inv_c > 0.0)) {
        set_error("render_traces: bad sizes or nonpositive fs / 1/c");
        return KKB_ERR_ARG;
    }
    if (!out || (n_sc > 0 && (!sx || !sz || !refl)) || !upos || !sin_t || !cos_t || !wave) {
        set_error("render_traces: null array");
        return KKB_ERR_ARG;
    }
    return render_traces(out, n_tx, n_el, n_t, sx, sz, refl, n_sc, upos, sin_t, cos_t, inv_c, fs,
                         t0, wave, n_w, half, spread, as_stream(stream));
}

// ------------------------------------------------------------- display / budgeting
namespace {
struct DevScratch {
    double *p = nullptr;
    ~DevScratch() {
        if (p) cudaFree(p);
    }
};
}  // namespace

extern "C" int kkb_max_f64(const double *x, long long n, double *max_host, void *stream) {
    if (!x || n <= 0 || !max_host) {
        set_error("max_f64: empty input");
        return KKB_ERR_ARG;
    }
    DevScratch sc;
    KKB_TRY_CUDA(cudaMalloc(&sc.p, sizeof(double) * 304), "cudaMalloc(scratch)");
    cudaStream_t s = as_stream(stream);
    int st = device_max(x, n, sc.p, sc.p + 300, s);
    if (st) return st;
    KKB_TRY_CUDA(cudaMemcpyAsync(max_host, sc.p + 300, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H max");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync max");
    return KKB_OK;
}

extern "C" int kkb_gamma_match(const double *image, const double *reference, long long n, double lo,
                               double hi, double tol, double *gamma_host, double *mapped,
                               void *stream) {
    if (!image || !reference || n <= 0 || !gamma_host || !(tol > 0.0)) {
        set_error("gamma_match: bad arguments");
        return KKB_ERR_ARG;
    }
    DevScratch sc;
    KKB_TRY_CUDA(cudaMalloc(&sc.p, sizeof(double) * 304), "cudaMalloc(scratch)");
    cudaStream_t s = as_stream(stream);
    double *imax = sc.p + 300, *rmax = sc.p + 301, *tmp = sc.p + 302;
    int st = device_max(image, n, sc.p, imax, s);
    if (!st) st = device_max(reference, n, sc.p, rmax, s);
    double h[2];
    if (!st) {
        KKB_TRY_CUDA(cudaMemcpyAsync(h, imax, 2 * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H max");
        KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync max");
        if (!(h[0] > 0.0) || !(h[1] > 0.0)) {
            set_error("gamma matching needs nonzero images");
            return KKB_ERR_SHAPE;
        }
    }
    double target = 0.0;
    if (!st) st = device_pow_mean(reference, n, rmax, 0.5, sc.p, tmp, &target, s);
    if (st) return st;
    int err = KKB_OK;
    auto objective = [&](double g) {
        double m = 0.0;
        if (!err) err = device_pow_mean(image, n, imax, g, sc.p, tmp, &m, s);
        return fabs(m - target);
    };
    // golden-section search of metrics.py:156-172, step for step
    const double invphi = (sqrt(5.0) - 1.0) / 2.0;
    double a = lo, b = hi;
    double c = b - invphi * (b - a), d = a + invphi * (b - a);
    double fc = objective(c), fd = objective(d);
    while (b - a > tol && !err) {
        if (fc < fd) {
            b = d;
            d = c;
            fd = fc;
            c = b - invphi * (b - a);
            fc = objective(c);
        } else {
            a = c;
            c = d;
            fc = fd;
            d = a + invphi * (b - a);
            fd = objective(d);
        }
    }
    if (err) return err;
    const double gamma = 0.5 * (a + b);
    *gamma_host = gamma;
    if (mapped) {
        st = pow_map(image, n, imax, gamma, mapped, s);
        if (st) return st;
        KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync map");  // scratch (imax) freed on return
    }
    return KKB_OK;
}

extern "C" int kkb_last_read_sample_max(const double *x, int nx, const double *z, int nz,
                                        const double *sin_t, const double *cos_t, int n_tx,
                                        const double *sin_r, const double *cos_r, int n_rx,
                                        double *max_host, void *stream) {
    if (!x || !z || nx <= 0 || nz <= 0 || n_tx <= 0 || n_rx <= 0 || !max_host) {
        set_error("last_read_sample: empty grid or angle set");
        return KKB_ERR_ARG;
    }
    DevScratch sc;
    KKB_TRY_CUDA(cudaMalloc(&sc.p, sizeof(double) * 304), "cudaMalloc(scratch)");
    cudaStream_t s = as_stream(stream);
    int st = last_read_max(x, nx, z, nz, sin_t, cos_t, n_tx, sin_r, cos_r, n_rx, sc.p, sc.p + 300, s);
    if (st) return st;
    KKB_TRY_CUDA(cudaMemcpyAsync(max_host, sc.p + 300, sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
    KKB_TRY_CUDA(cudaStreamSynchronize(s), "sync last read");
    return KKB_OK;
}
