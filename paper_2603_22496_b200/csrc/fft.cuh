// FFT plan and launchers shared by the spectral / decomposition paths.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <vector>

#define KKB_FFT_MAX_STAGES 16
#define KKB_FFT_MAX_RADIX 32
#define KKB_FFT_MAX_T 8192            // one transform per CTA in shared memory
#define KKB_FFT_MAX_T_TOTAL (1 << 20) // longer: four-step T = T1 x T2 (or direct DFT)
#define KKB_FFT_THREADS 256
#define KKB_FFT_TARGET_ELEMS 4096  // traces per CTA = max(1, this / T)

namespace kkb {

// Row-wise multi-destination store of a batched transform (fused trace
// all-gather): row r goes to dst[d] + off + (r / rows_per_frame) * frame_stride
// + (r % rows_per_frame) * out_stride for every d < ndst (complex64 elements).
#define KKB_ROW_SCATTER_MAX 8
struct RowScatter {
    int ndst = 0;
    int rows_per_frame = 1;
    long long frame_stride = 0;
    long long off = 0;
    float2 *dst[KKB_ROW_SCATTER_MAX] = {};
};

// Stage-1 handoff through an L2-resident ring (decomposer "ring" mode): K1
// writes the spectra of global row-tile t (tile_rows (frame, transmit) rows)
// into ring slot t % R once the persistent contraction has released the slot
// (con_done[t - R] == con_per_tile) and counts its transform pairs into
// fft_done[t]; the contraction consumes a tile when fft_done[t] reaches the
// tile's pair count.  Spins are bounded: on a timeout the kernel raises *err
// and proceeds (no hang; the result is then wrong and the caller fails).
struct Stage1Ring {
    int *fft_done = nullptr;
    int *con_done = nullptr;
    int R = 0;
    int con_per_tile = 0;
    long long traces_per_tile = 0;  // tile_rows * L
    unsigned *err = nullptr;
};

// wait until *p >= target (acquire); false after 2 s of %globaltimer (sets *err)
__device__ __forceinline__ bool ring_wait_geq(const int *p, int target, unsigned *err) {
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        int v;
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) return true;
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 2000000000ull) {
            atomicOr(err, 1u);
            return false;
        }
        __nanosleep(128);
    }
}

struct FftPlan {
    int T;
    int nstages;
    int direct;                      // 1: largest prime factor > 31 -> O(T^2) kernel
    int large;                       // 1: T > KKB_FFT_MAX_T, four-step with T = T1 * T2
    int T1, T2;
    int radix[KKB_FFT_MAX_STAGES];
    float2 *tw;                      // exp(-2 pi i k / T), k < T (device)
    float2 *tws;                     // stage-ordered twiddles of the compile-time plan (device; fft_ct_supported T only)
};

int get_fft_plan(int T, FftPlan *out);

// Batched C2C (forward exp(-), inverse exp(+) unnormalised, times `scale`).
int fft_c2c(const float2 *in, long long in_stride, int in_len, float2 *out, long long out_stride,
            int out_len, long long ntraces, int T, bool inverse, float scale, cudaStream_t s);

// Batched real-input FFT: bins [0, K) of each row, times bin_scale[k].
// Rows are paired (two real rows per complex transform) only within groups of
// group_rows consecutive rows (0: the whole batch is one group).
int fft_r2c(const float *in, long long ntraces, int T, float2 *out, long long out_stride, int K,
            const float *bin_scale, cudaStream_t s, float2 *scratch_c2c, long long group_rows = 0);

// compile-time-specialised twins (fft_ct.cu)
bool fft_ct_supported(int T);
// host copy of the stage-ordered twiddle table the *_ct kernels read
void fft_ct_twiddles(int T, std::vector<float2> &out);
// in_kind 0: float32 rows, 1: int16 rows (converted exactly to float32)
int fft_r2c_ct(const void *in, int in_kind, long long ntraces, int T, float2 *out,
               long long out_stride, int K, const float *bin_scale, const float2 *tws,
               cudaStream_t s, long long group_rows = 0);
// fft_r2c_ct writing through the stage-1 ring (even group_rows: pairs never
// straddle a (frame, transmit) row, so a row-tile's pairs are contiguous CTAs)
int fft_r2c_ct_ring(const void *in, int in_kind, long long ntraces, int T, float2 *ring,
                    long long out_stride, int K, const float *bin_scale, const float2 *tws,
                    cudaStream_t s, const Stage1Ring &rs);
int fft_c2c_ct(const float2 *in, long long in_stride, int in_len, float2 *out, long long out_stride,
               int out_len, long long ntraces, int T, bool inverse, float scale, const float2 *tw,
               cudaStream_t s, const RowScatter *sc = nullptr);
// K3 into the tensor-core gather's split planes (tcplanes.cuh) for rows
// (frame, pair) of the contracted bins Y; T in {1024, 1536, 2048}.  traces
// are written too when *nonfinite != 0.  planes: 4 x ceil(F/8)*8 x NM x T fp16.
int fft_c2c_planes(const float2 *Y, long long ldy, int K, int T, int n_frames, int NM, float scale,
                   const float2 *tws, const unsigned *fbound, const unsigned *nonfinite, float2 *traces,
                   __half *planes, cudaStream_t s);
// the per-frame bounds fft_c2c_planes scales by (max over rows of scale x the
// L1 norm of the row's bins), and the non-finite flag
int frame_bound(const float2 *Y, long long ldy, int K, long long rows, int rows_per_frame, float scale,
                unsigned *fbound, unsigned *nonfinite, cudaStream_t s);
// fft_c2c whose rows are stored through `sc` (out_stride = row pitch inside a
// frame): fused into the compile-time kernels' epilogue, otherwise one
// transform into scratch followed by a strided copy per destination.
int fft_c2c_scatter(const float2 *in, long long in_stride, int in_len, int out_len,
                    long long ntraces, int T, bool inverse, float scale, const RowScatter &sc,
                    cudaStream_t s);

}  // namespace kkb
