// K5 on the 5th-generation tensor cores: the kk pixel gather (_kk_kernel,
// beamform.py:212-236) as a sequence of small GEMMs, one per (tx, rx) pair.
//
// For a tile of 128 pixels (8 depth rows x 16 lateral columns) and a batch of
// up to 128 frames, the linear interpolation of pair (n, m) is
//     IQ[px, f] += sum_e  W_nm[px, e] * trace_nm[f, lo_nm + e],   e < KW
// where W_nm has at most two nonzeros per pixel row: w_m (1 - frac) at
// e = floor(fi) - lo and w_m frac at e + 1 (nearest: w_m at floor(fi + 0.5) - lo),
// and the row is all zero when the reference's in-window rule rejects the tap
// (beamform.py:226-235) — so the rule costs nothing in the product.  fi is the
// reference's float64 delay in its exact operation order (kk_delay /
// tap_index of kk_gather.cu; tap indices and the window predicate are the
// FMA kernels', bit for bit), frac its 23-bit weight.  The window
// [lo_nm, lo_nm + KW) is sized per plan from the tile's corner delays and
// proven for every (pixel, pair) at plan creation (kk_check_windows).
//
// One tcgen05.mma (kind::f16, M = 128 pixels, N = 2 x frames (re | im),
// K = 16 samples) per 16 window samples and split term: every operand is
// split into two fp16 halves x = hi + lo (traces first scaled by a per-frame
// power of two so the largest sample sits just under 2^15), and the product
// sums hi*hi + hi*lo + lo*hi with fp32 accumulation in TMEM (lo*lo ~ 2^-22 of
// the result is dropped): ~2^-21 relative per tap, the FP32 path's accuracy
// class (IQ within 1e-5 of the oracle).  Pairs accumulate in the reference's
// n-then-m order.  Each frame's column is an independent dot product, so an
// image does not depend on the batch it was gathered in.
//
// Pipeline per CTA: 8 producer warps build stage s's operands in shared
// memory (the tile's weight rows from the delay tables; the pair's trace
// windows for the batch, loaded with coalesced 64-byte runs, scaled and
// split) while one elected thread of a ninth warp issues the MMAs of the
// previous stages; full / empty mbarriers per stage (tcgen05.commit frees a
// stage).  The epilogue reads the 128 x N fp32 accumulator from TMEM and
// writes IQ (+ fused |IQ|^2, per-frame max) like the FMA kernels.

#include <algorithm>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kk.cuh"
#include "tc.cuh"

namespace kkb {

__device__ __forceinline__ double tc_kk_delay(double t1, double lz, double lx, double fs, double shift) {
    return __dadd_rn(__dmul_rn(__dsub_rn(__dadd_rn(t1, lz), lx), fs), shift);
}
#define TCG_MAGIC2 1572864.0   // 1.5 * 2^20 (kk_gather.cu KKB_FLOOR_MAGIC2)
#define TCG_MAGIC2_HI 0x41380000

#define TCG_PRODUCERS 256
#define TCG_WSCALE 4096.0f      // weights x 2^12: their fp16 low halves stay normal
#define TCG_TZ 8
#define TCG_TX 16

// per-frame max |re|, |im| of the traces (float bits; atomicMax on non-negative floats)
__global__ void k_frame_maxabs(const float2 *__restrict__ data, long long data_fs, long long per_frame,
                               unsigned *__restrict__ out) {
    const int f = blockIdx.y;
    const float2 *d = data + (long long)f * data_fs;
    float m = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per_frame;
         i += (long long)gridDim.x * blockDim.x) {
        const float2 v = __ldg(d + i);
        m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out + f, __float_as_uint(m));
}

struct TcgArgs {
    const float2 *data;
    long long data_fs;
    int N, M, T;
    const double *ltx, *ltzT, *lrx, *lrzT, *w;
    double fs, shift;
    int nx, nz;
    void *out;
    int out_kind;
    long long out_fs;
    float *inten;
    unsigned *fmax;
    int accum;
    int n_frames;
    const unsigned *maxabs;  // per-frame max |component| bits (scales)
    int FB;                  // frames per CTA (<= 128)
};

__device__ __forceinline__ float frame_scale(unsigned maxbits) {
    // 2^(14 - e) with e = floor(log2(max)): max * scale < 2^15 (fp16 max 65504)
    if (maxbits == 0u) return 1.0f;
    const int e = (int)((maxbits >> 23) & 0xff) - 127;
    const int s = min(max(14 - e, -120), 120);
    return __uint_as_float((unsigned)(127 + s) << 23);
}

__device__ __forceinline__ uint32_t pack_h2(__half a, __half b) {
    return (uint32_t)__half_as_ushort(a) | ((uint32_t)__half_as_ushort(b) << 16);
}

template <int KW, bool LINEAR>
__global__ void __launch_bounds__(TCG_PRODUCERS + 32, 1)
k_kk_gather_tc(const TcgArgs a) {
    constexpr int NSTAGE = KW <= 32 ? 3 : 2;
    constexpr int KC = KW / 8;                    // 16-byte K chunks (8 fp16) per row
    constexpr int NCOLS = 256;                    // B columns (re of 128 frames | im of 128 frames)
    constexpr int A_PLANE = KC * 128 * 16;        // one split half of the weight operand
    constexpr int B_PLANE = KC * NCOLS * 16;      // one split half of the trace operand (MN-major)
    constexpr int STAGE = 2 * A_PLANE + 2 * B_PLANE;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t full_bar[NSTAGE], empty_bar[NSTAGE], done_bar;
    __shared__ uint32_t tmem_base;
    __shared__ float fscale[128];
    int *lo_s = reinterpret_cast<int *>(sm + NSTAGE * STAGE);   // [N*M] window starts

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int N = a.N, M = a.M, T = a.T, nx = a.nx, nz = a.nz;
    const int tiles_z = (nz + TCG_TZ - 1) / TCG_TZ;
    const int iz0 = (blockIdx.x % tiles_z) * TCG_TZ, ix0 = (blockIdx.x / tiles_z) * TCG_TX;
    const int f0 = blockIdx.y * a.FB;
    const int FB = min(a.FB, a.n_frames - f0);
    const int NH = (a.FB + 7) & ~7;               // im columns start at NH (N = 2 NH, multiple of 16)
    const double fs = a.fs, shift = a.shift;

    // setup: barriers, TMEM, frame scales, window starts of every pair
    if (warp == 8) tc::tmem_alloc<256>(&tmem_base);
    if (t == 0) {
        for (int s = 0; s < NSTAGE; ++s) {
            tc::mbar_init(&full_bar[s], TCG_PRODUCERS);
            tc::mbar_init(&empty_bar[s], 1);
        }
        tc::mbar_init(&done_bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (t < 128) fscale[t] = t < FB ? frame_scale(a.maxabs[f0 + t]) : 1.0f;
    {
        const int rzb = min(TCG_TZ - 1, nz - 1 - iz0), cxb = min(TCG_TX - 1, nx - 1 - ix0);
        for (int i = t; i < N * M; i += blockDim.x) {
            const int n = i / M, m = i - n * M;
            double lo = 1e300;
            for (int cr = 0; cr < 2; ++cr)
                for (int cc = 0; cc < 2; ++cc) {
                    const int iz = iz0 + (cr ? rzb : 0), ix = ix0 + (cc ? cxb : 0);
                    const double t1 = __dadd_rn(a.ltx[(long long)ix * N + n], a.ltzT[(long long)n * nz + iz]);
                    lo = fmin(lo, tc_kk_delay(t1, a.lrzT[(long long)m * nz + iz], a.lrx[(long long)ix * M + m], fs, shift));
                }
            lo_s[i] = (int)fmax(fmin(floor(lo) - 1.0, 1.0e9), -1.0e9);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;
    const int npairs = N * M;

    if (warp < 8) {
        // ------------------------------------------------------------ producers
        // Loads of pair pr + PD are issued before pair pr's operands are
        // built (register prefetch, PD pairs deep), so the L2 latency of the
        // trace windows and delay tables overlaps the conversion work.
        // trace operand: warp w fills 8-frame groups g = w, w + 8, ...; lane k
        // holds window sample k (k + 32 for KW = 64) of the group's 8 frames, so
        // every load instruction reads one frame's window contiguously and
        // every store writes 8 frames of one sample (16 B, MN-major layout)
        constexpr int KP = KW / 32;                   // samples per lane
        constexpr int GPW = 2;                        // 8-frame groups per warp (NH <= 128)
        constexpr int PD = KW <= 32 ? 2 : 1;
        struct PairRegs {
            float2 v[GPW][KP][8];
            double tx, tz, lz, lx;
        };
        const int r = t & 127;                        // weight row (threads 0..127)
        const int ix = min(ix0 + r / TCG_TZ, nx - 1), iz = min(iz0 + r % TCG_TZ, nz - 1);
        auto fetch = [&](int pr, PairRegs &R) {
            const int n = pr / M, m = pr - n * M;
            const int lo = lo_s[pr];
            const float2 *base = a.data + (long long)f0 * a.data_fs + (long long)(n * M + m) * T;
#pragma unroll
            for (int g = 0; g < GPW; ++g)
#pragma unroll
                for (int kp = 0; kp < KP; ++kp) {
                    const int smp = lo + lane + 32 * kp;
                    const bool sok = (unsigned)smp < (unsigned)T;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const int f = (warp + 8 * g) * 8 + j;
                        R.v[g][kp][j] = sok && f < FB ? __ldg(base + (long long)f * a.data_fs + smp) : make_float2(0.f, 0.f);
                    }
                }
            if (t < 128) {
                R.tx = __ldg(a.ltx + (long long)ix * N + n);
                R.tz = __ldg(a.ltzT + (long long)n * nz + iz);
                R.lz = __ldg(a.lrzT + (long long)m * nz + iz);
                R.lx = __ldg(a.lrx + (long long)ix * M + m);
            }
        };
        PairRegs cur, nx1, nx2;
        fetch(0, cur);
        if (PD > 1 && npairs > 1) fetch(1, nx1);
        for (int pr = 0; pr < npairs; ++pr) {
            const int st = pr % NSTAGE, use = pr / NSTAGE;
            const int m = pr % M;
            if (PD > 1) {
                if (pr + 2 < npairs) fetch(pr + 2, nx2);
            } else if (pr + 1 < npairs) {
                fetch(pr + 1, nx1);
            }
            if (use > 0) tc::mbar_wait(&empty_bar[st], (use - 1) & 1);
            unsigned char *Ab = sm + st * STAGE;
            unsigned char *Bb = Ab + 2 * A_PLANE;
            const int lo = lo_s[pr];
            // trace operand (MN-major): (k, n) at (n/8) KC*128 + (k/8) 128 + (k%8) 16 + (n%8) 2
#pragma unroll
            for (int g = 0; g < GPW; ++g) {
                const int gg = warp + 8 * g;          // 8-frame group
                if (gg * 8 >= NH) break;              // uniform per warp
#pragma unroll
                for (int kp = 0; kp < KP; ++kp) {
                    const int k = lane + 32 * kp;
                    uint32_t rh[4], rl[4], ih[4], il[4];
#pragma unroll
                    for (int j = 0; j < 8; j += 2) {
                        const int f = gg * 8 + j;
                        const float s0 = f < FB ? fscale[f] : 1.0f, s1 = f + 1 < FB ? fscale[f + 1] : 1.0f;
                        const float x0 = cur.v[g][kp][j].x * s0, y0 = cur.v[g][kp][j].y * s0;
                        const float x1 = cur.v[g][kp][j + 1].x * s1, y1 = cur.v[g][kp][j + 1].y * s1;
                        const __half hx0 = __float2half_rn(x0), hx1 = __float2half_rn(x1);
                        const __half hy0 = __float2half_rn(y0), hy1 = __float2half_rn(y1);
                        rh[j / 2] = pack_h2(hx0, hx1);
                        ih[j / 2] = pack_h2(hy0, hy1);
                        rl[j / 2] = pack_h2(__float2half_rn(x0 - __half2float(hx0)), __float2half_rn(x1 - __half2float(hx1)));
                        il[j / 2] = pack_h2(__float2half_rn(y0 - __half2float(hy0)), __float2half_rn(y1 - __half2float(hy1)));
                    }
                    const int off_k = (k >> 3) * 128 + (k & 7) * 16;
                    unsigned char *bre = Bb + gg * (KC * 128) + off_k;
                    unsigned char *bim = Bb + (NH / 8 + gg) * (KC * 128) + off_k;
                    *reinterpret_cast<uint4 *>(bre) = make_uint4(rh[0], rh[1], rh[2], rh[3]);
                    *reinterpret_cast<uint4 *>(bim) = make_uint4(ih[0], ih[1], ih[2], ih[3]);
                    *reinterpret_cast<uint4 *>(bre + B_PLANE) = make_uint4(rl[0], rl[1], rl[2], rl[3]);
                    *reinterpret_cast<uint4 *>(bim + B_PLANE) = make_uint4(il[0], il[1], il[2], il[3]);
                }
            }
            // weight rows (scaled by 2^12 so the fp16 low halves stay normal)
            if (t < 128) {
                const double t1 = __dadd_rn(cur.tx, cur.tz);
                const double fi = tc_kk_delay(t1, cur.lz, cur.lx, fs, shift);
                const double sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), TCG_MAGIC2);
                const int F = __double2hiint(sv) - TCG_MAGIC2_HI;
                const bool ok = (unsigned)F <= (unsigned)(LINEAR ? T - 2 : T - 1);
                const int e = F - lo;
                const float wm = (a.w ? (float)a.w[m] : 1.0f) * TCG_WSCALE;
                float w0 = 0.f, w1 = 0.f;
                if (ok) {
                    if (LINEAR) {
                        const float fr = __uint_as_float(((unsigned)__double2loint(sv) >> 9) | 0x3F800000u) - 1.0f;
                        w0 = wm * (1.0f - fr);
                        w1 = wm * fr;
                    } else {
                        w0 = wm;
                    }
                }
                const __half h0 = __float2half_rn(w0), h1 = __float2half_rn(w1);
                const __half l0 = __float2half_rn(w0 - __half2float(h0)), l1 = __float2half_rn(w1 - __half2float(h1));
                const int c0 = ok ? e >> 3 : -2, p = e & 7;
                uint32_t wh[8], wl[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int q0 = 2 * i, q1 = 2 * i + 1;  // half positions in the 2-chunk window
                    const __half z = __ushort_as_half(0);
                    wh[i] = pack_h2(q0 == p ? h0 : (q0 == p + 1 ? h1 : z), q1 == p ? h0 : (q1 == p + 1 ? h1 : z));
                    wl[i] = pack_h2(q0 == p ? l0 : (q0 == p + 1 ? l1 : z), q1 == p ? l0 : (q1 == p + 1 ? l1 : z));
                }
#pragma unroll
                for (int c = 0; c < KC; ++c) {
                    uint4 vh = make_uint4(0, 0, 0, 0), vl = vh;
                    if (c == c0) {
                        vh = make_uint4(wh[0], wh[1], wh[2], wh[3]);
                        vl = make_uint4(wl[0], wl[1], wl[2], wl[3]);
                    } else if (c == c0 + 1) {
                        vh = make_uint4(wh[4], wh[5], wh[6], wh[7]);
                        vl = make_uint4(wl[4], wl[5], wl[6], wl[7]);
                    }
                    *reinterpret_cast<uint4 *>(Ab + (c * 128 + r) * 16) = vh;
                    *reinterpret_cast<uint4 *>(Ab + A_PLANE + (c * 128 + r) * 16) = vl;
                }
            }
            tc::fence_smem_to_async();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&full_bar[st]))
                         : "memory");
            cur = nx1;
            if (PD > 1) nx1 = nx2;
        }
    } else if (lane == 0) {
        // ------------------------------------------------------------ MMA issue
        const uint32_t idesc = tc::instr_desc(0, 128, 2 * NH, 1);
        const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
        for (int pr = 0; pr < npairs; ++pr) {
            const int st = pr % NSTAGE, use = pr / NSTAGE;
            tc::mbar_wait(&full_bar[st], use & 1);
            tc::fence_after_sync();
            const uint32_t sa = s0 + st * STAGE, sb = sa + 2 * A_PLANE;
            const uint64_t da = tc::smem_desc(sa, 128 * 16, 128), db = tc::smem_desc(sb, 128, KC * 128);
#pragma unroll
            for (int ks = 0; ks < KW / 16; ++ks) {
                const uint64_t ah = da + ((ks * 2 * 128 * 16) >> 4), al = ah + (A_PLANE >> 4);
                const uint64_t bh = db + ((ks * 2 * 128) >> 4), bl = bh + (B_PLANE >> 4);
                tc::mma_f16(tmem, ah, bh, idesc, pr > 0 || ks > 0);
                tc::mma_f16(tmem, ah, bl, idesc, true);
                tc::mma_f16(tmem, al, bh, idesc, true);
            }
            tc::commit(&empty_bar[st]);
        }
        tc::commit(&done_bar);
    }
    // ------------------------------------------------------------ epilogue
    if (warp < 8) {
        tc::mbar_wait(&done_bar, 0);
        tc::fence_after_sync();
        const int quarter = warp & 3, half = warp >> 2;
        const int r = quarter * 32 + lane;
        const int ix = ix0 + r / TCG_TZ, iz = iz0 + r % TCG_TZ;
        const bool pix = ix < nx && iz < nz;
        const int fb0 = half * (NH / 2), fb1 = min(FB, fb0 + NH / 2);
        for (int fc = fb0; fc < fb0 + NH / 2; fc += 8) {
            if (fc >= fb1) break;  // uniform across the warp
            float re[8], im[8];
            tc::tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + fc, re);
            tc::tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + NH + fc, im);
            tc::tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int f = fc + i;
                if (f >= fb1) break;
                const float inv = 1.0f / (fscale[f] * TCG_WSCALE);   // exact: a power of two
                const float vr = re[i] * inv, vi = im[i] * inv;
                float I = 0.f;
                if (pix) {
                    const long long px = (long long)(f0 + f) * a.out_fs + (long long)ix * nz + iz;
                    if (a.out) {
                        if (a.out_kind == KKB_OUT_C128)
                            reinterpret_cast<double2 *>(a.out)[px] = make_double2(vr, vi);
                        else
                            reinterpret_cast<float2 *>(a.out)[px] = make_float2(vr, vi);
                    }
                    if (a.inten) {
                        I = __fmaf_rn(vr, vr, __fmul_rn(vi, vi));
                        if (a.accum) I = __fadd_rn(I, a.inten[px]);
                        a.inten[px] = I;
                    }
                }
                if (a.fmax) {
                    for (int o = 16; o > 0; o >>= 1) I = fmaxf(I, __shfl_xor_sync(0xffffffffu, I, o));
                    if (lane == 0) atomicMax(a.fmax + f0 + f, __float_as_uint(I));
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 8) {
        __syncwarp();
        tc::tmem_free<256>(tmem);
    }
}

template <int KW, bool LINEAR>
static int launch_tc(const TcgArgs &a, cudaStream_t s) {
    constexpr int NSTAGE = KW <= 32 ? 3 : 2;
    constexpr int STAGE = 2 * (KW / 8) * 128 * 16 + 2 * (KW / 8) * 256 * 16;
    const size_t smem = (size_t)NSTAGE * STAGE + sizeof(int) * (size_t)a.N * a.M;
    if (smem > 227 * 1024) {
        set_error("kk tensor-core gather: %d pairs do not fit shared memory", a.N * a.M);
        return KKB_ERR_UNSUPPORTED;
    }
    auto fn = k_kk_gather_tc<KW, LINEAR>;
    KKB_TRY_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "smem attr kk tc");
    dim3 grid((unsigned)(ceil_div(a.nz, TCG_TZ) * ceil_div(a.nx, TCG_TX)), (unsigned)ceil_div(a.n_frames, a.FB));
    fn<<<grid, TCG_PRODUCERS + 32, smem, s>>>(a);
    KKB_CHECK_LAUNCH("k_kk_gather_tc");
    return KKB_OK;
}

int kk_gather_tc(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
                 const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
                 double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
                 long long out_fs, float *inten, unsigned *fmax, int W, int accum, cudaStream_t s) {
    if (W > 64 || W < 2) return KKB_ERR_UNSUPPORTED;
    unsigned *mx = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&mx, sizeof(unsigned) * (size_t)n_frames, s), "cudaMallocAsync(frame max)");
    struct Free {
        unsigned *p;
        cudaStream_t s;
        ~Free() { cudaFreeAsync(p, s); }
    } fr{mx, s};
    KKB_TRY_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned) * (size_t)n_frames, s), "zero frame max");
    const long long per = (long long)N * M * T;
    const int bx = (int)std::max<long long>(1, std::min<long long>(ceil_div(per, 256), std::max(1, 148 * 4 / n_frames)));
    k_frame_maxabs<<<dim3(bx, n_frames), 256, 0, s>>>(data, data_fs, per, mx);
    KKB_CHECK_LAUNCH("k_frame_maxabs");
    // frames per CTA: the largest batch (<= 128) that still gives every SM a tile
    const long long tiles = ceil_div(nz, TCG_TZ) * ceil_div(nx, TCG_TX);
    int FB = 128;
    while (FB > 8 && tiles * ceil_div(n_frames, FB) < sm_count()) FB /= 2;
    FB = std::min(FB, std::max(1, n_frames));
    TcgArgs a{data, data_fs, N, M, T, ltx, ltzT, lrx, lrzT, w, fs, shift, nx, nz,
              out, out_kind, out_fs, inten, fmax, accum, n_frames, mx, FB};
    const int KW = W <= 32 ? 32 : 64;  // one window sample per lane (two for 64)
    if (KW == 32) return linear ? launch_tc<32, true>(a, s) : launch_tc<32, false>(a, s);
    return linear ? launch_tc<64, true>(a, s) : launch_tc<64, false>(a, s);
}

}  // namespace kkb
