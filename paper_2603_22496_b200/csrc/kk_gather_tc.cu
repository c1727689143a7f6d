// K5 on the 5th-generation tensor cores: the kk pixel gather (_kk_kernel,
// beamform.py:212-236) as a sequence of small GEMMs, one per (tx, rx) pair.
//
// For a tile of 128 pixels (8 depth rows x 16 lateral columns) and a batch of
// 64 frames, the linear interpolation of pair (n, m) is
//     IQ[px, f] += sum_e  W_nm[px, e] * trace_nm[f, lo_nm + e],   e < 32
// where W_nm has at most two nonzeros per pixel row: w_m (1 - frac) at
// e = floor(fi) - lo and w_m frac at e + 1 (nearest: w_m at floor(fi + 0.5) - lo),
// and the row is all zero when the reference's in-window rule rejects the tap
// (beamform.py:226-235) — so the rule costs nothing in the product.  fi is the
// reference's float64 delay in its exact operation order (the FMA kernels'
// index arithmetic, bit for bit), frac its 23-bit weight.  The window
// [lo_nm, lo_nm + 32) comes from the tile's corner delays and is proven for
// every (pixel, pair) at plan creation (kk_check_windows).
//
// Operands: one tcgen05.mma (kind::f16, M = 128 pixels, N = 128 = re | im of
// 64 frames, K = 16 samples) per 16 window samples and split term.  Every
// operand is split into two fp16 halves x = hi + lo and the product sums
// hi*hi + hi*lo + lo*hi (lo*lo ~ 2^-22 dropped).  The traces are split ONCE
// per batch (k_split_planes: each frame scaled by a power of two so its
// largest sample sits just under 2^15) into four planes (hi/lo x re/im) laid
// out [frame group of 8][pair][sample][8 frames]: one 4-D TMA box (32 samples
// x 8 frames as one 512-byte row x 8 groups x 4 planes = 16 KB, cp.async.bulk.tensor)
// lands a pair's window for 64 frames directly in the MN-major operand layout,
// zero-filled where the window leaves the trace (the reference's out-of-window
// taps carry zero weight anyway).  Weights are scaled by 2^12 so their low
// halves stay normal.
//
// Accumulation: tensor-core adds into a TMEM accumulator truncate (measured,
// scripts/ubench/tc_accum.cu: ~3e-8 relative drift per MMA), so pairs are
// summed in groups of 8 into two ping-pong TMEM accumulators, and four drain
// warps add each finished group into float32 registers with round-to-nearest
// adds: the drift is bounded by one group's 48 MMAs.
//
// Warp roles (10 warps): 0-3 build the weight rows of each pair (one row per
// thread, delay tables staged in shared memory); 4 allocates TMEM and issues
// the TMA copies (one lane); 5 issues
// the MMAs (one lane); 6-9 drain the accumulators and run the epilogue (IQ,
// fused |IQ|^2, per-frame max).  Stages are guarded by full / empty
// mbarriers (tcgen05.commit frees a stage and publishes a group).

#include <algorithm>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kk.cuh"
#include "tc.cuh"

namespace kkb {

__device__ __forceinline__ double tc_kk_delay(double t1, double lz, double lx, double fs, double shift) {
    return __dadd_rn(__dmul_rn(__dsub_rn(__dadd_rn(t1, lz), lx), fs), shift);
}
#define TCG_MAGIC2 1572864.0   // 1.5 * 2^20 (kk_gather.cu KKB_FLOOR_MAGIC2)
#define TCG_MAGIC2_HI 0x41380000
#define TCG_WSCALE 4096.0f     // weights x 2^12: their fp16 low halves stay normal
#define TCG_TZ 8
#define TCG_TX 16
#define TCG_KW KKB_KK_TC_W     // window samples per pair (two K steps)
#define TCG_FB 64              // frames per CTA: N = 128 (re | im)
#define TCG_NA 4               // weight (A) stages
#define TCG_NB 8               // trace-window (B) stages: deeper, they hide the TMA latency
#define TCG_PB 2               // pairs per producer iteration (divides TCG_NA)
#define TCG_GROUP 8            // pairs per accumulator group
#define TCG_THREADS 320

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

__device__ __forceinline__ void split_h(float x, __half &hi, __half &lo) {
    hi = __float2half_rn(x);
    lo = __float2half_rn(x - __half2float(hi));
}

// planes[pl][g][q][t][8]: pl = re_hi, im_hi, re_lo, im_lo; frames 8g..8g+7
__global__ void k_split_planes(const float2 *__restrict__ data, long long data_fs, int n_frames, int NM, int T,
                               const unsigned *__restrict__ maxabs, long long ngroups, __half *__restrict__ planes) {
    const long long per_plane = ngroups * NM * (long long)T * 8;
    const long long total = ngroups * NM * (long long)T;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int t = (int)(i % T);
        const long long gq = i / T;
        const int q = (int)(gq % NM);
        const long long g = gq / NM;
        __half h[4][8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long f = g * 8 + j;
            float2 v = make_float2(0.f, 0.f);
            float sc = 1.0f;
            if (f < n_frames) {
                v = __ldg(data + f * data_fs + (long long)q * T + t);
                sc = frame_scale(maxabs[f]);
            }
            split_h(v.x * sc, h[0][j], h[2][j]);
            split_h(v.y * sc, h[1][j], h[3][j]);
        }
#pragma unroll
        for (int pl = 0; pl < 4; ++pl)
            reinterpret_cast<uint4 *>(planes + pl * per_plane)[i] =
                make_uint4(pack_h2(h[pl][0], h[pl][1]), pack_h2(h[pl][2], h[pl][3]), pack_h2(h[pl][4], h[pl][5]),
                           pack_h2(h[pl][6], h[pl][7]));
    }
}

struct TcgArgs {
    CUtensorMap planes;      // 4-D map of the split trace planes (64-byte aligned)
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
    const unsigned *maxabs;
};

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_4d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                       uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5}], [%6];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
        "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

template <bool LINEAR>
__global__ void __launch_bounds__(TCG_THREADS, 1)
k_kk_gather_tc(const __grid_constant__ TcgArgs a) {
    constexpr int KC = TCG_KW / 8;                 // 16-byte K chunks per weight row
    constexpr int A_PLANE = KC * 128 * 16;          // 8 KB: one split half of the weights (K-major)
    constexpr int B_PLANE = 16 * TCG_KW * 16;       // 8 KB: one split half of the traces (MN-major, 16 col groups)
    constexpr int ASTAGE = 2 * A_PLANE, BSTAGE = 2 * B_PLANE;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t a_full[TCG_NA], a_empty[TCG_NA], b_full[TCG_NB], b_empty[TCG_NB], dfull[2], dfree[2];
    __shared__ uint32_t tmem_base;
    __shared__ float fscale[TCG_FB];
    // delay tables of the tile (fp64) and the window starts, after the stages
    double *ltx_s = reinterpret_cast<double *>(sm + TCG_NA * ASTAGE + TCG_NB * BSTAGE);  // [N][TX]
    double *ltz_s = ltx_s + a.N * TCG_TX;                                  // [N][TZ]
    double *lrx_s = ltz_s + a.N * TCG_TZ;                                  // [M][TX]
    double *lrz_s = lrx_s + a.M * TCG_TX;                                  // [M][TZ]
    float *w_s = reinterpret_cast<float *>(lrz_s + a.M * TCG_TZ);        // [M] weights x 2^12
    int *lo_s = reinterpret_cast<int *>(w_s + a.M);                       // [N*M]

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int N = a.N, M = a.M, T = a.T, nx = a.nx, nz = a.nz;
    const int tiles_z = (nz + TCG_TZ - 1) / TCG_TZ;
    const int iz0 = (blockIdx.x % tiles_z) * TCG_TZ, ix0 = (blockIdx.x / tiles_z) * TCG_TX;
    const int f0 = blockIdx.y * TCG_FB;
    const int FB = min(TCG_FB, a.n_frames - f0);
    const double fs = a.fs, shift = a.shift;
    const int npairs = N * M;
    const int ngroups = (npairs + TCG_GROUP - 1) / TCG_GROUP;

    if (warp == 4) tc::tmem_alloc<256>(&tmem_base);
    if (t == 0) {
        for (int s = 0; s < TCG_NA; ++s) {
            tc::mbar_init(&a_full[s], 128);  // the 128 weight rows
            tc::mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < TCG_NB; ++s) {
            tc::mbar_init(&b_full[s], 1);    // the TMA issuer (expect_tx)
            tc::mbar_init(&b_empty[s], 1);
        }
        for (int d = 0; d < 2; ++d) {
            tc::mbar_init(&dfull[d], 1);
            tc::mbar_init(&dfree[d], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (t < TCG_FB) fscale[t] = t < FB ? frame_scale(a.maxabs[f0 + t]) : 1.0f;
    if (t == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.planes)) : "memory");
    // tile tables (edge tiles repeat the last row / column)
    for (int i = t; i < N * TCG_TX; i += blockDim.x) {
        const int n = i / TCG_TX, c = i - n * TCG_TX;
        ltx_s[i] = __ldg(a.ltx + (long long)min(ix0 + c, nx - 1) * N + n);
    }
    for (int i = t; i < N * TCG_TZ; i += blockDim.x) {
        const int n = i / TCG_TZ, r = i - n * TCG_TZ;
        ltz_s[i] = __ldg(a.ltzT + (long long)n * nz + min(iz0 + r, nz - 1));
    }
    for (int i = t; i < M * TCG_TX; i += blockDim.x) {
        const int m = i / TCG_TX, c = i - m * TCG_TX;
        lrx_s[i] = __ldg(a.lrx + (long long)min(ix0 + c, nx - 1) * M + m);
    }
    for (int i = t; i < M; i += blockDim.x) w_s[i] = (a.w ? (float)__ldg(a.w + i) : 1.0f) * TCG_WSCALE;
    for (int i = t; i < M * TCG_TZ; i += blockDim.x) {
        const int m = i / TCG_TZ, r = i - m * TCG_TZ;
        lrz_s[i] = __ldg(a.lrzT + (long long)m * nz + min(iz0 + r, nz - 1));
    }
    __syncthreads();
    {
        const int rzb = min(TCG_TZ - 1, nz - 1 - iz0), cxb = min(TCG_TX - 1, nx - 1 - ix0);
        for (int i = t; i < npairs; i += blockDim.x) {
            const int n = i / M, m = i - n * M;
            double lo = 1e300;
            for (int cr = 0; cr < 2; ++cr)
                for (int cc = 0; cc < 2; ++cc) {
                    const int r = cr ? rzb : 0, c = cc ? cxb : 0;
                    const double t1 = __dadd_rn(ltx_s[n * TCG_TX + c], ltz_s[n * TCG_TZ + r]);
                    lo = fmin(lo, tc_kk_delay(t1, lrz_s[m * TCG_TZ + r], lrx_s[m * TCG_TX + c], fs, shift));
                }
            // a live window (plan proof: lo in (-W, T - 1)) is never clamped; a
            // dead one (every tap rejected) is zero-filled by the TMA unit
            lo_s[i] = (int)fmax(fmin(floor(lo) - 1.0, (double)T), (double)-TCG_KW);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp < 4) {
        // ------------------------------------------------------------ weight rows
        // A row holds two nonzero halves (w0 at window sample e, w1 at e + 1)
        // in 32: the stage's A planes are zeroed once, then each pair writes
        // the two 32-bit words that carry them and clears the words it wrote
        // in the same stage one round earlier (4 x STS.32 per plane).
        const int r = t, cl = r / TCG_TZ, rl = r % TCG_TZ;
        unsigned char *row = sm + r * 16;
#pragma unroll
        for (int st = 0; st < TCG_NA; ++st)
#pragma unroll
            for (int c = 0; c < 2 * KC; ++c)
                *reinterpret_cast<uint4 *>(row + st * ASTAGE + c * 128 * 16) = make_uint4(0, 0, 0, 0);
        // byte offset of 32-bit word k (half pair 2k, 2k + 1) of the row
        auto word = [](int k) { return (k >> 2) * (128 * 16) + (k & 3) * 4; };
        uint32_t prevk = 0;  // per stage (4 bits each): first word written last round
        int n = 0, m = 0;
        // TCG_PB pairs per iteration: independent delay chains in flight and one
        // proxy fence per batch
        for (int pr0 = 0; pr0 < npairs; pr0 += TCG_PB) {
            uint32_t hA[TCG_PB], hB[TCG_PB], lA[TCG_PB], lB[TCG_PB];
            int kA[TCG_PB];
#pragma unroll
            for (int j = 0; j < TCG_PB; ++j) {
                const int pr = min(pr0 + j, npairs - 1);
                const double t1 = __dadd_rn(ltx_s[n * TCG_TX + cl], ltz_s[n * TCG_TZ + rl]);
                const double fi = tc_kk_delay(t1, lrz_s[m * TCG_TZ + rl], lrx_s[m * TCG_TX + cl], fs, shift);
                const float wm = w_s[m];
                const int lo = lo_s[pr];
                const double sv = __dadd_rd(LINEAR ? fi : __dadd_rn(fi, 0.5), TCG_MAGIC2);
                const int F = __double2hiint(sv) - TCG_MAGIC2_HI;
                const int e = F - lo;
                // the reference's in-window rule; (e < 32) holds for every live
                // window by the plan-time proof and only guards the stores
                const bool ok = (unsigned)F <= (unsigned)(LINEAR ? T - 2 : T - 1) && (unsigned)e < TCG_KW;
                float w0, w1 = 0.f;
                if (LINEAR) {
                    const float fr = __uint_as_float(((unsigned)__double2loint(sv) >> 9) | 0x3F800000u) - 1.0f;
                    w0 = wm * (1.0f - fr);
                    w1 = wm * fr;
                } else {
                    w0 = wm;
                }
                if (!ok) w0 = w1 = 0.f;
                __half h0, l0, h1, l1;
                split_h(w0, h0, l0);
                split_h(w1, h1, l1);
                const bool odd = e & 1;
                hA[j] = odd ? (uint32_t)__half_as_ushort(h0) << 16 : pack_h2(h0, h1);
                hB[j] = odd ? (uint32_t)__half_as_ushort(h1) : 0u;
                lA[j] = odd ? (uint32_t)__half_as_ushort(l0) << 16 : pack_h2(l0, l1);
                lB[j] = odd ? (uint32_t)__half_as_ushort(l1) : 0u;
                kA[j] = ok ? e >> 1 : 0;
                if (++m == M) {
                    m = 0;
                    ++n;
                }
            }
#pragma unroll
            for (int j = 0; j < TCG_PB; ++j) {
                const int pr = pr0 + j;
                if (pr >= npairs) break;
                const int st = pr % TCG_NA, use = pr / TCG_NA;
                unsigned char *Ab = row + st * ASTAGE;
                if (use > 0) {
                    tc::mbar_wait(&a_empty[st], (use - 1) & 1);
                    const int qA = (prevk >> (4 * st)) & 15, qB = qA == 15 ? 14 : qA + 1;
                    *reinterpret_cast<uint32_t *>(Ab + word(qA)) = 0u;
                    *reinterpret_cast<uint32_t *>(Ab + word(qB)) = 0u;
                    *reinterpret_cast<uint32_t *>(Ab + A_PLANE + word(qA)) = 0u;
                    *reinterpret_cast<uint32_t *>(Ab + A_PLANE + word(qB)) = 0u;
                }
                // kA == 15 (e >= 30) leaves hB / lB zero: their store to word 14 is a no-op
                const int kB = kA[j] == 15 ? 14 : kA[j] + 1;
                *reinterpret_cast<uint32_t *>(Ab + word(kB)) = hB[j];
                *reinterpret_cast<uint32_t *>(Ab + word(kA[j])) = hA[j];
                *reinterpret_cast<uint32_t *>(Ab + A_PLANE + word(kB)) = lB[j];
                *reinterpret_cast<uint32_t *>(Ab + A_PLANE + word(kA[j])) = lA[j];
                prevk = (prevk & ~(15u << (4 * st))) | ((uint32_t)kA[j] << (4 * st));
            }
            tc::fence_smem_to_async();
#pragma unroll
            for (int j = 0; j < TCG_PB; ++j)
                if (pr0 + j < npairs) mbar_arrive(&a_full[(pr0 + j) % TCG_NA]);
        }
    } else if (warp == 4) {
        // ------------------------------------------------------------ trace windows (TMA)
        // box [plane 4][group 8][sample 32][frame 8] = B hi (re groups | im
        // groups) then B lo: column group = im * 8 + g, 512 B apart
        if (lane == 0) {
            for (int pr = 0; pr < npairs; ++pr) {
                const int st = pr % TCG_NB, use = pr / TCG_NB;
                if (use > 0) tc::mbar_wait(&b_empty[st], (use - 1) & 1);
                mbar_arrive_tx(&b_full[st], BSTAGE);
                tma_4d(sm + TCG_NA * ASTAGE + st * BSTAGE, &a.planes, 8 * lo_s[pr], pr, f0 / 8, 0, &b_full[st]);
            }
        }
    } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issue
        // The whole warp runs the (warp-uniform) loop and one elected lane
        // issues a pair's six MMAs from one asm block: descriptors stay in
        // uniform registers, no per-MMA lane election.
        const uint32_t idesc = tc::instr_desc(0, 128, 2 * TCG_FB, 1);
        const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
        for (int pr = 0; pr < npairs; ++pr) {
            const int sa_ = pr % TCG_NA, sb_ = pr % TCG_NB;
            const int grp = pr / TCG_GROUP, d = grp & 1;
            const bool first = pr % TCG_GROUP == 0;
            if (first && grp >= 2) tc::mbar_wait(&dfree[d], ((grp >> 1) - 1) & 1);  // drained
            tc::mbar_wait(&a_full[sa_], (pr / TCG_NA) & 1);
            tc::mbar_wait(&b_full[sb_], (pr / TCG_NB) & 1);
            tc::fence_after_sync();
            const uint32_t sa = s0 + sa_ * ASTAGE, sb = s0 + TCG_NA * ASTAGE + sb_ * BSTAGE;
            const uint64_t da = tc::smem_desc(sa, 128 * 16, 128), db = tc::smem_desc(sb, 128, TCG_KW * 16);
            if (tc::elect_one()) {
                tc::mma_f16_split_pair<A_PLANE, B_PLANE, 2 * 128 * 16, 2 * 128>(tmem + d * 128, da, db, idesc,
                                                                                  !first);
                tc::commit(&a_empty[sa_]);
                tc::commit(&b_empty[sb_]);
                if (pr % TCG_GROUP == TCG_GROUP - 1 || pr == npairs - 1) tc::commit(&dfull[d]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ drains + epilogue
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        float S[2 * TCG_FB];
#pragma unroll
        for (int c = 0; c < 2 * TCG_FB; ++c) S[c] = 0.f;
        for (int grp = 0; grp < ngroups; ++grp) {
            const int d = grp & 1;
            tc::mbar_wait(&dfull[d], (grp >> 1) & 1);
            tc::fence_after_sync();
#pragma unroll
            for (int c0 = 0; c0 < 2 * TCG_FB; c0 += 8) {
                float v[8];
                tc::tmem_ld8(tmem + ((uint32_t)(quarter * 32) << 16) + d * 128 + c0, v);
                tc::tmem_ld_wait();
#pragma unroll
                for (int i = 0; i < 8; ++i) S[c0 + i] = __fadd_rn(S[c0 + i], v[i]);
            }
            tc::fence_before_sync();
            mbar_arrive(&dfree[d]);
        }
        const int ix = ix0 + r / TCG_TZ, iz = iz0 + r % TCG_TZ;
        const bool pix = ix < nx && iz < nz;
#pragma unroll
        for (int f = 0; f < TCG_FB; ++f) {
            if (f >= FB) break;
            const float inv = 1.0f / (fscale[f] * TCG_WSCALE);   // exact: a power of two
            const float vr = S[f] * inv, vi = S[TCG_FB + f] * inv;
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
                // non-negative floats order like their bit patterns: one redux per frame
                const unsigned mx = __reduce_max_sync(0xffffffffu, __float_as_uint(I));
                if (lane == 0) atomicMax(a.fmax + f0 + f, mx);
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 4) {
        __syncwarp();
        tc::tmem_free<256>(tmem);
    }
}

int kk_gather_tc(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
                 const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
                 double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
                 long long out_fs, float *inten, unsigned *fmax, int W, int accum, cudaStream_t s) {
    if (W > TCG_KW || W < 2) return KKB_ERR_UNSUPPORTED;
    const int NM = N * M;
    const long long ngroups = (n_frames + 7) / 8;
    const size_t plane_elems = (size_t)ngroups * NM * T * 8;
    unsigned *mx = nullptr;
    __half *planes = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&mx, sizeof(unsigned) * (size_t)n_frames, s), "cudaMallocAsync(frame max)");
    struct Free {
        void *p;
        cudaStream_t s;
        ~Free() {
            if (p) cudaFreeAsync(p, s);
        }
    } f1{mx, s};
    KKB_TRY_CUDA(cudaMallocAsync(&planes, sizeof(__half) * 4 * plane_elems, s), "cudaMallocAsync(trace planes)");
    Free f2{planes, s};
    KKB_TRY_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned) * (size_t)n_frames, s), "zero frame max");
    const long long per = (long long)NM * T;
    const int bx = (int)std::max<long long>(1, std::min<long long>(ceil_div(per, 256), std::max(1, 148 * 4 / n_frames)));
    k_frame_maxabs<<<dim3(bx, n_frames), 256, 0, s>>>(data, data_fs, per, mx);
    KKB_CHECK_LAUNCH("k_frame_maxabs");
    const long long units = ngroups * NM * (long long)T;
    k_split_planes<<<(unsigned)std::min<long long>(ceil_div(units, 256), 148LL * 64), 256, 0, s>>>(
        data, data_fs, n_frames, NM, T, mx, ngroups, planes);
    KKB_CHECK_LAUNCH("k_split_planes");
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        void *fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
            set_error("kk tensor-core gather: cuTensorMapEncodeTiled unavailable");
            return KKB_ERR_CUDA;
        }
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    TcgArgs a{};
    {
        // (sample, frame) flattened: a window is one 512-byte row of the box
        const cuuint64_t dims[4] = {8ull * T, (cuuint64_t)NM, (cuuint64_t)ngroups, 4};
        const cuuint64_t strides[3] = {16ull * T, 16ull * T * NM, 16ull * T * NM * ngroups};
        const cuuint32_t box[4] = {8 * TCG_KW, 1, 8, 4}, estr[4] = {1, 1, 1, 1};
        const CUresult r = encode(&a.planes, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, planes, dims, strides, box, estr,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            set_error("kk tensor-core gather: cuTensorMapEncodeTiled failed (%d)", (int)r);
            return KKB_ERR_CUDA;
        }
    }
    a.N = N, a.M = M, a.T = T, a.ltx = ltx, a.ltzT = ltzT, a.lrx = lrx, a.lrzT = lrzT, a.w = w;
    a.fs = fs, a.shift = shift, a.nx = nx, a.nz = nz, a.out = out, a.out_kind = out_kind, a.out_fs = out_fs;
    a.inten = inten, a.fmax = fmax, a.accum = accum, a.n_frames = n_frames, a.maxabs = mx;
    constexpr int ASTAGE = 2 * (TCG_KW / 8) * 128 * 16, BSTAGE = 2 * 16 * TCG_KW * 16;
    const size_t smem = (size_t)TCG_NA * ASTAGE + (size_t)TCG_NB * BSTAGE + sizeof(double) * (size_t)(N + M) * (TCG_TX + TCG_TZ) +
                        sizeof(float) * (size_t)M + sizeof(int) * (size_t)NM;
    if (smem > 227 * 1024) {
        set_error("kk tensor-core gather: %d pairs do not fit shared memory", NM);
        return KKB_ERR_UNSUPPORTED;
    }
    dim3 grid((unsigned)(ceil_div(nz, TCG_TZ) * ceil_div(nx, TCG_TX)), (unsigned)ceil_div(n_frames, TCG_FB));
    if (linear) {
        KKB_TRY_CUDA(cudaFuncSetAttribute(k_kk_gather_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                     "smem attr kk tc");
        k_kk_gather_tc<true><<<grid, TCG_THREADS, smem, s>>>(a);
    } else {
        KKB_TRY_CUDA(cudaFuncSetAttribute(k_kk_gather_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                     "smem attr kk tc");
        k_kk_gather_tc<false><<<grid, TCG_THREADS, smem, s>>>(a);
    }
    KKB_CHECK_LAUNCH("k_kk_gather_tc");
    return KKB_OK;
}

}  // namespace kkb
