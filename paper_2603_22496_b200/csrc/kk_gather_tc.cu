// K5 on the 5th-generation tensor cores: the kk pixel gather (_kk_kernel,
// beamform.py:212-236) as a sequence of small GEMMs, one per (tx, rx) pair.
//
// For a tile of 128 pixels (4 depth rows x 32 lateral columns) and a block of
// 64 frames, the linear interpolation of pair (n, m) is
//     IQ[px, f] += sum_e  W_nm[px, e] * trace_nm[f, lo_nm + e],   e < 16 or 32
// where W_nm has at most two nonzeros per pixel row: w_m (1 - frac) at
// e = floor(fi) - lo and w_m frac at e + 1 (nearest: w_m at floor(fi + 0.5) - lo),
// and the row is all zero when the reference's in-window rule rejects the tap
// (beamform.py:226-235) — so the rule costs nothing in the product.  fi is the
// reference's float64 delay in its exact operation order (the FMA kernels'
// index arithmetic, bit for bit), frac its 23-bit weight.  The window start
// lo_nm and its length (16 or 32 samples: one or two K = 16 steps) come from
// the plan (k_kk_tc_windows, kk_gather.cu): every pixel of the tile evaluated
// with this same arithmetic, so the window provably holds every live tap.
//
// Operands: per K = 16 window samples three tcgen05.mma (kind::f16, M = 128
// pixels, N = 16 x frame groups = re | im of up to 64 frames): every operand
// is split into two fp16 halves x = hi + lo and the product sums
// hi*hi + hi*lo + lo*hi (lo*lo ~ 2^-22 dropped).  The traces are split ONCE
// per batch (k_split_planes: each frame scaled by a power of two so its
// largest sample sits just under 2^15) into four planes (hi/lo x re/im) laid
// out [frame group of 8][pair][sample][8 frames]: one 4-D TMA box (16 or 32
// samples x 8 frames as one row x 8 groups x 4 planes, cp.async.bulk.tensor)
// lands a pair's window for 64 frames directly in the MN-major operand
// layout, zero-filled where the window leaves the trace.  Weights are scaled
// by 2^12 so their low halves stay normal.  A batch holding a NaN / Inf
// sample is left to the FMA gather (the standby launch in kk_gather.cu): a
// tensor-core product would multiply it by the zero weights of every other
// pixel of the tile, where the reference touches only the pixels that tap it.
//
// Accumulation: tensor-core adds into a TMEM accumulator truncate (measured,
// scripts/ubench/tc_accum.cu: ~3e-8 relative drift per MMA), so pairs are
// summed in groups of TCG_GROUP = 16 into four rotating TMEM accumulators,
// and four drain warps add each finished group into float32 registers with
// round-to-nearest adds: the drift is bounded by one group's <= 96 MMAs
// (measured 9e-7 rel L2 against the FMA gather on the bench batch; groups of
// 8: 5e-7 and 11% slower, of 32: 1.7e-6 and 1% faster;
// profiles/r02_gather_tc_sweep.jsonl).
//
// Work item = (pixel tile, TWO 64-frame blocks): the per-pair protocol (weight
// rows, ring handshakes, window copies) costs ~335 cycles per (tile, pair)
// whatever the MMA width (profiles/r02f_gather_tc_role_profile.json), so one
// weight build serves both blocks' windows and accumulators (the item's K5
// time per frame falls 13%).  Warp roles (16 warps = 4 warpgroups,
// persistent CTAs, setmaxnreg): warpgroup 0 builds the weight rows of each
// pair (one row per thread, delay tables staged in shared memory); in
// warpgroup 1, warp 4 allocates TMEM and issues the TMA copies (one lane, both
// blocks' windows into one 32 KB stage), warp 5 issues the MMAs (one elected
// lane), warp 6 builds the next item's tile tables; warpgroups 2 and 3 drain
// set 0's / set 1's accumulators (two each in TMEM) and run the epilogue (IQ,
// fused |IQ|^2, per-frame max) with 168 registers while the other two
// warpgroups give theirs back (88).  Stages are guarded by full / empty
// mbarriers (tcgen05.commit frees a stage and publishes a group).

#include <algorithm>
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "kk.cuh"
#include "tc.cuh"
#include "tcplanes.cuh"

namespace kkb {

__device__ __forceinline__ double tc_kk_delay(double t1, double lz, double lx, double fs, double shift) {
    return __dadd_rn(__dmul_rn(__dsub_rn(__dadd_rn(t1, lz), lx), fs), shift);
}
#define TCG_MAGIC2 1572864.0   // 1.5 * 2^20 (kk_gather.cu KKB_FLOOR_MAGIC2)
#define TCG_MAGIC2_HI 0x41380000
#define TCG_WSCALE 4096.0f     // weights x 2^12: their fp16 low halves stay normal
#define TCG_TZ KKB_KK_TC_TZ
#define TCG_TX KKB_KK_TC_TX
#define TCG_KW KKB_KK_TC_W     // window samples per pair (two K steps)
#define TCG_FB 64              // frames per CTA: N = 128 (re | im)
#ifndef TCG_NA
#define TCG_NA 4               // weight (A) stages
#endif
#ifndef TCG_NB
#define TCG_NB 4               // trace-window (B) stages (they hide the TMA latency), TCG_SETS windows each
#endif
#define TCG_SETS 2             // frame blocks per item: one weight build serves both
#ifndef TCG_PB
#define TCG_PB 2               // pairs per producer iteration
#endif
#ifndef TCG_GROUP
#define TCG_GROUP 16           // pairs per accumulator group
#endif
#define TCG_ND 4               // TMEM accumulators (128 columns each): 2 per frame-block set
#define TCG_NDS (TCG_ND / TCG_SETS)
#define TCG_THREADS 512        // 16 warps = 4 warpgroups (setmaxnreg per role)
#define TCG_REGS_LO 88         // producers, TMA / MMA / table warps
#define TCG_REGS_HI 168        // drains (128 fp32 partial sums each)
static_assert(2 * 128 * TCG_REGS_LO + 2 * 128 * TCG_REGS_HI == TCG_THREADS * 128, "register pool");
#ifndef TCG_EXP_SKIP2
#define TCG_EXP_SKIP2 0        // experiment builds: 1 = skip the second K step of two-step pairs
#endif

// A / TMEM row r -> tile pixel (column cl, depth row rl).  Lanes r, r+8,
// r+16, r+24 of a warp take the four depth rows of one column: their delays
// differ by a few samples, so the weight-row words they store (rows 16 B
// apart: the same bank quad) usually land in different banks, where rows 8
// apart at one depth (r = cl * 4 + rl) mostly collided 4-way.
static_assert(TCG_TZ == 4 && TCG_TX == 32, "row map assumes 4 x 32 tiles");
__device__ __forceinline__ int tcg_col(int r) { return (r & 7) + 8 * (r >> 5); }
__device__ __forceinline__ int tcg_row(int r) { return (r >> 3) & 3; }

// per-frame max |re|, |im| of the traces (float bits; atomicMax on
// non-negative floats).  V complex samples per load (2: 16-byte loads, when
// the frame stride and length are even and the base 16-byte aligned).
template <int V>
__global__ void __launch_bounds__(256) k_frame_maxabs(const float2 *__restrict__ data, long long data_fs,
                                                      long long per_frame, unsigned *__restrict__ out,
                                                      unsigned *__restrict__ nonfinite) {
    const int f = blockIdx.y;
    const float2 *d = data + (long long)f * data_fs;
    // max of the magnitude bits: finite < Inf (0x7f800000) < NaN
    unsigned m = 0;
    const long long nv = per_frame / V;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
        if (V == 2) {
            const float4 v = __ldg(reinterpret_cast<const float4 *>(d) + i);
            m = max(max(m, max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu)),
                    max(__float_as_uint(v.z) & 0x7fffffffu, __float_as_uint(v.w) & 0x7fffffffu));
        } else {
            const float2 v = __ldg(d + i);
            m = max(m, max(__float_as_uint(v.x) & 0x7fffffffu, __float_as_uint(v.y) & 0x7fffffffu));
        }
    }
    const unsigned mx = __reduce_max_sync(0xffffffffu, m);
    __shared__ unsigned wm[8];
    if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned r = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = max(r, wm[w]);
        if (r >= 0x7f800000u) atomicOr(nonfinite, 1u);
        else if (r) atomicMax(out + f, r);
    }
}

// planes[pl][g][q][t][8]: pl = re_hi, im_hi, re_lo, im_lo; frames 8g..8g+7.
// A thread owns V consecutive samples of one (g, q) row: 8 frame loads of
// V complex each, 4 planes x V 16-byte stores.
template <int V>
__global__ void __launch_bounds__(256) k_split_planes(const float2 *__restrict__ data, long long data_fs,
                                                      int n_frames, int NM, int T,
                                                      const unsigned *__restrict__ maxabs, long long ngroups,
                                                      __half *__restrict__ planes) {
    const long long per_plane = ngroups * NM * (long long)T * 8;
    const int TV = T / V;
    const long long total = ngroups * NM * (long long)TV;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int tv = (int)(i % TV);
        const long long gq = i / TV;
        const int q = (int)(gq % NM);
        const long long g = gq / NM;
        float2 v[8][V];
        float sc[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const long long f = g * 8 + j;
            sc[j] = 1.0f;
#pragma unroll
            for (int u = 0; u < V; ++u) v[j][u] = make_float2(0.f, 0.f);
            if (f < n_frames) {
                const float2 *src = data + f * data_fs + (long long)q * T + (long long)tv * V;
                if (V == 2) {
                    const float4 x = __ldg(reinterpret_cast<const float4 *>(src));
                    v[j][0] = make_float2(x.x, x.y);
                    v[j][V - 1] = make_float2(x.z, x.w);
                } else {
                    v[j][0] = __ldg(src);
                }
                sc[j] = frame_scale(__ldg(maxabs + f));
            }
        }
        uint4 *dst = reinterpret_cast<uint4 *>(planes) + gq * T + (long long)tv * V;
#pragma unroll
        for (int u = 0; u < V; ++u) {
            __half h[4][8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                split_h(v[j][u].x * sc[j], h[0][j], h[2][j]);
                split_h(v[j][u].y * sc[j], h[1][j], h[3][j]);
            }
#pragma unroll
            for (int pl = 0; pl < 4; ++pl)
                dst[pl * (per_plane / 8) + u] = make_uint4(pack_h2(h[pl][0], h[pl][1]), pack_h2(h[pl][2], h[pl][3]),
                                                           pack_h2(h[pl][4], h[pl][5]), pack_h2(h[pl][6], h[pl][7]));
        }
    }
}

struct TcgArgs {
    // 4-D maps of the split trace planes: [0] 32-sample windows, [1] 16-sample
    // windows (one K step); boxes of 8 frame groups, and of the last frame
    // block's gt groups for the tail maps
    CUtensorMap planes[2], tail[2];
    int gt;                  // frame groups (of 8) in the last frame block
    int nfb;                 // frame blocks
    const int *tc_lo;        // [tile][pair] window start * 2 + one-K-step flag (plan time, exact)
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
    const unsigned *maxabs;     // per-frame max |sample| (float bits)
    const unsigned *nonfinite;  // != 0: a NaN / Inf sample; the FMA gather runs instead
    int tiles_z;                // pixel tiles along depth
    long long tiles, items;     // work item = frame block * tiles + pixel tile
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

// per-slot delay tables of one pixel tile: [ltx N][TX] [ltz N][TZ] [lrx M][TX]
// [lrz M][TZ] (fp64) then the window starts lo [N*M] (int)
struct TcgTables {
    double *ltx, *ltz, *lrx, *lrz;
    int *lo;
};
__device__ __forceinline__ TcgTables tcg_tables(unsigned char *base, int N, int M) {
    TcgTables t;
    t.ltx = reinterpret_cast<double *>(base);
    t.ltz = t.ltx + N * TCG_TX;
    t.lrx = t.ltz + N * TCG_TZ;
    t.lrz = t.lrx + M * TCG_TX;
    t.lo = reinterpret_cast<int *>(t.lrz + M * TCG_TZ);
    return t;
}
__host__ __device__ __forceinline__ size_t tcg_slot_bytes(int N, int M) {
    return ((sizeof(double) * (size_t)(N + M) * (TCG_TX + TCG_TZ) + sizeof(int) * (size_t)N * M) + 15) & ~(size_t)15;
}

// Persistent: one CTA per SM walks work items (64-frame block, pixel tile)
// strided by the grid.  The rings, the accumulator
// sequence and the table slots run across items, so the drains' epilogue of
// one item overlaps the next item's MMAs (four TMEM accumulators give the
// MMA three groups of slack) and a table builder warp prepares the next
// item's tile tables while the current item runs.
template <bool LINEAR>
__global__ void __launch_bounds__(TCG_THREADS, 1)
k_kk_gather_tc(const __grid_constant__ TcgArgs a) {
    constexpr int KC = TCG_KW / 8;                 // 16-byte K chunks per weight row
    constexpr int A_PLANE = KC * 128 * 16;          // 8 KB: one split half of the weights (K-major)
    constexpr int B_PLANE = 16 * TCG_KW * 16;       // 8 KB: one split half of the traces (MN-major, 16 col groups)
    constexpr int ASTAGE = 2 * A_PLANE, BSET = 2 * B_PLANE, BSTAGE = TCG_SETS * BSET;
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint64_t a_full[TCG_NA], a_empty[TCG_NA], b_full[TCG_NB], b_empty[TCG_NB];
    __shared__ uint64_t dfull[TCG_ND], dfree[TCG_ND], tab_full[2], tab_empty[2];
    __shared__ uint32_t tmem_base;
    __shared__ int b_k16[TCG_NB];  // per B stage: 1 = a 16-sample window (one K step)
    __shared__ unsigned fm_s[TCG_SETS][2][4][TCG_FB];  // per set and item parity: each drain warp's frame maxima

    // a batch with a non-finite sample goes to the FMA gather (NaN x 0 would
    // spread it over the whole window); uniform, before any barrier
    if (*a.nonfinite) return;

    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    const int N = a.N, M = a.M, T = a.T, nx = a.nx, nz = a.nz;
    const double fs = a.fs, shift = a.shift;
    const int npairs = N * M;
    const int ngroups = (npairs + TCG_GROUP - 1) / TCG_GROUP;
    unsigned char *tab_base = sm + TCG_NA * ASTAGE + TCG_NB * BSTAGE;
    const size_t slot_bytes = tcg_slot_bytes(N, M);
    float *w_s = reinterpret_cast<float *>(tab_base + 2 * slot_bytes);  // [M] weights x 2^12
    // this CTA's items: blockIdx.x + k * gridDim.x.  Items run frame block
    // major, so the CTAs in flight share one frame block's trace planes in L2
    const int nit = (int)((a.items - blockIdx.x + gridDim.x - 1) / gridDim.x);
    auto item_of = [&](int k) { return (long long)blockIdx.x + (long long)k * gridDim.x; };
    auto tile_of = [&](int k) { return (int)(item_of(k) % a.tiles); };
    // item k covers frame blocks TCG_SETS * (item / tiles) + s, s < TCG_SETS
    auto fb_of = [&](int k, int set) { return (int)(item_of(k) / a.tiles) * TCG_SETS + set; };

    if (warp == 4) tc::tmem_alloc<32 * 4 * TCG_ND>(&tmem_base);
    if (t == 0) {
        for (int s = 0; s < TCG_NA; ++s) {
            tc::mbar_init(&a_full[s], 128);  // the 128 weight rows
            tc::mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < TCG_NB; ++s) {
            tc::mbar_init(&b_full[s], 1);    // the TMA issuer (expect_tx)
            tc::mbar_init(&b_empty[s], 1);
        }
        for (int d = 0; d < TCG_ND; ++d) {
            tc::mbar_init(&dfull[d], 1);
            tc::mbar_init(&dfree[d], 128);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&tab_full[s], 32);       // the builder warp
            tc::mbar_init(&tab_empty[s], 128 + 1); // weight rows + TMA issuer
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < 2; ++i) {
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.planes[i])) : "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&a.tail[i])) : "memory");
        }
    }
    for (int i = t; i < M; i += blockDim.x) w_s[i] = (a.w ? (float)__ldg(a.w + i) : 1.0f) * TCG_WSCALE;
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;

    if (warp < 4) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TCG_REGS_LO));
        // ------------------------------------------------------------ weight rows
        // A row holds two nonzero halves (w0 at window sample e, w1 at e + 1)
        // in 32: the A ring is zeroed once, then each pair writes the two
        // 32-bit words that carry them and clears the words it wrote in the
        // same stage one round earlier (4 x STS.32 per plane).
        const int r = t, cl = tcg_col(r), rl = tcg_row(r);
        unsigned char *row = sm + r * 16;
#pragma unroll
        for (int st = 0; st < TCG_NA; ++st)
#pragma unroll
            for (int c = 0; c < 2 * KC; ++c)
                *reinterpret_cast<uint4 *>(row + st * ASTAGE + c * 128 * 16) = make_uint4(0, 0, 0, 0);
        // byte offset of 32-bit word k (half pair 2k, 2k + 1) of the row
        auto word = [](int k) { return (k >> 2) * (128 * 16) + (k & 3) * 4; };
        uint32_t prevk = 0;  // per stage (4 bits each): first word written last round
        unsigned P = 0;      // pairs issued so far (the rings' sequence)
#ifdef TCG_EXP_PROFILE
        long long pprof[3] = {0, 0, 0};  // loop cycles, a_empty wait cycles, tab_full wait cycles
        const long long pt0 = clock64();
#endif
        for (int k = 0; k < nit; ++k) {
            const int slot = k & 1;
#ifdef TCG_EXP_PROFILE
            const long long tw0 = clock64();
#endif
            tc::mbar_wait(&tab_full[slot], (k >> 1) & 1);
#ifdef TCG_EXP_PROFILE
            pprof[2] += clock64() - tw0;
#endif
            const TcgTables tb = tcg_tables(tab_base + slot * slot_bytes, N, M);
            int n = 0, m = 0;
            // TCG_PB pairs per iteration: independent delay chains in flight
            // and one proxy fence per batch
            for (int pr0 = 0; pr0 < npairs; pr0 += TCG_PB) {
#ifdef TCG_EXP_NO_PROD  // experiment builds: the ring handshakes without weight rows
                {
                    const int nb = min(TCG_PB, npairs - pr0);
                    for (int j = 0; j < nb; ++j) {
                        const unsigned pp = P + j, use = pp / TCG_NA;
                        if (use > 0) tc::mbar_wait(&a_empty[(int)(pp % TCG_NA)], (uint32_t)((use - 1) & 1));
                    }
                    for (int j = 0; j < nb; ++j) mbar_arrive(&a_full[(int)((P + j) % TCG_NA)]);
                    P += nb;
                    continue;
                }
#endif
                uint32_t hA[TCG_PB], hB[TCG_PB], lA[TCG_PB], lB[TCG_PB];
                int kA[TCG_PB];
#pragma unroll
                for (int j = 0; j < TCG_PB; ++j) {
                    const int pr = min(pr0 + j, npairs - 1);
                    const double t1 = __dadd_rn(tb.ltx[n * TCG_TX + cl], tb.ltz[n * TCG_TZ + rl]);
                    const double fi = tc_kk_delay(t1, tb.lrz[m * TCG_TZ + rl], tb.lrx[m * TCG_TX + cl], fs, shift);
                    const float wm = w_s[m];
                    const int lo = tb.lo[pr] >> 1;  // bit 0: the one-K-step flag
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
                    uint32_t hw, lw;  // pack_h2(hi(w0), hi(w1)), pack_h2(lo(w0), lo(w1))
                    split_h2(w0, w1, hw, lw);
                    const bool odd = e & 1;
                    hA[j] = odd ? hw << 16 : hw;
                    hB[j] = odd ? hw >> 16 : 0u;
                    lA[j] = odd ? lw << 16 : lw;
                    lB[j] = odd ? lw >> 16 : 0u;
                    kA[j] = ok ? e >> 1 : 0;
                    if (++m == M) {
                        m = 0;
                        ++n;
                    }
                }
                const int nb = min(TCG_PB, npairs - pr0);
#pragma unroll
                for (int j = 0; j < TCG_PB; ++j) {
                    if (j >= nb) break;
                    const unsigned pp = P + j;
                    const int st = (int)(pp % TCG_NA);
                    const unsigned use = pp / TCG_NA;
                    unsigned char *Ab = row + st * ASTAGE;
                    if (use > 0) {
#ifdef TCG_EXP_PROFILE
                        const long long w0 = clock64();
#endif
                        tc::mbar_wait(&a_empty[st], (uint32_t)((use - 1) & 1));
#ifdef TCG_EXP_PROFILE
                        pprof[1] += clock64() - w0;
#endif
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
#ifndef TCG_EXP_NO_FENCE  // experiment builds: timing without the proxy fence (unsafe)
                tc::fence_smem_to_async();
#endif
#pragma unroll
                for (int j = 0; j < TCG_PB; ++j)
                    if (j < nb) mbar_arrive(&a_full[(int)((P + j) % TCG_NA)]);
                P += nb;
            }
            mbar_arrive(&tab_empty[slot]);  // this item's tables read
        }
#ifdef TCG_EXP_PROFILE
        pprof[0] = clock64() - pt0;
        if (t == 0)
            for (int i = 0; i < 3; ++i)
                atomicAdd(reinterpret_cast<unsigned long long *>(a.fmax) + 230 + i, (unsigned long long)pprof[i]);
#endif
    } else if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(TCG_REGS_LO));
      if (warp == 4) {
        // ------------------------------------------------------------ trace windows (TMA)
        // box [plane 4][group 8][sample 32 (or 16)][frame 8] = B hi (re
        // groups | im groups) then B lo: column group = im * 8 + g, 512 (256) B apart
        if (lane == 0) {
            unsigned P = 0;
#ifdef TCG_EXP_PROFILE
            long long bprof = 0;
            const long long bt0 = clock64();
#endif
            for (int k = 0; k < nit; ++k) {
                const int slot = k & 1;
                tc::mbar_wait(&tab_full[slot], (k >> 1) & 1);
                const int *lo = tcg_tables(tab_base + slot * slot_bytes, N, M).lo;
                // the item's frame blocks: set s is block fb_of(k, s) when it exists
                int fbs[TCG_SETS];
                uint32_t Gs[TCG_SETS];
#pragma unroll
                for (int st2 = 0; st2 < TCG_SETS; ++st2) {
                    fbs[st2] = fb_of(k, st2);
                    Gs[st2] = fbs[st2] >= a.nfb ? 0u : fbs[st2] == a.nfb - 1 ? (uint32_t)a.gt : TCG_FB / 8;
                }
                for (int pr = 0; pr < npairs; ++pr, ++P) {
                    const int st = (int)(P % TCG_NB);
                    const unsigned use = P / TCG_NB;
#ifdef TCG_EXP_PROFILE
                    const long long b0 = clock64();
#endif
                    if (use > 0) tc::mbar_wait(&b_empty[st], (uint32_t)((use - 1) & 1));
#ifdef TCG_EXP_PROFILE
                    bprof += clock64() - b0;
#endif
                    const int v = lo[pr], one = v & 1;
                    b_k16[st] = one;  // published to the MMA warp by the arrive below
                    // per set: 4 planes x G groups x (16 or 32) samples x 16 B
                    uint32_t bytes = 0;
#pragma unroll
                    for (int st2 = 0; st2 < TCG_SETS; ++st2) bytes += 4 * Gs[st2] * (one ? 16 : TCG_KW) * 16;
#ifdef TCG_EXP_NO_TMA  // experiment builds: the ring handshakes without the copies
                    (void)bytes;
                    mbar_arrive(&b_full[st]);
#else
                    mbar_arrive_tx(&b_full[st], bytes);
#pragma unroll
                    for (int st2 = 0; st2 < TCG_SETS; ++st2)
                        if (Gs[st2])
                            tma_4d(sm + TCG_NA * ASTAGE + st * BSTAGE + st2 * BSET,
                                   fbs[st2] == a.nfb - 1 ? &a.tail[one] : &a.planes[one], 8 * (v >> 1), pr,
                                   fbs[st2] * (TCG_FB / 8), 0, &b_full[st]);
#endif
                }
                mbar_arrive(&tab_empty[slot]);
            }
#ifdef TCG_EXP_PROFILE
            atomicAdd(reinterpret_cast<unsigned long long *>(a.fmax) + 233, (unsigned long long)(clock64() - bt0));
            atomicAdd(reinterpret_cast<unsigned long long *>(a.fmax) + 234, (unsigned long long)bprof);
#endif
        }
      } else if (warp == 5) {
        // ------------------------------------------------------------ MMA issue
        // The whole warp runs the (warp-uniform) loop and one elected lane
        // issues a pair's six MMAs from one asm block: descriptors stay in
        // uniform registers, no per-MMA lane election.
        const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(sm);
        unsigned P = 0, G = 0;  // pairs and accumulator groups so far
#ifdef TCG_EXP_PROFILE
        long long prof[5] = {0, 0, 0, 0, 0};
#endif
        for (int k = 0; k < nit; ++k) {
            // per set: N = 16 x frame groups, re columns [0, 8g), im [8g, 16g);
            // g = 0 when the item has no frame block for the set
            uint32_t gset[TCG_SETS], idesc[TCG_SETS];
#pragma unroll
            for (int st2 = 0; st2 < TCG_SETS; ++st2) {
                const int fb = fb_of(k, st2);
                gset[st2] = fb >= a.nfb ? 0u : fb == a.nfb - 1 ? (uint32_t)a.gt : TCG_FB / 8;
                idesc[st2] = tc::instr_desc(0, 128, 16 * (gset[st2] ? gset[st2] : 1), 1);
            }
            for (int pr = 0; pr < npairs; ++pr, ++P) {
                const int sa_ = (int)(P % TCG_NA), sb_ = (int)(P % TCG_NB), d = (int)(G % TCG_NDS);
                const bool first = pr % TCG_GROUP == 0, last = pr % TCG_GROUP == TCG_GROUP - 1 || pr == npairs - 1;
#ifdef TCG_EXP_PROFILE  // experiment builds: where the MMA warp's cycles go
                long long c_0 = clock64();
#endif
                if (first && G >= TCG_NDS) {  // both sets' accumulator d drained
#pragma unroll
                    for (int st2 = 0; st2 < TCG_SETS; ++st2)
                        tc::mbar_wait(&dfree[st2 * TCG_NDS + d], (uint32_t)((G / TCG_NDS - 1) & 1));
                }
#ifdef TCG_EXP_PROFILE
                long long c_1 = clock64();
#endif
                tc::mbar_wait(&a_full[sa_], (uint32_t)((P / TCG_NA) & 1));
#ifdef TCG_EXP_PROFILE
                long long c_2 = clock64();
#endif
                tc::mbar_wait(&b_full[sb_], (uint32_t)((P / TCG_NB) & 1));
#ifdef TCG_EXP_PROFILE
                long long c_3 = clock64();
#endif
                tc::fence_after_sync();
                const uint32_t sa = s0 + sa_ * ASTAGE;
                const bool one = b_k16[sb_] != 0;
                // B: column groups of (16 or 32 samples) x 16 B; B lo after the 2g hi groups
                const uint32_t kb = one ? 16 * 16 : TCG_KW * 16;
                const uint64_t ah = tc::smem_desc(sa, 128 * 16, 128), al = tc::smem_desc(sa + A_PLANE, 128 * 16, 128);
                if (tc::elect_one()) {
                    // one weight build (A) serves every set's frame block (B window, accumulator)
#pragma unroll
                    for (int st2 = 0; st2 < TCG_SETS; ++st2) {
                        if (!gset[st2]) continue;
                        const uint32_t sb = s0 + TCG_NA * ASTAGE + sb_ * BSTAGE + st2 * BSET;
                        const uint32_t dacc = tmem + (uint32_t)((st2 * TCG_NDS + d) * 128);
                        const uint64_t bh = tc::smem_desc(sb, 128, kb), bl = tc::smem_desc(sb + 2 * gset[st2] * kb, 128, kb);
#ifndef TCG_EXP_NO_MMA  // experiment builds: the pipeline without the MMAs
                        tc::mma_f16_split3(dacc, ah, al, bh, bl, idesc[st2], !first);
#endif
                        if (!one && !TCG_EXP_SKIP2)  // second K = 16 half: A + 2 chunks, B + 2 K groups
                            tc::mma_f16_split3(dacc, ah + ((2 * 128 * 16) >> 4), al + ((2 * 128 * 16) >> 4),
                                               bh + ((2 * 128) >> 4), bl + ((2 * 128) >> 4), idesc[st2], true);
                    }
                    tc::commit(&a_empty[sa_]);
                    tc::commit(&b_empty[sb_]);
                    if (last) {  // every set's drains run the group protocol, used or not
#pragma unroll
                        for (int st2 = 0; st2 < TCG_SETS; ++st2) tc::commit(&dfull[st2 * TCG_NDS + d]);
                    }
                }
                __syncwarp();
#ifdef TCG_EXP_PROFILE
                long long c_4 = clock64();
                prof[0] += c_1 - c_0;
                prof[1] += c_2 - c_1;
                prof[2] += c_3 - c_2;
                prof[3] += c_4 - c_3;
                prof[4] += 1;
#endif
                if (last) ++G;
            }
        }
#ifdef TCG_EXP_PROFILE
        if (lane == 0)
            for (int i = 0; i < 5; ++i) atomicAdd(reinterpret_cast<unsigned long long *>(a.fmax) + 220 + i, (unsigned long long)prof[i]);
#endif
      } else if (warp == 6) {
        // ------------------------------------------------------------ tile tables (next items)
        int held[2] = {-1, -1};  // tile held by each slot
        for (int k = 0; k < nit; ++k) {
            const int slot = k & 1, tile = tile_of(k);
            if (k >= 2) tc::mbar_wait(&tab_empty[slot], (uint32_t)(((k >> 1) - 1) & 1));
#ifdef TCG_EXP_NO_TAB  // experiment builds: stale tables (timing only)
            if (held[slot] != tile && held[slot] >= 0) held[slot] = tile;
#endif
            if (held[slot] != tile) {
                const TcgTables tb = tcg_tables(tab_base + slot * slot_bytes, N, M);
                const int iz0 = (tile % a.tiles_z) * TCG_TZ, ix0 = (tile / a.tiles_z) * TCG_TX;
                // edge tiles repeat the last row / column
                for (int i = lane; i < N * TCG_TX; i += 32) {
                    const int n = i / TCG_TX, c = i - n * TCG_TX;
                    tb.ltx[i] = __ldg(a.ltx + (long long)min(ix0 + c, nx - 1) * N + n);
                }
                for (int i = lane; i < N * TCG_TZ; i += 32) {
                    const int n = i / TCG_TZ, rr = i - n * TCG_TZ;
                    tb.ltz[i] = __ldg(a.ltzT + (long long)n * nz + min(iz0 + rr, nz - 1));
                }
                for (int i = lane; i < M * TCG_TX; i += 32) {
                    const int m = i / TCG_TX, c = i - m * TCG_TX;
                    tb.lrx[i] = __ldg(a.lrx + (long long)min(ix0 + c, nx - 1) * M + m);
                }
                for (int i = lane; i < M * TCG_TZ; i += 32) {
                    const int m = i / TCG_TZ, rr = i - m * TCG_TZ;
                    tb.lrz[i] = __ldg(a.lrzT + (long long)m * nz + min(iz0 + rr, nz - 1));
                }
                const int *src = a.tc_lo + (long long)tile * npairs;
                for (int i = lane; i < npairs; i += 32) tb.lo[i] = __ldg(src + i);
                held[slot] = tile;
            }
            mbar_arrive(&tab_full[slot]);
        }
      }  // warp 7: no role
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(TCG_REGS_HI));
        // ------------------------------------------------------------ drains + epilogue
        // warpgroup 2 drains set 0's accumulators, warpgroup 3 set 1's
        const int set = (warp - 8) >> 2, quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = tmem + ((uint32_t)(quarter * 32) << 16);
        unsigned G = 0;
        for (int k = 0; k < nit; ++k) {
            float S[2 * TCG_FB];
#pragma unroll
            for (int c = 0; c < 2 * TCG_FB; ++c) S[c] = 0.f;
            const int fbk = fb_of(k, set);
            // re [0, 8g), im [8g, 16g); g = 0: no frame block for this set (handshakes only)
            const uint32_t g = fbk >= a.nfb ? 0u : fbk == a.nfb - 1 ? (uint32_t)a.gt : TCG_FB / 8;
            for (int grp = 0; grp < ngroups; ++grp, ++G) {
                const int d = set * TCG_NDS + (int)(G % TCG_NDS);
                tc::mbar_wait(&dfull[d], (uint32_t)((G / TCG_NDS) & 1));
                tc::fence_after_sync();
                const uint32_t col = lane_base + d * 128;
#ifdef TCG_EXP_NO_DRAIN  // experiment builds: drains hand the accumulator straight back
                tc::fence_before_sync();
                mbar_arrive(&dfree[d]);
                continue;
#endif
#pragma unroll
                for (int c0 = 0; c0 < TCG_FB; c0 += 8) {
                    if (c0 < 8 * (int)g) {  // warp-uniform
                        float v[8], u[8];
                        tc::tmem_ld8(col + c0, v);
                        tc::tmem_ld8(col + 8 * g + c0, u);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            S[c0 + i] = __fadd_rn(S[c0 + i], v[i]);
                            S[TCG_FB + c0 + i] = __fadd_rn(S[TCG_FB + c0 + i], u[i]);
                        }
                    }
                }
                tc::fence_before_sync();
                mbar_arrive(&dfree[d]);
            }
#ifdef TCG_EXP_NO_EPI  // experiment builds: drains without the epilogue
            if (S[0] == 12345.f) a.fmax[0] = 1u;  // keep the drains' adds alive
            continue;
#endif
            if (!g) continue;
            // epilogue: straight-line passes over the 64 frames (IQ, |IQ|^2,
            // per-frame max), each frame independent of the others
            const int tile = tile_of(k), f0 = fbk * TCG_FB;
            const int FB = min(TCG_FB, a.n_frames - f0);
            const int ix = (tile / a.tiles_z) * TCG_TX + tcg_col(r), iz = (tile % a.tiles_z) * TCG_TZ + tcg_row(r);
            const bool pix = ix < nx && iz < nz;
            const long long px0 = (long long)f0 * a.out_fs + (long long)ix * nz + iz;
#pragma unroll
            for (int f = 0; f < TCG_FB; ++f) {
                // exact: the product of two powers of two
                const float sc = frame_scale(__ldg(a.maxabs + min(f0 + f, a.n_frames - 1)));
                const float inv = f < FB ? 1.0f / (sc * TCG_WSCALE) : 0.f;
                S[f] *= inv;
                S[TCG_FB + f] *= inv;
            }
            if (a.out && pix) {
                if (a.out_kind == KKB_OUT_C128) {
#pragma unroll
                    for (int f = 0; f < TCG_FB; ++f)
                        if (f < FB)
                            reinterpret_cast<double2 *>(a.out)[px0 + f * a.out_fs] = make_double2(S[f], S[TCG_FB + f]);
                } else {
#pragma unroll
                    for (int f = 0; f < TCG_FB; ++f)
                        if (f < FB)
                            reinterpret_cast<float2 *>(a.out)[px0 + f * a.out_fs] = make_float2(S[f], S[TCG_FB + f]);
                }
            }
            if (a.inten) {
#pragma unroll
                for (int f = 0; f < TCG_FB; ++f) S[f] = pix ? __fmaf_rn(S[f], S[f], __fmul_rn(S[TCG_FB + f], S[TCG_FB + f])) : 0.f;
                if (pix) {
                    if (a.accum) {
#pragma unroll
                        for (int f = 0; f < TCG_FB; ++f)
                            if (f < FB) S[f] = __fadd_rn(S[f], a.inten[px0 + f * a.out_fs]);
                    }
#pragma unroll
                    for (int f = 0; f < TCG_FB; ++f)
                        if (f < FB) a.inten[px0 + f * a.out_fs] = S[f];
                }
                if (a.fmax) {
                    // non-negative floats order like their bit patterns: one redux per
                    // frame and warp, the four drain warps combined in shared memory,
                    // then one atomic per frame and item (the CTAs in flight share a
                    // frame block, so per-warp atomics contend on 64 addresses)
                    unsigned *fm = fm_s[set][k & 1][quarter];
#pragma unroll
                    for (int f = 0; f < TCG_FB; ++f) {
                        const unsigned mx = __reduce_max_sync(0xffffffffu, __float_as_uint(S[f]));
                        if (lane == 0) fm[f] = mx;
                    }
                    // the set's four drain warps (named barrier 1 + set)
                    asm volatile("bar.sync %0, 128;" ::"r"(1 + set) : "memory");
                    const int dr = (warp - 8 - 4 * set) * 32 + lane;  // 0..127
                    if (dr < FB) {
                        const unsigned m4 = max(max(fm_s[set][k & 1][0][dr], fm_s[set][k & 1][1][dr]),
                                                max(fm_s[set][k & 1][2][dr], fm_s[set][k & 1][3][dr]));
                        atomicMax(a.fmax + f0 + dr, m4);
                    }
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 4) {
        __syncwarp();
        tc::tmem_free<32 * 4 * TCG_ND>(tmem);
    }
}

static size_t tcg_smem_bytes(int N, int M) {
    return (size_t)TCG_NA * (2 * (TCG_KW / 8) * 128 * 16) + (size_t)TCG_NB * TCG_SETS * (2 * 16 * TCG_KW * 16) +
           2 * tcg_slot_bytes(N, M) + sizeof(float) * (size_t)M;
}

// The gather proper on split planes (tcplanes.cuh) with per-frame scale bounds
// mx and the non-finite flag (the kernel stands down when it is set).
static int tcg_launch(const __half *planes, const unsigned *mx, const unsigned *nonfinite, int N, int M, int T,
                      const double *ltx, const double *ltzT, const double *lrx, const double *lrzT, int nx, int nz,
                      const double *w, double fs, double shift, int linear, void *out, int out_kind, int n_frames,
                      long long out_fs, float *inten, unsigned *fmax, const int *tc_lo, int accum, cudaStream_t s) {
    const int NM = N * M;
    const long long ngroups = (n_frames + 7) / 8;
    const size_t smem = tcg_smem_bytes(N, M);
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
        const cuuint32_t estr[4] = {1, 1, 1, 1};
        a.nfb = (int)ceil_div(ngroups, TCG_FB / 8);
        a.gt = (int)(ngroups - (long long)(a.nfb - 1) * (TCG_FB / 8));
        CUresult r = CUDA_SUCCESS;
        for (int one = 0; one < 2 && r == CUDA_SUCCESS; ++one)
            for (int tl = 0; tl < 2 && r == CUDA_SUCCESS; ++tl) {
                const cuuint32_t box[4] = {8u * (one ? 16u : (unsigned)TCG_KW), 1, tl ? (cuuint32_t)a.gt : 8u, 4};
                r = encode(tl ? &a.tail[one] : &a.planes[one], CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<__half *>(planes), dims,
                           strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
        if (r != CUDA_SUCCESS) {
            set_error("kk tensor-core gather: cuTensorMapEncodeTiled failed (%d)", (int)r);
            return KKB_ERR_CUDA;
        }
    }
    a.N = N, a.M = M, a.T = T, a.ltx = ltx, a.ltzT = ltzT, a.lrx = lrx, a.lrzT = lrzT, a.w = w;
    a.fs = fs, a.shift = shift, a.nx = nx, a.nz = nz, a.out = out, a.out_kind = out_kind, a.out_fs = out_fs;
    a.inten = inten, a.fmax = fmax, a.accum = accum, a.n_frames = n_frames, a.maxabs = mx;
    a.nonfinite = nonfinite;
    a.tc_lo = tc_lo;
    a.tiles_z = (int)ceil_div(nz, TCG_TZ);
    a.tiles = (long long)a.tiles_z * ceil_div(nx, TCG_TX);
    a.items = a.tiles * ceil_div(a.nfb, TCG_SETS);  // items of TCG_SETS frame blocks
    const unsigned grid = (unsigned)std::min<long long>(a.items, sm_count());
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

// The split planes are the size of the traces (~600 MB for the bench batch).
// Keep freed stream-ordered blocks in the device's pool across
// synchronisations (default release threshold 0 hands them back to the
// driver at every sync, and remapping them costs milliseconds per call).
static void keep_pool_blocks() {
    static int pool_kept = -1;
    if (pool_kept < 0) {
        int dev = 0;
        cudaMemPool_t pool;
        pool_kept = cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess;
        if (pool_kept) {
            unsigned long long keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        cudaGetLastError();
    }
}

int kk_gather_tc(const float2 *data, int N, int M, int T, const double *ltx, const double *ltzT,
                 const double *lrx, const double *lrzT, int nx, int nz, const double *w, double fs,
                 double shift, int linear, void *out, int out_kind, int n_frames, long long data_fs,
                 long long out_fs, float *inten, unsigned *fmax, const int *tc_lo, int accum,
                 cudaStream_t s, const std::function<int(const unsigned *)> &fma_fallback) {
    if (!tc_lo) return KKB_ERR_UNSUPPORTED;
    const int NM = N * M;
    const long long ngroups = (n_frames + 7) / 8;
    const size_t plane_elems = (size_t)ngroups * NM * T * 8;
    if (tcg_smem_bytes(N, M) > 227 * 1024) {
        set_error("kk tensor-core gather: %d pairs do not fit shared memory", NM);
        return KKB_ERR_UNSUPPORTED;
    }
    keep_pool_blocks();
    unsigned *mx = nullptr;  // [n_frames] frame max, then the non-finite flag
    __half *planes = nullptr;
    KKB_TRY_CUDA(cudaMallocAsync(&mx, sizeof(unsigned) * ((size_t)n_frames + 1), s), "cudaMallocAsync(frame max)");
    struct Free {
        void *p;
        cudaStream_t s;
        ~Free() {
            if (p) cudaFreeAsync(p, s);
        }
    } f1{mx, s};
    KKB_TRY_CUDA(cudaMallocAsync(&planes, sizeof(__half) * 4 * plane_elems, s), "cudaMallocAsync(trace planes)");
    Free f2{planes, s};
    unsigned *nonfinite = mx + n_frames;
    KKB_TRY_CUDA(cudaMemsetAsync(mx, 0, sizeof(unsigned) * ((size_t)n_frames + 1), s), "zero frame max");
    const long long per = (long long)NM * T;
    const bool v2 = (T % 2) == 0 && (data_fs % 2) == 0 && ((uintptr_t)data & 15) == 0;
    const int bx = (int)std::max<long long>(1, std::min<long long>(ceil_div(per, 512), ceil_div(148LL * 16, n_frames)));
    if (v2)
        k_frame_maxabs<2><<<dim3(bx, n_frames), 256, 0, s>>>(data, data_fs, per, mx, nonfinite);
    else
        k_frame_maxabs<1><<<dim3(bx, n_frames), 256, 0, s>>>(data, data_fs, per, mx, nonfinite);
    KKB_CHECK_LAUNCH("k_frame_maxabs");
    const long long units = ngroups * NM * (long long)(T / (v2 ? 2 : 1));
    const unsigned sblocks = (unsigned)std::min<long long>(ceil_div(units, 256), 148LL * 32);
    if (v2)
        k_split_planes<2><<<sblocks, 256, 0, s>>>(data, data_fs, n_frames, NM, T, mx, ngroups, planes);
    else
        k_split_planes<1><<<sblocks, 256, 0, s>>>(data, data_fs, n_frames, NM, T, mx, ngroups, planes);
    KKB_CHECK_LAUNCH("k_split_planes");
    int st = tcg_launch(planes, mx, nonfinite, N, M, T, ltx, ltzT, lrx, lrzT, nx, nz, w, fs, shift, linear, out,
                        out_kind, n_frames, out_fs, inten, fmax, tc_lo, accum, s);
    if (st) return st;
    // the FMA gather, live only when the batch held a non-finite sample
    return fma_fallback(nonfinite);
}

int kk_gather_tc_planes(const __half *planes, const unsigned *fbound, const unsigned *nonfinite, int N, int M,
                        int T, const double *ltx, const double *ltzT, const double *lrx, const double *lrzT, int nx,
                        int nz, const double *w, double fs, double shift, int linear, void *out, int out_kind,
                        int n_frames, long long out_fs, float *inten, unsigned *fmax, const int *tc_lo, int accum,
                        cudaStream_t s, const std::function<int(const unsigned *)> &fma_fallback) {
    if (!tc_lo || tcg_smem_bytes(N, M) > 227 * 1024) return KKB_ERR_UNSUPPORTED;
    int st = tcg_launch(planes, fbound, nonfinite, N, M, T, ltx, ltzT, lrx, lrzT, nx, nz, w, fs, shift, linear, out,
                        out_kind, n_frames, out_fs, inten, fmax, tc_lo, accum, s);
    if (st) return st;
    return fma_fallback(nonfinite);
}

}  // namespace kkb
