// K1 / K3 specialised for the trace lengths of the five workloads
// (T = 1024, 1536, 2048, 4096): the radix plan, thread count and every index
// are compile-time constants, so the Stockham stages are straight-line code.
//
// One CTA = one complex transform of length T (two real traces packed as
// re/im for the forward real FFT), three Stockham stages R0 x R1 x R2 with
// R0 = 16 (composite butterflies 16 = 4x4, 12 = 4x3, 8, 6 = 2x3 in registers).
// The transform is bound by L1/shared-memory wavefronts (ncu, r1: LSU data
// pipe 91-94% busy), so the layout minimises passes through shared memory:
//   - stage 0 reads its butterfly inputs straight from global memory (lane j
//     reads sample j + r T/R0: coalesced), no staging copy;
//   - stages 0 and 1 write in place into ONE shared buffer (8 B x T); stage 0
//     writes at stride 1 and goes through an XOR swizzle e ^ ((e >> 4) & 15)
//     that stage 1 reads back; from stage 1 on, output strides are >= 16;
//   - the last stage keeps its outputs in registers (natural order: lane j
//     holds bins j + r T/R2): the complex transform stores them to global
//     directly; the real-pair split writes them once to shared memory and
//     reads back only the mirrored bin T - k it needs.
// Twiddles: stage-ordered float32 table (stage_twiddles) so that lanes read
// consecutive entries; butterfly-internal twiddles are compile-time constants.
//
// Measured (r1, config 4, T = 1536, 28160 pairs): the previous four-stage
// radix-8 form with a staging pass and a length-T twiddle table took 224 us
// (177 us with the stage-ordered table); a persistent cp.async-pipelined
// variant was 22% slower and a multi-pair CTA with cp.async double-buffered
// staging 53% slower (register pressure), so one CTA per transform is kept.

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "fft.cuh"
#include "fft_ct.cuh"
#include "tcplanes.cuh"

namespace kkb {
namespace ct {

// Real-pair forward FFT: rows r0, r0+1 of `in` (length T) -> bins [0, K) of
// each row's spectrum at out + row*out_stride, times bin_scale[k].  Rows are
// paired only inside groups of `grp` rows (the L element traces of one
// (frame, transmit)); an odd group's last row pairs with zeros.  A row's
// rounding depends on its partner, so this keeps every trace independent of
// batch size, frame position and the transmit split across GPUs.
// Even groups pair exactly like the whole batch (rows 2p, 2p+1), so only odd
// groups take the GROUPED instance.
template <int T, typename InT, bool GROUPED = false, bool RING = false>
__global__ void __launch_bounds__(Plan<T>::NT)
k_r2c(const InT *__restrict__ in, long long ntraces, float2 *__restrict__ out,
      long long out_stride, int K, const float *__restrict__ bin_scale,
      const float2 *__restrict__ tw, int grp, const Stage1Ring rs = Stage1Ring{}) {
    using P = Plan<T>;
    __shared__ __align__(16) float2 buf[T];
    long long r0;
    bool l1;
    long long tile = 0;
    if constexpr (RING) {
        // wait until the contraction released this row-tile's ring slot
        tile = 2 * (long long)blockIdx.x / rs.traces_per_tile;
        if (tile >= rs.R) {
            if (threadIdx.x == 0) ring_wait_geq(rs.con_done + (tile - rs.R), rs.con_per_tile, rs.err);
            __syncthreads();
        }
    }
    if constexpr (GROUPED) {
        const unsigned ppg = (unsigned)(grp + 1) >> 1, gi = blockIdx.x / ppg, q = blockIdx.x - gi * ppg;
        r0 = (long long)gi * grp + 2 * q;
        if (r0 >= ntraces) return;
        l1 = (int)(2 * q + 1) < grp && r0 + 1 < ntraces;
    } else {
        r0 = 2 * (long long)blockIdx.x;
        l1 = r0 + 1 < ntraces;
    }
    const InT *x0 = in + r0 * T;
    const InT *x1 = in + (l1 ? r0 + 1 : r0) * T;
    using S0 = Stage<T, P::NT, P::R0>;
    S0 a;
#pragma unroll
    for (int t = 0; t < S0::ITER; ++t) {
        const int j = S0::lane_j(t);
        if (S0::ok(j)) {
#pragma unroll
            for (int r = 0; r < P::R0; ++r) {
                const int e = j + r * S0::TR;
                const float im = to_f(__ldg(x1 + e));
                a.v[t][r] = make_float2(to_f(__ldg(x0 + e)), l1 ? im : 0.f);
            }
        }
    }
    a.template compute<1, 0>(tw);
    a.template store<1, true>(buf);
    __syncthreads();
    using S2 = Stage<T, P::NT, P::R2>;
    S2 c;
    stages12<T>(buf, tw, c);
    __syncthreads();  // every stage-2 input read before the bins overwrite buf
#pragma unroll
    for (int t = 0; t < S2::ITER; ++t) {
        const int j = S2::lane_j(t);
        if (S2::ok(j)) {
#pragma unroll
            for (int r = 0; r < P::R2; ++r) buf[j + r * S2::TR] = c.v[t][r];
        }
    }
    __syncthreads();
    long long orow = r0;
    if constexpr (RING) orow = (tile % rs.R) * rs.traces_per_tile + (r0 - tile * rs.traces_per_tile);
    float2 *o0 = out + orow * out_stride;
    float2 *o1 = out + (orow + 1) * out_stride;
#pragma unroll
    for (int t = 0; t < S2::ITER; ++t) {
        const int j = S2::lane_j(t);
#pragma unroll
        for (int r = 0; r < P::R2; ++r) {
            const int k = j + r * S2::TR;
            if (S2::ok(j) && k < K) {
                const float2 zk = c.v[t][r];
                const float2 zn = buf[k == 0 ? 0 : T - k];
                const float s = 0.5f * (bin_scale ? __ldg(bin_scale + k) : 1.0f);
                // X0 = (Z_k + conj(Z_-k)) / 2 ; X1 = (Z_k - conj(Z_-k)) / (2i)
                o0[k] = make_float2(s * (zk.x + zn.x), s * (zk.y - zn.y));
                if (l1) o1[k] = make_float2(s * (zk.y + zn.y), -s * (zk.x - zn.x));
            }
        }
    }
    if constexpr (RING) {  // this pair's spectra are in the slot: count it (release)
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(rs.fft_done + tile, 1);
        }
    }
}

// Complex FFT of rows: input bins [0, in_len) (rest zero), output the first
// out_len points times `scale`; INV selects exp(+) via conjugation.  SC: the
// epilogue stores every row into each of sc.ndst buffers (peers' trace
// buffers mapped over NVLink) at sc.off + (row / rpf) * frame_stride +
// (row % rpf) * out_stride instead of `out` -- the fused trace all-gather of
// transmit-sharded stage 1.
// One complex transform of the row at src (bins [0, in_len), the rest zero)
// through buf; returns with the outputs (points j + r T/R2 of lane j) in c,
// conjugated on input for the inverse (the caller conjugates the output).
template <int T, bool INV, typename S2, bool SMEM_SRC = false>
__device__ __forceinline__ void c2c_row(const float2 *__restrict__ src, int in_len, const float2 *__restrict__ tw,
                                        float2 *buf, S2 &c, int bar = 0) {
    using P = Plan<T>;
    const float sg = INV ? -1.f : 1.f;
    using S0 = Stage<T, P::NT, P::R0>;
    S0 a;
#pragma unroll
    for (int t = 0; t < S0::ITER; ++t) {
        const int j = S0::lane_j(t);
        if (S0::ok(j)) {
#pragma unroll
            for (int r = 0; r < P::R0; ++r) {
                const int e = j + r * S0::TR;
                float2 v = make_float2(0.f, 0.f);
                if (e < in_len) v = SMEM_SRC ? src[e] : __ldg(src + e);
                a.v[t][r] = make_float2(v.x, sg * v.y);
            }
        }
    }
    a.template compute<1, 0>(tw);
    a.template store<1, true>(buf);
    xform_sync<P::NT>(bar);
    stages12<T>(buf, tw, c, bar);
}

template <int T, bool INV, bool SC = false>
__global__ void __launch_bounds__(Plan<T>::NT)
k_c2c(const float2 *__restrict__ in, long long in_stride, int in_len, float2 *__restrict__ out,
      long long out_stride, int out_len, float scale, const float2 *__restrict__ tw,
      RowScatter sc = RowScatter{}) {
    using P = Plan<T>;
    __shared__ __align__(16) float2 buf[T];
    const long long row = blockIdx.x;
    const float sg = INV ? -1.f : 1.f;
    using S2 = Stage<T, P::NT, P::R2>;
    S2 c;
    c2c_row<T, INV>(in + row * in_stride, in_len, tw, buf, c);
    const float sy = sg * scale;
    if constexpr (SC) {
        const long long o = sc.off + (row / sc.rows_per_frame) * sc.frame_stride +
                            (row % sc.rows_per_frame) * out_stride;
#pragma unroll 1
        for (int d = 0; d < sc.ndst; ++d) {
            float2 *dst = sc.dst[d] + o;
#pragma unroll
            for (int t = 0; t < S2::ITER; ++t) {
                const int j = S2::lane_j(t);
#pragma unroll
                for (int r = 0; r < P::R2; ++r) {
                    const int k = j + r * S2::TR;
                    if (S2::ok(j) && k < out_len) dst[k] = make_float2(c.v[t][r].x * scale, c.v[t][r].y * sy);
                }
            }
        }
    } else {
        float2 *dst = out + row * out_stride;
#pragma unroll
        for (int t = 0; t < S2::ITER; ++t) {
            const int j = S2::lane_j(t);
#pragma unroll
            for (int r = 0; r < P::R2; ++r) {
                const int k = j + r * S2::TR;
                if (S2::ok(j) && k < out_len) dst[k] = make_float2(c.v[t][r].x * scale, c.v[t][r].y * sy);
            }
        }
    }
}

// K3 into the tensor-core gather's split planes (tcplanes.cuh): inverse
// transforms of the contracted bins Y (rows (frame, pair), row stride ldy,
// bins [0, K)).  A CTA takes 4 frames (half a frame group) of one pair q:
// four transforms side by side (threads [i NT, (i + 1) NT) take frame i, each
// in its own T-point buffer with its own named barrier), each output scaled
// by its frame's power of two (from the frame bound fbound[f]) and split into
// fp16 halves, staged in the freed buffers as [frame][sample] 8-byte entries
// (the four planes' halves) and stored as the 8-byte halves of the planes'
// 16-byte rows (two CTAs fill a row; two CTAs per SM overlap their phases).
// Frames past n_frames stage zeros.  When *nonfinite is set the complex64
// traces are written too (the FMA gather, which then runs instead, reads them).
#ifndef KKB_C2C_PLANES_MINB
#define KKB_C2C_PLANES_MINB 2  // resident CTAs per SM the register budget is sized for
#endif
template <int T>
__global__ void __launch_bounds__(4 * Plan<T>::NT, KKB_C2C_PLANES_MINB)
k_c2c_planes(const float2 *__restrict__ Y, long long ldy, int K, int n_frames, int NM, float scale,
             const float2 *__restrict__ tw, const unsigned *__restrict__ fbound,
             const unsigned *__restrict__ nonfinite, float2 *__restrict__ traces, __half *__restrict__ planes,
             long long per_plane) {
    using P = Plan<T>;
    extern __shared__ __align__(16) unsigned char dsm[];
    float2 *bufs = reinterpret_cast<float2 *>(dsm);  // [4][T]; then the stage [4 frames][T] uint2
    uint2 *stage = reinterpret_cast<uint2 *>(dsm);
    // CTAs last to first: the frame bound just read the highest rows of Y
    // (L2-resident), and the gather starts from the lowest frames' planes
    const unsigned bid = gridDim.x - 1 - blockIdx.x;
    const int q = bid % NM;
    const long long gh = bid / NM, g = gh >> 1;
    const int half = (int)(gh & 1);
    const int i = threadIdx.x / P::NT;  // frame of the half group
    const long long f = g * 8 + half * 4 + i, row = f * NM + q;
    const bool live = f < n_frames;
    using S2 = Stage<T, P::NT, P::R2>;
    S2 c;
    c2c_row<T, true>(live ? Y + row * ldy : Y, live ? K : 0, tw, bufs + (size_t)i * T, c, 1 + i);
    const bool flag = *nonfinite != 0;
    const float sc = live ? frame_scale(__ldg(fbound + f)) : 0.f;
    // transform i's stage entries [i][k] occupy exactly its own buffer: once
    // its own threads have read it (named barrier 1 + i), the others need not wait
    xform_sync<P::NT>(1 + i);
#pragma unroll
    for (int t = 0; t < S2::ITER; ++t) {
        const int j = S2::lane_j(t);
#pragma unroll
        for (int r = 0; r < P::R2; ++r) {
            const int k = j + r * S2::TR;
            if (S2::ok(j)) {
                const float2 x = make_float2(c.v[t][r].x * scale, c.v[t][r].y * -scale);
                if (flag && live) traces[row * T + k] = x;
                uint32_t hi, lo;
                split_h2(x.x * sc, x.y * sc, hi, lo);
                stage[i * T + k] = make_uint2(hi, lo);  // consecutive k: conflict-free
            }
        }
    }
    __syncthreads();
    // per sample k: the 4 frames' 8-byte entries in, the four planes' 8-byte
    // half rows out (conflict-free 64-bit loads, coalesced 64-bit stores)
    uint2 *dst = reinterpret_cast<uint2 *>(planes) + ((g * NM + q) * T) * 2 + half;
    for (int k = threadIdx.x; k < T; k += blockDim.x) {
        uint2 e[4];
#pragma unroll
        for (int fi = 0; fi < 4; ++fi) e[fi] = stage[fi * T + k];
        // e.x = (re hi, im hi), e.y = (re lo, im lo) of one frame
        const long long o = 2LL * k;
        dst[0 * (per_plane / 4) + o] = make_uint2((e[0].x & 0xffffu) | (e[1].x << 16), (e[2].x & 0xffffu) | (e[3].x << 16));
        dst[1 * (per_plane / 4) + o] = make_uint2((e[0].x >> 16) | (e[1].x & 0xffff0000u), (e[2].x >> 16) | (e[3].x & 0xffff0000u));
        dst[2 * (per_plane / 4) + o] = make_uint2((e[0].y & 0xffffu) | (e[1].y << 16), (e[2].y & 0xffffu) | (e[3].y << 16));
        dst[3 * (per_plane / 4) + o] = make_uint2((e[0].y >> 16) | (e[1].y & 0xffff0000u), (e[2].y >> 16) | (e[3].y & 0xffff0000u));
    }
}

// K3 as a persistent kernel (2 CTAs per SM) whose CTAs walk the same units
// (4 frames of one pair) in the same order as k_c2c_planes, each unit's four
// rows of Y arriving by 1D bulk copies (cp.async.bulk, mbarrier complete_tx)
// into one of two shared slots while the previous unit transforms: the
// per-CTA load latency the one-shot kernel exposes at every CTA start is
// hidden behind the FFT.  Arithmetic and store order are those of
// k_c2c_planes, so the planes and traces are bit-identical.
template <int T>
__global__ void __launch_bounds__(4 * Plan<T>::NT, KKB_C2C_PLANES_MINB)
k_c2c_planes_pf(const float2 *__restrict__ Y, long long ldy, int K, int n_frames, int NM, float scale,
                const float2 *__restrict__ tw, const unsigned *__restrict__ fbound,
                const unsigned *__restrict__ nonfinite, float2 *__restrict__ traces, __half *__restrict__ planes,
                long long per_plane, int n_units, int row_bytes) {
    using P = Plan<T>;
    extern __shared__ __align__(128) unsigned char dsm[];
    float2 *bufs = reinterpret_cast<float2 *>(dsm);
    uint2 *stage = reinterpret_cast<uint2 *>(dsm);
    unsigned char *slots = dsm + sizeof(float2) * 4 * T;  // [2 slots][4 rows][row_bytes]
    uint64_t *mb = reinterpret_cast<uint64_t *>(slots + 8 * (size_t)row_bytes);
    const int i = threadIdx.x / P::NT;
    auto sa = [](const void *p) { return (uint32_t)__cvta_generic_to_shared(p); };
    // thread 0: the four live rows of unit u into slot sl
    auto fetch = [&](int u, int sl) {
        const int bid = n_units - 1 - u;
        const int q = bid % NM, gh = bid / NM, f0 = (gh >> 1) * 8 + (gh & 1) * 4;
        const int live = min(4, n_frames - f0);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mb[sl])),
                     "r"((uint32_t)(live * row_bytes))
                     : "memory");
        for (int fi = 0; fi < live; ++fi) {
            const long long row = (long long)(f0 + fi) * NM + q;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    sa(slots + ((size_t)sl * 4 + fi) * row_bytes)),
                "l"(Y + row * ldy), "r"((uint32_t)row_bytes), "r"(sa(&mb[sl]))
                : "memory");
        }
    };
    if (threadIdx.x == 0) {
        for (int k = 0; k < 2; ++k)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mb[k])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (blockIdx.x < n_units) fetch(blockIdx.x, 0);
        if (blockIdx.x + gridDim.x < n_units) fetch(blockIdx.x + gridDim.x, 1);
    }
    const bool flag = *nonfinite != 0;
    int it = 0;
#pragma unroll 1
    for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++it) {
        const int sl = it & 1;
        const int bid = n_units - 1 - u;
        const int q = bid % NM, gh = bid / NM, g = gh >> 1, half = gh & 1;
        const int f = g * 8 + half * 4 + i;
        const long long row = (long long)f * NM + q;
        const bool live = f < n_frames;
        {
            const uint32_t a = sa(&mb[sl]), par = (uint32_t)((it >> 1) & 1);
            asm volatile(
                "{\n\t.reg .pred P1;\n\tW_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                "@!P1 bra W_%=;\n\t}\n" ::"r"(a),
                "r"(par)
                : "memory");
        }
        using S2 = Stage<T, P::NT, P::R2>;
        S2 c;
        c2c_row<T, true, S2, true>(reinterpret_cast<const float2 *>(slots + ((size_t)sl * 4 + i) * row_bytes),
                                   live ? K : 0, tw, bufs + (size_t)i * T, c, 1 + i);
        const float sc = live ? frame_scale(__ldg(fbound + f)) : 0.f;
        __syncthreads();  // every transform's slot and buffer read
#pragma unroll
        for (int t = 0; t < S2::ITER; ++t) {
            const int j = S2::lane_j(t);
#pragma unroll
            for (int r = 0; r < P::R2; ++r) {
                const int k = j + r * S2::TR;
                if (S2::ok(j)) {
                    const float2 x = make_float2(c.v[t][r].x * scale, c.v[t][r].y * -scale);
                    if (flag && live) traces[row * T + k] = x;
                    uint32_t hi, lo;
                    split_h2(x.x * sc, x.y * sc, hi, lo);
                    stage[i * T + k] = make_uint2(hi, lo);
                }
            }
        }
        __syncthreads();
        // refill the slot (read before the first barrier above) with the unit
        // after next, here where the transform outputs are no longer live
        if (threadIdx.x == 0 && u + 2 * (int)gridDim.x < n_units) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            fetch(u + 2 * (int)gridDim.x, sl);
        }
        uint2 *dst = reinterpret_cast<uint2 *>(planes) + (((long long)g * NM + q) * T) * 2 + half;
        for (int k = threadIdx.x; k < T; k += blockDim.x) {
            uint2 e[4];
#pragma unroll
            for (int fi = 0; fi < 4; ++fi) e[fi] = stage[fi * T + k];
            const long long o = 2LL * k;
            dst[0 * (per_plane / 4) + o] = make_uint2((e[0].x & 0xffffu) | (e[1].x << 16), (e[2].x & 0xffffu) | (e[3].x << 16));
            dst[1 * (per_plane / 4) + o] = make_uint2((e[0].x >> 16) | (e[1].x & 0xffff0000u), (e[2].x >> 16) | (e[3].x & 0xffff0000u));
            dst[2 * (per_plane / 4) + o] = make_uint2((e[0].y & 0xffffu) | (e[1].y << 16), (e[2].y & 0xffffu) | (e[3].y << 16));
            dst[3 * (per_plane / 4) + o] = make_uint2((e[0].y >> 16) | (e[1].y & 0xffff0000u), (e[2].y >> 16) | (e[3].y & 0xffff0000u));
        }
        __syncthreads();  // stage read before the next unit's transforms reuse the buffers
    }
}

// Per-frame bound for the plane scale: max over the frame's rows of
// scale * sum_k (|Re Y_k| + |Im Y_k|) >= max_t |x_t| (the inverse transform
// of bins [0, K)), as float bits; a non-finite bin sets *nonfinite.  One warp
// per row.
__global__ void __launch_bounds__(256) k_frame_bound(const float2 *__restrict__ Y, long long ldy, int K,
                                                     long long rows, int rows_per_frame, float scale,
                                                     unsigned *__restrict__ fbound, unsigned *__restrict__ nonfinite) {
    // rows first to last: K2 runs its row tiles backwards, so the lowest rows
    // are the ones still in L2 (and K3 then starts from the highest)
    const long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
    if (row >= rows) return;
    const int lane = threadIdx.x & 31;
    const float2 *y = Y + row * ldy;
    float s = 0.f;
    for (int k = lane; k < K; k += 32) {
        const float2 v = __ldg(y + k);
        s += fabsf(v.x) + fabsf(v.y);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        // rounding margin: the sum and the transform's own roundings stay far
        // below 2^-10 relative, and a bound twice too large costs nothing
        const float b = s * fabsf(scale) * 1.001f;
        if (!(b <= 3.0e38f)) atomicOr(nonfinite, 1u);  // NaN or Inf
        else atomicMax(fbound + row / rows_per_frame, __float_as_uint(b));
    }
}

}  // namespace ct

bool fft_ct_supported(int T) { return T == 1024 || T == 1536 || T == 2048 || T == 4096; }

// Stage-ordered twiddle table of plan P, in the order fft<> reads it:
// for stages 1.. (input length NS, radix R): (R-1) x NS entries
// exp(-2 pi i r k / (NS R)), evaluated in double as the length-T table was.
template <int T>
static void stage_twiddles(std::vector<float2> &out) {
    using P = ct::Plan<T>;
    const int radix[4] = {P::R0, P::R1, P::R2, P::R3};
    int ns = radix[0];
    for (int s = 1; s < 4 && radix[s] > 1; ++s) {
        const int R = radix[s];
        for (int r = 1; r < R; ++r)
            for (int k = 0; k < ns; ++k) {
                const double a = -2.0 * M_PI * (double)(r * k * (T / (ns * R))) / (double)T;
                out.push_back(make_float2((float)cos(a), (float)sin(a)));
            }
        ns *= R;
    }
}

void fft_ct_twiddles(int T, std::vector<float2> &out) {
    out.clear();
    switch (T) {
        case 1024: stage_twiddles<1024>(out); break;
        case 1536: stage_twiddles<1536>(out); break;
        case 2048: stage_twiddles<2048>(out); break;
        case 4096: stage_twiddles<4096>(out); break;
    }
}

template <int T>
static int launch_r2c(const void *in, int in_kind, long long ntraces, float2 *out,
                      long long out_stride, int K, const float *bin_scale, const float2 *tw,
                      cudaStream_t s, int grp) {
    const unsigned npairs = (unsigned)(ceil_div(ntraces, grp) * ((grp + 1) / 2));
    const bool g = grp & 1;
    if (in_kind) {
        auto fn = g ? ct::k_r2c<T, short, true> : ct::k_r2c<T, short, false>;
        fn<<<npairs, ct::Plan<T>::NT, 0, s>>>(reinterpret_cast<const short *>(in), ntraces, out,
                                              out_stride, K, bin_scale, tw, grp, Stage1Ring{});
    } else {
        auto fn = g ? ct::k_r2c<T, float, true> : ct::k_r2c<T, float, false>;
        fn<<<npairs, ct::Plan<T>::NT, 0, s>>>(reinterpret_cast<const float *>(in), ntraces, out,
                                              out_stride, K, bin_scale, tw, grp, Stage1Ring{});
    }
    KKB_CHECK_LAUNCH("k_fft_r2c_ct");
    return KKB_OK;
}

template <int T>
static int launch_c2c(const float2 *in, long long in_stride, int in_len, float2 *out,
                      long long out_stride, int out_len, long long ntraces, bool inverse,
                      float scale, const float2 *tw, cudaStream_t s, const RowScatter *sc) {
    if (sc) {
        if (inverse)
            ct::k_c2c<T, true, true><<<(unsigned)ntraces, ct::Plan<T>::NT, 0, s>>>(
                in, in_stride, in_len, out, out_stride, out_len, scale, tw, *sc);
        else
            ct::k_c2c<T, false, true><<<(unsigned)ntraces, ct::Plan<T>::NT, 0, s>>>(
                in, in_stride, in_len, out, out_stride, out_len, scale, tw, *sc);
    } else if (inverse)
        ct::k_c2c<T, true><<<(unsigned)ntraces, ct::Plan<T>::NT, 0, s>>>(
            in, in_stride, in_len, out, out_stride, out_len, scale, tw);
    else
        ct::k_c2c<T, false><<<(unsigned)ntraces, ct::Plan<T>::NT, 0, s>>>(
            in, in_stride, in_len, out, out_stride, out_len, scale, tw);
    KKB_CHECK_LAUNCH("k_fft_c2c_ct");
    return KKB_OK;
}

int fft_r2c_ct(const void *in, int in_kind, long long ntraces, int T, float2 *out,
               long long out_stride, int K, const float *bin_scale, const float2 *tw,
               cudaStream_t s, long long group_rows) {
    if (ntraces <= 0) return KKB_OK;
    // pairing groups; the whole batch as one group pairs like groups of 2
    const int grp = group_rows > 0 && group_rows <= 0x7fffffffLL ? (int)group_rows : 2;
    if (ceil_div(ntraces, grp) * ((grp + 1) / 2) > 0x7fffffffLL) return KKB_ERR_UNSUPPORTED;
    switch (T) {
        case 1024: return launch_r2c<1024>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s, grp);
        case 1536: return launch_r2c<1536>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s, grp);
        case 2048: return launch_r2c<2048>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s, grp);
        case 4096: return launch_r2c<4096>(in, in_kind, ntraces, out, out_stride, K, bin_scale, tw, s, grp);
    }
    return KKB_ERR_UNSUPPORTED;
}

template <int T>
static int launch_r2c_ring(const void *in, int in_kind, long long ntraces, float2 *ring, long long out_stride,
                           int K, const float *bin_scale, const float2 *tw, cudaStream_t s, const Stage1Ring &rs) {
    const unsigned npairs = (unsigned)ceil_div(ntraces, 2);
    if (in_kind)
        ct::k_r2c<T, short, false, true><<<npairs, ct::Plan<T>::NT, 0, s>>>(
            reinterpret_cast<const short *>(in), ntraces, ring, out_stride, K, bin_scale, tw, 2, rs);
    else
        ct::k_r2c<T, float, false, true><<<npairs, ct::Plan<T>::NT, 0, s>>>(
            reinterpret_cast<const float *>(in), ntraces, ring, out_stride, K, bin_scale, tw, 2, rs);
    KKB_CHECK_LAUNCH("k_fft_r2c_ct_ring");
    return KKB_OK;
}

int fft_r2c_ct_ring(const void *in, int in_kind, long long ntraces, int T, float2 *ring,
                    long long out_stride, int K, const float *bin_scale, const float2 *tws,
                    cudaStream_t s, const Stage1Ring &rs) {
    if (ntraces <= 0) return KKB_OK;
    if ((ntraces & 1) || (rs.traces_per_tile & 1) || ceil_div(ntraces, 2) > 0x7fffffffLL) return KKB_ERR_UNSUPPORTED;
    switch (T) {
        case 1024: return launch_r2c_ring<1024>(in, in_kind, ntraces, ring, out_stride, K, bin_scale, tws, s, rs);
        case 1536: return launch_r2c_ring<1536>(in, in_kind, ntraces, ring, out_stride, K, bin_scale, tws, s, rs);
        case 2048: return launch_r2c_ring<2048>(in, in_kind, ntraces, ring, out_stride, K, bin_scale, tws, s, rs);
        case 4096: return launch_r2c_ring<4096>(in, in_kind, ntraces, ring, out_stride, K, bin_scale, tws, s, rs);
    }
    return KKB_ERR_UNSUPPORTED;
}

template <int T>
static int launch_c2c_planes(const float2 *Y, long long ldy, int K, int n_frames, int NM, float scale,
                             const float2 *tw, const unsigned *fbound, const unsigned *nonfinite, float2 *traces,
                             __half *planes, cudaStream_t s) {
    const long long groups = (n_frames + 7) / 8;
    const long long per_plane = groups * 8 * NM * (long long)T;
    const size_t smem = sizeof(float2) * 4 * (size_t)T;  // 4 transform buffers, then the fp16 stage
    // the prefetching persistent form, opt-in (KKB_K3_PREFETCH=1): bit-identical
    // and measured 0.18 ms slower per 400 frames than the one-shot kernel
    // (profiles/r02h_k3_prefetch_experiment.json: 276 B of spills at 64
    // registers).  Rows are copied whole in 16-byte units, so Y and its row
    // pitch must be 16-byte aligned and the pitch hold K rounded up to 2 bins.
    static const int pf_env = [] {
        const char *e = getenv("KKB_K3_PREFETCH");
        return e ? atoi(e) : 0;
    }();
    const int row_bytes = (int)(((long long)K * 8 + 15) / 16 * 16);
    if (pf_env && groups * 2 * NM < (1LL << 31) && ((uintptr_t)Y % 16) == 0 && (ldy * 8) % 16 == 0 && ldy * 8 >= row_bytes) {
        const int n_units = (int)(groups * 2 * NM);
        const size_t smem_pf = smem + 8 * (size_t)row_bytes + 16;
        KKB_TRY_CUDA(cudaFuncSetAttribute(ct::k_c2c_planes_pf<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem_pf),
                     "smem attr c2c planes pf");
        static int n_sm = 0;
        if (!n_sm) {
            int dev = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
        }
        const int grid = std::min(n_units, n_sm * KKB_C2C_PLANES_MINB);
        ct::k_c2c_planes_pf<T><<<(unsigned)grid, 4 * ct::Plan<T>::NT, smem_pf, s>>>(
            Y, ldy, K, n_frames, NM, scale, tw, fbound, nonfinite, traces, planes, per_plane, n_units, row_bytes);
        KKB_CHECK_LAUNCH("k_c2c_planes_pf");
        return KKB_OK;
    }
    KKB_TRY_CUDA(cudaFuncSetAttribute(ct::k_c2c_planes<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                 "smem attr c2c planes");
    ct::k_c2c_planes<T><<<(unsigned)(groups * 2 * NM), 4 * ct::Plan<T>::NT, smem, s>>>(
        Y, ldy, K, n_frames, NM, scale, tw, fbound, nonfinite, traces, planes, per_plane);
    KKB_CHECK_LAUNCH("k_c2c_planes");
    return KKB_OK;
}

int fft_c2c_planes(const float2 *Y, long long ldy, int K, int T, int n_frames, int NM, float scale,
                   const float2 *tws, const unsigned *fbound, const unsigned *nonfinite, float2 *traces,
                   __half *planes, cudaStream_t s) {
    if (n_frames <= 0) return KKB_OK;
    switch (T) {
        case 1024: return launch_c2c_planes<1024>(Y, ldy, K, n_frames, NM, scale, tws, fbound, nonfinite, traces, planes, s);
        case 1536: return launch_c2c_planes<1536>(Y, ldy, K, n_frames, NM, scale, tws, fbound, nonfinite, traces, planes, s);
        case 2048: return launch_c2c_planes<2048>(Y, ldy, K, n_frames, NM, scale, tws, fbound, nonfinite, traces, planes, s);
    }
    return KKB_ERR_UNSUPPORTED;
}

int frame_bound(const float2 *Y, long long ldy, int K, long long rows, int rows_per_frame, float scale,
                unsigned *fbound, unsigned *nonfinite, cudaStream_t s) {
    if (rows <= 0) return KKB_OK;
    ct::k_frame_bound<<<(unsigned)ceil_div(rows, 8), 256, 0, s>>>(Y, ldy, K, rows, rows_per_frame, scale, fbound,
                                                                   nonfinite);
    KKB_CHECK_LAUNCH("k_frame_bound");
    return KKB_OK;
}

int fft_c2c_ct(const float2 *in, long long in_stride, int in_len, float2 *out, long long out_stride,
               int out_len, long long ntraces, int T, bool inverse, float scale, const float2 *tw,
               cudaStream_t s, const RowScatter *sc) {
    if (ntraces <= 0) return KKB_OK;
    if (ntraces > 0x7fffffffLL) return KKB_ERR_UNSUPPORTED;
    switch (T) {
        case 1024: return launch_c2c<1024>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s, sc);
        case 1536: return launch_c2c<1536>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s, sc);
        case 2048: return launch_c2c<2048>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s, sc);
        case 4096: return launch_c2c<4096>(in, in_stride, in_len, out, out_stride, out_len, ntraces, inverse, scale, tw, s, sc);
    }
    return KKB_ERR_UNSUPPORTED;
}

}  // namespace kkb
