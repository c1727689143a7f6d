// tcgen05 / TMEM / mbarrier helpers (sm_100a inline PTX) for the tensor-core
// kernels of libkkb.  Operands live in shared memory in the canonical
// no-swizzle UMMA layouts.  K-major: 8-row x 16-byte core matrices, rows of a
// core matrix 16 B apart; the descriptor's SBO is the byte stride between
// 8-row groups, LBO the byte stride between the two 16-byte K halves of one
// MMA's 32-byte K step.  MN-major: core matrices of 8 K-rows x 16 bytes of
// consecutive M/N values; LBO = stride between 8-deep K groups, SBO = stride
// between 16-byte M/N groups.  Accumulators are fp32 in TMEM: row i of an M = 128
// tile is TMEM lane i, column j is TMEM column base + j.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace kkb {
namespace tc {

// Shared-memory matrix descriptor (UMMA SmemDescriptor, version 1 = sm_100,
// layout type 0 = no swizzle); addresses / offsets in bytes, 16-byte aligned.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

// Swizzled K-major shared-memory descriptor (layout 4 = 64-byte swizzle: rows
// of 64 bytes, 8-row atoms of 512; 6 = 32-byte swizzle: rows of 32 bytes,
// atoms of 256): sbo = the atom stride; the leading offset is unused.
__device__ __forceinline__ uint64_t smem_desc_sw(uint32_t saddr, uint32_t sbo, uint32_t layout) {
    return smem_desc(saddr, 16, sbo) | ((uint64_t)layout << 61);
}

// Instruction descriptor: fp32 accumulate, A/B format (0 f16, 1 bf16, 2 tf32),
// A K-major, B K-major (b_mn_major = 0) or MN-major (1), dense.
__host__ __device__ constexpr uint32_t instr_desc(int ab_format, int M, int N, int b_mn_major = 0) {
    return (1u << 4) | ((uint32_t)ab_format << 7) | ((uint32_t)ab_format << 10) |
           ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// D[tmem] (+)= A[smem] * B[smem]^T, issued by ONE thread.
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         bool accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)accumulate));
}

__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        bool accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"((uint32_t)accumulate));
}

// One K = 16 step of a split-fp16 product, hi*hi + hi*lo + lo*hi, as three
// MMAs from one asm block (descriptors of the A / B hi and lo halves);
// accumulate = false overwrites D with the first product.
__device__ __forceinline__ void mma_f16_split3(uint32_t d_tmem, uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl,
                                               uint32_t idesc, bool accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, q;\n\t"
        "setp.ne.b32 p, %6, 0;\n\t"
        "setp.eq.b32 q, 0, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %3, %5, p;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %4, %5, q;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %3, %5, q;\n\t}\n" ::"r"(d_tmem),
        "l"(ah), "l"(al), "l"(bh), "l"(bl), "r"(idesc), "r"((uint32_t)accumulate));
}

// one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
    uint32_t p = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n\t}" : "=r"(p));
    return p != 0;
}

// Arrive on an mbarrier once every MMA this thread issued so far completes.
__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)),
                 "r"(count)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy shared-memory writes visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_smem_to_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// TMEM allocation by one full warp; the base address is written to *dst (smem).
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t *dst) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "n"(COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

template <int COLS>
__device__ __forceinline__ void tmem_free(uint32_t base) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "n"(COLS) : "memory");
}

// 32 lanes x 8 consecutive 32-bit columns: thread t of the warp gets lane
// (warp's lane base + t), columns col .. col+7.
__device__ __forceinline__ void tmem_ld8(uint32_t addr, float (&v)[8]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                   "=r"(r[7])
                 : "r"(addr));
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// fp32 -> tf32 (round to nearest, ties away) as an fp32 bit pattern with the
// low 13 mantissa bits cleared; x = hi + lo with both exactly representable.
__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

}  // namespace tc
}  // namespace kkb
