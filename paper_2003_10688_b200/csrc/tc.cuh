// Shared tcgen05 / TMEM / TMA / mbarrier PTX wrappers and tensor-map encoders for the sm_100a
// kernels (igemm.cu, stem.cu).
#pragma once

#include <cuda.h>

#include <stdexcept>
#include <string>

#include "common.cuh"

namespace solb200 {
namespace tc {

constexpr int ROWB_ = 128;

// ---------------------------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------------------------

__device__ __forceinline__ void mbar_init(uint32_t addr, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(addr), "r"(count));
}

__device__ __forceinline__ void mbar_wait(uint32_t addr, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(addr),
        "r"(parity));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src),
                 "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::);
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::);
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::);
}

template <uint32_t COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t slot_addr) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(slot_addr),
                 "n"(COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
}
template <uint32_t COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "n"(COLS));
}

// UMMA shared-memory descriptor, SWIZZLE_128B (layout type 2), sm_100 version 1.
// K-major:  LBO unused (16 B), SBO = 1024 B between 8-row core-matrix groups.
// MN-major: LBO = stride between 64-element MN blocks, SBO = stride between 8-row K groups.
// Layout type 2 = SWIZZLE_128B; 1 = SWIZZLE_128B_BASE32B (32-byte swizzle atoms, used for the
// MN-major 32-bit (tf32) operands of wgrad).
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout = 2) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr & 0x3FFFF) >> 4);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // descriptor version (Blackwell)
    d |= static_cast<uint64_t>(layout) << 61;
    return d;
}

// Instruction descriptor: f32 accumulate, A/B format (1 = bf16, 2 = tf32), majors, N, M.
__host__ __device__ constexpr uint32_t make_idesc(int ab_fmt, int n, int m, int a_mn, int b_mn) {
    return (1u << 4) | (static_cast<uint32_t>(ab_fmt) << 7) | (static_cast<uint32_t>(ab_fmt) << 10) |
           (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
           (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

template <typename T>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                    uint32_t accum);
template <>
__device__ __forceinline__ void mma<__nv_bfloat16>(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                                   uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
template <>
__device__ __forceinline__ void mma<float>(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// The four K=16 steps of one 128-byte K block (descriptor start addresses advance by 32 B = 2
// units), issued by ONE elected lane of a CONVERGED warp from a single asm statement: with the
// loop run by the whole warp the operands stay warp-uniform, so ptxas issues back-to-back
// UTCHMMAs instead of a per-MMA elect/R2UR loop (measured: 48 vs ~110 cycles per N=64 MMA).
// KIND is "f16" or "tf32"; acc = 0 overwrites the accumulator on the first step.
template <typename T>
__device__ __forceinline__ void mma4_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc);
#define SOLB200_MMA4(KIND)                                                                         \
    asm volatile(                                                                                  \
        "{\n.reg .pred p, pa;\n.reg .b64 a1, a2, a3, b1, b2, b3;\n"                               \
        "elect.sync _|p, 0xffffffff;\n"                                                           \
        "setp.ne.b32 pa, %4, 0;\n"                                                                \
        "add.s64 a1, %1, 2;\nadd.s64 a2, %1, 4;\nadd.s64 a3, %1, 6;\n"                           \
        "add.s64 b1, %2, 2;\nadd.s64 b2, %2, 4;\nadd.s64 b3, %2, 6;\n"                           \
        "@p tcgen05.mma.cta_group::1.kind::" KIND " [%0], %1, %2, %3, pa;\n"                     \
        "@p tcgen05.mma.cta_group::1.kind::" KIND " [%0], a1, b1, %3, 1;\n"                      \
        "@p tcgen05.mma.cta_group::1.kind::" KIND " [%0], a2, b2, %3, 1;\n"                      \
        "@p tcgen05.mma.cta_group::1.kind::" KIND " [%0], a3, b3, %3, 1;\n"                      \
        "}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc))
template <>
__device__ __forceinline__ void mma4_elect<__nv_bfloat16>(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                                          uint32_t acc) {
    SOLB200_MMA4("f16");
}
template <>
__device__ __forceinline__ void mma4_elect<float>(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    SOLB200_MMA4("tf32");
}
#undef SOLB200_MMA4

// One filter row of a 3-tap convolution from shifted operands: taps dkw = 0..2 read A at
// +dkw rows (8 units of 16 B each) and B at +dkw * BSTR units, four K=16 steps each: twelve
// bf16 MMAs from one asm statement (immediate offsets -> uniform-register adds only).
template <int BSTR>
__device__ __forceinline__ void mma_row3_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
#define SOLB200_STEP(AI, BI) \
    "add.s64 ra, %1, " #AI ";\nadd.s64 rb, %2, %" #BI ";\n@p tcgen05.mma.cta_group::1.kind::f16 [%0], ra, rb, %3, 1;\n"
    asm volatile(
        "{\n.reg .pred p, pa;\n.reg .b64 ra, rb;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "setp.ne.b32 pa, %4, 0;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pa;\n"
        SOLB200_STEP(2, 5) SOLB200_STEP(4, 6) SOLB200_STEP(6, 7)
        SOLB200_STEP(8, 8) SOLB200_STEP(10, 9) SOLB200_STEP(12, 10) SOLB200_STEP(14, 11)
        SOLB200_STEP(16, 12) SOLB200_STEP(18, 13) SOLB200_STEP(20, 14) SOLB200_STEP(22, 15)
        "}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc),
        "n"(2), "n"(4), "n"(6), "n"(BSTR), "n"(BSTR + 2), "n"(BSTR + 4), "n"(BSTR + 6),
        "n"(2 * BSTR), "n"(2 * BSTR + 2), "n"(2 * BSTR + 4), "n"(2 * BSTR + 6));
#undef SOLB200_STEP
}

// Two consecutive K=16 bf16 MMAs (one 32-element K slice) for SWIZZLE_NONE operands whose
// second step starts ASTEP / BSTEP 16-byte units after the first; elected lane, converged warp.
template <int ASTEP, int BSTEP>
__device__ __forceinline__ void mma2_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p, pa;\n.reg .b64 a1, b1;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "setp.ne.b32 pa, %4, 0;\n"
        "add.s64 a1, %1, %5;\nadd.s64 b1, %2, %6;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n"
        "}\n" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc), "n"(ASTEP), "n"(BSTEP));
}

// tcgen05.commit from one elected lane of a converged warp.
__device__ __forceinline__ void mma_commit_elect(uint32_t mbar_addr) {
    asm volatile(
        "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
        "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(mbar_addr));
}

__device__ __forceinline__ void mma_commit(uint32_t mbar_addr) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
        mbar_addr));
}

// 32 lanes x 32 bits, 32 consecutive columns per thread; completion via tmem_wait_ld().
__device__ __forceinline__ void tmem_ld32_nowait(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

// 32 lanes x 32 bits, 16 consecutive columns per thread.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
        "[%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::);
}


__device__ __forceinline__ void tma_load_im2col_4d(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                                   uint16_t off_w, uint16_t off_h, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c), "r"(w), "r"(h), "r"(n), "h"(off_w), "h"(off_h)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t addr) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(addr));
}
__device__ __forceinline__ void mbar_arrive_tx(uint32_t addr, uint32_t bytes) {
    asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(addr),
                 "r"(bytes));
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint32_t addr) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(addr));
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(mbar)
        : "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}


// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link dependency).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

inline EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        SOL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// 2-D row-major [rows][cols] tensor, box = [box_rows][128 bytes], 128B swizzle (UMMA K-major atom).
inline CUtensorMap make_tmap_2d(const void* base, int dtype, uint64_t cols, uint64_t rows, uint64_t row_stride_elems,
                         uint32_t box_rows) {
    CUtensorMap m;
    const uint32_t es = dtype == DT_BF16 ? 2 : 4;
    cuuint64_t dims[2] = {cols, rows};
    cuuint64_t strides[1] = {row_stride_elems * es};
    cuuint32_t box[2] = {128 / es, box_rows};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, dtype == DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                                   2, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
}


}  // namespace tc
}  // namespace solb200
