// tcgen05 / TMEM implicit-GEMM kernels for sm_100a. See igemm.cuh for the semantics.
//
// Structure (one output tile per CTA, 128 threads = 4 warps):
//   * all 4 warps gather A (im2col / transposed-conv gather) and B (packed weights) tiles with
//     16-byte cp.async into a STAGES-deep ring of 128B-swizzled shared-memory tiles
//     (zero-fill implements conv padding, stride holes and ragged edges);
//   * one elected thread issues tcgen05.mma (M=128, N=BN, K=16 bf16 / K=8 tf32) reading both
//     operands through UMMA shared-memory descriptors, accumulating in TMEM; tcgen05.commit
//     arrives on the stage's mbarrier, which is what releases the slot for the next gather;
//   * the epilogue moves TMEM -> registers with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31,
//     i.e. output rows), adds the bias and stores NHWC rows.
#include "igemm.cuh"
#include "pack.cuh"
#include "tc.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace solb200 {
namespace {

using namespace tc;

constexpr int BM = 128;
constexpr int ROWB = 128;  // bytes per swizzle row
constexpr int THREADS = 128;
constexpr int SMEM_BUDGET = 200 * 1024;

template <typename T> struct AbFmt;
template <> struct AbFmt<__nv_bfloat16> { static constexpr int v = 1; };
template <> struct AbFmt<float> { static constexpr int v = 2; };

template <int STAGE_BYTES>
constexpr int stages_for() {
    return std::min(8, (SMEM_BUDGET - 2048) / STAGE_BYTES);
}

// Epilogue staging of the warp-specialised kernel: 8 KB per storing warp; when the tile has a
// single 128-byte output chunk per row (BN <= CW) only the first four epilogue warps store.
template <typename TO, int BN>
constexpr int ws_epi_bytes() {
    return (BN <= 128 / static_cast<int>(sizeof(TO)) ? 4 : 8) * 8192;
}
// pipeline depth: 227 KB minus 2 KB alignment/barriers and the epilogue staging
template <int STAGE_BYTES, int EPI_BYTES>
constexpr int ws_stages() {
    return std::min(12, (227 * 1024 - 2048 - EPI_BYTES - 1024) / STAGE_BYTES);
}

template <int BN>
constexpr uint32_t tmem_cols() {
    return BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));
}

// Epilogue store of 16 consecutive fp32 accumulators of one row.
// Columns in [nout, ld) are row padding and are written as zeros.
template <typename TO>
__device__ __forceinline__ void store_row16(TO* out, int n, int nout, int ld, const float* f) {
    if (n + 16 <= nout && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
        constexpr int V = 16 / sizeof(TO);
#pragma unroll
        for (int q = 0; q < 16; q += V) store16(out + q, f + q);
    } else {
        for (int q = 0; q < 16 && n + q < ld; ++q) out[q] = from_f32<TO>(n + q < nout ? f[q] : 0.f);
    }
}

// ---------------------------------------------------------------------------------------------
// wgrad: D[Cout][Ncol] += dy^T[Cout][P] * Xcol^T[P][Ncol]; both operands MN-major in smem.
// Tile layout per operand: [mn-block of 64 elems][k-group of 8 pixels][8 rows][128 B]
//   -> LBO (mn-block stride) = (BK/8)*1024 B, SBO (k-group stride) = 1024 B.
// Split-K over pixel ranges; partial tiles go to a workspace reduced by wgrad_reduce_kernel.
// ---------------------------------------------------------------------------------------------

template <typename T, int BN>
__global__ void __launch_bounds__(THREADS, 1) wgrad_kernel(WgradArgs a, int kb_per_split, int ncol) {
    constexpr int VEC = 16 / sizeof(T);
    constexpr int EPB = ROWB / sizeof(T);  // elements per 128B (MN block width)
    constexpr int BK = 64;                 // pixels per k-block (8 k-groups)
    constexpr int A_BLOCKS = BM / EPB;
    constexpr int B_BLOCKS = BN / EPB;
    constexpr int A_BYTES = A_BLOCKS * BK * ROWB;
    constexpr int B_BYTES = B_BLOCKS * BK * ROWB;
    constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    constexpr int STAGES = stages_for<STAGE_BYTES>();
    constexpr uint32_t TCOLS = tmem_cols<BN>();
    constexpr uint32_t IDESC = make_idesc(AbFmt<T>::v, BN, BM, 1, 1);
    constexpr int KPER_MMA = 32 / sizeof(T);  // 16 bf16 / 8 tf32 pixels per instruction
    // bf16: 128B-swizzle atoms of 8 K-rows (1024 B); tf32: 128B_BASE32B atoms of 4 K-rows (512 B)
    constexpr bool B32 = sizeof(T) == 4;
    constexpr int GR = B32 ? 4 : 8;
    constexpr int AT = GR * ROWB;
    constexpr uint32_t LAYOUT = B32 ? 1 : 2;
    constexpr uint32_t LBO = (BK / GR) * AT;
    static_assert(BN % EPB == 0, "BN must be a multiple of the 128B MN block");

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + STAGES);

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int m0 = blockIdx.x * BM;   // Cout block
    const int n0 = blockIdx.y * BN;   // (tap, ci) block
    const int split = blockIdx.z;
    const int P = a.N * a.OH * a.OW;
    const int total_kb = (P + BK - 1) / BK;
    const int kb_begin = split * kb_per_split;
    const int kb_end = min(total_kb, kb_begin + kb_per_split);
    const int num_kb = max(0, kb_end - kb_begin);

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(smem_u32(&mbar[s]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    if (warp == 0) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;

    const T* dy = static_cast<const T*>(a.dy);
    const T* x = static_cast<const T*>(a.x);
    const int j = tid & 7;
    const int rbase = tid >> 3;  // pixel row within k-block: rbase + 16*i, i < 4
    const int ohw = a.OH * a.OW;
    const int ntaps = a.kh * a.kw;

    auto load_stage = [&](int slot, int kb) {
        uint8_t* sa = smem + slot * STAGE_BYTES;
        uint8_t* sb = sa + A_BYTES;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int r = rbase + 16 * i;           // pixel within k-block
            const int p = kb * BK + r;
            const bool pv = p < P;
            int n = 0, oh = 0, ow = 0;
            if (pv) {
                n = p / ohw;
                const int rem = p - n * ohw;
                oh = rem / a.OW;
                ow = rem - oh * a.OW;
            }
            const int kg = r / GR, rr = r % GR;
            const int jp = B32 ? ((((j >> 1) ^ (r & 3)) << 1) | (j & 1)) : (j ^ (r & 7));
            // A: dy[p][m0 + blk*EPB + j*VEC]
#pragma unroll
            for (int blk = 0; blk < A_BLOCKS; ++blk) {
                const int co = m0 + blk * EPB + j * VEC;
                const bool ok = pv && co < a.Cout;
                const T* g = ok ? dy + static_cast<int64_t>(p) * a.ld_dy + co : dy;
                cp_async16(smem_u32(sa + (blk * (BK / GR) + kg) * AT + rr * ROWB + (jp << 4)), g, ok);
            }
            // B: x gathered at pixel p for column n0 + blk*EPB + j*VEC = (tap, ci)
#pragma unroll
            for (int blk = 0; blk < B_BLOCKS; ++blk) {
                const int col = n0 + blk * EPB + j * VEC;
                const int tap = col / a.SC;
                const int ci = col - tap * a.SC;
                const int dkh = tap / a.kw, dkw = tap - (tap / a.kw) * a.kw;
                const int hh = oh * a.sh - a.ph + dkh, ww = ow * a.sw - a.pw + dkw;
                const bool ok = pv && col < ncol && tap < ntaps && hh >= 0 && hh < a.SH && ww >= 0 && ww < a.SW;
                const T* g = ok ? x + ((static_cast<int64_t>(n) * a.SH + hh) * a.SW + ww) * a.SC + ci : x;
                cp_async16(smem_u32(sb + (blk * (BK / GR) + kg) * AT + rr * ROWB + (jp << 4)), g, ok);
            }
        }
    };

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < num_kb) load_stage(s, kb_begin + s);
        cp_async_commit();
    }
    for (int kb = 0; kb < num_kb; ++kb) {
        const int nk = kb + STAGES - 1;
        if (nk < num_kb) {
            const int ns = nk % STAGES;
            if (kb >= 1) mbar_wait(smem_u32(&mbar[ns]), ((kb - 1) / STAGES) & 1);
            load_stage(ns, kb_begin + nk);
        }
        cp_async_commit();
        cp_async_wait<STAGES - 1>();
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const int slot = kb % STAGES;
            const uint32_t a_addr = smem_u32(smem + slot * STAGE_BYTES);
            const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / KPER_MMA; ++k) {
                // K advance: KPER_MMA pixels = KPER_MMA/8 k-groups of 1024 B
                const uint32_t koff = (k * KPER_MMA / GR) * AT;
                const uint64_t ad = sw128_desc(a_addr + koff, LBO, AT, LAYOUT);
                const uint64_t bd = sw128_desc(b_addr + koff, LBO, AT, LAYOUT);
                mma<T>(tmem_d, ad, bd, IDESC, (kb | k) != 0);
            }
            mma_commit(smem_u32(&mbar[slot]));
        }
    }
    if (num_kb > 0) {
        const int last = num_kb - 1;
        mbar_wait(smem_u32(&mbar[last % STAGES]), (last / STAGES) & 1);
    }
    tc_fence_after();

    const int row = warp * 32 + lane;
    const int co = m0 + row;
    float* dst = a.workspace ? a.workspace + static_cast<int64_t>(split) * a.Cout * ncol : a.dw;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tmem_d + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
        const int n = n0 + c0;
        if (co < a.Cout && n < ncol) {
            float f[16];
#pragma unroll
            for (int q = 0; q < 16; ++q) f[q] = num_kb > 0 ? __uint_as_float(v[q]) : 0.0f;
            store_row16<float>(dst + static_cast<int64_t>(co) * ncol + n, n, ncol, ncol, f);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<TCOLS>(tmem_d);
    }
}

// split-K reduction straight into the canonical layout: canonical i = ((co*Cin + ci)*KH + kh)*KW + kw
// reads packed j = co*KH*KW*ld + (kh*KW + kw)*ld + ci of every split. Threads walk the PACKED
// index, so the `splits` partial reads are coalesced and only the one canonical write scatters
// (for a 3x3 the canonical walk read each partial with a stride of ld floats); the split sums
// keep their order (bit-identical), four partial loads in flight.
__global__ void wgrad_reduce_canon_kernel(const float* __restrict__ ws, float* __restrict__ w, int64_t n, int splits,
                                          int Cout, int Cin, int KH, int KW, int ld) {
    const int64_t rowlen = static_cast<int64_t>(KH) * KW * ld;
    const int64_t total = static_cast<int64_t>(Cout) * rowlen;
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < total;
         j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int co = static_cast<int>(j / rowlen);
        const int pcol = static_cast<int>(j - co * rowlen);
        const int tap = pcol / ld;
        const int ci = pcol - tap * ld;
        if (ci >= Cin) continue;
        const int kh = tap / KW, kw = tap - kh * KW;
        float acc = 0.f;
        int sp = 0;
        for (; sp + 4 <= splits; sp += 4) {
            const float v0 = __ldg(ws + static_cast<int64_t>(sp) * n + j);
            const float v1 = __ldg(ws + static_cast<int64_t>(sp + 1) * n + j);
            const float v2 = __ldg(ws + static_cast<int64_t>(sp + 2) * n + j);
            const float v3 = __ldg(ws + static_cast<int64_t>(sp + 3) * n + j);
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; sp < splits; ++sp) acc += __ldg(ws + static_cast<int64_t>(sp) * n + j);
        w[((static_cast<int64_t>(co) * Cin + ci) * KH + kh) * KW + kw] = acc;
    }
}

// Halo wgrad partials (wgrad_halo.cu): group g's spg partials are compact [N co][tiles x 128];
// each thread sums one partial position over the group's CTAs (contiguous, coalesced reads) and
// scatters it to the packed dW [Cout][tap * sc + ci] or the canonical dW [co][ci][kh][kw].
__global__ void wgrad_reduce_halo_kernel(const float* __restrict__ ws, float* __restrict__ dw_packed,
                                         float* __restrict__ dw_canon, int canon_cin, int spg, int sc,
                                         const WhPlan hp) {
    const int cols = wh_cols(hp);
    const int64_t pf = wh_partial_floats(hp);
    const int64_t total = static_cast<int64_t>(hp.groups) * pf;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int g = static_cast<int>(e / pf);
        const int64_t r = e - static_cast<int64_t>(g) * pf;
        const int co_l = static_cast<int>(r / cols), cl = static_cast<int>(r - static_cast<int64_t>(co_l) * cols);
        int co, tap, ci;
        if (hp.pairs) {
            co = co_l;
            tap = cl / sc;
            ci = cl - tap * sc;
            if (tap >= 9) continue;
        } else {
            const int os = g % hp.n_co, cs = (g / hp.n_co) % hp.n_ci, tg = g / (hp.n_co * hp.n_ci);
            tap = tg * hp.TT + cl / 128;
            if (tap >= 9) continue;
            ci = cs * 128 + (cl & 127);
            co = os * hp.N + co_l;
        }
        const float* src = ws + static_cast<int64_t>(g) * spg * pf + r;
        float acc = 0.f;
        int sp = 0;
        for (; sp + 4 <= spg; sp += 4) {  // four partial loads in flight, sums in split order
            const float v0 = __ldg(src + static_cast<int64_t>(sp) * pf);
            const float v1 = __ldg(src + static_cast<int64_t>(sp + 1) * pf);
            const float v2 = __ldg(src + static_cast<int64_t>(sp + 2) * pf);
            const float v3 = __ldg(src + static_cast<int64_t>(sp + 3) * pf);
            acc += v0;
            acc += v1;
            acc += v2;
            acc += v3;
        }
        for (; sp < spg; ++sp) acc += __ldg(src + static_cast<int64_t>(sp) * pf);
        if (dw_canon) {
            if (ci < canon_cin) dw_canon[((static_cast<int64_t>(co) * canon_cin + ci) * 3 + tap / 3) * 3 + tap % 3] = acc;
        } else {
            dw_packed[static_cast<int64_t>(co) * 9 * sc + tap * sc + ci] = acc;
        }
    }
}

__global__ void wgrad_reduce_kernel(const float* __restrict__ ws, float* __restrict__ dw, int64_t n,
                                    int splits) {
    const int64_t i4 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i4 >= n) return;
    if (i4 + 4 <= n) {
        float4 acc = make_float4(0, 0, 0, 0);
        for (int s = 0; s < splits; ++s) {
            float4 v = __ldg(reinterpret_cast<const float4*>(ws + s * n + i4));
            acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
        }
        *reinterpret_cast<float4*>(dw + i4) = acc;
    } else {
        for (int64_t i = i4; i < n; ++i) {
            float acc = 0.f;
            for (int s = 0; s < splits; ++s) acc += ws[s * n + i];
            dw[i] = acc;
        }
    }
}

// ---------------------------------------------------------------------------------------------
// Warp-specialised persistent implicit GEMM (fprop / dgrad).
//
//   warps 0-3  producers: 16-byte cp.async gathers of the A tile (im2col / transposed-conv
//              gather with zero-fill), cp.async.mbarrier.arrive.noinc on the stage's full barrier;
//              thread 0 also issues the TMA load of the B (packed weight) tile. When A is a plain
//              [M][C] matrix (1x1, stride 1, no padding) thread 0 TMA-loads A as well.
//   warps 4-7  epilogue: TMEM -> registers (tcgen05.ld, warp w%4 owns lanes 32(w%4)..), bias,
//              NHWC stores; releases the accumulator stage.
//   warp 8     TMEM allocation + the single-thread tcgen05.mma issuer.
// Barriers: full[S] (128 cp.async arrivals + 1 expect_tx), empty[S] (tcgen05.commit),
// tmem_full[2] (tcgen05.commit), tmem_empty[2] (128 epilogue arrivals). Two TMEM accumulator
// stages let the epilogue of tile i overlap the mainloop of tile i+1.
// ---------------------------------------------------------------------------------------------

constexpr int WS_THREADS = 416;  // 4 producer + 8 epilogue + 1 MMA warps
constexpr int WS_MMA_WARP = 12;
constexpr int IG_FPROP_TMA = 2;     // internal mode: A via TMA (1x1, stride 1, pad 0 fprop)
constexpr int IG_FPROP_IM2COL = 3;  // internal mode: A via TMA im2col (channels multiple of 128 B)
constexpr int IG_DUAL = 4;          // internal mode: two 1x1 convs summed in one accumulator (TMA)

template <int BN>
constexpr uint32_t ws_tmem_cols() {
    return 2 * BN <= 32 ? 32 : (2 * BN <= 64 ? 64 : (2 * BN <= 128 ? 128 : (2 * BN <= 256 ? 256 : 512)));
}

// RESB: the whole packed weight matrix of the single N tile (<= WS_RESB_MAX bytes) is loaded once
// per CTA and stays resident; pipeline stages then carry only the A tile (one third less
// L2 -> shared-memory traffic for the narrow 3x3 convolutions, whose im2col A is L2-bound).
constexpr int WS_RESB_MAX = 80 * 1024;

// EPI = 1: training dgrad epilogues with a ReLU-output mask (IgemmArgs::res_mode / mask);
// a separate instantiation so the inference residual epilogue keeps its register allocation
template <typename T, typename TO, int BN, int MODE, bool RESB = false, int EPI = 0>
__global__ void __launch_bounds__(WS_THREADS, 1)
    igemm_ws_kernel(const IgemmArgs a, const __grid_constant__ CUtensorMap tmap_b,
                    const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_c,
                    const __grid_constant__ CUtensorMap tmap_r, const __grid_constant__ CUtensorMap tmap_a2,
                    const __grid_constant__ CUtensorMap tmap_m) {
    constexpr int VEC = 16 / sizeof(T);
    constexpr int BK = ROWB / sizeof(T);
    constexpr int A_BYTES = BM * ROWB;
    constexpr int B_BYTES = BN * ROWB;
    constexpr int STAGE_BYTES = RESB ? A_BYTES : A_BYTES + B_BYTES;
    constexpr int EPI_BYTES = ws_epi_bytes<TO, BN>();
    constexpr int STAGES = ws_stages<STAGE_BYTES, EPI_BYTES + (RESB ? WS_RESB_MAX : 0)>();
    constexpr int NACC = 2;  // accumulator stages: the epilogue overlaps the next mainloop
    constexpr uint32_t TCOLS = NACC == 1 ? static_cast<uint32_t>(BN) : ws_tmem_cols<BN>();
    constexpr uint32_t IDESC = make_idesc(AbFmt<T>::v, BN, BM, 0, 0);
    constexpr int KSTEP_BYTES = 32;
    constexpr bool A_TMA = MODE == IG_FPROP_TMA || MODE == IG_FPROP_IM2COL || MODE == IG_DUAL;

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* rbar = tempty + 2;  // [8 epilogue warps][2 staging buffers]: residual TMA loads
    uint64_t* bres = rbar + 16;   // resident weights loaded (RESB)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bres + 1);
    uint8_t* bres_smem = smem + STAGES * STAGE_BYTES + 1024 + EPI_BYTES;

    const int tid = threadIdx.x;
    const int warp = tid >> 5, lane = tid & 31;
    const int M = a.N * a.OH * a.OW;
    const int m_tiles = (M + BM - 1) / BM;
    const int n_tiles = (a.Nout + BN - 1) / BN;
    const int tiles = m_tiles * n_tiles;
    const int num_kb = a.K_pad / BK;
    // Work order: tile v = start + k * stride, mapped to t = m * n_tiles + n. EPI == 2 (BN statistics)
    // pins every CTA to one N tile (the host sizes the grid as a multiple of n_tiles), so a warp's
    // columns never change and its statistics accumulate in registers across all its tiles.
    const int v_start = EPI == 2 ? static_cast<int>(blockIdx.x) / n_tiles : static_cast<int>(blockIdx.x);
    const int v_stride = EPI == 2 ? static_cast<int>(gridDim.x) / n_tiles : static_cast<int>(gridDim.x);
    const int v_end = EPI == 2 ? m_tiles : tiles;
    const int n_pin = static_cast<int>(blockIdx.x) % n_tiles;
    auto tile_of = [&](int v) { return EPI == 2 ? v * n_tiles + n_pin : v; };

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), A_TMA ? 1 : 129);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 256);
        }
        for (int s = 0; s < 16; ++s) mbar_init(smem_u32(&rbar[s]), 1);
        mbar_init(smem_u32(bres), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        tma_prefetch(&tmap_b);
        if (A_TMA) tma_prefetch(&tmap_a);
        if (MODE == IG_DUAL) tma_prefetch(&tmap_a2);
    }
    if (warp == WS_MMA_WARP) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        const T* src = static_cast<const T*>(a.src);
        const int j = tid & 7;
        const int rbase = tid >> 3;
        const int ohw = a.OH * a.OW;
        const int ntaps = a.kh * a.kw;
        int stage = 0;
        uint32_t phase = 0;
        if (RESB && tid == 0) {
            mbar_arrive_tx(smem_u32(bres), static_cast<uint32_t>(num_kb * B_BYTES));
            for (int kb = 0; kb < num_kb; ++kb)
                tma_load_2d(smem_u32(bres_smem + kb * B_BYTES), &tmap_b, kb * BK, 0, smem_u32(bres));
        }
        // With TMA operands only thread 0 produces. The other producer threads must not run the
        // loop: nothing waits for them, so a thread that fell a full ring cycle behind saw the
        // empty barrier's parity alias (phase p vs p + 2) and could wait for a completion that never
        // comes once the pipeline drained -- the rare end-of-kernel stall (one CTA left with one
        // producer warp in mbarrier.try_wait; found with cuda-gdb, scripts/diag/hang_hunt.sh)
        const int v_first = (A_TMA && tid != 0) ? v_end : v_start;
        for (int v = v_first; v < v_end; v += v_stride) {
            const int t = tile_of(v);
            const int m0 = (t / n_tiles) * BM;
            const int n0 = (t % n_tiles) * BN;
            int rn[8], rh[8], rw[8];
            if (!A_TMA) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int m = m0 + rbase + 16 * i;
                    if (m < M) {
                        const int n = m / ohw;
                        const int rem = m - n * ohw;
                        const int oh = rem / a.OW;
                        const int ow = rem - oh * a.OW;
                        rn[i] = n;
                        if (MODE == IG_FPROP) {
                            rh[i] = oh * a.sh - a.ph;
                            rw[i] = ow * a.sw - a.pw;
                        } else {
                            rh[i] = oh + a.ph;
                            rw[i] = ow + a.pw;
                        }
                    } else {
                        rn[i] = -1;
                        rh[i] = rw[i] = 0;
                    }
                }
            }
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                uint8_t* sa = smem + stage * STAGE_BYTES;
                uint8_t* sb = sa + A_BYTES;
                if (tid == 0) {
                    mbar_arrive_tx(smem_u32(&full[stage]), RESB ? A_BYTES : (A_TMA ? (A_BYTES + B_BYTES) : B_BYTES));
                    int kbb = kb;
                    if (MODE == IG_DUAL) {  // B columns follow the A source order above
                        const int kb2n = (a.K_pad - a.K1) / BK;
                        kbb = kb < kb2n ? a.K1 / BK + kb : kb - kb2n;
                    }
                    if (!RESB) tma_load_2d(smem_u32(sb), &tmap_b, kbb * BK, n0, smem_u32(&full[stage]));
                    if (MODE == IG_FPROP_TMA) tma_load_2d(smem_u32(sa), &tmap_a, kb * BK, m0, smem_u32(&full[stage]));
                    if (MODE == IG_DUAL) {
                        // the second source's k-blocks (packed at B columns [K1, K_pad)) go first: in
                        // the opposite order (cold downsample input last) the pipeline was observed to
                        // stall intermittently on B200 ("dual GEMM"); this order ran clean
                        // through 30k+ launches
                        const int kb2n = (a.K_pad - a.K1) / BK;
                        if (kb >= kb2n) {
                            tma_load_2d(smem_u32(sa), &tmap_a, (kb - kb2n) * BK, m0, smem_u32(&full[stage]));
                        } else if (a.s2 == 1) {
                            tma_load_2d(smem_u32(sa), &tmap_a2, kb * BK, m0, smem_u32(&full[stage]));
                        } else {
                            const int img = m0 / ohw, rem = m0 - img * ohw;
                            const int oh0 = rem / a.OW, ow0 = rem - (rem / a.OW) * a.OW;
                            tma_load_im2col_4d(smem_u32(sa), &tmap_a2, kb * BK, ow0 * a.s2, oh0 * a.s2, img, 0, 0,
                                               smem_u32(&full[stage]));
                        }
                    }
                    if (MODE == IG_FPROP_IM2COL) {
                        // hardware im2col: 128 output pixels from (n, oh, ow) of m0, one filter tap
                        // (im2col offsets) and one 128-byte channel block per k-block
                        const int cblocks = a.SC / BK;
                        const int tap = kb / cblocks;
                        const int cb = kb - tap * cblocks;
                        const int dkh = tap / a.kw, dkw = tap - (tap / a.kw) * a.kw;
                        const int img = m0 / ohw, rem = m0 - img * ohw;
                        const int oh0 = rem / a.OW, ow0 = rem - (rem / a.OW) * a.OW;
                        tma_load_im2col_4d(smem_u32(sa), &tmap_a, cb * BK, ow0 * a.sw - a.pw, oh0 * a.sh - a.ph, img,
                                           static_cast<uint16_t>(dkw), static_cast<uint16_t>(dkh),
                                           smem_u32(&full[stage]));
                    }
                }
                if (!A_TMA) {
                    const int k = kb * BK + j * VEC;
                    const int tap = k / a.SC;
                    const int c = k - tap * a.SC;
                    const int dkh = tap / a.kw;
                    const int dkw = tap - dkh * a.kw;
                    const bool tap_ok = tap < ntaps;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = rbase + 16 * i;
                        bool ok = tap_ok && rn[i] >= 0;
                        int hh, ww;
                        if (MODE == IG_FPROP) {
                            hh = rh[i] + dkh;
                            ww = rw[i] + dkw;
                        } else {
                            const int nh = rh[i] - dkh, nw = rw[i] - dkw;
                            ok = ok && nh >= 0 && nw >= 0 && (nh % a.sh) == 0 && (nw % a.sw) == 0;
                            hh = nh / a.sh;
                            ww = nw / a.sw;
                        }
                        ok = ok && hh >= 0 && hh < a.SH && ww >= 0 && ww < a.SW;
                        const T* g = ok ? src + ((static_cast<int64_t>(rn[i]) * a.SH + hh) * a.SW + ww) * a.SC + c : src;
                        cp_async16(smem_u32(sa + r * ROWB + ((j ^ (r & 7)) << 4)), g, ok);
                    }
                    cp_async_arrive_noinc(smem_u32(&full[stage]));
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
        if (!A_TMA) cp_async_wait<0>();
    } else if (warp == WS_MMA_WARP) {
        // ------------------------------------------------------------------ MMA issuer
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        if (RESB) mbar_wait(smem_u32(bres), 0);
        const uint64_t a_desc0 = sw128_desc(smem_u32(smem), 16, 1024);
        const uint64_t bres_desc0 = RESB ? sw128_desc(smem_u32(bres_smem), 16, 1024) : 0;
        const bool do_mma = !(a.dbg & 2);
        for (int v = v_start; v < v_end; v += v_stride) {
            mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
            tc_fence_after();
            const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * BN);
            // converged warp, one elected lane issues (tc::mma4_elect): operands stay uniform
            for (int kb = 0; kb < num_kb; ++kb) {
                mbar_wait(smem_u32(&full[stage]), phase);
                tc_fence_after();
                const uint64_t ad = a_desc0 + static_cast<uint32_t>(stage * (STAGE_BYTES >> 4));
                const uint64_t bd = RESB ? bres_desc0 + static_cast<uint32_t>(kb * (B_BYTES >> 4))
                                         : ad + static_cast<uint32_t>(A_BYTES >> 4);
                if (do_mma) mma4_elect<T>(dcol, ad, bd, IDESC, kb != 0);
                mma_commit_elect(smem_u32(&empty[stage]));
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            mma_commit_elect(smem_u32(&tfull[acc]));
            if (++acc == NACC) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue (warps 4-11)
        // TMEM -> registers -> 128B-swizzled smem staging (2 buffers per warp) -> TMA bulk-tensor
        // store of [32 rows x 128 bytes] boxes (OOB rows / columns are clipped by the TMA unit).
        // Two warps per TMEM lane quarter split the accumulator columns (alternate 128B chunks).
        constexpr int CW = 128 / static_cast<int>(sizeof(TO));  // columns per 128-byte box
        const int q = warp & 3;            // TMEM lane quarter
        const int half = (warp - 4) >> 2;  // column interleave
        // (with 4 staging slots the half-1 warps own no chunk and never touch their pointer)
        uint8_t* stage_buf = smem + STAGES * STAGE_BYTES + 1024 + (warp - 4) * 2 * 4096;
        const bool has_bias = a.bias != nullptr;
        const bool has_fold = a.ep_scale != nullptr;
        const bool has_res = a.residual != nullptr;
        const bool res_mask = EPI == 1 && a.res_mode == 1;
        const bool has_m2 = EPI == 1 && a.mask != nullptr;  // host guarantees one chunk per warp (SLOTS == 1)
        const int act = a.relu ? 1 : a.act;
        const bool no_sub_transpose = EPI == 3 && a.dbg & 4096;  // SOL_CONV_DBG=4096: scattered stores
        int acc = 0;
        uint32_t acc_phase = 0;
        int buf = 0;
        uint32_t rphase = 0;
        constexpr int SLOTS = (BN / CW + 1) / 2 > 0 ? (BN / CW + 1) / 2 : 1;
        // EPI == 2: this warp's running BN sums, per chunk slot and owned column pair
        float st_s[SLOTS][2], st_q[SLOTS][2];
#pragma unroll
        for (int k = 0; k < SLOTS; ++k) st_s[k][0] = st_s[k][1] = st_q[k][0] = st_q[k][1] = 0.f;
        for (int v = v_start; v < v_end; v += v_stride) {
            const int t = tile_of(v);
            const int m0 = (t / n_tiles) * BM;
            const int n0 = (t % n_tiles) * BN;
            constexpr int LCOLS = BN < CW ? BN : CW;  // TMEM columns per chunk (never past the tile)
            // residual boxes for this warp's first two chunks are TMA-loaded into the two staging
            // buffers before waiting for the accumulator, so their latency hides behind the mainloop
            if (has_res) {
                if (lane == 0) {
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                    for (int s = 0; s < 2 && s < SLOTS; ++s) {
                        const int cc = half * CW + s * 2 * CW;
                        if (cc >= BN || n0 + cc >= a.ldo) break;
                        const int bi = buf ^ s;
                        mbar_arrive_tx(smem_u32(&rbar[(warp - 4) * 2 + bi]), 4096);
                        tma_load_2d(smem_u32(stage_buf + bi * 4096), &tmap_r, n0 + cc, m0 + q * 32,
                                    smem_u32(&rbar[(warp - 4) * 2 + bi]));
                        if (has_m2) {  // the mask box goes to the other buffer
                            mbar_arrive_tx(smem_u32(&rbar[(warp - 4) * 2 + (bi ^ 1)]), 4096);
                            tma_load_2d(smem_u32(stage_buf + (bi ^ 1) * 4096), &tmap_m, n0 + cc, m0 + q * 32,
                                        smem_u32(&rbar[(warp - 4) * 2 + (bi ^ 1)]));
                        }
                    }
                }
                __syncwarp();
            }
            mbar_wait(smem_u32(&tfull[acc]), acc_phase);
            tc_fence_after();
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int cc = half * CW + s * 2 * CW;
                if (cc >= BN) break;
                const int n = n0 + cc;
                if (n >= a.ldo) break;
                uint32_t v[CW];
                const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + cc);
                if constexpr (LCOLS % 32 == 0) {
#pragma unroll
                    for (int h = 0; h < LCOLS; h += 32) tmem_ld32_nowait(taddr + h, v + h);
                } else {
#pragma unroll
                    for (int h = 0; h < LCOLS; h += 16) tmem_ld16_nowait(taddr + h, v + h);
                }
                tmem_wait_ld();
                float f[CW];
#pragma unroll
                for (int i = 0; i < CW; ++i) f[i] = i < LCOLS ? __uint_as_float(v[i]) : 0.0f;
                if (has_bias) {
                    if (n + CW <= a.Nout) {
#pragma unroll
                        for (int i = 0; i < CW; i += 4) {
                            const float4 bb = __ldg(reinterpret_cast<const float4*>(a.bias + n + i));
                            f[i] += bb.x; f[i + 1] += bb.y; f[i + 2] += bb.z; f[i + 3] += bb.w;
                        }
                    } else {
                        for (int i = 0; i < CW; ++i)
                            if (n + i < a.Nout) f[i] += __ldg(a.bias + n + i);
                    }
                }
                if (has_fold) {
                    if (n + CW <= a.Nout) {
#pragma unroll
                        for (int i = 0; i < CW; i += 4) {
                            const float4 sc = __ldg(reinterpret_cast<const float4*>(a.ep_scale + n + i));
                            const float4 sh = __ldg(reinterpret_cast<const float4*>(a.ep_shift + n + i));
                            f[i] = fmaf(f[i], sc.x, sh.x);
                            f[i + 1] = fmaf(f[i + 1], sc.y, sh.y);
                            f[i + 2] = fmaf(f[i + 2], sc.z, sh.z);
                            f[i + 3] = fmaf(f[i + 3], sc.w, sh.w);
                        }
                    } else {
                        for (int i = 0; i < CW; ++i)
                            if (n + i < a.Nout) f[i] = fmaf(f[i], __ldg(a.ep_scale + n + i), __ldg(a.ep_shift + n + i));
                    }
                }
                uint8_t* sb = stage_buf + buf * 4096;
                if (has_res) {
                    // residual box (zero-filled past the tensor edge) is in this chunk's staging
                    // buffer in the same swizzled layout the output is written in
                    if (s >= 2) {
                        if (lane == 0) {
                            asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                            mbar_arrive_tx(smem_u32(&rbar[(warp - 4) * 2 + buf]), 4096);
                            tma_load_2d(smem_u32(sb), &tmap_r, n, m0 + q * 32, smem_u32(&rbar[(warp - 4) * 2 + buf]));
                        }
                        __syncwarp();
                    }
                    mbar_wait(smem_u32(&rbar[(warp - 4) * 2 + buf]), (rphase >> buf) & 1);
                    rphase ^= 1u << buf;
                    if (has_m2) {
                        mbar_wait(smem_u32(&rbar[(warp - 4) * 2 + (buf ^ 1)]), (rphase >> (buf ^ 1)) & 1);
                        rphase ^= 1u << (buf ^ 1);
                    }
                    uint8_t* mb = stage_buf + (buf ^ 1) * 4096;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const uint32_t addr = smem_u32(sb + lane * 128 + ((j ^ (lane & 7)) << 4));
                        float rr[16 / sizeof(TO)];
                        uint32_t r0, r1, r2, r3;
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                                     : "r"(addr));
                        if constexpr (sizeof(TO) == 2) {
                            const uint32_t w[4] = {r0, r1, r2, r3};
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                rr[2 * k] = __uint_as_float(w[k] << 16);
                                rr[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
                            }
                        } else {
                            rr[0] = __uint_as_float(r0);
                            rr[1] = __uint_as_float(r1);
                            rr[2] = __uint_as_float(r2);
                            rr[3] = __uint_as_float(r3);
                        }
                        float mm[16 / sizeof(TO)];
                        if (has_m2) {
                            uint32_t m0r, m1r, m2r, m3r;
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];\n"
                                         : "=r"(m0r), "=r"(m1r), "=r"(m2r), "=r"(m3r)
                                         : "r"(smem_u32(mb + lane * 128 + ((j ^ (lane & 7)) << 4))));
                            if constexpr (sizeof(TO) == 2) {
                                const uint32_t w[4] = {m0r, m1r, m2r, m3r};
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    mm[2 * k] = __uint_as_float(w[k] << 16);
                                    mm[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
                                }
                            } else {
                                mm[0] = __uint_as_float(m0r);
                                mm[1] = __uint_as_float(m1r);
                                mm[2] = __uint_as_float(m2r);
                                mm[3] = __uint_as_float(m3r);
                            }
                        }
#pragma unroll
                        for (int k = 0; k < static_cast<int>(16 / sizeof(TO)); ++k) {
                            float& fv = f[j * (16 / sizeof(TO)) + k];
                            // Add + ReluBack: the unfused plan adds the stored (rounded) dgrad output
                            if constexpr (sizeof(TO) == 2)
                                if (has_m2) fv = __bfloat162float(__float2bfloat16_rn(fv));
                            fv = res_mask ? (rr[k] > 0.f ? fv : 0.f) : fv + rr[k];
                            if (has_m2) fv = mm[k] > 0.f ? fv : 0.f;
                        }
                    }
                }
                if (act != 0) {
#pragma unroll
                    for (int i = 0; i < CW; ++i) {
                        f[i] = fmaxf(f[i], 0.0f);
                        if (act == 2) f[i] = fminf(f[i], 6.0f);
                    }
                }
                if constexpr (EPI == 3) {
                    // sub-pixel dgrad class stored in place: this lane's row is one class-grid
                    // pixel; its 128 bytes go to the strided output pixel (and zeros to the rest
                    // of its stride cell when the other classes have no taps)
                    static_assert(sizeof(TO) == 2, "in-place sub-pixel classes are bf16");
                    const int m = m0 + q * 32 + lane;
                    if (n + CW <= a.ldo && !(a.dbg & 1) && !no_sub_transpose) {
                        // coalesced form: the warp's 32 rows go through the (idle) staging buffer,
                        // then every store instruction writes 4 whole output pixels (4 x 128 B)
                        // instead of 32 scattered 16-byte pieces. Per lane: its stride cell's
                        // origin and a mask of the cell positions inside the image
                        TO* cell = nullptr;
                        uint32_t pos_ok = 0;
                        if (m < M) {
                            const int ohw = a.OH * a.OW;
                            const int img = m / ohw, rem = m - img * ohw;
                            const int i = rem / a.OW, j = rem - i * a.OW;
                            const int oy = a.sub_sh * i, ox = a.sub_sw * j;
                            cell = static_cast<TO*>(a.out) + n + ((static_cast<int64_t>(img) * a.sub_H + oy) * a.sub_W + ox) * a.ldo;
                            for (int da = 0; da < a.sub_sh; ++da)
                                for (int db = 0; db < a.sub_sw; ++db)
                                    if (oy + da < a.sub_H && ox + db < a.sub_W) pos_ok |= 1u << (da * a.sub_sw + db);
                        }
                        uint8_t* sbuf = stage_buf;
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            __nv_bfloat162 p0 = __floats2bfloat162_rn(f[8 * k], f[8 * k + 1]);
                            __nv_bfloat162 p1 = __floats2bfloat162_rn(f[8 * k + 2], f[8 * k + 3]);
                            __nv_bfloat162 p2 = __floats2bfloat162_rn(f[8 * k + 4], f[8 * k + 5]);
                            __nv_bfloat162 p3 = __floats2bfloat162_rn(f[8 * k + 6], f[8 * k + 7]);
                            *reinterpret_cast<uint4*>(sbuf + lane * 128 + ((k ^ (lane & 7)) << 4)) =
                                make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                                           *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
                        }
                        __syncwarp();
                        const int k = lane & 7;
                        const int mine_pos = a.sub_a * a.sub_sw + a.sub_b;
#pragma unroll 2
                        for (int it = 0; it < 8; ++it) {
                            const int r = it * 4 + (lane >> 3);
                            const uint4 val = *reinterpret_cast<const uint4*>(sbuf + r * 128 + ((k ^ (r & 7)) << 4));
                            TO* cr = reinterpret_cast<TO*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(cell), r));
                            const uint32_t ok = __shfl_sync(0xffffffffu, pos_ok, r);
                            if (!a.sub_zero) {  // this class's own position only
                                if ((ok >> mine_pos) & 1u)
                                    *reinterpret_cast<uint4*>(cr + (static_cast<int64_t>(a.sub_a) * a.sub_W + a.sub_b) * a.ldo + 8 * k) = val;
                                continue;
                            }
                            for (int da = 0; da < a.sub_sh; ++da)
                                for (int db = 0; db < a.sub_sw; ++db) {
                                    const int ps = da * a.sub_sw + db;
                                    const bool mine = ps == mine_pos;
                                    if ((!mine && !a.sub_zero) || !((ok >> ps) & 1u)) continue;
                                    *reinterpret_cast<uint4*>(cr + (static_cast<int64_t>(da) * a.sub_W + db) * a.ldo + 8 * k) =
                                        mine ? val : make_uint4(0, 0, 0, 0);
                                }
                        }
                        __syncwarp();  // the rows are read before the next chunk rewrites the buffer
                        continue;
                    }
                    if (m < M && !(a.dbg & 1)) {
                        const int ohw = a.OH * a.OW;
                        const int img = m / ohw, rem = m - img * ohw;
                        const int i = rem / a.OW, j = rem - i * a.OW;
                        const int oy = a.sub_sh * i, ox = a.sub_sw * j;
                        TO* base = static_cast<TO*>(a.out) + n;
                        const bool full = n + CW <= a.ldo;
                        uint4 pk[8];
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            __nv_bfloat162 p0 = __floats2bfloat162_rn(f[8 * k], f[8 * k + 1]);
                            __nv_bfloat162 p1 = __floats2bfloat162_rn(f[8 * k + 2], f[8 * k + 3]);
                            __nv_bfloat162 p2 = __floats2bfloat162_rn(f[8 * k + 4], f[8 * k + 5]);
                            __nv_bfloat162 p3 = __floats2bfloat162_rn(f[8 * k + 6], f[8 * k + 7]);
                            pk[k] = make_uint4(*reinterpret_cast<uint32_t*>(&p0), *reinterpret_cast<uint32_t*>(&p1),
                                               *reinterpret_cast<uint32_t*>(&p2), *reinterpret_cast<uint32_t*>(&p3));
                        }
                        for (int da = 0; da < a.sub_sh; ++da) {
                            for (int db = 0; db < a.sub_sw; ++db) {
                                const bool mine = da == a.sub_a && db == a.sub_b;
                                if (!mine && !a.sub_zero) continue;
                                if (oy + da >= a.sub_H || ox + db >= a.sub_W) continue;
                                TO* o = base + ((static_cast<int64_t>(img) * a.sub_H + oy + da) * a.sub_W + ox + db) * a.ldo;
                                if (full) {
#pragma unroll
                                    for (int k = 0; k < 8; ++k)
                                        *reinterpret_cast<uint4*>(o + 8 * k) = mine ? pk[k] : make_uint4(0, 0, 0, 0);
                                } else {
                                    for (int k = 0; k < CW && n + k < a.ldo; ++k)
                                        o[k] = mine ? __float2bfloat16_rn(f[k]) : __float2bfloat16_rn(0.f);
                                }
                            }
                        }
                    }
                    continue;
                }
                // the staging buffer is free once the TMA store issued two chunks ago has read it
                // (with a residual, the buffer was drained before the residual load was issued)
                if (!has_res) {
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
                    __syncwarp();
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t addr = smem_u32(sb + lane * 128 + ((j ^ (lane & 7)) << 4));
                    const float* src = f + j * (16 / static_cast<int>(sizeof(TO)));
                    if constexpr (sizeof(TO) == 2) {
                        __nv_bfloat162 p0 = __floats2bfloat162_rn(src[0], src[1]);
                        __nv_bfloat162 p1 = __floats2bfloat162_rn(src[2], src[3]);
                        __nv_bfloat162 p2 = __floats2bfloat162_rn(src[4], src[5]);
                        __nv_bfloat162 p3 = __floats2bfloat162_rn(src[6], src[7]);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr),
                                     "r"(*reinterpret_cast<uint32_t*>(&p0)), "r"(*reinterpret_cast<uint32_t*>(&p1)),
                                     "r"(*reinterpret_cast<uint32_t*>(&p2)), "r"(*reinterpret_cast<uint32_t*>(&p3)));
                    } else {
                        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "f"(src[0]),
                                     "f"(src[1]), "f"(src[2]), "f"(src[3]));
                    }
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0 && !(a.dbg & 1)) {
                    asm volatile(
                        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                            reinterpret_cast<uint64_t>(&tmap_c)),
                        "r"(n), "r"(m0 + q * 32), "r"(smem_u32(sb))
                        : "memory");
                    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                }
                if constexpr (EPI == 2) {
                    // BN statistics of the stored chunk, read back from the staging buffer (the
                    // TMA store reads it concurrently): lane l owns columns n + 2l, n + 2l + 1;
                    // rows past M (zero-filled A) are excluded; sums of (y - shift) accumulate
                    // in registers until the CTA's last tile
                    static_assert(sizeof(TO) == 2, "BN statistics epilogue is bf16");
                    const int rv = min(32, M - (m0 + q * 32));
                    const int c0 = n + 2 * lane;
                    if (c0 < a.Nout && rv > 0) {
                        const float h0 = __ldg(a.stat_shift + c0);
                        const float h1 = c0 + 1 < a.Nout ? __ldg(a.stat_shift + c0 + 1) : 0.f;
                        const uint32_t base = smem_u32(sb) + static_cast<uint32_t>((lane & 3) * 4);
                        float s0 = 0.f, s1 = 0.f, q0 = 0.f, q1 = 0.f;
                        for (int r = 0; r < rv; ++r) {
                            uint32_t w;
                            asm volatile("ld.shared.b32 %0, [%1];\n"
                                         : "=r"(w)
                                         : "r"(base + static_cast<uint32_t>(r * 128 + (((lane >> 2) ^ (r & 7)) << 4))));
                            const float v0 = __uint_as_float(w << 16) - h0, v1 = __uint_as_float(w & 0xffff0000u) - h1;
                            s0 += v0;
                            q0 = fmaf(v0, v0, q0);
                            s1 += v1;
                            q1 = fmaf(v1, v1, q1);
                        }
                        st_s[s][0] += s0;
                        st_q[s][0] += q0;
                        st_s[s][1] += s1;
                        st_q[s][1] += q1;
                    }
                }
                buf ^= 1;
            }
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty[acc]));
            if (++acc == NACC) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        __syncwarp();
        if constexpr (EPI == 2) {
            // one partial block per (CTA, lane quarter): stat_partial[(c * MAXB + b) * 2 + {sum, sum sq}]
            // (MAXB = a.stat_blocks >= 4 * gridDim.x; CTA 0 zero-fills the blocks no CTA owns)
            const int64_t nblk = a.stat_blocks;
            const int64_t blk = static_cast<int64_t>(blockIdx.x) * 4 + q;
#pragma unroll
            for (int s = 0; s < SLOTS; ++s) {
                const int cc = half * CW + s * 2 * CW;
                if (cc >= BN) break;
                const int c0 = n_pin * BN + cc + 2 * lane;
                if (c0 < a.Nout) {
                    *reinterpret_cast<double2*>(a.stat_partial + (c0 * nblk + blk) * 2) = make_double2(st_s[s][0], st_q[s][0]);
                    if (c0 + 1 < a.Nout)
                        *reinterpret_cast<double2*>(a.stat_partial + ((c0 + 1) * nblk + blk) * 2) =
                            make_double2(st_s[s][1], st_q[s][1]);
                }
            }
            // blocks past 4 x gridDim.x belong to no CTA: zeroed, channels spread over the CTAs
            const int used = 4 * static_cast<int>(gridDim.x);
            for (int c = blockIdx.x; c < a.Nout; c += gridDim.x)
                for (int b = used + (tid - 128); b < static_cast<int>(nblk); b += 256)
                    *reinterpret_cast<double2*>(a.stat_partial + (static_cast<int64_t>(c) * nblk + b) * 2) =
                        make_double2(0.0, 0.0);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == WS_MMA_WARP) {
        tc_fence_after();
        tmem_dealloc<TCOLS>(tmem_base);
    }
}

// Im2col tensor map over the NHWC activation (dims {C, W, H, N}): pixelsPerColumn = 128 output
// pixels per load, channelsPerPixel = one 128-byte channel block, traversal strides = conv
// strides, bounding box corners (-pad, pad - (k-1)) so every window start of the convolution is
// enumerated in (n, oh, ow) order; OOB taps are zero-filled (the conv padding).
using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

CUtensorMap make_tmap_im2col(const IgemmArgs& a, int dtype, int rows = BM) {
    static EncodeIm2colFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        SOL_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw std::runtime_error("cuTensorMapEncodeIm2col unavailable");
        return reinterpret_cast<EncodeIm2colFn>(p);
    }();
    CUtensorMap m;
    const uint64_t es = dtype == DT_BF16 ? 2 : 4;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.SC), static_cast<cuuint64_t>(a.SW),
                          static_cast<cuuint64_t>(a.SH), static_cast<cuuint64_t>(a.N)};
    cuuint64_t strides[3] = {a.SC * es, static_cast<cuuint64_t>(a.SW) * a.SC * es,
                             static_cast<cuuint64_t>(a.SH) * a.SW * a.SC * es};
    // base positions run from `lower` to (S - 1 + upper) in steps of the stride: exactly O of them
    int lower[2] = {-a.pw, -a.ph};
    int upper[2] = {(a.OW - 1) * a.sw - (a.SW - 1) - a.pw, (a.OH - 1) * a.sh - (a.SH - 1) - a.ph};
    cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(a.sw), static_cast<cuuint32_t>(a.sh), 1};
    const CUresult r = fn(&m, dtype == DT_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                          const_cast<void*>(a.src), dims, strides, lower, upper, static_cast<cuuint32_t>(128 / es),
                          static_cast<cuuint32_t>(rows), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        throw std::runtime_error("cuTensorMapEncodeIm2col failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

template <typename T, typename TO, int BN, int MODE, bool RESB = false, int EPI = 0>
void launch_ws_t(const IgemmArgs& a, cudaStream_t s) {
    constexpr int STAGE_BYTES = RESB ? BM * ROWB : BM * ROWB + BN * ROWB;
    constexpr int EPI_BYTES = ws_epi_bytes<TO, BN>();
    constexpr int STAGES = ws_stages<STAGE_BYTES, EPI_BYTES + (RESB ? WS_RESB_MAX : 0)>();
    constexpr int SMEM = STAGES * STAGE_BYTES + 2048 + EPI_BYTES + (RESB ? WS_RESB_MAX : 0);
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(igemm_ws_kernel<T, TO, BN, MODE, RESB, EPI>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    });
    const int M = a.N * a.OH * a.OW;
    const int dt = sizeof(T) == 2 ? DT_BF16 : DT_F32;
    const int n_rows = static_cast<int>(ceil_div(a.Nout, BN)) * BN;  // packed B has >= Nout rows
    CUtensorMap tb = make_tmap_2d(a.wt, dt, a.K_pad, static_cast<uint64_t>(a.Nout), a.K_pad, BN);
    (void)n_rows;
    CUtensorMap ta = tb, ta2 = tb;
    if (MODE == IG_FPROP_TMA || MODE == IG_DUAL) ta = make_tmap_2d(a.src, dt, a.SC, static_cast<uint64_t>(M), a.SC, BM);
    if (MODE == IG_FPROP_IM2COL) ta = make_tmap_im2col(a, dt);
    if (MODE == IG_DUAL) {
        if (a.s2 == 1) {
            ta2 = make_tmap_2d(a.src2, dt, a.SC2, static_cast<uint64_t>(M), a.SC2, BM);
        } else {
            IgemmArgs g2 = a;
            g2.src = a.src2;
            g2.SH = a.SH2; g2.SW = a.SW2; g2.SC = a.SC2;
            g2.kh = g2.kw = 1; g2.sh = g2.sw = a.s2; g2.ph = g2.pw = 0;
            ta2 = make_tmap_im2col(g2, dt);
        }
    }
    const int tiles = static_cast<int>(ceil_div(M, BM) * ceil_div(a.Nout, BN));
    int grid = std::min(tiles, a.max_ctas > 0 ? std::min(a.max_ctas, num_sms()) : num_sms());
    if constexpr (EPI == 2) {  // every CTA pinned to one N tile (see the kernel's work order)
        const int nt = static_cast<int>(ceil_div(a.Nout, BN)), mt = static_cast<int>(ceil_div(M, BM));
        if (nt > num_sms() || a.stat_blocks < 4 * num_sms()) throw std::invalid_argument("igemm: BN statistics layout");
        grid = nt * std::max(1, std::min(mt, num_sms() / nt));
    }
    const int dto = sizeof(TO) == 2 ? DT_BF16 : DT_F32;
    CUtensorMap tc = make_tmap_2d(a.out, dto, a.ldo, static_cast<uint64_t>(M), a.ldo, 32);
    CUtensorMap tr = tc, tm = tc;
    if (a.residual) tr = make_tmap_2d(a.residual, dto, a.Nout, static_cast<uint64_t>(M), a.ld_res, 32);
    if (a.mask) {
        constexpr int CW = 128 / static_cast<int>(sizeof(TO));
        if ((BN / CW + 1) / 2 > 1 || !a.residual) throw std::logic_error("igemm: epilogue mask needs one chunk per warp");
        tm = make_tmap_2d(a.mask, dto, a.Nout, static_cast<uint64_t>(M), a.ld_res, 32);
    }
    igemm_ws_kernel<T, TO, BN, MODE, RESB, EPI><<<grid, WS_THREADS, SMEM, s>>>(a, tb, ta, tc, tr, ta2, tm);
    SOL_CUDA(cudaGetLastError());
}

template <typename T, typename TO, int MODE>
void dispatch_ws_mask(const IgemmArgs& a, cudaStream_t s) {
    // the add + mask form needs one epilogue chunk per warp: 128-wide tiles (bf16), 64 (f32); the
    // mask-only form (ReluBack) takes any tile, 256 included (bf16)
    constexpr int BNMAX = sizeof(TO) == 2 ? 128 : 64;
    const int lim = (sizeof(TO) == 2 && !a.mask) ? 256 : BNMAX;
    int bn = a.tile_n ? std::min(a.tile_n == 65 ? 64 : a.tile_n, lim) : std::min(igemm_block_n(a.Nout), lim);
    if (bn < 64) bn = 64;
    if constexpr (sizeof(TO) == 2) {
        if (bn == 256) return launch_ws_t<T, TO, 256, MODE, false, 1>(a, s);
    }
    if constexpr (BNMAX == 128) {
        if (bn == 128) return launch_ws_t<T, TO, 128, MODE, false, 1>(a, s);
    }
    launch_ws_t<T, TO, 64, MODE, false, 1>(a, s);
}

template <typename T, typename TO, int MODE>
void dispatch_ws_stats(const IgemmArgs& a, cudaStream_t s) {
    if constexpr (sizeof(T) == 2 && sizeof(TO) == 2 && (MODE == IG_FPROP_TMA || MODE == IG_FPROP_IM2COL)) {
        const int bn = a.tile_n ? (a.tile_n == 65 ? 64 : a.tile_n) : std::max(64, igemm_block_n(a.Nout));
        switch (bn) {
            case 64: return launch_ws_t<T, TO, 64, MODE, false, 2>(a, s);
            case 128: return launch_ws_t<T, TO, 128, MODE, false, 2>(a, s);
            default: return launch_ws_t<T, TO, 256, MODE, false, 2>(a, s);
        }
    }
    throw std::invalid_argument("igemm: BN statistics epilogue needs a bf16 TMA / TMA-im2col conv");
}

template <typename T, typename TO, int MODE>
void dispatch_ws_sub(const IgemmArgs& a, cudaStream_t s) {
    if constexpr (sizeof(T) == 2 && sizeof(TO) == 2 && (MODE == IG_FPROP_TMA || MODE == IG_FPROP_IM2COL)) {
        const int bn = a.tile_n ? (a.tile_n == 65 ? 64 : a.tile_n) : std::max(64, igemm_block_n(a.Nout));
        switch (bn) {
            case 64: return launch_ws_t<T, TO, 64, MODE, false, 3>(a, s);
            case 128: return launch_ws_t<T, TO, 128, MODE, false, 3>(a, s);
            default: return launch_ws_t<T, TO, 256, MODE, false, 3>(a, s);
        }
    }
    throw std::invalid_argument("igemm: in-place sub-pixel classes need a bf16 TMA / TMA-im2col conv");
}

template <typename T, typename TO, int MODE>
void dispatch_ws(const IgemmArgs& a, cudaStream_t s) {
    if (a.sub_sh) return dispatch_ws_sub<T, TO, MODE>(a, s);
    if (a.stat_partial) return dispatch_ws_stats<T, TO, MODE>(a, s);
    if constexpr (MODE == IG_FPROP_TMA || MODE == IG_FPROP_IM2COL || MODE == IG_FPROP) {
        if (a.mask || a.res_mode) return dispatch_ws_mask<T, TO, MODE>(a, s);
    }
    if (a.mask || a.res_mode) throw std::invalid_argument("igemm: masked epilogues are fprop-path only");
    if (a.tile_n) {  // autotuned choice
        if constexpr (sizeof(T) == 2 && sizeof(TO) == 2 && (MODE == IG_FPROP_TMA || MODE == IG_FPROP_IM2COL)) {
            if (a.tile_n == 65 && a.K_pad / 64 * 64 * ROWB <= WS_RESB_MAX) return launch_ws_t<T, TO, 64, MODE, true>(a, s);
        }
        switch (a.tile_n) {
            case 64: case 65: return launch_ws_t<T, TO, 64, MODE>(a, s);
            case 128: return launch_ws_t<T, TO, 128, MODE>(a, s);
            case 256: return launch_ws_t<T, TO, 256, MODE>(a, s);
            default: throw std::invalid_argument("igemm: tile_n must be 0, 64, 65, 128 or 256");
        }
    }
    if constexpr (sizeof(T) == 2 && sizeof(TO) == 2 && (MODE == IG_FPROP_TMA || MODE == IG_FPROP_IM2COL)) {
        const int bn = igemm_block_n(a.Nout);
        static const bool no_resb = std::getenv("SOL_NO_RESB") != nullptr;
        if (bn == 64 && a.K_pad / 64 * 64 * ROWB <= WS_RESB_MAX && a.K_pad >= 256 && !(a.dbg & 1024) && !no_resb)
            return launch_ws_t<T, TO, 64, MODE, true>(a, s);
    }
    int bn_sel = igemm_block_n(a.Nout);
    // small-M GEMMs (the classifier: M = batch): narrower N tiles put more SMs on the long K loop
    const int64_t m_tiles = ceil_div(static_cast<int64_t>(a.N) * a.OH * a.OW, BM);
    if (bn_sel > 64 && m_tiles * ceil_div(a.Nout, bn_sel) < num_sms() / 4) bn_sel = 64;
    switch (bn_sel) {
        case 16: return launch_ws_t<T, TO, 16, MODE>(a, s);
        case 32: return launch_ws_t<T, TO, 32, MODE>(a, s);
        case 64: return launch_ws_t<T, TO, 64, MODE>(a, s);
        case 128: return launch_ws_t<T, TO, 128, MODE>(a, s);
        default: return launch_ws_t<T, TO, 256, MODE>(a, s);
    }
}

template <typename T, typename TO>
void dispatch_mode(const IgemmArgs& a, cudaStream_t s) {
    const bool plain = a.mode == IG_FPROP && a.kh == 1 && a.kw == 1 && a.sh == 1 && a.sw == 1 && a.ph == 0 &&
                       a.pw == 0 && a.K_pad == a.SC;
    constexpr int BK = ROWB / sizeof(T);
    const bool im2col = a.mode == IG_FPROP && !plain && a.SC % BK == 0 && a.K_pad == a.kh * a.kw * a.SC &&
                        a.kh <= 8 && a.kw <= 8;
    if constexpr (sizeof(T) == 2 && sizeof(TO) == 2) {
        if (a.src2) {
            // 256-wide tiles with two accumulator stages (the whole TMEM) halve the A re-reads of
            // both sources: ResNet-50 l2.0 / l3.0 / l4.0 tails 107 / 91 / 84 -> 95 / 84 / 81 us.
            // (The intermittent stall once blamed on this configuration was the idle-producer
            // barrier aliasing fixed in igemm_ws_kernel.) SOL_DUAL_BN256=0/1 forces off/on
            static const char* bn256_env = std::getenv("SOL_DUAL_BN256");
            const bool bn256 = a.tile_n ? a.tile_n == 256 : (bn256_env ? bn256_env[0] == '1' : true);
            if (a.Nout > 128 && bn256) return launch_ws_t<T, TO, 256, IG_DUAL>(a, s);
            if (a.Nout > 64) return launch_ws_t<T, TO, 128, IG_DUAL>(a, s);
            return dispatch_ws<T, TO, IG_DUAL>(a, s);
        }
    }
    if (a.src2) throw std::invalid_argument("igemm: dual GEMM is bf16 only");
    if (plain) dispatch_ws<T, TO, IG_FPROP_TMA>(a, s);
    else if (im2col) dispatch_ws<T, TO, IG_FPROP_IM2COL>(a, s);
    else if (a.mode == IG_FPROP) dispatch_ws<T, TO, IG_FPROP>(a, s);
    else dispatch_ws<T, TO, IG_DGRAD>(a, s);
}

// ---------------------------------------------------------------------------------------------
// host dispatch
// ---------------------------------------------------------------------------------------------

template <typename T, int BN>
void launch_wgrad_t(const WgradArgs& a, int ncol, int splits, int kb_per_split, cudaStream_t s) {
    constexpr int EPB = ROWB / sizeof(T);
    constexpr int STAGE_BYTES = (BM / EPB) * 64 * ROWB + (BN / EPB) * 64 * ROWB;
    constexpr int STAGES = stages_for<STAGE_BYTES>();
    constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + STAGES * 8 + 16;
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(wgrad_kernel<T, BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    });
    dim3 grid(static_cast<unsigned>(ceil_div(a.Cout, BM)), static_cast<unsigned>(ceil_div(ncol, BN)),
              static_cast<unsigned>(splits));
    wgrad_kernel<T, BN><<<grid, THREADS, SMEM, s>>>(a, kb_per_split, ncol);
    SOL_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------------
// wgrad, bf16 fast path: persistent warp-specialised tcgen05 GEMM with both operands by TMA.
//   D[M][N] = sum_p A[p][m] * B[p][n], both operands MN-major in shared memory (pixels = K):
//     dy    [P][Cout]        2-D tiled TMA, boxes of 64 channels x 64 pixels
//     xcol  [P][(tap, ci)]   TMA im2col, one box = 64 pixels x 64 channels of one tap
//   normal:  M = Cout (dy), N = columns (xcol);  swapped (Cout < 128): M = columns, N = Cout.
// Work items = (m tile, n tile, pixel split); each writes its f32 tile to the split's slice of
// the workspace [split][Cout][ncol] (or straight to dW with one split), reduced afterwards.
//   warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue (TMEM double-buffered).
// ---------------------------------------------------------------------------------------------
constexpr int WG_THREADS = 192;
constexpr int WG_BK = 64;  // pixels per k-block

template <int BN>
constexpr int wg_stages() {
    return std::min(8, (227 * 1024 - 2048) / (128 * WG_BK * 2 + BN * WG_BK * 2));
}

template <int BN, bool SWAP>
__global__ void __launch_bounds__(WG_THREADS, 1)
    wgrad_ws_kernel(const WgradArgs a, const __grid_constant__ CUtensorMap tm_dy,
                    const __grid_constant__ CUtensorMap tm_x, int ncol, int m_tiles, int n_tiles, int splits,
                    int kb_per_split) {
    constexpr int A_BYTES = 128 * WG_BK * 2;
    constexpr int B_BYTES = BN * WG_BK * 2;
    constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    constexpr int STAGES = wg_stages<BN>();
    constexpr uint32_t TCOLS = ws_tmem_cols<BN>();
    constexpr uint32_t IDESC = make_idesc(1, BN, 128, 1, 1);
    constexpr uint32_t LBO = (WG_BK / 8) * 1024;  // stride between 64-element MN blocks

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int P = a.N * a.OH * a.OW;
    const int total_kb = (P + WG_BK - 1) / WG_BK;
    const int items = m_tiles * n_tiles * splits;
    const int ohw = a.OH * a.OW;

    if (tid == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        tma_prefetch(&tm_dy);
        tma_prefetch(&tm_x);
    }
    if (warp == 1) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    // tile-fastest order: the CTAs running at once cover every tile of a few pixel splits, so the
    // dy rows and the (tap-shifted) x rows of a split are fetched from HBM once and re-read from L2
    // by the other tiles (split-fastest order re-read them from HBM once per tile: ~9x for 3x3)
    const int tiles = m_tiles * n_tiles;
    auto decode = [&](int it, int& tm, int& tn, int& kb0, int& kb1) {
        const int sp = it / tiles;
        const int t = it - sp * tiles;
        tm = t / n_tiles;
        tn = t - tm * n_tiles;
        kb0 = sp * kb_per_split;
        kb1 = min(total_kb, kb0 + kb_per_split);
    };

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int it = blockIdx.x; it < items; it += gridDim.x) {
                int tm, tn, kb0, kb1;
                decode(it, tm, tn, kb0, kb1);
                const int co_base = SWAP ? tn * BN : tm * 128;
                const int col_base = SWAP ? tm * 128 : tn * BN;
                constexpr int CO_BLOCKS = SWAP ? BN / 64 : 2;
                constexpr int COL_BLOCKS = SWAP ? 2 : BN / 64;
                for (int kb = kb0; kb < kb1; ++kb) {
                    mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                    uint8_t* sa = smem + stage * STAGE_BYTES;
                    uint8_t* sb = sa + A_BYTES;
                    uint8_t* s_dy = SWAP ? sb : sa;
                    uint8_t* s_x = SWAP ? sa : sb;
                    const uint32_t fb = smem_u32(&full[stage]);
                    mbar_arrive_tx(fb, STAGE_BYTES);
                    const int p0 = kb * WG_BK;
#pragma unroll
                    for (int j = 0; j < CO_BLOCKS; ++j)
                        tma_load_2d(smem_u32(s_dy + j * WG_BK * 128), &tm_dy, co_base + 64 * j, p0, fb);
                    const int img = p0 / ohw, rem = p0 - img * ohw;
                    const int oh0 = rem / a.OW, ow0 = rem - (rem / a.OW) * a.OW;
#pragma unroll
                    for (int j = 0; j < COL_BLOCKS; ++j) {
                        int col = col_base + 64 * j;
                        if (col >= ncol) col = 0;  // tile padding: any in-range box (discarded)
                        const int tap = col / a.SC, ci = col - tap * a.SC;
                        const int dkh = tap / a.kw, dkw = tap - dkh * a.kw;
                        tma_load_im2col_4d(smem_u32(s_x + j * WG_BK * 128), &tm_x, ci, ow0 * a.sw - a.pw,
                                           oh0 * a.sh - a.ph, img, static_cast<uint16_t>(dkw),
                                           static_cast<uint16_t>(dkh), fb);
                    }
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        int stage = 0, acc = 0;
        uint32_t phase = 0, acc_phase = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int tm, tn, kb0, kb1;
            decode(it, tm, tn, kb0, kb1);
            mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
            tc_fence_after();
            const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * BN);
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(smem_u32(&full[stage]), phase);
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t a_addr = smem_u32(smem + stage * STAGE_BYTES);
                    const uint32_t b_addr = a_addr + A_BYTES;
#pragma unroll
                    for (int k = 0; k < WG_BK / 16; ++k) {
                        const uint64_t ad = sw128_desc(a_addr + k * 2048, LBO, 1024);
                        const uint64_t bd = sw128_desc(b_addr + k * 2048, LBO, 1024);
                        mma<__nv_bfloat16>(dcol, ad, bd, IDESC, (kb > kb0 || k > 0) ? 1u : 0u);
                    }
                    mma_commit(smem_u32(&empty[stage]));
                }
                __syncwarp();
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (lane == 0) mma_commit(smem_u32(&tfull[acc]));
            __syncwarp();
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue
        const int q = warp & 3;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int it = blockIdx.x; it < items; it += gridDim.x) {
            int tm, tn, kb0, kb1;
            decode(it, tm, tn, kb0, kb1);
            const int sp = it / tiles;
            float* dst = a.workspace ? a.workspace + static_cast<int64_t>(sp) * a.Cout * ncol : a.dw;
            mbar_wait(smem_u32(&tfull[acc]), acc_phase);
            tc_fence_after();
            const int row = tm * 128 + q * 32 + lane;  // M index
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t v[32];
                tmem_ld32_nowait(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + c0), v);
                tmem_wait_ld();
                const int nb = tn * BN + c0;  // first N index of this chunk
                if (!SWAP) {
                    if (row < a.Cout) {
                        float* o = dst + static_cast<int64_t>(row) * ncol + nb;
                        if (nb + 32 <= ncol) {
#pragma unroll
                            for (int i = 0; i < 32; i += 4)
                                *reinterpret_cast<float4*>(o + i) =
                                    make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
                        } else {
                            for (int i = 0; i < 32 && nb + i < ncol; ++i) o[i] = __uint_as_float(v[i]);
                        }
                    }
                } else if (row < ncol) {
                    // row = column of dW, the chunk's 32 values = 32 consecutive Cout
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (nb + i < a.Cout) dst[static_cast<int64_t>(nb + i) * ncol + row] = __uint_as_float(v[i]);
                }
            }
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty[acc]));
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<TCOLS>(tmem_base);
    }
}

struct WgradPlan {
    int ncol, bn, splits, kb_per_split;
    bool fast = false, swap = false, halo = false;
    int spg = 0;           // reduction: partials per group (0: one group of all splits)
    WhPlan hp{};           // halo wgrad grouping (hp.pairs = 1: a single group)
    int m_tiles = 1, n_tiles = 1;
};

WgradPlan plan_wgrad(const WgradArgs& a) {
    WgradPlan p;
    p.ncol = a.kh * a.kw * a.SC;
    const int total_kb = static_cast<int>(ceil_div(static_cast<int64_t>(a.N) * a.OH * a.OW, 64));
    if (wgrad_halo_supported(a)) {  // one partial per CTA (wgrad_halo.cu)
        p.halo = true;
        p.bn = 64;
        p.splits = wgrad_halo_splits(a, &p.spg);
        p.hp = wgrad_halo_plan(a);
        p.kb_per_split = 0;
        return p;
    }
    if (a.dtype == DT_BF16 && a.SC % 64 == 0 && (a.ld_dy * 2) % 16 == 0) {
        p.fast = true;
        p.swap = a.Cout < 128 && p.ncol > a.Cout;
        const int Mt = p.swap ? p.ncol : a.Cout, Nt = p.swap ? a.Cout : p.ncol;
        p.bn = Nt <= 64 ? 64 : (Nt <= 128 ? 128 : 256);
        p.m_tiles = static_cast<int>(ceil_div(Mt, 128));
        p.n_tiles = static_cast<int>(ceil_div(Nt, p.bn));
        const int tiles = p.m_tiles * p.n_tiles;
        // work items per SM, each at least 4 k-blocks deep: one for the few-tile (<= 4) layers with
        // long pixel reductions (ResNet-50 layers 1-2 1x1: half the split-K partial traffic, 6-16 us
        // faster each), two otherwise (the epilogue of one item overlaps the next item's mainloop);
        // SOL_WG_ITEMS_PER_SM forces a count
        static const int ips_env = std::getenv("SOL_WG_ITEMS_PER_SM") ? std::atoi(std::getenv("SOL_WG_ITEMS_PER_SM")) : 0;
        const int ips = ips_env > 0 ? ips_env : (tiles <= 4 ? 1 : 2);
        int splits = std::max(1, std::min(std::max(1, total_kb / 4), (ips * num_sms() + tiles - 1) / tiles));
        p.kb_per_split = static_cast<int>(ceil_div(total_kb, splits));
        p.splits = static_cast<int>(ceil_div(total_kb, p.kb_per_split));
        return p;
    }
    const int epb = a.dtype == DT_BF16 ? 64 : 32;
    p.bn = p.ncol <= epb ? epb : (p.ncol <= 2 * epb ? 2 * epb : 256);
    if (a.dtype == DT_F32 && p.bn > 128) p.bn = 128;
    const int tiles = static_cast<int>(ceil_div(a.Cout, BM) * ceil_div(p.ncol, p.bn));
    int splits = std::max(1, std::min(total_kb, (2 * num_sms() + tiles - 1) / tiles));
    p.kb_per_split = static_cast<int>(ceil_div(total_kb, splits));
    p.splits = static_cast<int>(ceil_div(total_kb, p.kb_per_split));
    return p;
}

template <int BN, bool SWAP>
void launch_wgrad_ws(const WgradArgs& a, const WgradPlan& p, cudaStream_t s) {
    constexpr int STAGE_BYTES = 128 * WG_BK * 2 + BN * WG_BK * 2;
    constexpr int SMEM = wg_stages<BN>() * STAGE_BYTES + 2048;
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(wgrad_ws_kernel<BN, SWAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    });
    const int P = a.N * a.OH * a.OW;
    const CUtensorMap tdy = make_tmap_2d(a.dy, DT_BF16, a.Cout, static_cast<uint64_t>(P), a.ld_dy, WG_BK);
    IgemmArgs g;
    g.src = a.x;
    g.N = a.N; g.SH = a.SH; g.SW = a.SW; g.SC = a.SC;
    g.OH = a.OH; g.OW = a.OW;
    g.kh = a.kh; g.kw = a.kw; g.sh = a.sh; g.sw = a.sw; g.ph = a.ph; g.pw = a.pw;
    const CUtensorMap tx = make_tmap_im2col(g, DT_BF16, WG_BK);
    const int items = p.m_tiles * p.n_tiles * p.splits;
    const int grid = std::min(items, num_sms());
    wgrad_ws_kernel<BN, SWAP><<<grid, WG_THREADS, SMEM, s>>>(a, tdy, tx, p.ncol, p.m_tiles, p.n_tiles, p.splits,
                                                            p.kb_per_split);
    SOL_CUDA(cudaGetLastError());
}

}  // namespace

int igemm_block_n(int nout) {
    if (nout <= 16) return 16;
    if (nout <= 32) return 32;
    if (nout <= 64) return 64;
    if (nout <= 128) return 128;
    return 256;
}

bool igemm_stats_supported(const IgemmArgs& a) {
    if (a.dtype != DT_BF16 || a.out_dtype != DT_BF16 || a.mode != IG_FPROP || a.src2) return false;
    if (a.residual || a.mask || a.res_mode || a.ep_scale || a.act || a.relu) return false;
    const bool plain = a.kh == 1 && a.kw == 1 && a.sh == 1 && a.sw == 1 && a.ph == 0 && a.pw == 0 && a.K_pad == a.SC;
    const bool im2col = !plain && a.SC % 64 == 0 && a.K_pad == a.kh * a.kw * a.SC && a.kh <= 8 && a.kw <= 8;
    // the halo path (stride-1 3x3 on 64/128 channels) stores from registers: keep it, unfused
    return (plain || im2col) && !halo_supported(a) && a.ldo % 8 == 0 && (a.Nout + 63) / 64 <= num_sms();
}

int igemm_stat_blocks(const IgemmArgs&) { return 4 * num_sms(); }

bool igemm_sub_supported(const IgemmArgs& a) {
    static const bool off = std::getenv("SOL_NO_SUBPIXEL_INPLACE") != nullptr;
    if (off || a.dtype != DT_BF16 || a.out_dtype != DT_BF16 || a.mode != IG_FPROP || a.src2) return false;
    if (a.residual || a.mask || a.res_mode || a.ep_scale || a.bias || a.act || a.relu || a.stat_partial) return false;
    const bool plain = a.kh == 1 && a.kw == 1 && a.sh == 1 && a.sw == 1 && a.ph == 0 && a.pw == 0 && a.K_pad == a.SC;
    const bool im2col = !plain && a.SC % 64 == 0 && a.K_pad == a.kh * a.kw * a.SC && a.kh <= 8 && a.kw <= 8;
    return (plain || im2col) && a.ldo % 8 == 0;
}

void igemm_launch(const IgemmArgs& a_in, cudaStream_t s) {
    // profiling only: SOL_CONV_DBG ORs debug flags into every plan conv (1 = skip stores, 2 = skip MMA)
    static const int env_dbg = std::getenv("SOL_CONV_DBG") ? std::atoi(std::getenv("SOL_CONV_DBG")) : 0;
    IgemmArgs a = a_in;
    a.dbg |= env_dbg;
    const int vec = a.dtype == DT_BF16 ? 8 : 4;
    const int bk = a.dtype == DT_BF16 ? 64 : 32;
    if (a.SC % vec != 0) throw std::invalid_argument("igemm: channel count must be a multiple of 16 bytes");
    if (a.K_pad % bk != 0) throw std::invalid_argument("igemm: K_pad must be a multiple of the k-block");
    const int out_es = a.out_dtype == DT_BF16 ? 2 : 4;
    if ((a.ldo * out_es) % 16 != 0) throw std::invalid_argument("igemm: output row stride must be a multiple of 16 bytes");
    if (a.residual && ((a.ld_res * out_es) % 16 != 0 || (reinterpret_cast<uintptr_t>(a.residual) & 15) != 0))
        throw std::invalid_argument("igemm: residual must be 16-byte aligned with a 16-byte multiple row stride");
    if (a.N * a.OH * a.OW <= 0 || a.Nout <= 0) return;
    if (a.src2 && (a.SC % 64 || a.SC2 % 64 || a.K1 != a.SC || a.K_pad != a.SC + a.SC2 || a.mode != IG_FPROP))
        throw std::invalid_argument("igemm: dual GEMM needs two 1x1 convs over 128-byte channel blocks");
    if (!a.src2 && !a.mask && !a.stat_partial && !a.sub_sh && a.tile_n == 0 && halo_supported(a)) return halo_launch(a, s);  // a forced tile: im2col path
    if (a.dtype == DT_BF16) {
        if (a.out_dtype == DT_BF16) dispatch_mode<__nv_bfloat16, __nv_bfloat16>(a, s);
        else dispatch_mode<__nv_bfloat16, float>(a, s);
    } else {
        if (a.out_dtype != DT_F32) throw std::invalid_argument("igemm: tf32 path writes f32");
        dispatch_mode<float, float>(a, s);
    }
}

size_t wgrad_workspace_floats(const WgradArgs& a) {
    WgradPlan p = plan_wgrad(a);
    if (p.halo) return static_cast<size_t>(p.splits) * wh_partial_floats(p.hp);
    return p.splits > 1 ? static_cast<size_t>(p.splits) * a.Cout * p.ncol : 0;
}

void wgrad_launch(const WgradArgs& a_in, cudaStream_t s) {
    WgradArgs a = a_in;
    const int vec = a.dtype == DT_BF16 ? 8 : 4;
    if (a.SC % vec != 0 || a.ld_dy % vec != 0)
        throw std::invalid_argument("wgrad: channel counts must be multiples of 16 bytes");
    WgradPlan p = plan_wgrad(a);
    if (p.splits <= 1 && !p.halo) a.workspace = nullptr;  // the halo path always reduces its partials
    else if (a.workspace == nullptr) throw std::invalid_argument("wgrad: workspace required");
    if (p.halo) {
        wgrad_halo_launch(a, s);
    } else if (p.fast) {
        if (p.swap) {
            switch (p.bn) {
                case 64: launch_wgrad_ws<64, true>(a, p, s); break;
                case 128: launch_wgrad_ws<128, true>(a, p, s); break;
                default: launch_wgrad_ws<256, true>(a, p, s); break;
            }
        } else {
            switch (p.bn) {
                case 64: launch_wgrad_ws<64, false>(a, p, s); break;
                case 128: launch_wgrad_ws<128, false>(a, p, s); break;
                default: launch_wgrad_ws<256, false>(a, p, s); break;
            }
        }
    } else if (a.dtype == DT_BF16) {
        switch (p.bn) {
            case 64: launch_wgrad_t<__nv_bfloat16, 64>(a, p.ncol, p.splits, p.kb_per_split, s); break;
            case 128: launch_wgrad_t<__nv_bfloat16, 128>(a, p.ncol, p.splits, p.kb_per_split, s); break;
            default: launch_wgrad_t<__nv_bfloat16, 256>(a, p.ncol, p.splits, p.kb_per_split, s); break;
        }
    } else {
        switch (p.bn) {
            case 32: launch_wgrad_t<float, 32>(a, p.ncol, p.splits, p.kb_per_split, s); break;
            case 64: launch_wgrad_t<float, 64>(a, p.ncol, p.splits, p.kb_per_split, s); break;
            default: launch_wgrad_t<float, 128>(a, p.ncol, p.splits, p.kb_per_split, s); break;
        }
    }
    if (p.halo) {
        const int64_t total = static_cast<int64_t>(p.hp.groups) * wh_partial_floats(p.hp);
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 8L * num_sms())));
        wgrad_reduce_halo_kernel<<<grid, 256, 0, s>>>(a.workspace, a.dw, a.dw_canon, a.canon_cin, p.spg, a.SC, p.hp);
        SOL_CUDA(cudaGetLastError());
    } else if (p.splits > 1 && a.dw_canon) {
        const int64_t n = static_cast<int64_t>(a.Cout) * p.ncol;
        const int64_t total = static_cast<int64_t>(a.Cout) * a.kh * a.kw * a.SC;  // packed walk
        const unsigned grid = static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 8L * num_sms())));
        wgrad_reduce_canon_kernel<<<grid, 256, 0, s>>>(a.workspace, a.dw_canon, n, p.splits, a.Cout, a.canon_cin,
                                                       a.kh, a.kw, a.SC);
        SOL_CUDA(cudaGetLastError());
    } else if (p.splits > 1) {
        const int64_t n = static_cast<int64_t>(a.Cout) * p.ncol;
        const int threads = 256;
        wgrad_reduce_kernel<<<static_cast<unsigned>(ceil_div(ceil_div(n, 4), threads)), threads, 0, s>>>(
            a.workspace, a.dw, n, p.splits);
        SOL_CUDA(cudaGetLastError());
    } else if (a.dw_canon) {
        unpack_conv_grad(a.dw, a.dw_canon, a.Cout, a.canon_cin, a.kh, a.kw, a.SC, s);
    }
}

}  // namespace solb200
