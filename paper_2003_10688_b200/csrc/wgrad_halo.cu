// Halo weight gradient for stride-1 "same" 3x3 convolutions on 64 input and 64 output channels
// (ResNet-50 layer 1). The TMA-im2col wgrad re-fetches every x pixel row from L2 once per filter
// tap pair and every dy row once per tap-pair tile (24 KB per 4 MMAs: ~3x the L2 bandwidth at the
// MMA rate). Here one work unit is R whole output rows of one image in the row-padded pixel order
// of the forward halo kernel (halo.cu: Wp = W + 2 columns, the last two junk):
//   dy  [K = 128 pixel rows][64 co]  one 4-D TMA box (junk columns are out of bounds = 0; rows past
//                                    R * Wp stay zero in shared memory)
//   x   [HX rows * Wp][64 ci]        one 4-D TMA box from (row - 1, col - 1) (padding = OOB zeros)
// and tap t = (dkh, dkw) pairs dy pixel p with x halo row p + dkh * Wp + dkw. The 576 columns
// (tap, ci) of dW are five M = 128 tiles of two taps each: both 64-channel halves of a tile's A
// operand are the same halo buffer at two shifts, so a tile is ONE MN-major descriptor whose
// leading-byte offset is the shift difference (the 128B swizzle is a function of the absolute
// shared-memory address, as the forward halo kernel relies on). B = dy (N = 64).
// Every CTA accumulates all five tiles (320 TMEM columns) over a contiguous range of units and
// writes one f32 partial [Cout][576] to the split-K workspace; the existing ordered reduction
// (wgrad_reduce_canon) sums the partials: deterministic, like every other wgrad path.
//   warp 0 TMA producer, warp 1 MMA issuer, warps 2-5 epilogue (once, at the end)
// Semantics: reference.cpp Conv2dBackW (igemm.cuh WgradArgs).
#include "igemm.cuh"
#include "tc.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace solb200 {
namespace {

using namespace tc;

constexpr int WH_THREADS = 192;
constexpr int WH_K = 128;  // pixel rows per unit (MMA K), row-padded
constexpr int WH_BLK = WH_K * 128;  // one 64-channel block of the dy buffer: [128 px][64 ch] bf16

// Two shapes (ResNet-50 layers 1 and 2):
//   64 -> 64:   five M tiles of two taps each (A halves = one halo at two shifts), N = 64,
//               5 x 64 TMEM columns, one tap group
//   128 -> 128: one tap per M tile (A halves = the two 64-channel halo blocks), N = 128; the nine
//               taps need 1152 TMEM columns, so each CTA takes one filter row (3 taps, 384
//               columns) and the work is (filter row, unit range)
struct WhGeo {
    int Wp, R, HX, ncx, ncd, cb_bytes, x_bytes, dy_bytes, stage_bytes, row_blocks, units;
    int tiles, groups;  // M tiles per CTA, tap groups
};

__host__ __device__ inline WhGeo wh_geo(const WgradArgs& a) {
    WhGeo g;
    g.Wp = a.OW + 2;
    g.R = WH_K / g.Wp;
    // x rows read: pixel rows up to K - 1 shifted by up to 2 * Wp + 2
    g.HX = (WH_K - 1 + 2 * g.Wp + 2) / g.Wp + 1;
    g.ncx = a.SC / 64;
    g.ncd = a.Cout / 64;
    g.cb_bytes = (g.HX * g.Wp * 128 + 1023) / 1024 * 1024;
    g.x_bytes = g.ncx * g.cb_bytes;
    g.dy_bytes = g.ncd * WH_BLK;
    g.stage_bytes = g.dy_bytes + g.x_bytes;
    g.row_blocks = g.R > 0 ? (a.OH + g.R - 1) / g.R : 0;
    g.units = a.N * g.row_blocks;
    g.tiles = g.ncx == 1 ? 5 : 3;
    g.groups = g.ncx == 1 ? 1 : 3;
    return g;
}

__host__ __device__ inline int wh_shift(int t, int Wp) { return (t / 3) * Wp + t % 3; }

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                            uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(mbar)
        : "memory");
}

// One K = 16 step of all five tap-pair tiles (accumulators at d + 64 * mt) from ONE asm
// statement, issued by one elected lane of the converged warp (uniform operands: back-to-back
// UTCHMMAs; a per-MMA single-lane issue loop ran at ~110 instead of 48 cycles per N=64 MMA)
__device__ __forceinline__ void wh_mma5(uint32_t d, uint64_t a0, uint64_t a1, uint64_t a2, uint64_t a3, uint64_t a4,
                                        uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p, pa;\n.reg .b32 d1, d2, d3, d4;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "setp.ne.b32 pa, %8, 0;\n"
        "add.u32 d1, %0, 64;\nadd.u32 d2, %0, 128;\nadd.u32 d3, %0, 192;\nadd.u32 d4, %0, 256;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %6, %7, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [d1], %2, %6, %7, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [d2], %3, %6, %7, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [d3], %4, %6, %7, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [d4], %5, %6, %7, pa;\n"
        "}\n" ::"r"(d), "l"(a0), "l"(a1), "l"(a2), "l"(a3), "l"(a4), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void wh_mma3(uint32_t d, uint64_t a0, uint64_t a1, uint64_t a2, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p, pa;\n.reg .b32 d1, d2;\n"
        "elect.sync _|p, 0xffffffff;\n"
        "setp.ne.b32 pa, %6, 0;\n"
        "add.u32 d1, %0, 128;\nadd.u32 d2, %0, 256;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %4, %5, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [d1], %2, %4, %5, pa;\n"
        "@p tcgen05.mma.cta_group::1.kind::f16 [d2], %3, %4, %5, pa;\n"
        "}\n" ::"r"(d), "l"(a0), "l"(a1), "l"(a2), "l"(b), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(WH_THREADS, 1)
    wgrad_halo_kernel(const WgradArgs a, const __grid_constant__ CUtensorMap tm_dy,
                      const __grid_constant__ CUtensorMap tm_x, int stages, int per_cta, int splits_per_group) {
    const WhGeo G = wh_geo(a);
    const int ncol = 9 * a.SC;
    const uint32_t idesc = make_idesc(1, a.Cout, 128, 1, 1);

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * G.stage_bytes);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int grp = static_cast<int>(blockIdx.x) / splits_per_group;  // filter row (128 channels) or 0
    const int u_begin = min(G.units, (static_cast<int>(blockIdx.x) - grp * splits_per_group) * per_cta);
    const int u_end = min(G.units, u_begin + per_cta);

    // dy rows past R * Wp are never written by the TMA boxes: zero them once per stage and block
    for (int s = 0; s < stages; ++s)
        for (int cb = 0; cb < G.ncd; ++cb) {
            uint4* z = reinterpret_cast<uint4*>(smem + s * G.stage_bytes + cb * WH_BLK + G.R * G.Wp * 128);
            for (int i = tid; i < (WH_K - G.R * G.Wp) * 8; i += WH_THREADS) z[i] = make_uint4(0, 0, 0, 0);
        }
    if (tid == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        mbar_init(smem_u32(tfull), 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        tma_prefetch(&tm_dy);
        tma_prefetch(&tm_x);
    }
    if (warp == 1) tmem_alloc<512>(smem_u32(tmem_slot));
    fence_proxy_async();  // the zeroed rows are read by the tensor core (async proxy)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int u = u_begin; u < u_end; ++u) {
                const int img = u / G.row_blocks, rb = u - img * G.row_blocks;
                mbar_wait(smem_u32(&empty[stage]), phase ^ 1);
                uint8_t* sd = smem + stage * G.stage_bytes;
                const uint32_t fb = smem_u32(&full[stage]);
                mbar_arrive_tx(fb, static_cast<uint32_t>((G.ncd * G.R + G.ncx * G.HX) * G.Wp * 128));
                for (int cb = 0; cb < G.ncd; ++cb)
                    tma_load_4d(smem_u32(sd + cb * WH_BLK), &tm_dy, cb * 64, 0, rb * G.R, img, fb);
                for (int cb = 0; cb < G.ncx; ++cb)
                    tma_load_4d(smem_u32(sd + G.dy_bytes + cb * G.cb_bytes), &tm_x, cb * 64, -1, rb * G.R - 1, img, fb);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        // ---------------------------------------------------------------- MMA issuer
        // the whole warp runs the loop; descriptors are warp-uniform and advance by 16 pixel rows
        // (2048 B = 128 units) per K step
        int stage = 0;
        uint32_t phase = 0;
        uint32_t acc = 0;
        uint64_t ad[5];
        for (int u = u_begin; u < u_end; ++u) {
            mbar_wait(smem_u32(&full[stage]), phase);
            tc_fence_after();
            const uint32_t dy_addr = smem_u32(smem + stage * G.stage_bytes);
            const uint32_t x_addr = dy_addr + G.dy_bytes;
            const uint64_t bd = sw128_desc(dy_addr, WH_BLK, 1024);  // N atoms: the 64-channel dy blocks
            if (G.ncx == 1) {
#pragma unroll
                for (int mt = 0; mt < 5; ++mt) {
                    const int s0 = wh_shift(2 * mt, G.Wp);
                    const int s1 = 2 * mt + 1 < 9 ? wh_shift(2 * mt + 1, G.Wp) : s0 + 1;
                    ad[mt] = sw128_desc(x_addr + s0 * 128, (s1 - s0) * 128, 1024);
                }
#pragma unroll
                for (int k = 0; k < WH_K / 16; ++k) {
                    const uint64_t o = static_cast<uint64_t>(k * 128);
                    wh_mma5(tmem_base, ad[0] + o, ad[1] + o, ad[2] + o, ad[3] + o, ad[4] + o, bd + o, idesc, acc);
                    acc = 1;
                }
            } else {
#pragma unroll
                for (int j = 0; j < 3; ++j)  // tap (grp, j): both channel blocks at the same shift
                    ad[j] = sw128_desc(x_addr + wh_shift(3 * grp + j, G.Wp) * 128, G.cb_bytes, 1024);
#pragma unroll
                for (int k = 0; k < WH_K / 16; ++k) {
                    const uint64_t o = static_cast<uint64_t>(k * 128);
                    wh_mma3(tmem_base, ad[0] + o, ad[1] + o, ad[2] + o, bd + o, idesc, acc);
                    acc = 1;
                }
            }
            mma_commit_elect(smem_u32(&empty[stage]));
            if (++stage == stages) {
                stage = 0;
                phase ^= 1;
            }
        }
        mma_commit_elect(smem_u32(tfull));
    } else {
        // ---------------------------------------------------------------- epilogue (once)
        // TMEM lane = dW column (tap, ci) of tile mt, the Cout accumulator columns = co; a CTA of
        // tap group grp writes only its group's columns of its partial
        const int q = warp & 3;
        float* dst = a.workspace + static_cast<int64_t>(blockIdx.x) * a.Cout * ncol;
        mbar_wait(smem_u32(tfull), 0);
        tc_fence_after();
#pragma unroll 1
        for (int mt = 0; mt < G.tiles; ++mt) {
            const int row = q * 32 + lane;
            const int col = G.ncx == 1 ? mt * 128 + row : (3 * grp + mt) * a.SC + row;
#pragma unroll 1
            for (int c0 = 0; c0 < a.Cout; c0 += 32) {
                uint32_t v[32];
                tmem_ld32_nowait(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(mt * a.Cout + c0), v);
                tmem_wait_ld();
                if (col < ncol) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) dst[static_cast<int64_t>(c0 + i) * ncol + col] = __uint_as_float(v[i]);
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem_base);
    }
}

CUtensorMap wh_tmap(const void* base, const WgradArgs& a, int C, int ld, int box_w, int box_h) {
    CUtensorMap m;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(C), static_cast<cuuint64_t>(a.OW), static_cast<cuuint64_t>(a.OH),
                          static_cast<cuuint64_t>(a.N)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(a.OW) * ld * 2,
                             static_cast<cuuint64_t>(a.OH) * a.OW * ld * 2};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_w), static_cast<cuuint32_t>(box_h), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("wgrad halo: cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

int wh_stages(const WhGeo& G) { return std::min(8, (227 * 1024 - 2048) / G.stage_bytes); }

// CTAs per tap group: contiguous ranges of per_cta units, none empty
int wh_splits_per_group(const WhGeo& G, int* per_cta_out) {
    const int grid = std::max(1, std::min(G.units, num_sms() / G.groups));
    const int per_cta = (G.units + grid - 1) / grid;
    if (per_cta_out) *per_cta_out = per_cta;
    return (G.units + per_cta - 1) / per_cta;
}

}  // namespace

bool wgrad_halo_supported(const WgradArgs& a) {
    static const bool off = std::getenv("SOL_NO_WGRAD_HALO") != nullptr;
    if (off || a.dtype != DT_BF16) return false;
    if (!((a.SC == 64 && a.Cout == 64) || (a.SC == 128 && a.Cout == 128)) || a.ld_dy % 8 != 0) return false;
    if (a.kh != 3 || a.kw != 3 || a.sh != 1 || a.sw != 1 || a.ph != 1 || a.pw != 1) return false;
    if (a.OH != a.SH || a.OW != a.SW) return false;
    const WhGeo G = wh_geo(a);
    return G.R >= 1 && G.Wp <= 256 && G.HX <= 256 && wh_stages(G) >= 2;
}

// partials (= CTAs): splits_per_group per tap group; group g writes only its columns
// [g * cols_per_group, (g + 1) * cols_per_group) of its partials
int wgrad_halo_splits(const WgradArgs& a, int* splits_per_group, int* cols_per_group) {
    const WhGeo G = wh_geo(a);
    const int spg = wh_splits_per_group(G, nullptr);
    if (splits_per_group) *splits_per_group = spg;
    if (cols_per_group) *cols_per_group = 9 * a.SC / G.groups;
    return spg * G.groups;
}

void wgrad_halo_launch(const WgradArgs& a, cudaStream_t s) {
    const WhGeo G = wh_geo(a);
    const int stages = wh_stages(G);
    const int smem = stages * G.stage_bytes + 1024 + 1024;
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(wgrad_halo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    });
    int per_cta = 0;
    const int spg = wh_splits_per_group(G, &per_cta);
    const CUtensorMap tdy = wh_tmap(a.dy, a, a.Cout, a.ld_dy, G.Wp, G.R);
    const CUtensorMap tx = wh_tmap(a.x, a, a.SC, a.SC, G.Wp, G.HX);
    wgrad_halo_kernel<<<spg * G.groups, WH_THREADS, smem, s>>>(a, tdy, tx, stages, per_cta, spg);
    SOL_CUDA(cudaGetLastError());
}

}  // namespace solb200
