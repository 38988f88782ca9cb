// Halo weight gradient for stride-1 "same" 3x3 convolutions (ResNet-50 layers 1-4). The TMA-im2col
// wgrad re-fetches every x pixel row from L2 once per filter tap pair and every dy row once per
// tap-pair tile (24 KB per 4 N=64 MMAs at layer 1: ~3x the L2 bandwidth at the MMA rate). Here one
// work unit is R whole output rows of one image in the row-padded pixel order of the forward halo
// kernel (halo.cu: Wp = W + 2 columns, the last two junk), K = 64 or 128 pixel rows:
//   dy  [K pixel rows][co slice]   one 4-D TMA box per 64 channels (junk columns are out of bounds
//                                  = 0; rows past R * Wp stay zero in shared memory)
//   x   [HX rows * Wp][ci slice]   one 4-D TMA box per 64 channels from (row - 1, col - 1)
//                                  (the padding = OOB zeros)
// and tap t = (dkh, dkw) pairs dy pixel p with x halo row p + dkh * Wp + dkw. dW's columns
// (tap, ci) are M = 128 tiles whose two MN-major 64-channel halves are either
//   * one halo at two tap shifts (64 input channels: five tiles of two taps), or
//   * two 64-channel halo blocks at one tap shift (>= 128 input channels: one tap per tile),
// so a tile is ONE descriptor whose leading-byte offset is the shift difference / the block stride
// (the 128B swizzle is a function of the absolute shared-memory address, as the forward halo kernel
// relies on). B = dy (N = the co slice, <= 256).
// Work = (tap group, ci slice, co slice) x units: each CTA accumulates its group's tiles in TMEM
// (<= 512 columns) over a contiguous unit range and writes one f32 partial of its group's dW
// entries; the ordered split-K reduction sums each entry over its group's CTAs (deterministic).
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

__host__ __device__ inline int wh_shift(int t, int Wp) { return (t / 3) * Wp + t % 3; }

WhPlan wh_plan_make(const WgradArgs& a) {
    WhPlan g{};
    g.Wp = a.OW + 2;
    // K = 128 pixel rows per unit, or 64 when a whole (small) image fits in 64
    g.K = a.OH * g.Wp <= 64 ? 64 : 128;
    g.R = std::min(g.K / g.Wp, a.OH);
    // x rows read: pixel rows up to K - 1 shifted by up to 2 * Wp + 2
    g.HX = (g.K - 1 + 2 * g.Wp + 2) / g.Wp + 1;
    g.pairs = a.SC == 64 ? 1 : 0;
    g.ncx = g.pairs ? 1 : 2;                       // x channel blocks per unit (the ci slice)
    g.N = std::min(a.Cout, 256);                   // co slice
    g.ncd = g.N / 64;
    g.n_ci = g.pairs ? 1 : a.SC / 128;
    g.n_co = a.Cout / g.N;
    g.TT = g.pairs ? 9 : std::min(3, 512 / g.N);   // taps per CTA: tiles x N <= 512 TMEM columns
    g.tap_groups = g.pairs ? 1 : (9 + g.TT - 1) / g.TT;
    g.groups = g.tap_groups * g.n_ci * g.n_co;
    g.cb_bytes = (g.HX * g.Wp * 128 + 1023) / 1024 * 1024;
    g.dy_blk = g.K * 128;
    g.stage_bytes = g.ncd * g.dy_blk + g.ncx * g.cb_bytes;
    g.row_blocks = g.R > 0 ? (a.OH + g.R - 1) / g.R : 0;
    g.units = a.N * g.row_blocks;
    return g;
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                            uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(mbar)
        : "memory");
}

// One K = 16 step of CNT tiles (accumulators d + j * ds) from ONE asm statement, issued by one
// elected lane of the converged warp (uniform operands: back-to-back UTCHMMAs; a per-MMA
// single-lane issue loop ran at ~110 instead of 48 cycles per N=64 MMA)
#define WH_MMA(D, A) "@p tcgen05.mma.cta_group::1.kind::f16 [" D "], " A ", %7, %8, pa;\n"
template <int CNT>
__device__ __forceinline__ void wh_mma(uint32_t d, uint32_t ds, const uint64_t* ad, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
    if constexpr (CNT == 1) {
        asm volatile("{\n.reg .pred p, pa;\nelect.sync _|p, 0xffffffff;\nsetp.ne.b32 pa, %9, 0;\n" WH_MMA("%0", "%2") "}\n"
                     ::"r"(d), "r"(ds), "l"(ad[0]), "l"(0ull), "l"(0ull), "l"(0ull), "l"(0ull), "l"(b), "r"(idesc), "r"(acc));
    } else if constexpr (CNT == 2) {
        asm volatile("{\n.reg .pred p, pa;\n.reg .b32 d1;\nelect.sync _|p, 0xffffffff;\nsetp.ne.b32 pa, %9, 0;\n"
                     "add.u32 d1, %0, %1;\n" WH_MMA("%0", "%2") WH_MMA("d1", "%3") "}\n"
                     ::"r"(d), "r"(ds), "l"(ad[0]), "l"(ad[1]), "l"(0ull), "l"(0ull), "l"(0ull), "l"(b), "r"(idesc), "r"(acc));
    } else if constexpr (CNT == 3) {
        asm volatile("{\n.reg .pred p, pa;\n.reg .b32 d1, d2;\nelect.sync _|p, 0xffffffff;\nsetp.ne.b32 pa, %9, 0;\n"
                     "add.u32 d1, %0, %1;\nadd.u32 d2, d1, %1;\n" WH_MMA("%0", "%2") WH_MMA("d1", "%3") WH_MMA("d2", "%4") "}\n"
                     ::"r"(d), "r"(ds), "l"(ad[0]), "l"(ad[1]), "l"(ad[2]), "l"(0ull), "l"(0ull), "l"(b), "r"(idesc), "r"(acc));
    } else {
        static_assert(CNT == 5, "tiles");
        asm volatile("{\n.reg .pred p, pa;\n.reg .b32 d1, d2, d3, d4;\nelect.sync _|p, 0xffffffff;\nsetp.ne.b32 pa, %9, 0;\n"
                     "add.u32 d1, %0, %1;\nadd.u32 d2, d1, %1;\nadd.u32 d3, d2, %1;\nadd.u32 d4, d3, %1;\n"
                     WH_MMA("%0", "%2") WH_MMA("d1", "%3") WH_MMA("d2", "%4") WH_MMA("d3", "%5") WH_MMA("d4", "%6") "}\n"
                     ::"r"(d), "r"(ds), "l"(ad[0]), "l"(ad[1]), "l"(ad[2]), "l"(ad[3]), "l"(ad[4]), "l"(b), "r"(idesc), "r"(acc));
    }
}
#undef WH_MMA

__global__ void __launch_bounds__(WH_THREADS, 1)
    wgrad_halo_kernel(const WgradArgs a, const WhPlan G, const __grid_constant__ CUtensorMap tm_dy,
                      const __grid_constant__ CUtensorMap tm_x, int stages, int per_cta, int spg) {
    const int ncol = 9 * a.SC;
    const uint32_t idesc = make_idesc(1, G.N, 128, 1, 1);

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + stages * G.stage_bytes);
    uint64_t* empty = full + 8;
    uint64_t* tfull = empty + 8;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tfull + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // group = (tap group, ci slice, co slice), co slice fastest
    const int grp = static_cast<int>(blockIdx.x) / spg;
    const int co_s = grp % G.n_co, ci_s = (grp / G.n_co) % G.n_ci, tg = grp / (G.n_co * G.n_ci);
    const int tap0 = tg * G.TT;
    const int ntiles = G.pairs ? 5 : min(G.TT, 9 - tap0);
    const int u_begin = min(G.units, (static_cast<int>(blockIdx.x) - grp * spg) * per_cta);
    const int u_end = min(G.units, u_begin + per_cta);
    const int dy_bytes = G.ncd * G.dy_blk;

    // dy rows past R * Wp are never written by the TMA boxes: zero them once per stage and block
    for (int s = 0; s < stages; ++s)
        for (int cb = 0; cb < G.ncd; ++cb) {
            uint4* z = reinterpret_cast<uint4*>(smem + s * G.stage_bytes + cb * G.dy_blk + G.R * G.Wp * 128);
            for (int i = tid; i < (G.K - G.R * G.Wp) * 8; i += WH_THREADS) z[i] = make_uint4(0, 0, 0, 0);
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
                    tma_load_4d(smem_u32(sd + cb * G.dy_blk), &tm_dy, co_s * G.N + cb * 64, 0, rb * G.R, img, fb);
                for (int cb = 0; cb < G.ncx; ++cb)
                    tma_load_4d(smem_u32(sd + dy_bytes + cb * G.cb_bytes), &tm_x, ci_s * 128 + cb * 64, -1,
                                rb * G.R - 1, img, fb);
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
            const uint32_t x_addr = dy_addr + dy_bytes;
            const uint64_t bd = sw128_desc(dy_addr, G.dy_blk, 1024);  // N atoms: the 64-channel dy blocks
#pragma unroll
            for (int j = 0; j < 5; ++j) {
                if (G.pairs) {
                    const int s0 = wh_shift(2 * j, G.Wp);
                    const int s1 = 2 * j + 1 < 9 ? wh_shift(2 * j + 1, G.Wp) : s0 + 1;
                    ad[j] = sw128_desc(x_addr + s0 * 128, (s1 - s0) * 128, 1024);
                } else {  // tap tap0 + j: both channel blocks of the slice at the same shift
                    const int t = min(tap0 + j, 8);
                    ad[j] = sw128_desc(x_addr + wh_shift(t, G.Wp) * 128, G.cb_bytes, 1024);
                }
            }
            for (int k = 0; k < G.K / 16; ++k) {
                const uint64_t o = static_cast<uint64_t>(k * 128);
                uint64_t ak[5];
#pragma unroll
                for (int j = 0; j < 5; ++j) ak[j] = ad[j] + o;
                switch (ntiles) {
                    case 1: wh_mma<1>(tmem_base, G.N, ak, bd + o, idesc, acc); break;
                    case 2: wh_mma<2>(tmem_base, G.N, ak, bd + o, idesc, acc); break;
                    case 3: wh_mma<3>(tmem_base, G.N, ak, bd + o, idesc, acc); break;
                    default: wh_mma<5>(tmem_base, G.N, ak, bd + o, idesc, acc); break;
                }
                acc = 1;
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
        // TMEM lane = dW column (tap, ci) of tile j, accumulator columns = the co slice; a CTA
        // writes only its group's entries of its partial
        const int q = warp & 3;
        const int cols = wh_cols(G);
        float* dst = a.workspace + static_cast<int64_t>(blockIdx.x) * wh_partial_floats(G);
        mbar_wait(smem_u32(tfull), 0);
        tc_fence_after();
        const int row = q * 32 + lane;
#pragma unroll 1
        for (int j = 0; j < ntiles; ++j) {
            const int col = j * 128 + row;  // partial column; dW column (tap0 + j or pair j, ci_s)
            const bool live = G.pairs ? col < ncol : true;
#pragma unroll 1
            for (int c0 = 0; c0 < G.N; c0 += 32) {
                uint32_t v[32];
                tmem_ld32_nowait(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(j * G.N + c0), v);
                tmem_wait_ld();
                if (live) {
                    float* o = dst + static_cast<int64_t>(c0) * cols + col;
#pragma unroll
                    for (int i = 0; i < 32; ++i) o[static_cast<int64_t>(i) * cols] = __uint_as_float(v[i]);
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

int wh_stages(const WhPlan& G) { return std::min(8, (227 * 1024 - 2048) / G.stage_bytes); }

// CTAs per group: contiguous ranges of per_cta units, none empty
int wh_splits_per_group(const WhPlan& G, int* per_cta_out) {
    const int grid = std::max(1, std::min(G.units, num_sms() / G.groups));
    const int per_cta = (G.units + grid - 1) / grid;
    if (per_cta_out) *per_cta_out = per_cta;
    return (G.units + per_cta - 1) / per_cta;
}

}  // namespace

WhPlan wgrad_halo_plan(const WgradArgs& a) { return wh_plan_make(a); }

bool wgrad_halo_supported(const WgradArgs& a) {
    static const bool off = std::getenv("SOL_NO_WGRAD_HALO") != nullptr;
    static const bool no_wide = std::getenv("SOL_NO_WGRAD_HALO_WIDE") != nullptr;
    if (off || a.dtype != DT_BF16 || a.ld_dy % 8 != 0) return false;
    if (a.kh != 3 || a.kw != 3 || a.sh != 1 || a.sw != 1 || a.ph != 1 || a.pw != 1) return false;
    if (a.OH != a.SH || a.OW != a.SW) return false;
    const bool c64 = a.SC == 64 && a.Cout == 64;
    const bool c128 = a.SC == 128 && a.Cout == 128;
    const bool wide = !no_wide && a.SC >= 256 && a.SC % 128 == 0 && a.Cout % 256 == 0;
    if (!c64 && !c128 && !wide) return false;
    const WhPlan G = wh_plan_make(a);
    return G.R >= 1 && G.Wp <= 256 && G.HX <= 256 && wh_stages(G) >= 2 && G.groups <= num_sms();
}

// partials (= CTAs): splits_per_group per group; a group's CTAs write only the group's entries
int wgrad_halo_splits(const WgradArgs& a, int* splits_per_group) {
    const WhPlan G = wh_plan_make(a);
    const int spg = wh_splits_per_group(G, nullptr);
    if (splits_per_group) *splits_per_group = spg;
    return spg * G.groups;
}

void wgrad_halo_launch(const WgradArgs& a, cudaStream_t s) {
    const WhPlan G = wh_plan_make(a);
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
    wgrad_halo_kernel<<<spg * G.groups, WH_THREADS, smem, s>>>(a, G, tdy, tx, stages, per_cta, spg);
    SOL_CUDA(cudaGetLastError());
}

}  // namespace solb200
