// Stride-2 stem convolution straight from the canonical NCHW f32 graph input, without an im2col
// matrix (ResNet-50's 7x7/2 3->64 conv; the reference's conv semantics, reference.cpp:138-161).
//
// One tile = one output row (OW <= 124 pixels of the M = 128 MMA rows). For kernel row kh the
// im2col row of output pixel ox is 8 horizontally adjacent input pixels x 4 channels starting at
// input column 2*ox - pw: with the input row stored "compact" (4 bf16 channels = 8 bytes per pixel,
// pixel k = column + pw at byte 8k) that row is the 64 contiguous bytes at 16*ox. Consecutive A rows
// therefore overlap, 16 bytes apart, which is exactly the K-major SWIZZLE_NONE UMMA layout with
// core-matrix rows 16 B apart (LBO = 16 B to the next 8-element K chunk, SBO = 128 B to the next 8
// rows): the tensor core reads the compact halo directly, two K=16 MMAs per kernel row.
//
//   warp 0      TMA: weights once as [64 cout][16 B] K-chunk planes; per tile one f32 box
//               {nbw cols, kh rows, Cin planes} of the NCHW input (zero fill = padding), ring of NH
//   warps 1-8   converters: one box column each -> compact bf16 rows [kh][RS px][4 ch]
//   warp 9      MMA issuer (converged warp, elected lane): 2 * kh MMAs, M = 128, N = 64, K = 16
//   warps 10-13 epilogue: TMEM -> bias / folded BN / activation -> bf16 -> 128B-swizzled staging ->
//               TMA store of {64 ch, 32 px} boxes (pixels past OW are clipped by the TMA unit;
//               measured: direct per-lane 16-byte global stores were 35% slower)
// Shared-memory traffic per tile: the tensor core's operand reads (~84 KB) + the f32 box written and
// read once + ~15 KB of compact rows + the 16 KB output staging written and read once.
#include "igemm.cuh"
#include "tc.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace solb200 {
namespace {

using namespace tc;

constexpr int SR_THREADS = 448;
constexpr int SR_BN = 64;
constexpr int SR_KH_MAX = 8;
constexpr int SR_RS = 264;                                // compact row stride (pixels): 2*127 + 8 + pad
constexpr int SR_CMP_BYTES = SR_KH_MAX * SR_RS * 8;       // 16.5 KB
constexpr int SR_B_BYTES = SR_KH_MAX * 4 * SR_BN * 16;    // 32 K-chunk planes of [64][16 B]
constexpr int SR_HALO_MAX = 4 * SR_KH_MAX * 256 * 4;  // f32 box, <= 4 planes x kh rows x 256 cols
constexpr int SR_NCMP = 2, SR_NH_MAX = 8, SR_NACC = 4;
constexpr int OFF_B = 0;
constexpr int OFF_CMP = OFF_B + SR_B_BYTES;
constexpr int OFF_STG = OFF_CMP + SR_NCMP * SR_CMP_BYTES;  // epilogue staging, 4 warps x 4 KB
constexpr int SR_ROW_BYTES = 128 * 128;                    // one conv output row (<= 128 px x 64 ch bf16)
constexpr int OFF_RING = OFF_STG + 4 * 4096;               // pool mode: last 3 conv rows
constexpr int OFF_BAR = OFF_RING + 3 * SR_ROW_BYTES;
constexpr int OFF_HALO = OFF_BAR + 1024;  // ring of NH halo slots (runtime slot size) to the end
constexpr int SR_SMEM = 227 * 1024;

__device__ __forceinline__ void tma_load_4d_f(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                              uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(mbar)
        : "memory");
}

__device__ __forceinline__ uint64_t plain_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return sw128_desc(saddr, lbo, sbo, 0);  // layout type 0 = SWIZZLE_NONE (K-major core matrices)
}

// Work order. Plain: tile t = (image, conv row), strided over CTAs. Pool mode: CTAs take bands of
// BP pooled rows; a band computes conv rows 2*p0-1 .. 2*(p0+BP)-1 in order (one recomputed row).
struct RowTasks {
    int N, OH, pool, BP, nbands;
    __device__ RowTasks(const IgemmArgs& a, int bp) : N(a.N), OH(a.OH), pool(a.pool3s2), BP(bp) {
        nbands = pool ? (OH / 2 + BP - 1) / BP : 0;
    }
    // visits (n, oy, p0) for every conv row this CTA computes, in order
    template <typename F>
    __device__ void each(F&& f) const {
        if (!pool) {
            for (int t = blockIdx.x; t < N * OH; t += gridDim.x) f(t / OH, t % OH, 0);
            return;
        }
        for (int g = blockIdx.x; g < N * nbands; g += gridDim.x) {
            const int n = g / nbands, p0 = (g - n * nbands) * BP;
            const int r0 = max(0, 2 * p0 - 1), r1 = min(OH - 1, 2 * (p0 + BP) - 1);
            for (int oy = r0; oy <= r1; ++oy) f(n, oy, p0);
        }
    }
};

__global__ void __launch_bounds__(SR_THREADS, 1)
    stem_row_kernel(const IgemmArgs a, const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                    const __grid_constant__ CUtensorMap tm_o, int nbw, int delta, int slot_bytes, int NH, int BP) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* b_full = bar;
    uint64_t* halo_full = bar + 1;                  // [SR_NH_MAX]
    uint64_t* halo_empty = halo_full + SR_NH_MAX;   // [SR_NH_MAX]
    uint64_t* cmp_full = halo_empty + SR_NH_MAX;    // [SR_NCMP]
    uint64_t* cmp_empty = cmp_full + SR_NCMP;       // [SR_NCMP]
    uint64_t* tfull = cmp_empty + SR_NCMP;          // [SR_NACC]
    uint64_t* tempty = tfull + SR_NACC;             // [SR_NACC]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + SR_NACC);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const RowTasks tasks(a, BP);
    const int C = a.SC;
    const uint32_t halo_bytes = static_cast<uint32_t>(C * a.kh * nbw * 4);

    if (tid == 0) {
        mbar_init(smem_u32(b_full), 1);
        for (int s = 0; s < SR_NH_MAX; ++s) {
            mbar_init(smem_u32(&halo_full[s]), 1);
            mbar_init(smem_u32(&halo_empty[s]), 256);
        }
        for (int s = 0; s < SR_NCMP; ++s) {
            mbar_init(smem_u32(&cmp_full[s]), 256);
            mbar_init(smem_u32(&cmp_empty[s]), 1);
        }
        for (int s = 0; s < SR_NACC; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        tma_prefetch(&tm_x);
        tma_prefetch(&tm_w);
        tma_prefetch(&tm_o);
    }
    if (warp == 9) tmem_alloc<SR_NACC * SR_BN>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (lane == 0) {
            const int nchunks = a.kh * 4;
            mbar_arrive_tx(smem_u32(b_full), static_cast<uint32_t>(nchunks * SR_BN * 16));
            for (int j = 0; j < nchunks; ++j)
                tma_load_2d(smem_u32(smem + OFF_B + j * SR_BN * 16), &tm_w, j * 8, 0, smem_u32(b_full));
            int hb = 0;
            uint32_t hph = 0;
            tasks.each([&](int n, int oy, int) {
                mbar_wait(smem_u32(&halo_empty[hb]), hph ^ 1);
                mbar_arrive_tx(smem_u32(&halo_full[hb]), halo_bytes);
                tma_load_4d_f(smem_u32(smem + OFF_HALO + hb * slot_bytes), &tm_x, -a.pw - delta, oy * a.sh - a.ph, 0,
                              n, smem_u32(&halo_full[hb]));
                if (++hb == NH) {
                    hb = 0;
                    hph ^= 1;
                }
            });
        }
    } else if (warp <= 8) {
        // ---------------------------------------------------------------- converters (8 warps)
        // thread b converts box column e = b (compact pixel e - delta) of every kernel row
        const int e = tid - 32;
        const int k = e - delta;
        const bool active = e < nbw && k >= 0;
        const int pstride = a.kh * nbw;
        int hb = 0, cb = 0;
        uint32_t hph = 0, cph = 0;
        tasks.each([&](int, int, int) {
            mbar_wait(smem_u32(&halo_full[hb]), hph);
            const float* plane = reinterpret_cast<const float*>(smem + OFF_HALO + hb * slot_bytes);
            float f[SR_KH_MAX][4];
            if (active) {
#pragma unroll
                for (int r = 0; r < SR_KH_MAX; ++r) {
                    if (r < a.kh) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) f[r][c] = c < C ? plane[c * pstride + r * nbw + e] : 0.f;
                    }
                }
            }
            mbar_arrive(smem_u32(&halo_empty[hb]));
            if (++hb == NH) {
                hb = 0;
                hph ^= 1;
            }
            mbar_wait(smem_u32(&cmp_empty[cb]), cph ^ 1);
            uint2* cmp = reinterpret_cast<uint2*>(smem + OFF_CMP + cb * SR_CMP_BYTES);
            if (active) {
#pragma unroll
                for (int r = 0; r < SR_KH_MAX; ++r) {
                    if (r < a.kh) {
                        const __nv_bfloat162 lo = __floats2bfloat162_rn(f[r][0], f[r][1]);
                        const __nv_bfloat162 hi = __floats2bfloat162_rn(f[r][2], f[r][3]);
                        cmp[r * SR_RS + k] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo),
                                                        *reinterpret_cast<const uint32_t*>(&hi));
                    }
                }
            }
            fence_proxy_async();  // generic-proxy stores -> tcgen05 operand reads
            mbar_arrive(smem_u32(&cmp_full[cb]));
            if (++cb == SR_NCMP) {
                cb = 0;
                cph ^= 1;
            }
        });
    } else if (warp == 9) {
        // ---------------------------------------------------------------- MMA issuer
        constexpr uint32_t IDESC = make_idesc(1, SR_BN, 128, 0, 0);
        mbar_wait(smem_u32(b_full), 0);
        const uint64_t bdesc0 = plain_desc(smem_u32(smem + OFF_B), SR_BN * 16, 128);
        const uint64_t adesc0 = plain_desc(smem_u32(smem + OFF_CMP), 16, 128);
        int cb = 0, acc = 0;
        uint32_t cph = 0, aph = 0;
        tasks.each([&](int, int, int) {
            mbar_wait(smem_u32(&tempty[acc]), aph ^ 1);
            mbar_wait(smem_u32(&cmp_full[cb]), cph);
            tc_fence_after();
            const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * SR_BN);
            const uint64_t ad0 = adesc0 + static_cast<uint32_t>(cb * (SR_CMP_BYTES >> 4));
            for (int kh = 0; kh < a.kh; ++kh) {
                // A: compact row kh (+32 B for the second K16 step); B: K-chunk planes 4kh, 4kh+2
                const uint64_t ad = ad0 + static_cast<uint32_t>(kh * (SR_RS * 8 / 16));
                const uint64_t bd = bdesc0 + static_cast<uint32_t>(kh * 4 * (SR_BN * 16 / 16));
                mma2_elect<2, 2 * SR_BN>(dcol, ad, bd, IDESC, kh != 0);  // +32 B in A, +2 K-chunk planes in B
            }
            mma_commit_elect(smem_u32(&cmp_empty[cb]));
            mma_commit_elect(smem_u32(&tfull[acc]));
            if (++cb == SR_NCMP) {
                cb = 0;
                cph ^= 1;
            }
            if (++acc == SR_NACC) {
                acc = 0;
                aph ^= 1;
            }
        });
    } else {
        // ---------------------------------------------------------------- epilogue (warps 10-13)
        const int q = warp & 3;  // TMEM lane quarter = output pixels 32q .. 32q + 31
        uint8_t* stage = smem + OFF_STG + q * 4096;
        const bool has_bias = a.bias != nullptr, has_fold = a.ep_scale != nullptr;
        const int act = a.relu ? 1 : a.act;
        uint32_t aph = 0;
        int acc = 0;
        const int PH = a.OH / 2, PW = a.OW / 2;
        uint8_t* ring = smem + OFF_RING;
        tasks.each([&](int n, int oy, int p0) {
            mbar_wait(smem_u32(&tfull[acc]), aph);
            tc_fence_after();
            uint32_t v[SR_BN];
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * SR_BN);
            tmem_ld32_nowait(taddr, v);
            tmem_ld32_nowait(taddr + 32, v + 32);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty[acc]));
            if (++acc == SR_NACC) {
                acc = 0;
                aph ^= 1;
            }
            if (!a.pool3s2 && q * 32 >= a.OW) return;  // this quarter holds only junk rows
            float f[SR_BN];
#pragma unroll
            for (int i = 0; i < SR_BN; ++i) f[i] = __uint_as_float(v[i]);
            if (has_bias) {
#pragma unroll
                for (int i = 0; i < SR_BN; i += 4) {
                    const float4 bb = __ldg(reinterpret_cast<const float4*>(a.bias + i));
                    f[i] += bb.x; f[i + 1] += bb.y; f[i + 2] += bb.z; f[i + 3] += bb.w;
                }
            }
            if (has_fold) {
#pragma unroll
                for (int i = 0; i < SR_BN; i += 4) {
                    const float4 sc = __ldg(reinterpret_cast<const float4*>(a.ep_scale + i));
                    const float4 sh = __ldg(reinterpret_cast<const float4*>(a.ep_shift + i));
                    f[i] = fmaf(f[i], sc.x, sh.x);
                    f[i + 1] = fmaf(f[i + 1], sc.y, sh.y);
                    f[i + 2] = fmaf(f[i + 2], sc.z, sh.z);
                    f[i + 3] = fmaf(f[i + 3], sc.w, sh.w);
                }
            }
            if (act != 0) {
#pragma unroll
                for (int i = 0; i < SR_BN; ++i) {
                    f[i] = fmaxf(f[i], 0.f);
                    if (act == 2) f[i] = fminf(f[i], 6.f);
                }
            }
            if (a.pool3s2) {
                // conv row -> ring slot oy % 3 ([px][8 x 16-byte chunks], chunk j at j ^ (px & 7));
                // after an odd row 2py+1 the 128 epilogue threads max-pool rows 2py-1..2py+1
                const int ox = q * 32 + lane;
                uint8_t* slot = ring + (oy % 3) * SR_ROW_BYTES;
                if (ox < a.OW) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float* src = f + j * 8;
                        __nv_bfloat162 p0v = __floats2bfloat162_rn(src[0], src[1]);
                        __nv_bfloat162 p1v = __floats2bfloat162_rn(src[2], src[3]);
                        __nv_bfloat162 p2v = __floats2bfloat162_rn(src[4], src[5]);
                        __nv_bfloat162 p3v = __floats2bfloat162_rn(src[6], src[7]);
                        *reinterpret_cast<uint4*>(slot + ox * 128 + ((j ^ (ox & 7)) << 4)) =
                            make_uint4(*reinterpret_cast<uint32_t*>(&p0v), *reinterpret_cast<uint32_t*>(&p1v),
                                       *reinterpret_cast<uint32_t*>(&p2v), *reinterpret_cast<uint32_t*>(&p3v));
                    }
                }
                asm volatile("bar.sync 2, 128;\n" ::: "memory");
                const int py = (oy - 1) / 2;
                if ((oy & 1) && py >= p0) {
                    const int et = tid - 320;  // 0..127
                    __nv_bfloat16* orow = static_cast<__nv_bfloat16*>(a.out) + (static_cast<int64_t>(n) * PH + py) * PW * a.ldo;
                    for (int item = et; item < PW * 8; item += 128) {
                        const int px = item >> 3, j = item & 7;
                        // window taps clamped onto in-window ones (a duplicate never changes a max;
                        // OH, OW even: only the top / left edges clip), all nine loads in flight,
                        // packed bf16x2 max (NaN taps ignored, as fmaxf does), then min_init
                        const uint8_t* rs[3];
                        int cs[3];
#pragma unroll
                        for (int k = 0; k < 3; ++k) {
                            rs[k] = ring + (max(2 * py + k - 1, 0) % 3) * SR_ROW_BYTES;
                            cs[k] = max(2 * px + k - 1, 0);
                        }
                        uint4 tv[9];
#pragma unroll
                        for (int kr = 0; kr < 3; ++kr)
#pragma unroll
                            for (int kc = 0; kc < 3; ++kc)
                                tv[kr * 3 + kc] = *reinterpret_cast<const uint4*>(rs[kr] + cs[kc] * 128 + ((j ^ (cs[kc] & 7)) << 4));
                        __nv_bfloat162 mx[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i) mx[i] = reinterpret_cast<const __nv_bfloat162*>(&tv[0])[i];
#pragma unroll
                        for (int t = 1; t < 9; ++t)
#pragma unroll
                            for (int i = 0; i < 4; ++i) mx[i] = __hmax2(mx[i], reinterpret_cast<const __nv_bfloat162*>(&tv[t])[i]);
                        float m[8];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float2 t2 = __bfloat1622float2(mx[i]);
                            m[2 * i] = fmaxf(t2.x, a.pool_min_init);
                            m[2 * i + 1] = fmaxf(t2.y, a.pool_min_init);
                        }
                        store16(orow + px * a.ldo + j * 8, m);
                    }
                    asm volatile("bar.sync 2, 128;\n" ::: "memory");
                }
                return;
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float* src = f + j * 8;
                __nv_bfloat162 p0 = __floats2bfloat162_rn(src[0], src[1]);
                __nv_bfloat162 p1 = __floats2bfloat162_rn(src[2], src[3]);
                __nv_bfloat162 p2 = __floats2bfloat162_rn(src[4], src[5]);
                __nv_bfloat162 p3 = __floats2bfloat162_rn(src[6], src[7]);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                 smem_u32(stage + lane * 128 + ((j ^ (lane & 7)) << 4))),
                             "r"(*reinterpret_cast<uint32_t*>(&p0)), "r"(*reinterpret_cast<uint32_t*>(&p1)),
                             "r"(*reinterpret_cast<uint32_t*>(&p2)), "r"(*reinterpret_cast<uint32_t*>(&p3)));
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(
                        reinterpret_cast<uint64_t>(&tm_o)),
                    "r"(0), "r"(q * 32), "r"(oy), "r"(n), "r"(smem_u32(stage))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
        });
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc<SR_NACC * SR_BN>(tmem_base);
    }
}

// f32 NCHW input map: box {nbw cols, kh rows, C planes, 1 image}
CUtensorMap sr_tmap_x(const IgemmArgs& a, int nbw) {
    CUtensorMap m;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.SW), static_cast<cuuint64_t>(a.SH), static_cast<cuuint64_t>(a.SC),
                          static_cast<cuuint64_t>(a.N)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.SW) * 4, static_cast<cuuint64_t>(a.SH) * a.SW * 4,
                             static_cast<cuuint64_t>(a.SC) * a.SH * a.SW * 4};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(nbw), static_cast<cuuint32_t>(a.kh), static_cast<cuuint32_t>(a.SC), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(a.src), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("stem_row: input tensor map failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

// packed weights [64][K_pad] bf16 -> 16-byte K-chunk boxes {8 elements, 64 rows}, no swizzle
CUtensorMap sr_tmap_w(const IgemmArgs& a) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.K_pad), static_cast<cuuint64_t>(SR_BN)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.K_pad) * 2};
    cuuint32_t box[2] = {8, static_cast<cuuint32_t>(SR_BN)};
    cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.wt), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("stem_row: weight tensor map failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

// output [N][OH][OW][64] bf16, box {64 ch, 32 px, 1, 1}, 128B swizzle (matches the staging layout)
CUtensorMap sr_tmap_o(const IgemmArgs& a) {
    CUtensorMap m;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.ldo), static_cast<cuuint64_t>(a.OW), static_cast<cuuint64_t>(a.OH),
                          static_cast<cuuint64_t>(a.N)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.ldo) * 2, static_cast<cuuint64_t>(a.OW) * a.ldo * 2,
                             static_cast<cuuint64_t>(a.OH) * a.OW * a.ldo * 2};
    cuuint32_t box[4] = {64, 32, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, a.out, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("stem_row: output tensor map failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

void sr_geometry(const IgemmArgs& a, int& nbw, int& delta) {
    delta = (4 - a.pw % 4) % 4;  // box starts 16-byte aligned, `delta` columns before -pw
    nbw = (2 * (a.OW - 1) + 8 + delta + 3) / 4 * 4;  // all 8 kw slots of the last pixel
}

}  // namespace

bool stem_row_supported(const IgemmArgs& a) {
    static const bool disabled = std::getenv("SOL_STEM_LEGACY") != nullptr;
    if (disabled || !a.src_nchw_f32 || a.mode != IG_FPROP || a.dtype != DT_BF16 || a.out_dtype != DT_BF16) return false;
    if (a.SC < 1 || a.SC > 4 || a.Nout != SR_BN || a.ldo != SR_BN || a.residual != nullptr) return false;
    if (a.sw != 2 || a.kw > 8 || a.kh > SR_KH_MAX || a.K_pad != stem_kpad(a.kh) || a.OW > 124 || a.OW < 1) return false;
    if (a.pool3s2 && (a.OH % 2 || a.OW % 2 || a.OH < 2)) return false;
    int nbw, delta;
    sr_geometry(a, nbw, delta);
    return nbw <= 256 && a.SC * a.kh * nbw * 4 <= SR_HALO_MAX && a.N > 0 && a.OH > 0;  // one converter per column
}

void stem_row_launch(const IgemmArgs& a, cudaStream_t s) {
    int nbw, delta;
    sr_geometry(a, nbw, delta);
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(stem_row_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SR_SMEM));
    });
    const CUtensorMap tx = sr_tmap_x(a, nbw);
    const CUtensorMap tw = sr_tmap_w(a);
    IgemmArgs ao = a;  // pool mode stores pooled rows directly; the output map is a dummy
    if (a.pool3s2) ao.OH = ao.OW = 1;
    const CUtensorMap to = sr_tmap_o(ao);
    // pool mode: bands of BP pooled rows (~14: one recomputed conv row per 28, CTAs balanced)
    const int PH = a.OH / 2;
    const int nb = (PH + 13) / 14;
    const int BP = a.pool3s2 ? (PH + nb - 1) / nb : 0;
    const int tiles = a.pool3s2 ? a.N * ((PH + BP - 1) / BP) : a.N * a.OH;
    const int grid = std::min(tiles, num_sms());
    const int slot = (a.SC * a.kh * nbw * 4 + 1023) / 1024 * 1024;
    const int nh = std::min(SR_NH_MAX, (SR_SMEM - 1024 - OFF_HALO) / slot);
    stem_row_kernel<<<grid, SR_THREADS, SR_SMEM, s>>>(a, tx, tw, to, nbw, delta, slot, nh, BP);
    SOL_CUDA(cudaGetLastError());
}

}  // namespace solb200
