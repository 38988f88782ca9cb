// Stem convolution for images with few channels (Cin <= 4, stored as 8-channel NHWC pixels),
// e.g. ResNet-50's 7x7/2 3->64 conv. The generic implicit GEMM gathers one 16-byte (pixel, tap)
// vector per A element group, which for Cin = 3 is 49 scattered loads per output pixel; here each
// 8x16 output tile instead loads its input halo ONCE with a 4-D TMA box, and the im2col matrix is
// built in shared memory:
//
//   warp 0      TMA: packed weights once, then one halo box [HH][HWp][8 ch] per tile
//   warps 1-8   builders: halo -> compact [HH][HWp][4 ch] (8 B / pixel) -> A tile rows in the
//               UMMA K-major SWIZZLE_128B layout, K ordered (kh, kw in 8 slots, c in 4), i.e. one
//               16-byte chunk = two horizontally adjacent taps x 4 channels
//   warp 9      tcgen05.mma issuer (M = 128 pixels, N = Cout = 64, K = kh * 32)
//   warps 10-13 epilogue: TMEM -> (bias, folded BN, activation) -> bf16 -> 128B-swizzled staging ->
//               TMA store of [2 rows][16 cols][64 ch] boxes
//
// Semantics are exactly the generic fprop's (reference.cpp:138-161): zero padding comes from the
// TMA out-of-bounds fill, the accumulation is f32 over bf16 operands.
#include "igemm.cuh"
#include "tc.cuh"

#include <algorithm>
#include <mutex>

namespace solb200 {
namespace {

using namespace tc;

constexpr int ST_TH = 8, ST_TW = 16;  // output tile: 8 rows x 16 columns = 128 pixels
constexpr int ST_BN = 64;             // Cout
constexpr int ST_THREADS = 448;  // TMA warp, 8 builder warps, MMA warp, 4 epilogue warps
constexpr int ST_A_BYTES = 65536;     // 4 k-blocks x 128 rows x 128 B
constexpr int ST_B_BYTES = 4 * ST_BN * 128;
constexpr int ST_STAGE_BYTES = 4 * 4096;      // epilogue staging: 4 warps x 1 buffer
constexpr int ST_HALO_MAX = 13312;            // raw halo bytes (16 B / pixel), double-buffered
constexpr int ST_COMPACT_MAX = 8192 + 64;     // compact halo (8 B / pixel, + overrun pad)
constexpr int OFF_A = 0;
constexpr int OFF_B = OFF_A + 2 * ST_A_BYTES;
constexpr int OFF_STG = OFF_B + ST_B_BYTES;
constexpr int OFF_HALO = OFF_STG + ST_STAGE_BYTES;
constexpr int OFF_CMP = OFF_HALO + 2 * ST_HALO_MAX;
constexpr int OFF_BAR = OFF_CMP + ST_COMPACT_MAX;
constexpr int ST_SMEM = OFF_BAR + 256 + 1024;  // barriers + 1 KB alignment slack

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                            uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(mbar)
        : "memory");
}

__device__ __forceinline__ void builders_sync() { asm volatile("bar.sync 1, 256;\n" ::: "memory"); }

// WG: weight gradient instead of fprop. The im2col tile the builders produce is, read per 64-column
// block, exactly the MN-major operand of dW = xcol^T dy (pixels = K), and the dy tile arrives by a
// [8 rows][16 cols][64 ch] TMA box (tm_w holds dy's map); every CTA accumulates dW^T over all its
// tiles in TMEM (2 M tiles of 128 K columns x 64 Cout) and writes one f32 partial to `ws`.
template <bool SW2, bool WG>
__global__ void __launch_bounds__(ST_THREADS, 1)
    stem_kernel(const IgemmArgs a, const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                const __grid_constant__ CUtensorMap tm_o, int HH, int HWp, float* ws, int nbw, int ndelta) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* b_full = bar + 0;
    uint64_t* halo_full = bar + 15;   // [2]
    uint64_t* halo_empty = bar + 17;  // [2]
    uint64_t* a_full = bar + 3;   // [2]
    uint64_t* a_empty = bar + 5;  // [2]
    uint64_t* tfull = bar + 7;    // [2]
    uint64_t* tempty = bar + 9;   // [2]
    uint64_t* dy_full = bar + 11;   // [2] (WG)
    uint64_t* dy_empty = bar + 13;  // [2] (WG)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 19);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_y = (a.OH + ST_TH - 1) / ST_TH, tiles_x = (a.OW + ST_TW - 1) / ST_TW;
    const int tiles = a.N * tiles_y * tiles_x;
    const int nkb = (a.kh * 32 + 63) / 64;
    const int ksteps = a.kh * 2;  // k16 steps over the kh * 32 real K elements
    // NCHW f32 halo: TMA boxes must start on 16-byte boundaries along W, so the box starts
    // `ndelta` columns early (constant per conv: tile origins are multiples of 16 columns) and is
    // `nbw` columns wide; the repack shifts it back
    const uint32_t halo_bytes =
        static_cast<uint32_t>(a.src_nchw_f32 ? HH * nbw * 4 * a.SC : HH * HWp * 16);

    if (tid == 0) {
        mbar_init(smem_u32(b_full), 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&halo_full[s]), 1);
            mbar_init(smem_u32(&halo_empty[s]), 256);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(smem_u32(&a_full[s]), 256);
            mbar_init(smem_u32(&a_empty[s]), 1);
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 128);
            mbar_init(smem_u32(&dy_full[s]), 1);
            mbar_init(smem_u32(&dy_empty[s]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        tma_prefetch(&tm_x);
        tma_prefetch(&tm_w);
        tma_prefetch(&tm_o);
    }
    if (warp == 9) tmem_alloc<2 * ST_BN>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ---------------------------------------------------------------- TMA producer
        if (lane == 0) {
            if (!WG) {
                mbar_arrive_tx(smem_u32(b_full), static_cast<uint32_t>(nkb * ST_BN * 128));
                for (int kb = 0; kb < nkb; ++kb)
                    tma_load_2d(smem_u32(smem + OFF_B + kb * ST_BN * 128), &tm_w, kb * 64, 0, smem_u32(b_full));
            }
            uint32_t hphase = 0, dphase = 0;
            int ds = 0, hb = 0;
            for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
                const int n = t / (tiles_y * tiles_x);
                const int rem = t - n * tiles_y * tiles_x;
                const int oy0 = (rem / tiles_x) * ST_TH, ox0 = (rem % tiles_x) * ST_TW;
                if (WG) {
                    // dy tile [8][16][64] -> 128 pixel rows x 128 B (MN-major operand)
                    mbar_wait(smem_u32(&dy_empty[ds]), dphase ^ 1);
                    mbar_arrive_tx(smem_u32(&dy_full[ds]), 16384);
                    tma_load_4d(smem_u32(smem + OFF_B + ds * 16384), &tm_w, 0, ox0, oy0, n, smem_u32(&dy_full[ds]));
                    if (++ds == 2) {
                        ds = 0;
                        dphase ^= 1;
                    }
                }
                mbar_wait(smem_u32(&halo_empty[hb]), hphase ^ 1);
                mbar_arrive_tx(smem_u32(&halo_full[hb]), halo_bytes);
                if (a.src_nchw_f32)  // box {nbw, HH, Cin, 1} over the NCHW f32 input
                    tma_load_4d(smem_u32(smem + OFF_HALO + hb * ST_HALO_MAX), &tm_x, ox0 * a.sw - a.pw - ndelta,
                                oy0 * a.sh - a.ph, 0, n, smem_u32(&halo_full[hb]));
                else
                    tma_load_4d(smem_u32(smem + OFF_HALO + hb * ST_HALO_MAX), &tm_x, 0, ox0 * a.sw - a.pw,
                                oy0 * a.sh - a.ph, n, smem_u32(&halo_full[hb]));
                if (++hb == 2) {
                    hb = 0;
                    hphase ^= 1;
                }
            }
        }
    } else if (warp <= 8) {
        // ---------------------------------------------------------------- builders (8 warps)
        const int b = tid - 32;
        const int r = b & 127;   // A row = output pixel of the tile
        const int kh_first = b >> 7;  // the two builder halves take alternate kernel rows
        const int ty = r / ST_TW, tx = r % ST_TW;
        int hb = 0;
        uint2* cmp = reinterpret_cast<uint2*>(smem + OFF_CMP);
        const int npix = HH * HWp;
        const int nchw = a.src_nchw_f32;
        const int cin = a.SC;
        uint32_t hphase = 0, aphase = 0;
        int s = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            builders_sync();  // every builder is done reading the previous compact halo
            mbar_wait(smem_u32(&halo_full[hb]), hphase);
            if (nchw) {
                // f32 planes [Cin][HH][HWp] -> 4 bf16 channels per pixel (channels >= Cin zero)
                const float* plane = reinterpret_cast<const float*>(smem + OFF_HALO + hb * ST_HALO_MAX);
                const int pplane = HH * nbw;
                for (int i = b; i < npix; i += 256) {
                    const int hy = i / HWp, hx = i - (i / HWp) * HWp;
                    const int src = hy * nbw + hx + ndelta;
                    float f[4];
#pragma unroll
                    for (int ch = 0; ch < 4; ++ch) f[ch] = ch < cin ? plane[ch * pplane + src] : 0.f;
                    const __nv_bfloat162 lo = __floats2bfloat162_rn(f[0], f[1]);
                    const __nv_bfloat162 hi = __floats2bfloat162_rn(f[2], f[3]);
                    cmp[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&lo), *reinterpret_cast<const uint32_t*>(&hi));
                }
            } else {
                const uint4* raw = reinterpret_cast<const uint4*>(smem + OFF_HALO + hb * ST_HALO_MAX);
                for (int i = b; i < npix; i += 256) {
                    const uint4 v = raw[i];
                    cmp[i] = make_uint2(v.x, v.y);  // channels 0..3
                }
            }
            builders_sync();
            mbar_arrive(smem_u32(&halo_empty[hb]));
            if (++hb == 2) {
                hb = 0;
                hphase ^= 1;
            }
            mbar_wait(smem_u32(&a_empty[s]), aphase ^ 1);
            uint8_t* A = smem + OFF_A + s * ST_A_BYTES;
            for (int khi = kh_first; khi < a.kh; khi += 2) {
                const int pix = (ty * a.sh + khi) * HWp + tx * a.sw;
#pragma unroll
                for (int jc = 0; jc < 4; ++jc) {
                    uint4 v;
                    if (SW2) {
                        v = *reinterpret_cast<const uint4*>(cmp + pix + 2 * jc);
                    } else {
                        const uint2 p0 = cmp[pix + 2 * jc], p1 = cmp[pix + 2 * jc + 1];
                        v = make_uint4(p0.x, p0.y, p1.x, p1.y);
                    }
                    const int q = khi * 4 + jc;
                    const uint32_t dst =
                        smem_u32(A + (q >> 3) * 16384 + r * 128 + (((q & 7) ^ (r & 7)) << 4));
                    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(dst), "r"(v.x), "r"(v.y),
                                 "r"(v.z), "r"(v.w));
                }
            }
            fence_proxy_async();
            mbar_arrive(smem_u32(&a_full[s]));
            if (++s == 2) {
                s = 0;
                aphase ^= 1;
            }
        }
    } else if (warp == 9 && WG) {
        // ---------------------------------------------------------------- MMA issuer (dW^T)
        constexpr uint32_t IDESC = make_idesc(1, ST_BN, 128, 1, 1);
        uint32_t aphase = 0;
        int s = 0;
        bool first = true;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(smem_u32(&a_full[s]), aphase);
            mbar_wait(smem_u32(&dy_full[s]), aphase);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t a_addr = smem_u32(smem + OFF_A + s * ST_A_BYTES);
                const uint32_t d_addr = smem_u32(smem + OFF_B + s * 16384);
                for (int ks = 0; ks < 8; ++ks) {  // 16 pixels per step
                    const uint64_t bd = sw128_desc(d_addr + ks * 2048, 16384, 1024);
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        if (mt * 128 >= a.kh * 32) break;
                        const uint64_t ad = sw128_desc(a_addr + mt * 2 * 16384 + ks * 2048, 16384, 1024);
                        mma<__nv_bfloat16>(tmem_base + static_cast<uint32_t>(mt * ST_BN), ad, bd, IDESC,
                                           (first && ks == 0) ? 0u : 1u);
                    }
                }
                mma_commit(smem_u32(&a_empty[s]));
                mma_commit(smem_u32(&dy_empty[s]));
            }
            first = false;
            __syncwarp();
            if (++s == 2) {
                s = 0;
                aphase ^= 1;
            }
        }
        if (lane == 0) mma_commit(smem_u32(&tfull[0]));
        __syncwarp();
    } else if (warp >= 10 && WG) {
        // ---------------------------------------------------------------- dW^T partial -> ws
        const int q = warp & 3;
        mbar_wait(smem_u32(&tfull[0]), 0);
        tc_fence_after();
        for (int mt = 0; mt < 2; ++mt) {
            uint32_t v[ST_BN];
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(mt * ST_BN);
            tmem_ld32_nowait(taddr, v);
            tmem_ld32_nowait(taddr + 32, v + 32);
            tmem_wait_ld();
            const int kcol = mt * 128 + q * 32 + lane;
            float* dst = ws + (static_cast<int64_t>(blockIdx.x) * 256 + kcol) * ST_BN;
#pragma unroll
            for (int i = 0; i < ST_BN; i += 4)
                *reinterpret_cast<float4*>(dst + i) = make_float4(__uint_as_float(v[i]), __uint_as_float(v[i + 1]),
                                                                  __uint_as_float(v[i + 2]), __uint_as_float(v[i + 3]));
        }
    } else if (warp == 9) {
        // ---------------------------------------------------------------- MMA issuer
        constexpr uint32_t IDESC = make_idesc(1, ST_BN, 128, 0, 0);
        mbar_wait(smem_u32(b_full), 0);
        uint32_t aphase = 0, acc_phase = 0;
        int s = 0, acc = 0;
        const uint32_t b_addr = smem_u32(smem + OFF_B);
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
            mbar_wait(smem_u32(&a_full[s]), aphase);
            tc_fence_after();
            if (lane == 0) {
                const uint32_t a_addr = smem_u32(smem + OFF_A + s * ST_A_BYTES);
                const uint32_t dcol = tmem_base + static_cast<uint32_t>(acc * ST_BN);
                for (int ks = 0; ks < ksteps; ++ks) {
                    const uint64_t ad = sw128_desc(a_addr + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024);
                    const uint64_t bd = sw128_desc(b_addr + (ks >> 2) * (ST_BN * 128) + (ks & 3) * 32, 16, 1024);
                    mma<__nv_bfloat16>(dcol, ad, bd, IDESC, ks > 0);
                }
                mma_commit(smem_u32(&a_empty[s]));
                mma_commit(smem_u32(&tfull[acc]));
            }
            __syncwarp();
            if (++s == 2) {
                s = 0;
                aphase ^= 1;
            }
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue
        const int q = warp & 3;  // TMEM lane quarter this warp may access = tile rows 2q, 2q+1
        uint8_t* stage = smem + OFF_STG + q * 4096;
        const bool has_bias = a.bias != nullptr, has_fold = a.ep_scale != nullptr;
        const int act = a.relu ? 1 : a.act;
        uint32_t acc_phase = 0;
        int acc = 0, buf = 0;
        for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
            const int n = t / (tiles_y * tiles_x);
            const int rem = t - n * tiles_y * tiles_x;
            const int oy0 = (rem / tiles_x) * ST_TH, ox0 = (rem % tiles_x) * ST_TW;
            mbar_wait(smem_u32(&tfull[acc]), acc_phase);
            tc_fence_after();
            uint32_t v[ST_BN];
            const uint32_t taddr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * ST_BN);
            tmem_ld32_nowait(taddr, v);
            tmem_ld32_nowait(taddr + 32, v + 32);
            tmem_wait_ld();
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty[acc]));
            float f[ST_BN];
#pragma unroll
            for (int i = 0; i < ST_BN; ++i) f[i] = __uint_as_float(v[i]);
            if (has_bias) {
#pragma unroll
                for (int i = 0; i < ST_BN; i += 4) {
                    const float4 b = __ldg(reinterpret_cast<const float4*>(a.bias + i));
                    f[i] += b.x; f[i + 1] += b.y; f[i + 2] += b.z; f[i + 3] += b.w;
                }
            }
            if (has_fold) {
#pragma unroll
                for (int i = 0; i < ST_BN; i += 4) {
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
                for (int i = 0; i < ST_BN; ++i) {
                    f[i] = fmaxf(f[i], 0.f);
                    if (act == 2) f[i] = fminf(f[i], 6.f);
                }
            }
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            __syncwarp();
            uint8_t* sb = stage;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float* src = f + j * 8;
                __nv_bfloat162 p0 = __floats2bfloat162_rn(src[0], src[1]);
                __nv_bfloat162 p1 = __floats2bfloat162_rn(src[2], src[3]);
                __nv_bfloat162 p2 = __floats2bfloat162_rn(src[4], src[5]);
                __nv_bfloat162 p3 = __floats2bfloat162_rn(src[6], src[7]);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                                 smem_u32(sb + lane * 128 + ((j ^ (lane & 7)) << 4))),
                             "r"(*reinterpret_cast<uint32_t*>(&p0)), "r"(*reinterpret_cast<uint32_t*>(&p1)),
                             "r"(*reinterpret_cast<uint32_t*>(&p2)), "r"(*reinterpret_cast<uint32_t*>(&p3)));
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                asm volatile(
                    "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];\n" ::"l"(
                        reinterpret_cast<uint64_t>(&tm_o)),
                    "r"(0), "r"(ox0), "r"(oy0 + 2 * q), "r"(n), "r"(smem_u32(sb))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
            }
            buf ^= 1;
            if (++acc == 2) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
        if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc<2 * ST_BN>(tmem_base);
    }
}

CUtensorMap tmap_4d(const void* base, uint64_t c, uint64_t w, uint64_t h, uint64_t n, uint32_t bc, uint32_t bw,
                    uint32_t bh, CUtensorMapSwizzle swz) {
    CUtensorMap m;
    cuuint64_t dims[4] = {c, w, h, n};
    cuuint64_t strides[3] = {c * 2, w * c * 2, h * w * c * 2};
    cuuint32_t box[4] = {bc, bw, bh, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("stem: cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

void stem_geometry(const IgemmArgs& a, int& HH, int& HWp, int* nbw = nullptr, int* ndelta = nullptr) {
    HH = (ST_TH - 1) * a.sh + a.kh;
    const int HW = (ST_TW - 1) * a.sw + a.kw;
    HWp = HW + (HW & 1);
    // NCHW f32 box: start aligned down to 4 floats (tile origins are 16 * sw columns apart)
    const int delta = ((a.pw % 4) == 0) ? 0 : 4 - a.pw % 4;
    if (ndelta) *ndelta = delta;
    if (nbw) *nbw = (HWp + 1 + delta + 3) / 4 * 4;  // covers column HWp (cmp over-read pad)
}

CUtensorMap tmap_nchw_f32(const void* base, int N, int C, int H, int W, int bw, int bh) {
    CUtensorMap m;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H), static_cast<cuuint64_t>(C),
                          static_cast<cuuint64_t>(N)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(W) * 4, static_cast<cuuint64_t>(H) * W * 4,
                             static_cast<cuuint64_t>(C) * H * W * 4};
    cuuint32_t box[4] = {static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh), static_cast<cuuint32_t>(C), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("stem: NCHW tensor map failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

}  // namespace

int stem_kpad(int kh) { return (kh * 32 + 63) / 64 * 64; }

bool stem_supported(const IgemmArgs& a) {
    if (a.mode != IG_FPROP || a.dtype != DT_BF16 || a.out_dtype != DT_BF16) return false;
    if ((a.src_nchw_f32 ? (a.SC < 1 || a.SC > 4) : a.SC != 8) || a.Nout != ST_BN || a.ldo != ST_BN ||
        a.residual != nullptr)
        return false;
    if (a.kw > 8 || a.kh * 32 > 256 || a.K_pad != stem_kpad(a.kh)) return false;
    int HH, HWp, nbw, nd;
    stem_geometry(a, HH, HWp, &nbw, &nd);
    const int halo = a.src_nchw_f32 ? HH * nbw * 4 * a.SC : HH * HWp * 16;
    return halo <= ST_HALO_MAX && HWp <= 256 && HH <= 256 && a.N > 0 && a.OH > 0 && a.OW > 0;
}

void stem_launch(const IgemmArgs& a, cudaStream_t s) {
    if (!stem_supported(a)) throw std::invalid_argument("stem conv: unsupported shape");
    if (stem_row_supported(a)) return stem_row_launch(a, s);
    int HH, HWp, nbw, nd;
    stem_geometry(a, HH, HWp, &nbw, &nd);
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(stem_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM));
        SOL_CUDA(cudaFuncSetAttribute(stem_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM));
    });
    const CUtensorMap tx = a.src_nchw_f32 ? tmap_nchw_f32(a.src, a.N, a.SC, a.SH, a.SW, nbw, HH)
                                          : tmap_4d(a.src, 8, a.SW, a.SH, a.N, 8, HWp, HH, CU_TENSOR_MAP_SWIZZLE_NONE);
    const CUtensorMap tw = make_tmap_2d(a.wt, DT_BF16, a.K_pad, ST_BN, a.K_pad, ST_BN);
    const CUtensorMap to = tmap_4d(a.out, a.ldo, a.OW, a.OH, a.N, 64, ST_TW, 2, CU_TENSOR_MAP_SWIZZLE_128B);
    const int tiles = a.N * ((a.OH + ST_TH - 1) / ST_TH) * ((a.OW + ST_TW - 1) / ST_TW);
    const int grid = std::min(tiles, num_sms());
    if (a.sw % 2 == 0) stem_kernel<true, false><<<grid, ST_THREADS, ST_SMEM, s>>>(a, tx, tw, to, HH, HWp, nullptr, nbw, nd);
    else stem_kernel<false, false><<<grid, ST_THREADS, ST_SMEM, s>>>(a, tx, tw, to, HH, HWp, nullptr, nbw, nd);
    SOL_CUDA(cudaGetLastError());
}

namespace {
// dW[co][c][kh][kw] = sum over CTA partials of dW^T[kh*32 + kw*4 + c][co]
__global__ void stem_wgrad_reduce(const float* __restrict__ ws, int parts, float* __restrict__ dw, int Cout, int Cin,
                                  int KH, int KW) {
    const int total = Cout * Cin * KH * KW;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int kw = i % KW, kh = (i / KW) % KH, c = (i / (KW * KH)) % Cin, co = i / (KW * KH * Cin);
        const int kcol = kh * 32 + kw * 4 + c;
        float acc = 0.f;
        for (int p = 0; p < parts; ++p) acc += ws[(static_cast<int64_t>(p) * 256 + kcol) * ST_BN + co];
        dw[i] = acc;
    }
}
}  // namespace

bool stem_wgrad_supported(const IgemmArgs& a, int ld_dy) {
    IgemmArgs f = a;
    f.mode = IG_FPROP;
    f.Nout = ST_BN;
    f.ldo = ST_BN;
    f.K_pad = stem_kpad(a.kh);
    f.out_dtype = DT_BF16;
    f.residual = nullptr;
    return ld_dy == ST_BN && stem_supported(f);
}

size_t stem_wgrad_workspace_floats() { return static_cast<size_t>(num_sms()) * 256 * ST_BN; }

void stem_wgrad_launch(const IgemmArgs& a, const void* dy, int Cin, float* ws, float* dw, cudaStream_t s) {
    int HH, HWp, nbw, nd;
    stem_geometry(a, HH, HWp, &nbw, &nd);
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(stem_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM));
        SOL_CUDA(cudaFuncSetAttribute(stem_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, ST_SMEM));
    });
    const CUtensorMap tx = a.src_nchw_f32 ? tmap_nchw_f32(a.src, a.N, a.SC, a.SH, a.SW, nbw, HH)
                                          : tmap_4d(a.src, 8, a.SW, a.SH, a.N, 8, HWp, HH, CU_TENSOR_MAP_SWIZZLE_NONE);
    const CUtensorMap tdy = tmap_4d(dy, ST_BN, a.OW, a.OH, a.N, 64, ST_TW, ST_TH, CU_TENSOR_MAP_SWIZZLE_128B);
    const int tiles = a.N * ((a.OH + ST_TH - 1) / ST_TH) * ((a.OW + ST_TW - 1) / ST_TW);
    const int grid = std::min(tiles, num_sms());
    if (a.sw % 2 == 0) stem_kernel<true, true><<<grid, ST_THREADS, ST_SMEM, s>>>(a, tx, tdy, tdy, HH, HWp, ws, nbw, nd);
    else stem_kernel<false, true><<<grid, ST_THREADS, ST_SMEM, s>>>(a, tx, tdy, tdy, HH, HWp, ws, nbw, nd);
    SOL_CUDA(cudaGetLastError());
    const int total = ST_BN * Cin * a.kh * a.kw;
    stem_wgrad_reduce<<<(total + 255) / 256, 256, 0, s>>>(ws, grid, dw, ST_BN, Cin, a.kh, a.kw);
    SOL_CUDA(cudaGetLastError());
}

}  // namespace solb200
