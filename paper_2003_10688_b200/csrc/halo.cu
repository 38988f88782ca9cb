// Halo-tile implicit GEMM for stride-1 "same" convolutions with one or two 64-channel blocks
// (ResNet-50's 56x56x64 and 28x28x128 3x3 convs). The TMA-im2col path re-reads every input pixel from L2 once per filter tap
// (9x for 3x3) and is bound by the TMA im2col request rate; here one tile covers R whole output
// rows in a row-padded pixel order (Wp = W + k - 1 columns, the last k - 1 of them junk), so the A
// operand of tap (dkh, dkw) is simply the halo box shifted by dkh * Wp + dkw rows: the halo
// [R + k - 1][Wp][64 ch] is loaded ONCE per tile by a 4-D TMA box (out-of-bounds fill = the zero
// padding) and every tap's MMA reads it through a shifted UMMA descriptor (the SW128 swizzle is a
// function of the absolute smem address, so 128-byte-row shifts need no re-layout).
//
//   warp 0      producer: resident weights once, then one halo TMA box per tile (ring of NH)
//   warp 4      tcgen05.mma issuer: the whole warp runs the loop, one elected lane issues a filter
//               row's 12 MMAs per asm statement (M = 128 row-padded pixels, N = BN, K = 9 x 64)
//   warps 5-8   epilogue: TMEM -> bias / folded BN / residual / activation -> bf16 -> global
//               (junk columns and rows past the tile are skipped)
// Measured (B200, B=256, 3x3): 56x56x64 75 us vs 130 us, 28x28x128 55 us vs 75 us for TMA
// im2col, bit-identical output.
//
// Semantics are the generic fprop's (reference.cpp:138-161; igemm.cuh).
#include "igemm.cuh"
#include "tc.cuh"

#include <algorithm>
#include <cstdlib>
#include <mutex>

namespace solb200 {
namespace {

using namespace tc;
using T_BF16 = __nv_bfloat16;

constexpr int HL_THREADS = 416;  // 4 producer warps (1 active), MMA warp, 8 epilogue warps
constexpr int HL_HALO_MAX = 49152;  // bytes of one halo buffer (all channel blocks)
constexpr int HL_PCACHE = 512;      // channels of cached epilogue parameters (3 x 2 KB after the barriers)

__device__ __forceinline__ void tma_load_4d_tile(uint32_t dst, const CUtensorMap* map, int c, int w, int h, int n,
                                                 uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c), "r"(w), "r"(h), "r"(n), "r"(mbar)
        : "memory");
}

struct HaloGeo {
    int Wp, R, HR, ncb, cb_bytes, halo_bytes, row_blocks;
};

__host__ __device__ inline HaloGeo halo_geo(const IgemmArgs& a) {
    HaloGeo g;
    g.Wp = a.OW + a.kw - 1;
    g.R = 128 / g.Wp;
    g.HR = g.R + a.kh - 1;
    g.ncb = a.SC / 64;
    g.cb_bytes = (g.HR * g.Wp * 128 + 1023) / 1024 * 1024;
    g.halo_bytes = g.ncb * g.cb_bytes;
    g.row_blocks = g.R > 0 ? (a.OH + g.R - 1) / g.R : 0;
    return g;
}

template <int BN>
constexpr int hl_stages() {
    return std::min(12, (227 * 1024 - 2 * HL_HALO_MAX - 2048 - 12 * HL_PCACHE) / (BN * 128));
}

// RESB: the whole weight matrix of the (single) N tile stays resident in shared memory, loaded
// once per CTA; otherwise [BN][64] weight blocks stream through a TMA ring.
constexpr int HL_NH_MAX = 8;  // halo ring depth bound

template <int BN, bool RESB>
__global__ void __launch_bounds__(HL_THREADS, 1)
    halo_kernel(const IgemmArgs a, const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w,
                int base_mode, int NH) {
    constexpr int B_BYTES = BN * 128;
    constexpr int STAGES = RESB ? 1 : hl_stages<BN>();
    constexpr int NA = 4 * BN <= 512 ? 4 : 2;  // TMEM accumulator stages
    constexpr uint32_t TCOLS = NA * BN <= 128 ? 128 : (NA * BN <= 256 ? 256 : 512);
    constexpr uint32_t IDESC = make_idesc(1, BN, 128, 0, 0);
    const HaloGeo G = halo_geo(a);

    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int HB = G.halo_bytes;                 // one halo buffer
    const int taps = a.kh * a.kw;
    uint8_t* halo = smem;                        // NH x HB (ring)
    uint8_t* bring = smem + NH * HB;             // RESB: taps x ncb blocks, else STAGES blocks
    uint64_t* bar = reinterpret_cast<uint64_t*>(bring + (RESB ? taps * G.ncb : STAGES) * B_BYTES);
    uint64_t* hfull = bar;                       // [HL_NH_MAX]
    uint64_t* hempty = bar + HL_NH_MAX;          // [HL_NH_MAX]
    uint64_t* tfull = bar + 2 * HL_NH_MAX;       // [4]
    uint64_t* tempty = tfull + 4;                // [4]
    uint64_t* bfull = tempty + 4;                // [STAGES]
    uint64_t* bempty = bfull + STAGES;  // [STAGES]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bempty + STAGES);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int n_tiles = (a.Nout + BN - 1) / BN;
    const int tiles = a.N * G.row_blocks * n_tiles;
    // contiguous tile ranges per CTA: consecutive row blocks of an image share halo rows, so the
    // overlap is served from L2 by the same SM instead of racing other SMs to DRAM
    const int per_cta = (tiles + gridDim.x - 1) / gridDim.x;
    const int t_begin = min(tiles, static_cast<int>(blockIdx.x) * per_cta);
    const int t_end = min(tiles, t_begin + per_cta);
    // tiles in order (the next tile's halo overlaps this one's in L2); debug flag 8192: even
    // offsets first, then odd
    const int n_even = (a.dbg & 8192) ? (t_end - t_begin + 1) / 2 : 1 << 30;
    auto tile_at = [&](int j) { return t_begin + (j < n_even ? ((a.dbg & 8192) ? 2 * j : j) : 2 * (j - n_even) + 1); };

    if (tid == 0) {
        for (int s = 0; s < NH; ++s) {
            mbar_init(smem_u32(&hfull[s]), 1);
            mbar_init(smem_u32(&hempty[s]), 1);
        }
        for (int s = 0; s < NA; ++s) {
            mbar_init(smem_u32(&tfull[s]), 1);
            mbar_init(smem_u32(&tempty[s]), 256);
        }
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(smem_u32(&bfull[s]), 1);
            mbar_init(smem_u32(&bempty[s]), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
        tma_prefetch(&tm_x);
        tma_prefetch(&tm_w);
    }
    if (warp == 4) tmem_alloc<TCOLS>(smem_u32(tmem_slot));
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp < 4 && RESB) {
        // ---------------------------------------------------------------- producer (RESB):
        // weights once, then per tile the whole halo as one 4-D TMA box per channel block
        // (out-of-bounds rows/columns zero-filled = the conv padding)
        if (tid == 0) {
            mbar_arrive_tx(smem_u32(&bfull[0]), static_cast<uint32_t>(taps * G.ncb * B_BYTES));
            for (int j = 0; j < taps * G.ncb; ++j)
                tma_load_2d(smem_u32(bring + j * B_BYTES), &tm_w, j * 64, 0, smem_u32(&bfull[0]));
            int hb = 0;
            uint32_t hph = 0;
            for (int j = 0; j < t_end - t_begin; ++j) {
                const int t = tile_at(j);
                const int rb = (t / n_tiles) % G.row_blocks;
                const int img = t / (n_tiles * G.row_blocks);
                mbar_wait(smem_u32(&hempty[hb]), ((hph >> hb) & 1) ^ 1);
                if (a.dbg & 16384) {  // profiling: skip the halo loads
                    mbar_arrive(smem_u32(&hfull[hb]));
                } else {
                    mbar_arrive_tx(smem_u32(&hfull[hb]), static_cast<uint32_t>(G.ncb * G.HR * G.Wp * 128));
                    for (int cb = 0; cb < G.ncb; ++cb)
                        tma_load_4d_tile(smem_u32(halo + hb * HB + cb * G.cb_bytes), &tm_x, cb * 64, -a.pw,
                                         rb * G.R - a.ph, img, smem_u32(&hfull[hb]));
                }
                hph ^= 1u << hb;
                if (++hb == NH) hb = 0;
            }
        }
    } else if (warp < 4) {
        // ---------------------------------------------------------------- TMA producer (streamed B)
        if (warp == 0 && lane == 0) {
            int stage = 0, hb = 0;
            uint32_t phase = 0, hph = 0;  // hph bit b = phase of halo buffer b
            for (int j = 0; j < t_end - t_begin; ++j) {
                const int t = tile_at(j);
                const int nt = t % n_tiles;
                const int rb = (t / n_tiles) % G.row_blocks;
                const int img = t / (n_tiles * G.row_blocks);
                mbar_wait(smem_u32(&hempty[hb]), ((hph >> hb) & 1) ^ 1);
                mbar_arrive_tx(smem_u32(&hfull[hb]), static_cast<uint32_t>(G.ncb * G.HR * G.Wp * 128));
                for (int cb = 0; cb < G.ncb; ++cb)
                    tma_load_4d_tile(smem_u32(halo + hb * HB + cb * G.cb_bytes), &tm_x, cb * 64, -a.pw,
                                     rb * G.R - a.ph, img, smem_u32(&hfull[hb]));
                hph ^= 1u << hb;
                if (++hb == NH) hb = 0;
                for (int tap = 0; tap < taps; ++tap) {
                    for (int cb = 0; cb < G.ncb; ++cb) {
                        mbar_wait(smem_u32(&bempty[stage]), phase ^ 1);
                        mbar_arrive_tx(smem_u32(&bfull[stage]), B_BYTES);
                        tma_load_2d(smem_u32(bring + stage * B_BYTES), &tm_w, tap * a.SC + cb * 64, nt * BN,
                                    smem_u32(&bfull[stage]));
                        if (++stage == STAGES) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                }
            }
        }
    } else if (warp == 4) {
        // ---------------------------------------------------------------- MMA issuer
        // The whole warp runs the loop (converged, operands warp-uniform); one elected lane
        // issues each K block's four MMAs (tc::mma4_elect). Descriptors are precomputed and
        // advanced by adds (the 14-bit start-address field is smem address >> 4).
        {
            int stage = 0, hb = 0, acc = 0;
            uint32_t phase = 0, hph = 0, acc_phase = 0;
            if (RESB) mbar_wait(smem_u32(&bfull[0]), 0);
            const uint64_t bdesc0 = sw128_desc(smem_u32(bring), 16, 1024);
            const uint32_t cb_units = static_cast<uint32_t>(G.cb_bytes) >> 4;
            const uint32_t row_skip = static_cast<uint32_t>(G.Wp - a.kw) * 8u;  // to the next filter row
            const bool do_mma = !(a.dbg & 2);
            for (int j = 0; j < t_end - t_begin; ++j) {
                mbar_wait(smem_u32(&tempty[acc]), acc_phase ^ 1);
                mbar_wait(smem_u32(&hfull[hb]), (hph >> hb) & 1);
                tc_fence_after();
                if ((a.dbg & 64) && blockIdx.x == 0 && lane == 0 && j < 64)
                    reinterpret_cast<long long*>(a.out)[64 + j] = clock64();
                const uint32_t dcol = __shfl_sync(0xffffffffu, tmem_base + static_cast<uint32_t>(acc * BN), 0);
                const uint64_t adesc0 = sw128_desc(smem_u32(halo + hb * HB), 16, 1024);
                uint32_t aoff = 0;  // (dkh * Wp + dkw) * 128 B, in 16-byte units
                uint32_t boff = 0;
                uint32_t accum = 0;
                if (RESB && a.kh == 3 && a.kw == 3 && G.ncb == 1 && G.Wp == 58 && do_mma) {
                    // ResNet-50 layer 1 (56x56): row pitch known at compile time, so every
                    // descriptor is base + immediate and stays in uniform registers
                    constexpr uint32_t WP8 = 58 * 8, BU = B_BYTES >> 4;
                    mma_row3_elect<BU>(dcol, adesc0, bdesc0, IDESC, 0);
                    mma_row3_elect<BU>(dcol, adesc0 + WP8, bdesc0 + 3 * BU, IDESC, 1);
                    mma_row3_elect<BU>(dcol, adesc0 + 2 * WP8, bdesc0 + 6 * BU, IDESC, 1);
                } else if (RESB && a.kw == 3 && (G.ncb == 1 || G.ncb == 2)) {
                    // 3x3 fast path: one asm statement per (channel block, filter row)
                    for (int cb = 0; cb < G.ncb; ++cb) {
                        for (int dkh = 0; dkh < a.kh; ++dkh) {
                            const uint64_t ad = adesc0 + static_cast<uint32_t>(dkh * G.Wp * 8) + cb * cb_units;
                            const uint64_t bd = bdesc0 + static_cast<uint32_t>((dkh * 3 * G.ncb + cb) * (B_BYTES >> 4));
                            if (do_mma) {
                                if (G.ncb == 1) mma_row3_elect<(B_BYTES >> 4)>(dcol, ad, bd, IDESC, accum);
                                else mma_row3_elect<2 * (B_BYTES >> 4)>(dcol, ad, bd, IDESC, accum);
                            }
                            accum = 1;
                        }
                    }
                } else
                for (int dkh = 0; dkh < a.kh; ++dkh) {
                    for (int dkw = 0; dkw < a.kw; ++dkw) {
                        for (int cb = 0; cb < G.ncb; ++cb) {
                            uint64_t bd;
                            if (RESB) {
                                bd = bdesc0 + boff;
                                boff += B_BYTES >> 4;
                            } else {
                                mbar_wait(smem_u32(&bfull[stage]), phase);
                                tc_fence_after();
                                bd = bdesc0 + static_cast<uint32_t>(stage * (B_BYTES >> 4));
                            }
                            if (do_mma) mma4_elect<__nv_bfloat16>(dcol, adesc0 + aoff + cb * cb_units, bd, IDESC, accum);
                            accum = 1;
                            if (!RESB) {
                                mma_commit_elect(smem_u32(&bempty[stage]));
                                if (++stage == STAGES) {
                                    stage = 0;
                                    phase ^= 1;
                                }
                            }
                        }
                        aoff += 8;
                    }
                    aoff += row_skip;
                }
                mma_commit_elect(smem_u32(&hempty[hb]));
                mma_commit_elect(smem_u32(&tfull[acc]));
                hph ^= 1u << hb;
                if (++hb == NH) hb = 0;
                if (++acc == NA) {
                    acc = 0;
                    acc_phase ^= 1;
                }
            }
        }
    } else {
        // ---------------------------------------------------------------- epilogue
        // two warps per TMEM lane quarter, each taking half of the tile's columns
        const int q = warp & 3;
        const int half = (warp - 5) >> 2;
        const bool has_bias = a.bias != nullptr, has_fold = a.ep_scale != nullptr, has_res = a.residual != nullptr;
        const bool res_mask = a.res_mode == 1;
        const int act = a.relu ? 1 : a.act;
        __nv_bfloat16* out = static_cast<__nv_bfloat16*>(a.out);
        const __nv_bfloat16* res = static_cast<const __nv_bfloat16*>(a.residual);
        int acc = 0;
        uint32_t acc_phase = 0;
        // per-channel epilogue parameters cached in shared memory once per CTA (warp-uniform reads
        // are broadcasts; the global loads' latency sat on every tile's critical path)
        float* p_bias = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(bar) + 1024);
        float* p_scale = p_bias + HL_PCACHE;
        float* p_shift = p_scale + HL_PCACHE;
        const bool cached = a.Nout <= HL_PCACHE;
        if (cached) {
            for (int c = tid - 160; c < a.Nout; c += 256) {
                p_bias[c] = has_bias ? a.bias[c] : 0.f;
                p_scale[c] = has_fold ? a.ep_scale[c] : 1.f;
                p_shift[c] = has_fold ? a.ep_shift[c] : 0.f;
            }
            asm volatile("bar.sync 3, 256;\n" ::: "memory");
        }
        const int i = q * 32 + lane;  // tile row (row-padded pixel order)
        const int oyl = i / G.Wp, ox = i - (i / G.Wp) * G.Wp;
        for (int j = 0; j < t_end - t_begin; ++j) {
            const int t = tile_at(j);
            const int nt = t % n_tiles;
            const int rb = (t / n_tiles) % G.row_blocks;
            const int img = t / (n_tiles * G.row_blocks);
            const int oy = rb * G.R + oyl;
            const bool valid = oyl < G.R && ox < a.OW && oy < a.OH;
            const int64_t m = (static_cast<int64_t>(img) * a.OH + oy) * a.OW + ox;
            mbar_wait(smem_u32(&tfull[acc]), acc_phase);
            tc_fence_after();
            if ((a.dbg & 64) && blockIdx.x == 0 && q == 0 && lane == 0 && j < 64)
                reinterpret_cast<long long*>(a.out)[128 + j] = clock64();
#pragma unroll 1
            for (int c0 = half * 32; c0 < BN; c0 += 64) {
                uint32_t v[32];
                tmem_ld32_nowait(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN + c0), v);
                tmem_wait_ld();
                const int n = nt * BN + c0;
                if (!valid || n >= a.ldo || (a.dbg & 1)) continue;
                float f[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) f[j] = __uint_as_float(v[j]);
                const bool full = n + 32 <= a.Nout;
                // every loop is unrolled so f[] stays in registers (a dynamic index would put it in
                // local memory); full chunks use float4 parameter loads (the addresses are warp-uniform)
                if (has_bias) {
                    if (full && cached) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 bb = *reinterpret_cast<const float4*>(p_bias + n + j);
                            f[j] += bb.x; f[j + 1] += bb.y; f[j + 2] += bb.z; f[j + 3] += bb.w;
                        }
                    } else if (full) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 bb = __ldg(reinterpret_cast<const float4*>(a.bias + n + j));
                            f[j] += bb.x; f[j + 1] += bb.y; f[j + 2] += bb.z; f[j + 3] += bb.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n + j < a.Nout) f[j] += __ldg(a.bias + n + j);
                    }
                }
                if (has_fold) {
                    if (full && cached) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 sc = *reinterpret_cast<const float4*>(p_scale + n + j);
                            const float4 sh = *reinterpret_cast<const float4*>(p_shift + n + j);
                            f[j] = fmaf(f[j], sc.x, sh.x);
                            f[j + 1] = fmaf(f[j + 1], sc.y, sh.y);
                            f[j + 2] = fmaf(f[j + 2], sc.z, sh.z);
                            f[j + 3] = fmaf(f[j + 3], sc.w, sh.w);
                        }
                    } else if (full) {
#pragma unroll
                        for (int j = 0; j < 32; j += 4) {
                            const float4 sc = __ldg(reinterpret_cast<const float4*>(a.ep_scale + n + j));
                            const float4 sh = __ldg(reinterpret_cast<const float4*>(a.ep_shift + n + j));
                            f[j] = fmaf(f[j], sc.x, sh.x);
                            f[j + 1] = fmaf(f[j + 1], sc.y, sh.y);
                            f[j + 2] = fmaf(f[j + 2], sc.z, sh.z);
                            f[j + 3] = fmaf(f[j + 3], sc.w, sh.w);
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n + j < a.Nout) f[j] = fmaf(f[j], __ldg(a.ep_scale + n + j), __ldg(a.ep_shift + n + j));
                    }
                }
                if (has_res) {
                    const __nv_bfloat16* rp = res + m * a.ld_res + n;
                    if (full) {
#pragma unroll
                        for (int j = 0; j < 32; j += 8) {
                            float r8[8];
                            load16(rp + j, r8);
#pragma unroll
                            for (int k = 0; k < 8; ++k) f[j + k] = res_mask ? (r8[k] > 0.f ? f[j + k] : 0.f) : f[j + k] + r8[k];
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (n + j < a.Nout) {
                                const float r = __bfloat162float(rp[j]);
                                f[j] = res_mask ? (r > 0.f ? f[j] : 0.f) : f[j] + r;
                            }
                    }
                }
                if (act != 0) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        f[j] = fmaxf(f[j], 0.f);
                        if (act == 2) f[j] = fminf(f[j], 6.f);
                    }
                }
                __nv_bfloat16* op = out + m * a.ldo + n;
                if (full && n + 32 <= a.ldo) {
#pragma unroll
                    for (int j = 0; j < 32; j += 8) store16(op + j, f + j);
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (n + j < a.ldo) op[j] = __float2bfloat16_rn(n + j < a.Nout ? f[j] : 0.f);
                }
            }
            tc_fence_before();
            mbar_arrive(smem_u32(&tempty[acc]));
            if (++acc == NA) {
                acc = 0;
                acc_phase ^= 1;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        tmem_dealloc<TCOLS>(tmem_base);
    }
}

CUtensorMap halo_tmap_x(const IgemmArgs& a, const HaloGeo& G) {
    CUtensorMap m;
    cuuint64_t dims[4] = {static_cast<cuuint64_t>(a.SC), static_cast<cuuint64_t>(a.SW), static_cast<cuuint64_t>(a.SH),
                          static_cast<cuuint64_t>(a.N)};
    cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.SC) * 2, static_cast<cuuint64_t>(a.SW) * a.SC * 2,
                             static_cast<cuuint64_t>(a.SH) * a.SW * a.SC * 2};
    cuuint32_t box[4] = {64, static_cast<cuuint32_t>(G.Wp), static_cast<cuuint32_t>(G.HR), 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(a.src), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("halo: cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
    return m;
}

bool halo_resident_b(const IgemmArgs& a, int bn) {
    const HaloGeo G = halo_geo(a);
    return a.Nout <= bn && a.kh * a.kw * G.ncb * bn * 128 + 2 * G.halo_bytes + 4096 <= 227 * 1024;
}

template <int BN, bool RESB>
void halo_launch_t(const IgemmArgs& a, cudaStream_t s) {
    const HaloGeo G = halo_geo(a);
    const int bbytes = (RESB ? a.kh * a.kw * G.ncb : hl_stages<BN>()) * BN * 128;
    const int nh = std::max(2, std::min(HL_NH_MAX, (227 * 1024 - bbytes - 2048 - 12 * HL_PCACHE) / G.halo_bytes));
    const int smem = nh * G.halo_bytes + bbytes + 1024 + 1024 + 12 * HL_PCACHE;
    static std::once_flag once;
    std::call_once(once, [] {
        SOL_CUDA(cudaFuncSetAttribute(halo_kernel<BN, RESB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    });
    const CUtensorMap tx = halo_tmap_x(a, G);
    const CUtensorMap tw = make_tmap_2d(a.wt, DT_BF16, a.K_pad, static_cast<uint64_t>(a.Nout), a.K_pad, BN);
    const int tiles = a.N * G.row_blocks * ((a.Nout + BN - 1) / BN);
    const int grid = std::min(tiles, num_sms());
    halo_kernel<BN, RESB><<<grid, HL_THREADS, smem, s>>>(a, tx, tw, (a.dbg & 32) ? 1 : 0, nh);
    SOL_CUDA(cudaGetLastError());
}

template <int BN>
void halo_dispatch(const IgemmArgs& a, cudaStream_t s) {
    if (halo_resident_b(a, BN)) halo_launch_t<BN, true>(a, s);
    else halo_launch_t<BN, false>(a, s);
}

}  // namespace

bool halo_supported(const IgemmArgs& a) {
    // On by default for 64- and 128-channel inputs (ResNet-50's 56x56x64 and 28x28x128 3x3 convs:
    // 1.7x / 1.35x faster than TMA im2col, bit-identical: same k-block order). 64 channels keep the
    // weights resident; at 128 they stream through the TMA ring (288 KB per tile of L2 reads, still
    // well under im2col's 9x re-read of the input). Off: conv debug flag 512 or SOL_NO_HALO=1.
    static const bool disabled = std::getenv("SOL_NO_HALO") != nullptr;
    if ((a.dbg & 512) || disabled) return false;
    if (a.SC != 64 && a.SC != 128) return false;
    if (a.mode != IG_FPROP || a.dtype != DT_BF16 || a.out_dtype != DT_BF16 || (a.dbg & 16)) return false;
    if (a.sh != 1 || a.sw != 1 || a.kh != a.kw || a.kh % 2 == 0 || a.kh < 3 || a.kh > 7) return false;
    if (a.ph != a.kh / 2 || a.pw != a.kw / 2 || a.OH != a.SH || a.OW != a.SW) return false;
    if (a.SC % 64 != 0 || a.K_pad != a.kh * a.kw * a.SC || a.ldo % 8 != 0) return false;
    if (a.residual && (a.ld_res % 8 != 0)) return false;
    const HaloGeo G = halo_geo(a);
    // worthwhile while the halo fits, the row padding wastes little of each tile and the weights
    // stay resident (streaming them per tile costs as much L2 traffic as im2col saves)
    return G.R >= 1 && G.halo_bytes <= HL_HALO_MAX && G.R * a.OW >= 96 &&
           (a.SC == 128 || halo_resident_b(a, igemm_block_n(a.Nout) < 64 ? 64 : igemm_block_n(a.Nout)));
}

void halo_launch(const IgemmArgs& a, cudaStream_t s) {
    switch (igemm_block_n(a.Nout)) {
        case 16:
        case 32:
        case 64: return halo_dispatch<64>(a, s);
        case 128: return halo_dispatch<128>(a, s);
        default: return halo_dispatch<256>(a, s);
    }
}

}  // namespace solb200
