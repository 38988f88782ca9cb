// tcgen05/TMEM implicit-GEMM for Conv2d / Linear (fprop, dgrad) and the wgrad GEMM, sm_100a.
//
// Semantics follow the reference's heavy-layer providers and oracle:
//   fprop   y[n,oh,ow,co] = b[co] + sum_{kh,kw,ci} x[n, oh*sh-ph+kh, ow*sw-pw+kw, ci] W[co,ci,kh,kw]
//           (proj/src/reference.cpp:138-161; dnn_providers.cpp:104-183)
//   dgrad   dx[n,ih,iw,ci] = sum_{kh,kw,co} dy[n,(ih+ph-kh)/sh,(iw+pw-kw)/sw,co] W[co,ci,kh,kw]
//           over exactly divisible, in-range positions (reference.cpp:482-506; dnn_providers.cpp:185-215)
//   wgrad   dW[co,(kh,kw,ci)] = sum_{n,oh,ow} dy[n,oh,ow,co] x[n,oh*sh-ph+kh,ow*sw-pw+kw,ci]
//           (reference.cpp:507-533; dnn_providers.cpp:217-241)
// Layout: activations NHWC (ActLayout::ChannelsLast), weights packed K-major [rows][K_pad].
#pragma once

#include "common.cuh"

namespace solb200 {

enum IgemmMode : int {
    IG_FPROP = 0,   // A = im2col(x) gathered K-major; B = W packed [Cout][kh][kw][Cin_pad]
    IG_DGRAD = 1,   // A = transposed-conv gather of dy; B = W packed [Cin][kh][kw][Cout_pad]
};

struct IgemmArgs {
    int mode = IG_FPROP;
    int dtype = DT_BF16;       // element type of A/B (bf16 -> kind::f16, f32 -> kind::tf32)
    int out_dtype = DT_BF16;   // element type of the output
    const void* src = nullptr; // gathered operand source, NHWC [N, SH, SW, SC]
    const void* wt = nullptr;  // packed B, [n_rows][K_pad]
    const float* bias = nullptr;
    void* out = nullptr;       // [M][ldo]
    int N = 0, SH = 0, SW = 0, SC = 0;
    int OH = 0, OW = 0;
    int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
    int Nout = 0;              // GEMM N
    int K_pad = 0;             // padded reduction extent of the packed operand
    int ldo = 0;
    int relu = 0;              // fused epilogue ReLU (unused by the reference path)
    int max_ctas = 0;          // cap on the persistent grid (0 = one CTA per SM); concurrent launches share the SMs
    int dbg = 0;               // profiling knobs: 1 = skip output stores, 2 = skip MMA issue
    // fused epilogue (inference BN folding, beyond the reference pass set):
    //   y = act( (acc + bias) * ep_scale[c] + ep_shift[c] [+ residual[m, c]] )
    const float* ep_scale = nullptr;
    const float* ep_shift = nullptr;
    const void* residual = nullptr;  // same dtype as the output, row stride ld_res
    int ld_res = 0;
    int act = 0;                     // 0 none, 1 relu, 2 relu6 (applied after the residual add)
    // 1: the residual is a ReLU OUTPUT used as a backward mask instead of an addend:
    //    y = residual > 0 ? acc : 0 (ReluBack(delta, relu(x)) fused into the dgrad epilogue)
    int res_mode = 0;
    // optional second epilogue input: y = mask > 0 ? acc + residual : 0 (Add + ReluBack fused into
    // a dgrad epilogue; mask = the ReLU output, same layout as the residual; N tiles of one chunk
    // per epilogue warp so both boxes fit the warp's two staging buffers)
    const void* mask = nullptr;
    // optional BatchNorm statistics of the stored (bf16) output, for a training BN that consumes it
    // (sol_b200_plan_link_bn_stats): per channel c and block b = (CTA, 32-row lane quarter),
    //   stat_partial[(c * stat_blocks + b) * 2 + {0, 1}] = sum over the block's rows of (y - shift[c])^{1,2}
    // with shift = stat_shift (the previous step's batch mean); blocks no CTA owns are zeroed
    double* stat_partial = nullptr;
    const float* stat_shift = nullptr;
    int stat_blocks = 0;  // partial blocks allocated (igemm_stat_blocks)
    // strided dgrad by sub-pixel classes, stored in place: GEMM row (n, i, j) of the class grid
    // (N, OH, OW) goes to pixel (n, sub_sh * i + sub_a, sub_sw * j + sub_b) of the [N, sub_H, sub_W]
    // output with direct 16-byte stores; sub_zero: the class also zeroes the other positions of its
    // sub_sh x sub_sw cell (the classes without taps). 0 = ordinary output.
    int sub_sh = 0, sub_sw = 0, sub_a = 0, sub_b = 0, sub_H = 0, sub_W = 0, sub_zero = 0;
    // dual GEMM (inference bottleneck-block fusion): K = [0, K1) reads A from `src` as a 1x1
    // stride-1 conv, K = [K1, K_pad) reads a second 1x1 conv with stride s2 over src2
    // [N, SH2, SW2, SC2] on the same output grid; B packs both weight matrices side by side.
    const void* src2 = nullptr;
    int SH2 = 0, SW2 = 0, SC2 = 0, s2 = 1, K1 = 0;
    // stem only: `src` is the canonical NCHW f32 input with SC = Cin channels (the layout
    // conversion of the graph input is folded into the stem's halo load)
    int src_nchw_f32 = 0;
    // stem_row only: fused 3x3 / stride-2 / pad-1 max pool after the epilogue; `out` is then the
    // pooled tensor [N, OH/2, OW/2, ldo] (OH, OW = the conv's output grid, both even)
    int pool3s2 = 0;
    float pool_min_init = -INFINITY;  // the MaxPool2d min_init (0 after the relu-into-pool pass)
    // autotune override (SOL_MODOPT_TILE_N): 0 = heuristic; 64 / 128 / 256 = that N-tile width;
    // 65 = 64-wide with the weights resident in shared memory (RESB)
    int tile_n = 0;
};

// Launches on `stream`. Throws on unsupported shapes (no fallback path exists).
void igemm_launch(const IgemmArgs& a, cudaStream_t stream);
// whether igemm_launch can emit BN statistics (IgemmArgs::stat_partial) for this conv
bool igemm_stats_supported(const IgemmArgs& a);
// whether igemm_launch can store a sub-pixel dgrad class in place (IgemmArgs::sub_*)
bool igemm_sub_supported(const IgemmArgs& a);
int igemm_stat_blocks(const IgemmArgs& a);  // one per (CTA, lane quarter): 4 x SM count

// Few-channel stem convolution (stem.cu): bf16, input pixels of 8 channels holding Cin <= 4,
// Cout = 64, kw <= 8, K packed (kh, kw in 8 slots, c in 4) to stem_kpad(kh) (pack_stem_weight).
bool stem_supported(const IgemmArgs& a);
void stem_launch(const IgemmArgs& a, cudaStream_t stream);
int stem_kpad(int kh);
// Stride-2 stem from the NCHW f32 input without an im2col matrix (stem_row.cu): the MMA reads
// overlapping 64-byte windows of compact bf16 input rows (K-major SWIZZLE_NONE operand).
bool stem_row_supported(const IgemmArgs& a);
void stem_row_launch(const IgemmArgs& a, cudaStream_t stream);
// Stem weight gradient (same halo / im2col machinery): dW canonical [Cout=64][Cin][kh][kw] f32 from
// dy [N, OH, OW, 64] and x (a.src); `ws` holds stem_wgrad_workspace_floats() partial sums.
bool stem_wgrad_supported(const IgemmArgs& a, int ld_dy);
size_t stem_wgrad_workspace_floats();
void stem_wgrad_launch(const IgemmArgs& a, const void* dy, int Cin, float* ws, float* dw, cudaStream_t stream);

// Row-padded halo-tile path for stride-1 "same" k x k convolutions with <= 48 KB halos (halo.cu).
bool halo_supported(const IgemmArgs& a);
void halo_launch(const IgemmArgs& a, cudaStream_t stream);

// Tile configuration chosen for a GEMM (exposed for the roofline/bench bookkeeping).
int igemm_block_n(int nout);

// wgrad: dW[Cout][K_pad] (f32) = dy^T x im2col(x), both operands MN-major.
struct WgradArgs {
    int dtype = DT_BF16;
    const void* dy = nullptr;  // [N, OH, OW, Cout] (Cout padded/strided by ld_dy)
    const void* x = nullptr;   // [N, SH, SW, SC]
    float* dw = nullptr;       // [Cout][kh*kw*SC] f32 (packed order kh, kw, ci)
    int N = 0, SH = 0, SW = 0, SC = 0, OH = 0, OW = 0, Cout = 0;
    int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
    int ld_dy = 0;
    float* workspace = nullptr;  // split-K partials (size from wgrad_workspace_floats)
    // optional canonical output dW[co][ci][kh][kw] (ci < canon_cin): the split-K reduction writes
    // it directly (one pass instead of reduce + unpack); without splits dw is unpacked into it
    float* dw_canon = nullptr;
    int canon_cin = 0;
};
void wgrad_launch(const WgradArgs& a, cudaStream_t stream);
// halo weight gradient (wgrad_halo.cu): stride-1 3x3, bf16; 64 -> 64, 128 -> 128 and >= 256-channel
// shapes. Work = (tap group, ci slice, co slice) x pixel units; every CTA writes one compact partial
// [co slice][its tiles x 128] of its group's dW entries (wh_group_of maps an entry to its group and
// offset).
struct WhPlan {
    int Wp, K, R, HX;          // row pitch (W + 2), pixel rows per unit (64 / 128), output rows, x rows
    int pairs;                 // 64 input channels: five M tiles of two taps
    int ncx, ncd, N;           // x / dy 64-channel blocks per unit, co slice width
    int n_ci, n_co, TT;        // ci slices (128), co slices, taps per CTA
    int tap_groups, groups;
    int cb_bytes, dy_blk, stage_bytes;
    int row_blocks, units;
};
WhPlan wgrad_halo_plan(const WgradArgs& a);
// columns of one CTA's partial (its tiles x 128) and the partial's size in floats (co slice rows)
__host__ __device__ inline int wh_cols(const WhPlan& g) { return (g.pairs ? 5 : g.TT) * 128; }
__host__ __device__ inline int64_t wh_partial_floats(const WhPlan& g) { return static_cast<int64_t>(g.N) * wh_cols(g); }
// group of dW entry (co, packed column = tap * sc + ci) and its offset inside a partial
__host__ __device__ inline int wh_group_of(const WhPlan& g, int sc, int co, int col, int64_t* off) {
    if (g.pairs) {
        *off = static_cast<int64_t>(co) * wh_cols(g) + col;
        return 0;
    }
    const int tap = col / sc, ci = col - tap * sc;
    const int tg = tap / g.TT, cs = ci / 128, os = co / g.N;
    *off = static_cast<int64_t>(co - os * g.N) * wh_cols(g) + (tap - tg * g.TT) * 128 + (ci - cs * 128);
    return (tg * g.n_ci + cs) * g.n_co + os;
}
bool wgrad_halo_supported(const WgradArgs& a);
int wgrad_halo_splits(const WgradArgs& a, int* splits_per_group = nullptr);
void wgrad_halo_launch(const WgradArgs& a, cudaStream_t stream);
size_t wgrad_workspace_floats(const WgradArgs& a);

}  // namespace solb200
