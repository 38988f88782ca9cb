// Fused DFP (depth-first parallelism) kernels for sm_100a.
//
// The reference lowers each fused unit to a KernelIR loop nest whose body is an expression tree,
// with producers inlined depth-first (proj/src/dfp_lower.cpp:392-796) and interprets it per
// output element (proj/src/dfp_interp.cpp:40-164). Here a unit compiles (module.cpp) to one of a
// few hand-written kernel families over NHWC tensors, each parameterised by small per-channel
// "programs": straight-line, vectorised (16 bytes = 8 bf16 / 4 f32 channels per thread) register
// code evaluated at a pixel. The loop nest becomes the grid; the expression tree becomes the
// program; reductions (pool windows, global average, per-channel statistics) are explicit.
#pragma once

#include "common.cuh"

namespace solb200 {

constexpr int DFP_MAX_INS = 24;
constexpr int DFP_MAX_IN = 8;
constexpr int DFP_MAX_P = 16;
constexpr int DFP_MAX_CAT = 40;

enum PwOp : uint8_t {
    PW_LD = 0,     // r[dst] = input[a] at the current pixel
    PW_AFF,        // r[dst] = r[dst] * P[arg][c] + P[arg+1][c]
    PW_AXPBY,      // r[dst] = r[dst] * P[arg][c] + r[b] * P[arg+1][c] + P[arg+2][c]
    PW_RELU,       // r[dst] = max(r[dst], 0)
    PW_RELU6,      // r[dst] = min(max(r[dst], 0), 6)
    PW_ADD,        // r[dst] = r[a] + r[b]
    PW_MASK,       // r[dst] = r[a] * (r[b] > 0)
    PW_MASK6,      // r[dst] = r[a] * (r[b] > 0 && r[b] < 6)
    PW_MOV,        // r[dst] = r[a]
    PW_SCALE,      // r[dst] = r[dst] * imm
    PW_PARAM,      // r[dst] = P[arg][c]
    PW_BN,         // r[dst] = ((r[dst] - P[arg][c]) - P[arg+1][c]) * P[arg+2][c] + P[arg+3][c]
                   //   (BatchNorm apply; the mean is split hi+lo so x - mean keeps f64-grade accuracy)
};

struct PwInstr {
    uint8_t op = 0, dst = 0, a = 0, b = 0;
    int16_t arg = 0;
    int16_t pad = 0;
    float imm = 0.f;
};

struct Program {
    int n = 0;
    PwInstr ins[DFP_MAX_INS];
};

enum InKind : int {
    IN_PIX = 0,    // NHWC tensor on the program's grid: ptr + pixel*ld + coff + c
    IN_NC = 1,     // [N, C] tensor broadcast over pixels: ptr + n*ld + c
    IN_CAT = 2,    // concat over channel segments (cat_* fields)
    IN_FLAT = 3,   // canonical-order flattened [N, C*HW] read at pixel p, channel c (FlattenBack)
};

enum Family : int {
    FAM_POINTWISE = 0,  // out[p, c] = post(p, c)
    FAM_POOL,           // out[o, c] = post(reduce_{window(o)} pre(i, c))          (Max/AvgPool2d)
    FAM_GAP,            // out[n, c] = post(mean_{h,w} pre((n,h,w), c))             (GlobalAvgPool)
    FAM_DWCONV,         // out[o, c] = post(sum_{window} pre(i, c) * w[kh,kw,c] (+b)) (depthwise Conv2d)
    FAM_CHAN_REDUCE,    // S1[c] = sum_p pre.r0, S2[c] = sum_p pre.r0 * pre.r1      (BN statistics / grads)
    FAM_MAXPOOL_BACK,   // dx[i, c] = post(sum_{o: argmax(o)==i} pre(o, c))         (MaxPool2dBack)
    FAM_AVGPOOL_BACK,   // dx[i, c] = post(sum_{o: i in window(o)} pre(o, c) / cnt(o))
};

struct DfpArgs {
    int family = FAM_POINTWISE;
    int dtype = DT_BF16;
    // source grid (where `pre` runs) and output grid (where `post` runs); NHWC
    int N = 0, H = 1, W = 1, C = 0;
    int OH = 1, OW = 1;
    int kh = 1, kw = 1, sh = 1, sw = 1, ph = 0, pw = 0;
    float min_init = 0.f;
    int count_padding = 0;
    // inputs
    int n_in = 0;
    const void* in[DFP_MAX_IN] = {};
    int in_kind[DFP_MAX_IN] = {};
    int in_ld[DFP_MAX_IN] = {};
    int in_coff[DFP_MAX_IN] = {};
    int in_f32[DFP_MAX_IN] = {};   // input stored as f32 even in a bf16 plan
    int in_hw[DFP_MAX_IN] = {};    // IN_FLAT: H*W of the unflattened tensor
    int n_cat = 0;
    const void* cat_ptr[DFP_MAX_CAT] = {};
    int cat_off[DFP_MAX_CAT + 1] = {};
    // per-channel f32 parameter arrays
    const float* P[DFP_MAX_P] = {};
    // extra operands
    const float* dw_w = nullptr;   // FAM_DWCONV: [kh][kw][C] f32
    const float* dw_b = nullptr;
    int pool_x = -1;               // FAM_MAXPOOL_BACK: input slot holding the forward pool input
    int pool_max = 1;              // FAM_POOL: 1 = max, 0 = average
    Program pre, post;
    // outputs
    void* out = nullptr;
    int out_ld = 0, out_coff = 0;
    int out_f32 = 0;               // output stored as f32 even in a bf16 plan
    double* partial = nullptr;     // FAM_CHAN_REDUCE: [C][blocks][2] (f64, channel-major)
    uint8_t* argmax = nullptr;     // FAM_MAXPOOL_BACK scratch: [windows][C] first-max tap (255 = none)
    void* out2 = nullptr;          // straight-line chains: second output act2(value) (sibling ReLU unit)
    int act2 = 0;
    int reduce_blocks = 0;
};

void dfp_launch(const DfpArgs& a, cudaStream_t s);
int dfp_reduce_blocks(int64_t pixels, int C, int dtype);  // partial blocks used by FAM_CHAN_REDUCE
struct ReduceGeo {
    int blocks;  // pixel blocks (the partials' block dimension)
    int cvb;     // channel vectors per block (grid.y = ceil(C / V / cvb))
};
ReduceGeo reduce_geo(int64_t pixels, int C, int V);

// Small fixed-function kernels (rows of [N, C], BN finalisation, SGD, layout conversion).
void softmax_rows(int dtype, const void* x, void* y, int rows, int cols, int ld, cudaStream_t s);
// loss = -sum(t * log(p)) / rows  (reference.cpp CrossEntropyLoss); writes one f32
void ce_loss(int dtype, const void* p, const void* t, float* loss, int rows, int cols, int ld, cudaStream_t s);
// dx = (p - t) / rows (SoftmaxCeBack) or -t / (p * rows) (CeBack)
void ce_back(int dtype, int fused_softmax, const void* p, const void* t, void* dx, int rows, int cols, int ld,
             cudaStream_t s);
// dx = y * (delta - sum_c delta*y)  (SoftmaxBack)
void softmax_back(int dtype, const void* delta, const void* y, void* dx, int rows, int cols, int ld, cudaStream_t s);

// Per-channel finalisation of FAM_CHAN_REDUCE partials (in f64).
enum FinalizeMode : int {
    FIN_BN_STATS = 0,   // mean/var from shifted sums -> stats[2C] = (mean, rstd),
                        // coef[4C] = (mean_hi, mean_lo, gamma*rstd, beta) for PW_BN; optional running update
    FIN_SUMS = 1,       // out0[c] = S1, out1[c] = S2 (f32)
    FIN_BN_BACK = 2,    // dbeta = S1, dgamma = S2 (over xhat); coef[3C] for dx = dy*A + x*B + Cc
    FIN_BN_BACK4 = 3,   // from bn_back_reduce's 4 sums: x statistics (mean, rstd) and the BN backward
                        // sums in one pass; out0 = dbeta, out1 = dgamma, coef[3C] (A, B, Cc) and
                        // xhat[3C] = (mean_hi, mean_lo, rstd) for bn_back_apply
};
struct FinalizeArgs {
    int mode = FIN_BN_STATS;
    int C = 0;
    int Cstride = 0;               // channel stride of the partial sums (>= C; 0 = C)
    int blocks = 0;
    const double* partial = nullptr;
    double count = 1.0;
    float eps = 1e-5f;
    float momentum = 0.1f;
    const float* shift = nullptr;  // per-channel shift used by the stats reduction (FIN_BN_STATS)
    const float* gamma = nullptr;
    const float* beta = nullptr;
    const float* stats = nullptr;  // (mean, rstd) for FIN_BN_BACK
    float* running_mean = nullptr;
    float* running_var = nullptr;
    float* stats_out = nullptr;
    float* coef = nullptr;
    float* out0 = nullptr;
    float* out1 = nullptr;
    float* xhat = nullptr;         // FIN_BN_BACK4
    const void* shift_x = nullptr; // FIN_BN_BACK4 with shift == nullptr: the shift is x's first pixel
    int shift_dtype = DT_BF16;
};
void dfp_finalize(const FinalizeArgs& a, cudaStream_t s);
// A FAM_CHAN_REDUCE launch followed by its finalisation: one cooperative kernel when the reduction
// has a fast path and its grid is co-resident, else the two launches.
void dfp_reduce_finalize(const DfpArgs& a, const FinalizeArgs& f, cudaStream_t s);

// BatchNorm backward in two HBM passes (training; autodiff BNBackX/Gamma/Beta,
// dfp_lower.cpp:709-753, 806-851): one reduction over (dy, x) producing, per channel and block,
// [sum dy, sum dy*(x - shift), sum (x - shift), sum (x - shift)^2] (f64 partials [blocks][C][4]),
// then (after FIN_BN_BACK4) dx = A*dy + B*xhat + Cc with xhat = ((x - mean_hi) - mean_lo) * rstd.
// Returns 0 (reduction only), 1 (+ the finalisation `fin`, fused in one cooperative launch) or
// 2 (+ also the BatchNormBackX apply into `apply_out`, over each block's own rows, same launch).
int bn_back_reduce(int dtype, const void* dy, const void* x, int C, int64_t pixels, const float* shift,
                   double* partial, int blocks, cudaStream_t s, const FinalizeArgs* fin = nullptr,
                   void* apply_out = nullptr);
void bn_back_apply(int dtype, const void* dy, const void* x, int C, int64_t pixels, const float* coef,
                   const float* xhat, void* dx, cudaStream_t s);

// BN inference coefficients for PW_BN: coef[4C] = (mean, 0, gamma/sqrt(var+eps), beta).
void bn_infer_coef(const float* gamma, const float* beta, const float* mean, const float* var, float eps,
                   float* coef, int C, cudaStream_t s);
// Shift vector for shifted-sum statistics: shift[c] = x[0, c] (first pixel).
void bn_shift(int dtype, const void* x, int ld, int C, float* shift, cudaStream_t s);

// w -= lr * g over n f32 elements (SgdUpdate, reference.cpp:580-584); optional bf16 mirror.
// lr_dev (optional): the learning rate read from device memory at run time (plan_set_lr), else lr
void sgd_update(float* w, const float* g, int64_t n, float lr, void* mirror_bf16, cudaStream_t s,
                const float* lr_dev = nullptr);
// One launch updating many parameters: w_i -= lr * g_i for i < count (multi-tensor SGD).
constexpr int SGD_MULTI_MAX = 512;
struct SgdMultiArgs {
    int count = 0;
    float lr = 0.f;
    const float* lr_dev = nullptr;  // when set, the learning rate is read from device memory
    float* w[SGD_MULTI_MAX];
    const float* g[SGD_MULTI_MAX];
    int64_t n[SGD_MULTI_MAX];
    int block0[SGD_MULTI_MAX + 1];  // first block of each tensor (prefix over ceil(n / 1024))
};
void sgd_multi(const SgdMultiArgs& a, cudaStream_t s);

// Strided dgrad: dx[n, h, w, :] = cls[(h % sh) * sw + w % sw][n, h / sh, w / sw, :] (zero where the
// class pointer is null); class c has grid ch[c] x cw[c], all rows `ld` elements.
struct InterleaveArgs {
    const void* cls[16] = {};
    int ch[16] = {}, cw[16] = {};
    int sh = 1, sw = 1, N = 0, H = 0, W = 0, ld = 0;
    void* out = nullptr;
};
void subpixel_interleave(int dtype, const InterleaveArgs& a, cudaStream_t s);

// Layout/dtype conversion between canonical NCHW f32 (host-facing) and NHWC plan storage.
// c_pad >= C channels; padded channels are zero.
void nchw_to_nhwc(const float* src, void* dst, int dtype, int N, int C, int H, int W, int c_pad,
                  cudaStream_t s);
void nhwc_to_nchw(const void* src, float* dst, int dtype, int N, int C, int H, int W, int ld,
                  cudaStream_t s);
// Flatten in canonical (reference) order: out[n, c*H*W + h*W + w] = x[n, h, w, c]
// (dfp_lower.cpp:1098-1112; reference.cpp:245-254) and its inverse (FlattenBack).
void flatten_nhwc(int dtype, const void* x, void* y, int N, int C, int H, int W, int inverse,
                  cudaStream_t s);
// dtype cast (f32 <-> bf16) of n elements.
void cast_copy(const void* src, int src_dtype, void* dst, int dst_dtype, int64_t n, cudaStream_t s);

}  // namespace solb200
