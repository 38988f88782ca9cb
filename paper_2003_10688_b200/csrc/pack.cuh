#pragma once

#include <algorithm>

#include "common.cuh"

namespace solb200 {

void pack_conv_weight(const float* w, void* packed, int dtype, int Cout, int Cin, int kh, int kw, int ld, int kpad,
                      cudaStream_t s);
// stem K order: packed[co][kh*32 + kw*4 + c] (kw < 8 slots, c < 4), zero elsewhere (stem.cu)
void pack_stem_weight(const float* w, void* packed, int Cout, int Cin, int kh, int kw, int kpad, cudaStream_t s);
// Strided dgrad, parity class (a, b): packed[ci][(th, tw)][co] = w[co][ci][kh][kw] with
// kh = a + ph - sh * (off_h + th), kw = b + pw - sw * (off_w + tw) (sub-pixel decomposition).
void pack_dgrad_class(const float* w, void* packed, int dtype, int Cout, int Cin, int KH, int KW, int ld_o, int kpad,
                      int TH, int TW, int kh0, int kw0, int sh, int sw, cudaStream_t s);
// Dual-GEMM bottleneck fusion (inference): packed[co][0:C1] = W1[co][:] * s1[co],
// packed[co][C1:C1+C2] = W2[co][:] * s2[co] (bf16) with s = gamma / sqrt(var + eps) of each branch's
// BatchNorm, and bias[co] = sum over branches of (conv_bias - mean) * s + beta (f32).
struct DualFold {
    const float *w1, *cb1, *g1, *b1, *m1, *v1;
    const float *w2, *cb2, *g2, *b2, *m2, *v2;
    float eps1, eps2;
    int Cout, C1, C2;
};
void pack_dual_weight(const DualFold& f, void* packed, float* bias, cudaStream_t s);
void pack_conv_weight_t(const float* w, void* packed, int dtype, int Cout, int Cin, int kh, int kw, int ld_o,
                        int kpad, cudaStream_t s, bool flip = false);
void unpack_conv_grad(const float* packed, float* w, int Cout, int Cin, int kh, int kw, int ld, cudaStream_t s);
void pack_dw_weight(const float* w, float* packed, int C, int kh, int kw, cudaStream_t s);
// Batched packing: between begin and end, pack_conv_weight / _t / pack_stem_weight /
// pack_dgrad_class record jobs instead of launching; end() issues them as one launch on `s`.
void pack_batch_begin();
void pack_batch_end(cudaStream_t s);

}  // namespace solb200
