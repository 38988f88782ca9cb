// Weight (re)packing between the reference's canonical parameter layouts and the K-major
// layouts the tcgen05 kernels read. Canonical conv weights are [Cout][Cin][kh][kw] f32
// (tests/builders.hpp:65-80; reference.cpp:138-161); Linear weights [Cout][Cin].
#include "pack.cuh"

namespace solb200 {
namespace {

// packed[co][(kh*KW + kw)*ld + ci] = w[co][ci][kh][kw]; zero for ci >= Cin and k >= K
template <typename T>
__global__ void pack_fwd_kernel(const float* __restrict__ w, T* __restrict__ p, int Cout, int Cin, int KH, int KW,
                                int ld, int kpad) {
    const int64_t total = static_cast<int64_t>(Cout) * kpad;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int co = static_cast<int>(i / kpad);
        const int k = static_cast<int>(i - static_cast<int64_t>(co) * kpad);
        const int tap = k / ld, ci = k - tap * ld;
        float v = 0.f;
        if (tap < KH * KW && ci < Cin) {
            const int kh = tap / KW, kw = tap - kh * KW;
            v = w[((static_cast<int64_t>(co) * Cin + ci) * KH + kh) * KW + kw];
        }
        p[i] = from_f32<T>(v);
    }
}

// packed_t[ci][(kh*KW + kw)*ld_o + co] = w[co][ci][kh][kw]  (dgrad B operand); with flip the
// taps are mirrored, w[co][ci][KH-1-kh][KW-1-kw], so a stride-1 dgrad runs as a forward conv of dy
template <typename T>
__global__ void pack_t_kernel(const float* __restrict__ w, T* __restrict__ p, int Cout, int Cin, int KH, int KW,
                              int ld_o, int kpad, bool flip) {
    const int64_t total = static_cast<int64_t>(Cin) * kpad;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int ci = static_cast<int>(i / kpad);
        const int k = static_cast<int>(i - static_cast<int64_t>(ci) * kpad);
        const int tap = k / ld_o, co = k - tap * ld_o;
        float v = 0.f;
        if (tap < KH * KW && co < Cout) {
            int kh = tap / KW, kw = tap - kh * KW;
            if (flip) {
                kh = KH - 1 - kh;
                kw = KW - 1 - kw;
            }
            v = w[((static_cast<int64_t>(co) * Cin + ci) * KH + kh) * KW + kw];
        }
        p[i] = from_f32<T>(v);
    }
}

__global__ void pack_stem_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ p, int Cout, int Cin,
                                 int KH, int KW, int kpad) {
    const int total = Cout * kpad;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int co = i / kpad, k = i - co * kpad;
        const int kh = k / 32, kw = (k % 32) / 4, c = k % 4;
        float v = 0.f;
        if (kh < KH && kw < KW && c < Cin) v = w[((static_cast<int64_t>(co) * Cin + c) * KH + kh) * KW + kw];
        p[i] = __float2bfloat16_rn(v);
    }
}

template <typename T>
__global__ void pack_class_kernel(const float* __restrict__ w, T* __restrict__ p, int Cout, int Cin, int KH, int KW,
                                  int ld_o, int kpad, int TW, int ntap, int kh0, int kw0, int sh, int sw) {
    const int64_t total = static_cast<int64_t>(Cin) * kpad;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int ci = static_cast<int>(i / kpad);
        const int k = static_cast<int>(i - static_cast<int64_t>(ci) * kpad);
        const int tap = k / ld_o, co = k - tap * ld_o;
        float v = 0.f;
        if (tap < ntap && co < Cout) {
            const int th = tap / TW, tw = tap - th * TW;
            const int kh = kh0 - sh * th, kw = kw0 - sw * tw;  // kh0 = a + ph - sh * off_h
            if (kh >= 0 && kh < KH && kw >= 0 && kw < KW)
                v = w[((static_cast<int64_t>(co) * Cin + ci) * KH + kh) * KW + kw];
        }
        p[i] = from_f32<T>(v);
    }
}

__global__ void pack_dual_kernel(const DualFold f, __nv_bfloat16* __restrict__ p, float* __restrict__ bias) {
    const int K = f.C1 + f.C2;
    const int64_t total = static_cast<int64_t>(f.Cout) * K;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int co = static_cast<int>(i / K), k = static_cast<int>(i - static_cast<int64_t>(co) * K);
        float v;
        if (k < f.C1) {
            const double sc = static_cast<double>(f.g1[co]) / sqrt(static_cast<double>(f.v1[co]) + f.eps1);
            v = static_cast<float>(f.w1[static_cast<int64_t>(co) * f.C1 + k] * sc);
        } else {
            const double sc = static_cast<double>(f.g2[co]) / sqrt(static_cast<double>(f.v2[co]) + f.eps2);
            v = static_cast<float>(f.w2[static_cast<int64_t>(co) * f.C2 + (k - f.C1)] * sc);
        }
        p[i] = __float2bfloat16_rn(v);
        if (k == 0) {
            const double s1 = static_cast<double>(f.g1[co]) / sqrt(static_cast<double>(f.v1[co]) + f.eps1);
            const double s2 = static_cast<double>(f.g2[co]) / sqrt(static_cast<double>(f.v2[co]) + f.eps2);
            const double t1 = ((f.cb1 ? f.cb1[co] : 0.f) - static_cast<double>(f.m1[co])) * s1 + f.b1[co];
            const double t2 = ((f.cb2 ? f.cb2[co] : 0.f) - static_cast<double>(f.m2[co])) * s2 + f.b2[co];
            bias[co] = static_cast<float>(t1 + t2);
        }
    }
}

// canonical dw[co][ci][kh][kw] = packed[co][(kh*KW + kw)*ld + ci]
__global__ void unpack_grad_kernel(const float* __restrict__ p, float* __restrict__ w, int Cout, int Cin, int KH,
                                   int KW, int ld) {
    const int64_t total = static_cast<int64_t>(Cout) * Cin * KH * KW;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int kw = static_cast<int>(i % KW);
        const int kh = static_cast<int>((i / KW) % KH);
        const int ci = static_cast<int>((i / (KW * KH)) % Cin);
        const int co = static_cast<int>(i / (static_cast<int64_t>(KW) * KH * Cin));
        w[i] = p[static_cast<int64_t>(co) * KH * KW * ld + (kh * KW + kw) * ld + ci];
    }
}

// depthwise [C][1][kh][kw] -> [kh][kw][C]
__global__ void pack_dw_kernel(const float* __restrict__ w, float* __restrict__ p, int C, int KH, int KW) {
    const int total = C * KH * KW;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        const int c = i % C, tap = i / C;
        p[i] = w[c * KH * KW + tap];
    }
}

unsigned grid_of(int64_t n) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 4096)));
}

}  // namespace

void pack_conv_weight(const float* w, void* packed, int dtype, int Cout, int Cin, int kh, int kw, int ld, int kpad,
                      cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(Cout) * kpad;
    if (dtype == DT_BF16)
        pack_fwd_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, kh, kw, ld, kpad);
    else
        pack_fwd_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<float*>(packed), Cout, Cin, kh, kw, ld, kpad);
    SOL_CUDA(cudaGetLastError());
}

void pack_conv_weight_t(const float* w, void* packed, int dtype, int Cout, int Cin, int kh, int kw, int ld_o,
                        int kpad, cudaStream_t s, bool flip) {
    const int64_t n = static_cast<int64_t>(Cin) * kpad;
    if (dtype == DT_BF16)
        pack_t_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, kh, kw, ld_o, kpad,
                                                 flip);
    else
        pack_t_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<float*>(packed), Cout, Cin, kh, kw, ld_o, kpad, flip);
    SOL_CUDA(cudaGetLastError());
}

void pack_stem_weight(const float* w, void* packed, int Cout, int Cin, int kh, int kw, int kpad, cudaStream_t s) {
    pack_stem_kernel<<<grid_of(static_cast<int64_t>(Cout) * kpad), 256, 0, s>>>(
        w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, kh, kw, kpad);
    SOL_CUDA(cudaGetLastError());
}

void pack_dgrad_class(const float* w, void* packed, int dtype, int Cout, int Cin, int KH, int KW, int ld_o, int kpad,
                      int TH, int TW, int kh0, int kw0, int sh, int sw, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(Cin) * kpad;
    if (dtype == DT_BF16)
        pack_class_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, KH, KW, ld_o,
                                                     kpad, TW, TH * TW, kh0, kw0, sh, sw);
    else
        pack_class_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<float*>(packed), Cout, Cin, KH, KW, ld_o, kpad,
                                                     TW, TH * TW, kh0, kw0, sh, sw);
    SOL_CUDA(cudaGetLastError());
}

void pack_dual_weight(const DualFold& f, void* packed, float* bias, cudaStream_t s) {
    pack_dual_kernel<<<grid_of(static_cast<int64_t>(f.Cout) * (f.C1 + f.C2)), 256, 0, s>>>(
        f, static_cast<__nv_bfloat16*>(packed), bias);
    SOL_CUDA(cudaGetLastError());
}

void unpack_conv_grad(const float* packed, float* w, int Cout, int Cin, int kh, int kw, int ld, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(Cout) * Cin * kh * kw;
    unpack_grad_kernel<<<grid_of(n), 256, 0, s>>>(packed, w, Cout, Cin, kh, kw, ld);
    SOL_CUDA(cudaGetLastError());
}

void pack_dw_weight(const float* w, float* packed, int C, int kh, int kw, cudaStream_t s) {
    pack_dw_kernel<<<grid_of(static_cast<int64_t>(C) * kh * kw), 256, 0, s>>>(w, packed, C, kh, kw);
    SOL_CUDA(cudaGetLastError());
}

}  // namespace solb200
