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

// ---- batched packing: every pack of a plan run in ONE launch (module prepack, runtime.cu) ----
enum PackKind { PK_FWD = 0, PK_T = 1, PK_STEM = 2, PK_CLASS = 3 };
struct PackJob {
    int kind, dtype;
    const float* w;
    void* p;
    int Cout, Cin, KH, KW, ld, kpad;
    int TW, ntap, kh0, kw0, sh, sw, flip;
    int64_t total;
};
constexpr int PACK_BATCH_MAX = 128;
struct PackBatchArgs {
    int count;
    int block0[PACK_BATCH_MAX + 1];  // first block of each job (1024 elements per block)
    PackJob job[PACK_BATCH_MAX];
};

__device__ __forceinline__ float pack_value(const PackJob& j, int64_t i) {
    switch (j.kind) {
        case PK_FWD: {
            const int co = static_cast<int>(i / j.kpad);
            const int k = static_cast<int>(i - static_cast<int64_t>(co) * j.kpad);
            const int tap = k / j.ld, ci = k - tap * j.ld;
            if (tap >= j.KH * j.KW || ci >= j.Cin) return 0.f;
            const int kh = tap / j.KW, kw = tap - kh * j.KW;
            return j.w[((static_cast<int64_t>(co) * j.Cin + ci) * j.KH + kh) * j.KW + kw];
        }
        case PK_T: {
            const int ci = static_cast<int>(i / j.kpad);
            const int k = static_cast<int>(i - static_cast<int64_t>(ci) * j.kpad);
            const int tap = k / j.ld, co = k - tap * j.ld;
            if (tap >= j.KH * j.KW || co >= j.Cout) return 0.f;
            int kh = tap / j.KW, kw = tap - kh * j.KW;
            if (j.flip) {
                kh = j.KH - 1 - kh;
                kw = j.KW - 1 - kw;
            }
            return j.w[((static_cast<int64_t>(co) * j.Cin + ci) * j.KH + kh) * j.KW + kw];
        }
        case PK_STEM: {
            const int co = static_cast<int>(i / j.kpad), k = static_cast<int>(i - static_cast<int64_t>(co) * j.kpad);
            const int kh = k / 32, kw = (k % 32) / 4, c = k % 4;
            if (kh >= j.KH || kw >= j.KW || c >= j.Cin) return 0.f;
            return j.w[((static_cast<int64_t>(co) * j.Cin + c) * j.KH + kh) * j.KW + kw];
        }
        default: {  // PK_CLASS
            const int ci = static_cast<int>(i / j.kpad);
            const int k = static_cast<int>(i - static_cast<int64_t>(ci) * j.kpad);
            const int tap = k / j.ld, co = k - tap * j.ld;
            if (tap >= j.ntap || co >= j.Cout) return 0.f;
            const int th = tap / j.TW, tw = tap - th * j.TW;
            const int kh = j.kh0 - j.sh * th, kw = j.kw0 - j.sw * tw;
            if (kh < 0 || kh >= j.KH || kw < 0 || kw >= j.KW) return 0.f;
            return j.w[((static_cast<int64_t>(co) * j.Cin + ci) * j.KH + kh) * j.KW + kw];
        }
    }
}

__global__ void __launch_bounds__(256) pack_batch_kernel(const __grid_constant__ PackBatchArgs a) {
    int lo = 0, hi = a.count;
    while (hi - lo > 1) {
        const int mid = (lo + hi) / 2;
        if (a.block0[mid] <= static_cast<int>(blockIdx.x)) lo = mid;
        else hi = mid;
    }
    const PackJob& j = a.job[lo];
    const int64_t base = static_cast<int64_t>(blockIdx.x - a.block0[lo]) * 1024;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        const int64_t i = base + r * 256 + threadIdx.x;
        if (i >= j.total) break;
        const float v = pack_value(j, i);
        if (j.dtype == DT_BF16) static_cast<__nv_bfloat16*>(j.p)[i] = __float2bfloat16_rn(v);
        else static_cast<float*>(j.p)[i] = v;
    }
}

thread_local bool t_batching = false;
thread_local PackBatchArgs t_batch;

void batch_flush(cudaStream_t s) {
    if (t_batch.count == 0) return;
    int blocks = 0;
    for (int k = 0; k < t_batch.count; ++k) {
        t_batch.block0[k] = blocks;
        blocks += static_cast<int>(ceil_div(t_batch.job[k].total, static_cast<int64_t>(1024)));
    }
    t_batch.block0[t_batch.count] = blocks;
    pack_batch_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(t_batch);
    SOL_CUDA(cudaGetLastError());
    t_batch.count = 0;
}

// true: recorded into the open batch (flushed when full)
bool batch_add(const PackJob& j, cudaStream_t s) {
    if (!t_batching) return false;
    if (t_batch.count == PACK_BATCH_MAX) batch_flush(s);
    t_batch.job[t_batch.count++] = j;
    return true;
}

unsigned grid_of(int64_t n) {
    return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 4096)));
}

}  // namespace

void pack_conv_weight(const float* w, void* packed, int dtype, int Cout, int Cin, int kh, int kw, int ld, int kpad,
                      cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(Cout) * kpad;
    if (batch_add(PackJob{PK_FWD, dtype, w, packed, Cout, Cin, kh, kw, ld, kpad, 0, 0, 0, 0, 0, 0, 0, n}, s)) return;
    if (dtype == DT_BF16)
        pack_fwd_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, kh, kw, ld, kpad);
    else
        pack_fwd_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<float*>(packed), Cout, Cin, kh, kw, ld, kpad);
    SOL_CUDA(cudaGetLastError());
}

void pack_conv_weight_t(const float* w, void* packed, int dtype, int Cout, int Cin, int kh, int kw, int ld_o,
                        int kpad, cudaStream_t s, bool flip) {
    const int64_t n = static_cast<int64_t>(Cin) * kpad;
    if (batch_add(PackJob{PK_T, dtype, w, packed, Cout, Cin, kh, kw, ld_o, kpad, 0, 0, 0, 0, 0, 0, flip ? 1 : 0, n}, s))
        return;
    if (dtype == DT_BF16)
        pack_t_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, kh, kw, ld_o, kpad,
                                                 flip);
    else
        pack_t_kernel<<<grid_of(n), 256, 0, s>>>(w, static_cast<float*>(packed), Cout, Cin, kh, kw, ld_o, kpad, flip);
    SOL_CUDA(cudaGetLastError());
}

void pack_stem_weight(const float* w, void* packed, int Cout, int Cin, int kh, int kw, int kpad, cudaStream_t s) {
    if (batch_add(PackJob{PK_STEM, DT_BF16, w, packed, Cout, Cin, kh, kw, 0, kpad, 0, 0, 0, 0, 0, 0, 0,
                          static_cast<int64_t>(Cout) * kpad},
                  s))
        return;
    pack_stem_kernel<<<grid_of(static_cast<int64_t>(Cout) * kpad), 256, 0, s>>>(
        w, static_cast<__nv_bfloat16*>(packed), Cout, Cin, kh, kw, kpad);
    SOL_CUDA(cudaGetLastError());
}

void pack_dgrad_class(const float* w, void* packed, int dtype, int Cout, int Cin, int KH, int KW, int ld_o, int kpad,
                      int TH, int TW, int kh0, int kw0, int sh, int sw, cudaStream_t s) {
    const int64_t n = static_cast<int64_t>(Cin) * kpad;
    if (batch_add(PackJob{PK_CLASS, dtype, w, packed, Cout, Cin, KH, KW, ld_o, kpad, TW, TH * TW, kh0, kw0, sh, sw, 0, n},
                  s))
        return;
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

void pack_batch_begin() {
    t_batch.count = 0;
    t_batching = true;
}

void pack_batch_end(cudaStream_t s) {
    t_batching = false;
    batch_flush(s);
}

}  // namespace solb200
