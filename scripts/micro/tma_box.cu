// Micro-benchmark: TMA tiled-box load throughput for halo-shaped boxes (not part of the library).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_box tma_box.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void box_kernel(const __grid_constant__ CUtensorMap m, int loads, int bytes, int w0, int dims4, int nbuf) {
    extern __shared__ __align__(1024) uint8_t sm[];
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + nbuf * 32768);
    if (threadIdx.x != 0) return;
    for (int i = 0; i < nbuf; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    uint32_t ph = 0;
    for (int i = 0; i < loads; ++i) {
        const int b = i % nbuf;
        if (i >= nbuf) {
            const uint32_t par = ((i / nbuf) - 1) & 1;
            asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}\n" ::"r"(su32(&bar[b])), "r"(par));
        }
        asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(su32(&bar[b])), "r"(bytes));
        const int tile = blockIdx.x + i * gridDim.x;  // distinct 4-row blocks: DRAM-sourced
        const int img = (tile / 14) % 256, rb = tile % 14;
        if (dims4 == 2)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(su32(sm + b * 32768)), "l"(&m), "r"(-3), "r"(rb * 4 - 3), "r"(0), "r"(img), "r"(su32(&bar[b])) : "memory");
        else if (dims4)
            asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(su32(sm + b * 32768)), "l"(&m), "r"(0), "r"(w0), "r"(rb * 4), "r"(img), "r"(su32(&bar[b])) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(sm + b * 32768)), "l"(&m), "r"(0), "r"((img * 14 + rb) * 224), "r"(su32(&bar[b])) : "memory");
    }
    for (int i = loads - nbuf; i < loads; ++i) {
        const int b = i % nbuf;
        const uint32_t par = (i / nbuf) & 1;
        asm volatile("{\n.reg .pred P;\nW2: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}\n" ::"r"(su32(&bar[b])), "r"(par));
    }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* fn; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    Enc enc = (Enc)fn;
    const int N = 256, H = 56, W = 56, C = 64;
    void* x; cudaMalloc(&x, (size_t)N * 3 * 224 * 224 * 4 + (size_t)N * H * W * C * 2);
    cudaMemset(x, 0, (size_t)N * H * W * C * 2);
    cudaFuncSetAttribute(box_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg { const char* name; int dims4, bw, bh, w0, nbuf; };
    const int bwv = getenv("BW") ? atoi(getenv("BW")) : 40, bhv = getenv("BH") ? atoi(getenv("BH")) : 21;
    Cfg cfgs[] = {{"nchw f32", 2, bwv, bhv, 0, 5}, {"4d 64x58x4 w0=-1", 1, 58, 4, -1, 5}, {"4d 64x56x4 w0=0", 1, 56, 4, 0, 5}, {"4d 64x58x4 nbuf2", 1, 58, 4, -1, 2},
                  {"2d 64x224", 0, 0, 0, 0, 5}, {"4d 64x56x4 nbuf6", 1, 56, 4, 0, 6}, {"2d 64x224 nbuf2", 0, 0, 0, 0, 2}};
    for (auto& c : cfgs) {
        CUtensorMap m;
        if (c.dims4 == 2) {
            cuuint64_t dims[4] = {224, 224, 3, (cuuint64_t)N};
            cuuint64_t str[3] = {224 * 4, 224 * 224 * 4, 3ull * 224 * 224 * 4};
            cuuint32_t box[4] = {(cuuint32_t)c.bw, (cuuint32_t)c.bh, 3, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            CUresult rr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            fprintf(stderr, "encode %d box %u %u %u\n", (int)rr, box[0], box[1], box[2]);
        } else if (c.dims4) {
            cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
            cuuint64_t str[3] = {(cuuint64_t)C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
            cuuint32_t box[4] = {64, (cuuint32_t)c.bw, (cuuint32_t)c.bh, 1};
            cuuint32_t es[4] = {1, 1, 1, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        } else {
            cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)N * H * W};
            cuuint64_t str[1] = {(cuuint64_t)C * 2};
            cuuint32_t box[2] = {64, 224};
            cuuint32_t es[2] = {1, 1};
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, x, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        const int bytes = c.dims4 == 2 ? 4 * 3 * c.bw * c.bh : (c.dims4 ? 128 * c.bw * c.bh : 128 * 224);
        const int loads = 24;
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int r = 0; r < 1; ++r) {
            cudaEventRecord(e0);
            box_kernel<<<148, 32, 200 * 1024>>>(m, loads, bytes, c.w0, c.dims4, c.nbuf);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("%-22s %6.1f us  %6.2f TB/s  (err %s)\n", c.name, ms * 1e3, 148.0 * loads * bytes / (ms * 1e-3) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
