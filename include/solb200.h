/* solb200 — B200 (sm_100a) execution backend for SOL, C ABI.
 *
 * This is the drop-in boundary behind the reference's three device-backend interfaces
 * (reference = /root/reference/proj):
 *
 *   1. DFP module compile + launch, replacing
 *        sol::dfp::lower_group -> KernelIR        include/sol/dfp.hpp:43-45, src/dfp_lower.cpp:923-1139
 *        sol::dfp::interpret(KernelIR, inputs, output)   include/sol/dfp.hpp:53, src/dfp_interp.cpp:152-164
 *      -> sol_b200_module_create / sol_b200_module_run / sol_b200_launch
 *   2. the heavy-layer plugin sol::dnn::KernelProvider::execute   include/sol/dnn.hpp:44-64
 *      (Conv2d, Conv2dBackX, Conv2dBackW, Linear, LinearBackX, LinearBackW)
 *      -> the same module calls with a single heavy op (plus sol_b200_conv_* raw entry points)
 *   3. the device queue sol::rt::CommandQueue                    include/sol/runtime.hpp:95-145
 *        malloc_async / free_async / memcpy_h2d / memcpy_d2h / launch / barrier / synchronize / stats
 *      -> sol_b200_queue_* with the same VirtualPtr encoding (ref << 32 | offset,
 *         include/sol/runtime.hpp:28-55) and deferred first-error semantics (src/runtime.cpp:157-256)
 *
 * plus the execution-plan layer the reference declares but does not implement
 * (fe::DevicePlan / Step / run_device, include/sol/frontend.hpp:41-61, :148-150) and NCCL
 * gradient all-reduce for batch-sharded data parallelism.
 *
 * All functions are noexcept, return an int status (SOL_OK = 0) and record a message retrievable
 * with sol_b200_last_error(). No torch types cross this boundary: plain pointers and sizes.
 */
#ifndef SOLB200_H
#define SOLB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror rt::QueueError and sol/errors.hpp) ---------------------------- */
enum {
    SOL_OK = 0,
    SOL_E_USE_AFTER_FREE = 1,     /* rt::QueueError::UseAfterFree */
    SOL_E_UNKNOWN_REF = 2,        /* rt::QueueError::UnknownRef   */
    SOL_E_OUT_OF_BOUNDS = 3,      /* rt::QueueError::OutOfBounds  */
    SOL_E_INVALID_ARGUMENT = 10,  /* std::invalid_argument        */
    SOL_E_SHAPE_MISMATCH = 11,    /* ShapeMismatchError           */
    SOL_E_UNSUPPORTED = 12,       /* UnsupportedInGroupError / NoProviderError (no fallback) */
    SOL_E_OVERFLOW = 13,          /* ArithmeticOverflowError      */
    SOL_E_OUT_OF_REFS = 14,       /* OutOfRefsError               */
    SOL_E_NCCL = 50,
    SOL_E_CUDA = 100              /* + cudaError_t                */
};

/* ---- element types ------------------------------------------------------------------------ */
enum { SOL_DT_F32 = 0, SOL_DT_BF16 = 1 };

/* ---- op kinds: sol::OpKind order (include/sol/model.hpp:24-57) + extensions --------------- */
enum {
    SOL_OP_CONV2D = 0, SOL_OP_LINEAR, SOL_OP_RELU, SOL_OP_MAXPOOL2D, SOL_OP_AVGPOOL2D,
    SOL_OP_BATCHNORM2D, SOL_OP_ADD, SOL_OP_FLATTEN, SOL_OP_GLOBALAVGPOOL, SOL_OP_SOFTMAX,
    SOL_OP_CROSSENTROPYLOSS, SOL_OP_COPY,
    SOL_OP_RELUBACK, SOL_OP_MAXPOOL2DBACK, SOL_OP_AVGPOOL2DBACK, SOL_OP_GLOBALAVGPOOLBACK,
    SOL_OP_FLATTENBACK, SOL_OP_SOFTMAXBACK, SOL_OP_SOFTMAXCEBACK, SOL_OP_CEBACK,
    SOL_OP_BATCHNORMBACKX, SOL_OP_BATCHNORMBACKGAMMA, SOL_OP_BATCHNORMBACKBETA,
    SOL_OP_CONV2DBACKX, SOL_OP_CONV2DBACKW, SOL_OP_CONV2DBACKB, SOL_OP_LINEARBACKX,
    SOL_OP_LINEARBACKW, SOL_OP_LINEARBACKB, SOL_OP_SGDUPDATE,
    /* extensions beyond the reference IR */
    SOL_OP_CONCAT, SOL_OP_RELU6, SOL_OP_RELU6BACK, SOL_OP_CONCATBACK,
    SOL_OP_COUNT,
    /* plan-internal layout steps (fe::Step::Kind::Reorder, frontend.hpp:41-50) */
    SOL_OP_REORDER_IN = 100,  /* canonical f32 (NCHW / NC) -> NHWC plan storage */
    SOL_OP_REORDER_OUT = 101  /* NHWC plan storage -> canonical f32 */
};

/* sol::Attrs (include/sol/model.hpp:64-80) */
typedef struct {
    int64_t out_channels, out_features;
    int64_t kh, kw, sh, sw, ph, pw;
    int64_t groups;
    int32_t has_bias;
    float min_init;
    int32_t count_padding;
    float eps, momentum;
    int32_t training;
    float lr;
    int64_t offset; /* ConcatBack channel offset */
} sol_attrs;

#define SOL_MAX_OP_IN 40
/* One member op of an execution unit. Operand refs: r >= 0 is boundary binding r;
 * r < 0 is the output of member op (-r - 1). Params are binding indices. */
typedef struct {
    int32_t op;
    int32_t n_inputs;
    int32_t inputs[SOL_MAX_OP_IN];
    int32_t n_params;
    int32_t params[4];
    sol_attrs attrs;
    int64_t saved_dims[4]; /* LayerNode::saved_meta for gradient ops (canonical dims) */
    int32_t saved_rank;
    int64_t out_dims[4];   /* LayerNode::out_meta (canonical dims) */
    int32_t out_rank;
} sol_unit_op;

/* Boundary tensor binding (KernelIR::TensorBinding, include/sol/kernel_ir.hpp:99-105).
 * dims are canonical ([N,C,H,W] / [N,C] / [] / plain param extents); activations are stored
 * NHWC (ActLayout::ChannelsLast) with row stride `ld` elements (>= C); params are plain f32. */
typedef struct {
    int32_t is_param;   /* 0 activation (plan layout), 1 parameter (canonical f32), 2 activation in
                           the canonical host layout (NCHW f32), accepted by few-channel stem convs */
    int32_t dtype;
    int32_t rank;
    int64_t dims[4];
    int64_t ld;
} sol_binding;

typedef struct {
    int32_t kind; /* 0 = DfpGroup, 1 = DnnNode (dfp::ExecUnit::Kind) */
    int32_t n_ops;
    const sol_unit_op* ops;
    int32_t n_bindings; /* activations first, then params (KernelIR input order) */
    const sol_binding* bindings;
    sol_binding output;
    int32_t dtype;      /* plan compute dtype */
} sol_unit_desc;

typedef struct sol_b200_module_s* sol_b200_module_t;
typedef struct sol_b200_queue_s* sol_b200_queue_t;
typedef struct sol_b200_plan_s* sol_b200_plan_t;

typedef struct {
    char family[32];      /* kernel family selected for the unit */
    int32_t n_args;       /* bindings + 1 output */
    uint64_t scratch_bytes;
    int64_t launches;     /* kernels launched per run */
    double algo_bytes;    /* algorithmic HBM bytes per run (inputs + output, roofline) */
    double algo_flops;    /* algorithmic FLOPs per run (GEMMs) */
    int64_t launches_frozen; /* kernels per run once the plan is frozen (weight packing / BN folding
                                cached: inference) */
} sol_module_info;

/* rt::TransferStats (include/sol/runtime.hpp:72-82) */
typedef struct {
    uint64_t h2d_bytes, d2h_bytes, h2d_ops, d2h_ops, packed_transfers, launches;
    double device_time_us;
    /* allocator evidence (B200): pinned host slabs ever allocated for copy staging (a reusable
       pool: constant once warm) and device arena slabs (the arena grows stream-ordered instead of
       failing when full) */
    uint64_t pinned_slabs, device_slabs;
} sol_transfer_stats;

const char* sol_b200_last_error(void);
int sol_b200_device_count(int* count);
int sol_b200_set_device(int device);

/* ---- module compile / run ----------------------------------------------------------------- */
int sol_b200_module_create(const sol_unit_desc* desc, sol_b200_module_t* out);
int sol_b200_module_destroy(sol_b200_module_t m);
int sol_b200_module_info(sol_b200_module_t m, sol_module_info* info);
/* Sibling-unit fusion: a BatchNormBackX module additionally writes the outputs of the sibling
 * BatchNormBackGamma (mask bit 0) / BatchNormBackBeta (bit 1) units over the same (dy, x) from its
 * single reduction pass; their buffers follow the output in the run arguments (n_args grows).
 * Returns SOL_E_UNSUPPORTED for modules that cannot. */
int sol_b200_module_set_sibling_outputs(sol_b200_module_t m, int32_t mask);
/* Module options. SOL_MODOPT_UPDATE_BN_RUNNING_STATS (value 0/1, default 0): a training
 * BatchNorm2d unit also applies autodiff::update_bn_running_stats (autodiff.cpp:356-384: momentum,
 * unbiased variance) to its running_mean / running_var parameters, in place, from the batch
 * statistics it computes anyway. Off by default so module_run keeps interpret's purity contract;
 * training plans turn it on. SOL_E_UNSUPPORTED when the option does not apply to the module. */
/* SOL_MODOPT_TILE_N (conv / linear forward and the dual GEMM): the tcgen05 tile configuration,
 * chosen by autotune: 0 = built-in heuristic (incl. the halo kernel for 64-channel 3x3 convs),
 * 64 / 128 / 256 = N-tile width on the im2col / TMA path, 65 = 64-wide with resident weights. */
enum { SOL_MODOPT_UPDATE_BN_RUNNING_STATS = 1, SOL_MODOPT_TILE_N = 2 };
int sol_b200_module_set_option(sol_b200_module_t m, int32_t key, int32_t value);
/* Raw-pointer launch on a CUDA stream (cudaStream_t passed as void*): args = bindings in order,
 * then the output; scratch must hold info.scratch_bytes. `frozen_params` lets a module cache
 * parameter-derived constants (BN coefficients, packed weights) across runs. */
int sol_b200_module_run(sol_b200_module_t m, void* const* args, int32_t nargs, void* scratch,
                        void* stream, int32_t frozen_params);

/* ---- device queue (rt::CommandQueue) ------------------------------------------------------ */
int sol_b200_queue_create(int device, uint64_t arena_bytes, int32_t coalesce, sol_b200_queue_t* out);
int sol_b200_queue_destroy(sol_b200_queue_t q);
int sol_b200_malloc_async(sol_b200_queue_t q, uint64_t bytes, uint64_t* vptr);
int sol_b200_free_async(sol_b200_queue_t q, uint64_t vptr);
int sol_b200_vptr_add(uint64_t vptr, uint64_t delta, uint64_t* out);
int sol_b200_memcpy_h2d(sol_b200_queue_t q, uint64_t dst, const void* src, uint64_t bytes);
int sol_b200_memcpy_d2h(sol_b200_queue_t q, void* dst, uint64_t src, uint64_t bytes);
int sol_b200_launch(sol_b200_queue_t q, sol_b200_module_t m, const uint64_t* args, int32_t nargs);
int sol_b200_barrier(sol_b200_queue_t q);
/* Waits for all enqueued work; returns the first deferred error (SOL_OK if none). */
int sol_b200_synchronize(sol_b200_queue_t q, char* msg, size_t msg_len);
int sol_b200_stats(sol_b200_queue_t q, sol_transfer_stats* out);
int sol_b200_queue_stream(sol_b200_queue_t q, void** stream);

/* ---- execution plans (fe::DevicePlan) ----------------------------------------------------- */
int sol_b200_plan_create(int device, sol_b200_plan_t* out);
int sol_b200_plan_destroy(sol_b200_plan_t p);
/* persistent buffers survive the whole plan (params, inputs, outputs); others are placed by
 * liveness into one arena slab. */
int sol_b200_plan_add_buffer(sol_b200_plan_t p, uint64_t bytes, int32_t persistent, int32_t* id);
/* Adds a step running `m` on buffers ids[0..n) (bindings then output). The plan owns m. */
int sol_b200_plan_add_step(sol_b200_plan_t p, sol_b200_module_t m, const int32_t* ids, int32_t n);
/* Sum-all-reduce `count` elements of buffer `id` across ranks, then scale (1/G averaging). */
int sol_b200_plan_add_allreduce(sol_b200_plan_t p, int32_t id, uint64_t count, int32_t dtype, float scale);
int sol_b200_plan_finalize(sol_b200_plan_t p);
int sol_b200_plan_buffer_ptr(sol_b200_plan_t p, int32_t id, void** dptr);
int sol_b200_plan_set_frozen(sol_b200_plan_t p, int32_t frozen);
/* Runs every step on the plan stream (or replays the captured CUDA graph when use_graph). */
int sol_b200_plan_run(sol_b200_plan_t p, int32_t use_graph);
int sol_b200_plan_stream(sol_b200_plan_t p, void** stream);
int sol_b200_plan_sync(sol_b200_plan_t p);
/* Per-step device timing (CUDA events around every step); times_us has n_steps entries. */
int sol_b200_plan_profile(sol_b200_plan_t p, double* times_us, int32_t n);
int sol_b200_plan_num_steps(sol_b200_plan_t p, int32_t* n);
int sol_b200_plan_step_info(sol_b200_plan_t p, int32_t i, sol_module_info* info);
int sol_b200_plan_arena_bytes(sol_b200_plan_t p, uint64_t* bytes);
/* Host <-> plan buffer copies, ordered on the plan stream (src/dst should be pinned host memory). */
int sol_b200_plan_h2d(sol_b200_plan_t p, int32_t id, const void* src, uint64_t bytes);
int sol_b200_plan_d2h(sol_b200_plan_t p, void* dst, int32_t id, uint64_t bytes);
/* Pipelined input staging (serving): copies `src` (pinned) into a device staging area for buffer
 * `id` on the plan's copy stream, after the previous staged copy of that buffer was consumed; the
 * next plan_run starts by moving it into the buffer. The host-to-device copy of step i+1 thus
 * overlaps the kernels of step i (the reference queue's copy/compute overlap, runtime.hpp:95-145). */
int sol_b200_plan_stage_h2d(sol_b200_plan_t p, int32_t id, const void* src, uint64_t bytes);
/* Copy-stream fences for pinned-source reuse: a ticket taken after stage_h2d() calls completes once
   those copies have read their host sources; copy_wait blocks the host until then (the refill of a
   pinned staging buffer must not race the copy still reading it). */
int sol_b200_plan_copy_fence(sol_b200_plan_t p, uint64_t* ticket);
int sol_b200_plan_copy_wait(sol_b200_plan_t p, uint64_t ticket);
/* CUDA events on the plan stream (slots 0..15) for device-side timing. */
int sol_b200_plan_event_record(sol_b200_plan_t p, int32_t slot);
int sol_b200_plan_event_elapsed(sol_b200_plan_t p, int32_t a, int32_t b, float* ms);
/* pinned host memory */
int sol_b200_host_alloc(uint64_t bytes, void** ptr);
int sol_b200_host_free(void* ptr);

/* ---- NCCL (batch-sharded data parallelism) ------------------------------------------------ */
int sol_b200_nccl_unique_id(uint8_t id[128]);
int sol_b200_plan_set_comm(sol_b200_plan_t p, const uint8_t id[128], int32_t rank, int32_t nranks);
/* The plan communicator as NCCL sees it (ncclCommCount / ncclCommUserRank / ncclCommCuDevice);
   1 / 0 / the plan device when no communicator is attached. Bench evidence that N ranks really
   share one communicator on N distinct GPUs. */
int sol_b200_plan_comm_info(sol_b200_plan_t p, int32_t* nranks, int32_t* rank, int32_t* cuda_device);

/* ---- runtime knobs (fe::OptimizedModel::train_step(batch, lr, mode), autotune) ------------ */
/* Sets the learning rate every SgdUpdate step of the plan reads at run time (a stream-ordered
   device write, so captured graph replays see it); *n_steps = how many steps took it. */
int sol_b200_plan_set_lr(sol_b200_plan_t p, float lr, int32_t* n_steps);
/* Median device time (us) of module step `step` run alone `reps` times (after one warm-up run),
   on the plan's buffers as they are: the measurement behind autotune (dnn.cpp:214-290). */
int sol_b200_plan_time_step(sol_b200_plan_t p, int32_t step, int32_t reps, double* us);
/* BatchNorm statistics from the producing convolution's GEMM epilogue (training plans): the conv
 * step writes per-(M tile, row quarter) partial sums of (y - shift) and (y - shift)^2 of its stored
 * bf16 output, shift = the BN's previous batch mean; the BN step then skips its statistics pass
 * over y and finalises from those partials. bn_binding = the index of the conv output among the
 * BN unit's bindings. SOL_E_UNSUPPORTED when the conv's kernel path cannot (halo / stem / fused
 * epilogue / not bf16) or the unit has no training BN on that binding. */
int sol_b200_plan_link_bn_stats(sol_b200_plan_t p, int32_t conv_step, int32_t bn_step, int32_t bn_binding);
/* sol_b200_module_set_option on the module a plan step owns (the plan owns added modules). */
int sol_b200_plan_step_set_option(sol_b200_plan_t p, int32_t step, int32_t key, int32_t value);

/* ---- raw heavy-layer entry points (KernelProvider::execute on device pointers) ------------ */
typedef struct {
    int32_t N, Cin, H, W, Cout, OH, OW;
    int32_t kh, kw, sh, sw, ph, pw;
    int32_t cin_ld;   /* stored channel stride of x (>= Cin, multiple of 16 bytes) */
    int32_t dtype;
    int32_t cout_ld;  /* stored channel stride of y (>= Cout, multiple of 16 bytes; 0 = Cout) */
} sol_conv_desc;

/* W canonical f32 [Cout][Cin][kh][kw] -> packed [Cout][kh][kw][cin_ld] (K padded) in dtype
 * (transposed = 0), or [Cin][kh][kw][Cout] for dgrad (transposed = 1). */
int sol_b200_conv_packed_elems(const sol_conv_desc* d, int32_t transposed, int64_t* elems);
int sol_b200_conv_pack_weight(const sol_conv_desc* d, const float* w, void* packed, int32_t transposed, void* stream);
int sol_b200_conv_fprop(const sol_conv_desc* d, const void* x, const void* wpacked, const float* bias, void* y,
                        int32_t y_dtype, void* stream);
int sol_b200_conv_dgrad(const sol_conv_desc* d, const void* dy, const void* wtpacked, void* dx, void* stream);
int sol_b200_conv_wgrad_workspace(const sol_conv_desc* d, uint64_t* bytes);
/* profiling knob for sol_b200_conv_fprop: 1 = skip output stores, 2 = skip MMA issue (0 = normal) */
int sol_b200_set_conv_debug(int32_t flags);
/* dW canonical f32 [Cout][Cin][kh][kw] */
int sol_b200_conv_wgrad(const sol_conv_desc* d, const void* dy, const void* x, float* dw, void* workspace,
                        void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SOLB200_H */
