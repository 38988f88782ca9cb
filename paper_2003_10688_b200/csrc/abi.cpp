// extern "C" boundary (include/solb200.h). Every entry point is noexcept: C++ exceptions map to
// status codes mirroring the reference's error classes (proj/include/sol/errors.hpp:11-57) and
// the message is kept per thread for sol_b200_last_error().
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "../../include/solb200.h"
#include "dfp.cuh"
#include "igemm.cuh"
#include "module.hpp"
#include "pack.cuh"
#include "runtime.hpp"

struct sol_b200_module_s {
    std::unique_ptr<solb200::Module> m;
};
struct sol_b200_queue_s {
    std::unique_ptr<solb200::Queue> q;
};
struct sol_b200_plan_s {
    std::unique_ptr<solb200::Plan> p;
};

namespace solb200 {

int num_sms() {
    static int n = [] {
        int dev = 0, v = 148;
        if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        return v;
    }();
    return n;
}

}  // namespace solb200

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) noexcept {
    try {
        f();
        return SOL_OK;
    } catch (const solb200::CudaError& e) {
        g_err = e.what();
        return SOL_E_CUDA + e.code;
    } catch (const solb200::UnsupportedError& e) {
        g_err = e.what();
        return SOL_E_UNSUPPORTED;
    } catch (const solb200::ShapeError& e) {
        g_err = e.what();
        return SOL_E_SHAPE_MISMATCH;
    } catch (const std::overflow_error& e) {
        g_err = e.what();
        return SOL_E_OUT_OF_REFS;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SOL_E_INVALID_ARGUMENT;
    } catch (const std::exception& e) {
        g_err = e.what();
        return std::string(e.what()).rfind("NCCL", 0) == 0 ? SOL_E_NCCL : SOL_E_INVALID_ARGUMENT;
    }
}

solb200::IgemmArgs conv_args(const sol_conv_desc* d) {
    solb200::IgemmArgs a;
    a.dtype = d->dtype;
    a.out_dtype = d->dtype;
    a.N = d->N;
    a.SH = d->H;
    a.SW = d->W;
    a.SC = d->cin_ld;
    a.OH = d->OH;
    a.OW = d->OW;
    a.kh = d->kh; a.kw = d->kw; a.sh = d->sh; a.sw = d->sw; a.ph = d->ph; a.pw = d->pw;
    a.Nout = d->Cout;
    const int bk = d->dtype == SOL_DT_BF16 ? 64 : 32;
    a.K_pad = static_cast<int>(solb200::round_up(static_cast<int64_t>(d->kh) * d->kw * d->cin_ld, bk));
    a.ldo = d->cout_ld > 0 ? d->cout_ld : d->Cout;
    return a;
}

}  // namespace

extern "C" {

const char* sol_b200_last_error(void) { return g_err.c_str(); }

int sol_b200_device_count(int* count) {
    return guard([&] { SOL_CUDA(cudaGetDeviceCount(count)); });
}

int sol_b200_set_device(int device) {
    return guard([&] { SOL_CUDA(cudaSetDevice(device)); });
}

// ---- modules ---------------------------------------------------------------------------------

int sol_b200_module_create(const sol_unit_desc* desc, sol_b200_module_t* out) {
    return guard([&] {
        if (!desc || !out) throw std::invalid_argument("null argument");
        auto h = std::make_unique<sol_b200_module_s>();
        h->m = solb200::compile_unit(*desc);
        *out = h.release();
    });
}

int sol_b200_module_destroy(sol_b200_module_t m) {
    return guard([&] { delete m; });
}

static void fill_info(const solb200::Module* m, sol_module_info* info) {
    std::memset(info, 0, sizeof(*info));
    std::strncpy(info->family, m->family.c_str(), sizeof(info->family) - 1);
    info->n_args = m->n_args;
    info->scratch_bytes = m->scratch_bytes();
    info->launches = m->launches;
    info->launches_frozen = m->launches_frozen >= 0 ? m->launches_frozen : m->launches;
    info->algo_bytes = m->algo_bytes;
    info->algo_flops = m->algo_flops;
}

int sol_b200_module_info(sol_b200_module_t m, sol_module_info* info) {
    return guard([&] {
        if (!m || !info) throw std::invalid_argument("null argument");
        fill_info(m->m.get(), info);
    });
}

int sol_b200_module_set_option(sol_b200_module_t m, int32_t key, int32_t value) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null module");
        if (!m->m->set_option(key, value)) throw solb200::UnsupportedError("module option does not apply");
    });
}

int sol_b200_module_set_sibling_outputs(sol_b200_module_t m, int32_t mask) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null module");
        if (!m->m->set_sibling_outputs(mask)) throw solb200::UnsupportedError("module has no sibling outputs");
    });
}

int sol_b200_module_run(sol_b200_module_t m, void* const* args, int32_t nargs, void* scratch, void* stream,
                        int32_t frozen) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null module");
        m->m->run(args, nargs, scratch, static_cast<cudaStream_t>(stream), frozen != 0);
    });
}

// ---- queue -----------------------------------------------------------------------------------

int sol_b200_queue_create(int device, uint64_t arena_bytes, int32_t coalesce, sol_b200_queue_t* out) {
    return guard([&] {
        auto h = std::make_unique<sol_b200_queue_s>();
        h->q = std::make_unique<solb200::Queue>(device, arena_bytes, coalesce != 0);
        *out = h.release();
    });
}

int sol_b200_queue_destroy(sol_b200_queue_t q) {
    return guard([&] { delete q; });
}

int sol_b200_malloc_async(sol_b200_queue_t q, uint64_t bytes, uint64_t* vptr) {
    return guard([&] { *vptr = q->q->malloc_async(bytes); });
}

int sol_b200_free_async(sol_b200_queue_t q, uint64_t vptr) {
    return guard([&] { q->q->free_async(vptr); });
}

int sol_b200_vptr_add(uint64_t vptr, uint64_t delta, uint64_t* out) {
    // VirtualPtr::operator+ (runtime.cpp:19-24): offset arithmetic never carries into the ref
    const uint64_t off = (vptr & 0xffffffffull) + delta;
    if (delta > 0xffffffffull || off > 0xffffffffull) {
        g_err = "virtual pointer offset overflow: " + std::to_string(off);
        return SOL_E_OVERFLOW;
    }
    *out = (vptr & 0xffffffff00000000ull) | off;
    return SOL_OK;
}

int sol_b200_memcpy_h2d(sol_b200_queue_t q, uint64_t dst, const void* src, uint64_t bytes) {
    return guard([&] { q->q->memcpy_h2d(dst, src, bytes); });
}

int sol_b200_memcpy_d2h(sol_b200_queue_t q, void* dst, uint64_t src, uint64_t bytes) {
    return guard([&] { q->q->memcpy_d2h(dst, src, bytes); });
}

int sol_b200_launch(sol_b200_queue_t q, sol_b200_module_t m, const uint64_t* args, int32_t nargs) {
    return guard([&] {
        if (!m) throw std::invalid_argument("launch: null module");
        q->q->launch(m->m.get(), args, nargs);
    });
}

int sol_b200_barrier(sol_b200_queue_t q) {
    return guard([&] { q->q->barrier(); });
}

int sol_b200_synchronize(sol_b200_queue_t q, char* msg, size_t msg_len) {
    std::string m;
    int code = SOL_OK;
    const int rc = guard([&] { code = q->q->synchronize(&m); });
    if (rc != SOL_OK) return rc;
    if (msg && msg_len) {
        std::strncpy(msg, m.c_str(), msg_len - 1);
        msg[msg_len - 1] = 0;
    }
    if (code != SOL_OK) g_err = m;
    return code;
}

int sol_b200_stats(sol_b200_queue_t q, sol_transfer_stats* out) {
    return guard([&] { *out = q->q->stats(); });
}

int sol_b200_queue_stream(sol_b200_queue_t q, void** stream) {
    return guard([&] { *stream = q->q->stream(); });
}

// ---- plans -----------------------------------------------------------------------------------

int sol_b200_plan_create(int device, sol_b200_plan_t* out) {
    return guard([&] {
        auto h = std::make_unique<sol_b200_plan_s>();
        h->p = std::make_unique<solb200::Plan>(device);
        *out = h.release();
    });
}

int sol_b200_plan_destroy(sol_b200_plan_t p) {
    return guard([&] { delete p; });
}

int sol_b200_plan_add_buffer(sol_b200_plan_t p, uint64_t bytes, int32_t persistent, int32_t* id) {
    return guard([&] { *id = p->p->add_buffer(bytes, persistent != 0); });
}

int sol_b200_plan_add_step(sol_b200_plan_t p, sol_b200_module_t m, const int32_t* ids, int32_t n) {
    return guard([&] {
        if (!m) throw std::invalid_argument("null module");
        p->p->add_step(std::move(m->m), ids, n);
        delete m;
    });
}

int sol_b200_plan_add_allreduce(sol_b200_plan_t p, int32_t id, uint64_t count, int32_t dtype, float scale) {
    return guard([&] { p->p->add_allreduce(id, count, dtype, scale); });
}

int sol_b200_plan_finalize(sol_b200_plan_t p) {
    return guard([&] { p->p->finalize(); });
}

int sol_b200_plan_buffer_ptr(sol_b200_plan_t p, int32_t id, void** dptr) {
    return guard([&] { *dptr = p->p->buffer_ptr(id); });
}

int sol_b200_plan_set_frozen(sol_b200_plan_t p, int32_t frozen) {
    return guard([&] { p->p->set_frozen(frozen != 0); });
}

int sol_b200_plan_run(sol_b200_plan_t p, int32_t use_graph) {
    return guard([&] { p->p->run(use_graph != 0); });
}

int sol_b200_plan_stream(sol_b200_plan_t p, void** stream) {
    return guard([&] { *stream = p->p->stream(); });
}

int sol_b200_plan_sync(sol_b200_plan_t p) {
    return guard([&] { p->p->sync(); });
}

int sol_b200_plan_profile(sol_b200_plan_t p, double* times_us, int32_t n) {
    return guard([&] { p->p->profile(times_us, n); });
}

int sol_b200_plan_num_steps(sol_b200_plan_t p, int32_t* n) {
    return guard([&] { *n = p->p->num_steps(); });
}

int sol_b200_plan_step_info(sol_b200_plan_t p, int32_t i, sol_module_info* info) {
    return guard([&] {
        if (i < 0 || i >= p->p->num_steps()) throw std::invalid_argument("bad step index");
        const solb200::Module* m = p->p->step_module(i);
        if (m) {
            fill_info(m, info);
        } else {
            std::memset(info, 0, sizeof(*info));
            std::strncpy(info->family, "nccl_allreduce", sizeof(info->family) - 1);
            info->n_args = 1;
        }
    });
}

int sol_b200_plan_arena_bytes(sol_b200_plan_t p, uint64_t* bytes) {
    return guard([&] { *bytes = p->p->arena_bytes(); });
}

int sol_b200_plan_h2d(sol_b200_plan_t p, int32_t id, const void* src, uint64_t bytes) {
    return guard([&] { p->p->h2d(id, src, bytes); });
}

int sol_b200_plan_stage_h2d(sol_b200_plan_t p, int32_t id, const void* src, uint64_t bytes) {
    return guard([&] { p->p->stage_h2d(id, src, bytes); });
}

int sol_b200_plan_copy_fence(sol_b200_plan_t p, uint64_t* ticket) {
    return guard([&] { *ticket = p->p->copy_fence(); });
}

int sol_b200_plan_copy_wait(sol_b200_plan_t p, uint64_t ticket) {
    return guard([&] { p->p->copy_wait(ticket); });
}

int sol_b200_plan_d2h(sol_b200_plan_t p, void* dst, int32_t id, uint64_t bytes) {
    return guard([&] { p->p->d2h(dst, id, bytes); });
}

int sol_b200_plan_event_record(sol_b200_plan_t p, int32_t slot) {
    return guard([&] { p->p->event_record(slot); });
}

int sol_b200_plan_event_elapsed(sol_b200_plan_t p, int32_t a, int32_t b, float* ms) {
    return guard([&] { *ms = p->p->event_elapsed(a, b); });
}

int sol_b200_host_alloc(uint64_t bytes, void** ptr) {
    return guard([&] { SOL_CUDA(cudaMallocHost(ptr, bytes)); });
}

int sol_b200_host_free(void* ptr) {
    return guard([&] { SOL_CUDA(cudaFreeHost(ptr)); });
}

// ---- NCCL ------------------------------------------------------------------------------------

int sol_b200_nccl_unique_id(uint8_t id[128]) {
    return guard([&] {
        ncclUniqueId uid;
        const ncclResult_t r = ncclGetUniqueId(&uid);
        if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL id: ") + ncclGetErrorString(r));
        static_assert(sizeof(uid) == 128, "ncclUniqueId size");
        std::memcpy(id, &uid, 128);
    });
}

int sol_b200_plan_set_comm(sol_b200_plan_t p, const uint8_t id[128], int32_t rank, int32_t nranks) {
    return guard([&] { p->p->set_comm(id, rank, nranks); });
}

int sol_b200_plan_set_lr(sol_b200_plan_t p, float lr, int32_t* n_steps) {
    return guard([&] {
        const int n = p->p->set_lr(lr);
        if (n_steps) *n_steps = n;
    });
}

int sol_b200_plan_time_step(sol_b200_plan_t p, int32_t step, int32_t reps, double* us) {
    return guard([&] { *us = p->p->time_step(step, reps); });
}

int sol_b200_plan_step_set_option(sol_b200_plan_t p, int32_t step, int32_t key, int32_t value) {
    return guard([&] {
        if (!p->p->step_set_option(step, key, value)) throw solb200::UnsupportedError("module option does not apply");
    });
}

int sol_b200_plan_link_bn_stats(sol_b200_plan_t p, int32_t conv_step, int32_t bn_step, int32_t bn_binding) {
    return guard([&] {
        if (!p->p->link_bn_stats(conv_step, bn_step, bn_binding))
            throw solb200::UnsupportedError("the conv cannot emit this BatchNorm's statistics");
    });
}

int sol_b200_plan_comm_info(sol_b200_plan_t p, int32_t* nranks, int32_t* rank, int32_t* cuda_device) {
    return guard([&] {
        int n = 1, r = 0, d = 0;
        p->p->comm_info(&n, &r, &d);
        *nranks = n;
        *rank = r;
        *cuda_device = d;
    });
}

// ---- raw heavy-layer entry points ------------------------------------------------------------

int sol_b200_conv_packed_elems(const sol_conv_desc* d, int32_t transposed, int64_t* elems) {
    return guard([&] {
        const int bk = d->dtype == SOL_DT_BF16 ? 64 : 32;
        if (!transposed)
            *elems = static_cast<int64_t>(d->Cout) * solb200::round_up(static_cast<int64_t>(d->kh) * d->kw * d->cin_ld, bk);
        else
            *elems = static_cast<int64_t>(d->Cin) * solb200::round_up(static_cast<int64_t>(d->kh) * d->kw * d->Cout, bk);
    });
}

int sol_b200_conv_pack_weight(const sol_conv_desc* d, const float* w, void* packed, int32_t transposed, void* stream) {
    return guard([&] {
        const int bk = d->dtype == SOL_DT_BF16 ? 64 : 32;
        auto s = static_cast<cudaStream_t>(stream);
        if (!transposed)
            solb200::pack_conv_weight(w, packed, d->dtype, d->Cout, d->Cin, d->kh, d->kw, d->cin_ld,
                                      static_cast<int>(solb200::round_up(static_cast<int64_t>(d->kh) * d->kw * d->cin_ld, bk)), s);
        else
            solb200::pack_conv_weight_t(w, packed, d->dtype, d->Cout, d->Cin, d->kh, d->kw, d->Cout,
                                        static_cast<int>(solb200::round_up(static_cast<int64_t>(d->kh) * d->kw * d->Cout, bk)), s);
    });
}

static int g_conv_dbg = 0;

int sol_b200_set_conv_debug(int32_t flags) {
    g_conv_dbg = flags;
    return SOL_OK;
}

int sol_b200_conv_fprop(const sol_conv_desc* d, const void* x, const void* wpacked, const float* bias, void* y,
                        int32_t y_dtype, void* stream) {
    return guard([&] {
        solb200::IgemmArgs a = conv_args(d);
        a.dbg = g_conv_dbg;
        a.mode = solb200::IG_FPROP;
        a.src = x;
        a.wt = wpacked;
        a.bias = bias;
        a.out = y;
        a.out_dtype = y_dtype;
        solb200::igemm_launch(a, static_cast<cudaStream_t>(stream));
    });
}

int sol_b200_conv_dgrad(const sol_conv_desc* d, const void* dy, const void* wtpacked, void* dx, void* stream) {
    return guard([&] {
        solb200::IgemmArgs a;
        a.mode = solb200::IG_DGRAD;
        a.dtype = d->dtype;
        a.out_dtype = d->dtype;
        a.src = dy;
        a.wt = wtpacked;
        a.out = dx;
        a.N = d->N;
        a.SH = d->OH;
        a.SW = d->OW;
        a.SC = d->Cout;
        a.OH = d->H;
        a.OW = d->W;
        a.kh = d->kh; a.kw = d->kw; a.sh = d->sh; a.sw = d->sw; a.ph = d->ph; a.pw = d->pw;
        a.Nout = d->Cin;
        const int bk = d->dtype == SOL_DT_BF16 ? 64 : 32;
        a.K_pad = static_cast<int>(solb200::round_up(static_cast<int64_t>(d->kh) * d->kw * d->Cout, bk));
        a.ldo = d->cin_ld;
        solb200::igemm_launch(a, static_cast<cudaStream_t>(stream));
    });
}

static solb200::WgradArgs wgrad_args(const sol_conv_desc* d) {
    solb200::WgradArgs w;
    w.dtype = d->dtype;
    w.N = d->N;
    w.SH = d->H;
    w.SW = d->W;
    w.SC = d->cin_ld;
    w.OH = d->OH;
    w.OW = d->OW;
    w.Cout = d->Cout;
    w.kh = d->kh; w.kw = d->kw; w.sh = d->sh; w.sw = d->sw; w.ph = d->ph; w.pw = d->pw;
    w.ld_dy = d->Cout;
    return w;
}

int sol_b200_conv_wgrad_workspace(const sol_conv_desc* d, uint64_t* bytes) {
    return guard([&] {
        solb200::WgradArgs w = wgrad_args(d);
        const uint64_t packed = static_cast<uint64_t>(d->Cout) * d->kh * d->kw * d->cin_ld;
        *bytes = (solb200::round_up(packed, 64) + solb200::wgrad_workspace_floats(w)) * 4 + 256;
    });
}

int sol_b200_conv_wgrad(const sol_conv_desc* d, const void* dy, const void* x, float* dw, void* workspace,
                        void* stream) {
    return guard([&] {
        auto s = static_cast<cudaStream_t>(stream);
        solb200::WgradArgs w = wgrad_args(d);
        float* packed = static_cast<float*>(workspace);
        const int64_t pk = static_cast<int64_t>(d->Cout) * d->kh * d->kw * d->cin_ld;
        w.dy = dy;
        w.x = x;
        w.dw = packed;
        w.workspace = packed + solb200::round_up(pk, 64);
        solb200::wgrad_launch(w, s);
        solb200::unpack_conv_grad(packed, dw, d->Cout, d->Cin, d->kh, d->kw, d->cin_ld, s);
    });
}

}  // extern "C"
