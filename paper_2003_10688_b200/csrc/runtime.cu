// Device runtime (see runtime.hpp).
//
// Queue semantics mirror the reference rt::CommandQueue (proj/src/runtime.cpp):
//   * malloc_async never blocks and hands out VirtualPtr = ref << 32 | offset   (:287-302)
//   * bytes must be in (0, 2^32); free requires offset 0 (eager invalid_argument) (:288, :305)
//   * resolution errors (use-after-free, unknown ref, out-of-bounds) are deferred: the first one
//     wins, later commands are skipped, synchronize() reports it                 (:128-141, :157-256)
//   * adjacent H2D copies coalesce: a run of >= 64 KiB becomes one packed transfer (:144-155) —
//     here a real one: one pinned->device DMA of the whole run plus one scatter kernel.
#include "runtime.hpp"
#include "pack.cuh"

#include <cstdio>
#include <cstdlib>

#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <tuple>

#include "../../include/solb200.h"

namespace solb200 {

constexpr uint64_t kPackThreshold = 65536;
constexpr size_t kAlign = 256;

// ---------------------------------------------------------------------------------------------
// Arena
// ---------------------------------------------------------------------------------------------

Arena::~Arena() {
    if (base_) cudaFree(base_);
}

void Arena::init(size_t bytes, cudaStream_t stream) {
    cap_ = round_up(static_cast<int64_t>(std::max<size_t>(bytes, kAlign)), kAlign);
    if (stream) SOL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&base_), cap_, stream));
    else SOL_CUDA(cudaMalloc(&base_, cap_));
    free_.clear();
    live_.clear();
    free_[0] = cap_;
    used_ = 0;
}

int64_t Arena::alloc(size_t bytes) {
    const size_t need = round_up(static_cast<int64_t>(std::max<size_t>(bytes, 1)), kAlign);
    for (auto it = free_.begin(); it != free_.end(); ++it) {
        if (it->second >= need) {
            const int64_t off = it->first;
            const size_t rest = it->second - need;
            free_.erase(it);
            if (rest) free_[off + static_cast<int64_t>(need)] = rest;
            live_[off] = need;
            used_ += need;
            return off;
        }
    }
    return -1;
}

void Arena::free(int64_t off) {
    auto it = live_.find(off);
    if (it == live_.end()) return;
    size_t sz = it->second;
    used_ -= sz;
    live_.erase(it);
    auto nx = free_.lower_bound(off);
    if (nx != free_.end() && off + static_cast<int64_t>(sz) == nx->first) {
        sz += nx->second;
        nx = free_.erase(nx);
    }
    if (nx != free_.begin()) {
        auto pv = std::prev(nx);
        if (pv->first + static_cast<int64_t>(pv->second) == off) {
            pv->second += sz;
            return;
        }
    }
    free_[off] = sz;
}

// ---------------------------------------------------------------------------------------------
// Queue
// ---------------------------------------------------------------------------------------------

namespace {

struct ScatterEntry {
    uint64_t dst;
    uint64_t src_off;
    uint64_t bytes;
};

__global__ void scatter_kernel(const uint8_t* __restrict__ staging, int n) {
    const ScatterEntry* tab = reinterpret_cast<const ScatterEntry*>(staging);
    for (int e = blockIdx.x; e < n; e += gridDim.x) {
        const ScatterEntry t = tab[e];
        uint8_t* dst = reinterpret_cast<uint8_t*>(t.dst);
        const uint8_t* src = staging + t.src_off;
        if (((t.dst | t.src_off | t.bytes) & 15) == 0) {
            for (uint64_t i = threadIdx.x * 16ull; i < t.bytes; i += blockDim.x * 16ull)
                *reinterpret_cast<uint4*>(dst + i) = *reinterpret_cast<const uint4*>(src + i);
        } else {
            for (uint64_t i = threadIdx.x; i < t.bytes; i += blockDim.x) dst[i] = src[i];
        }
    }
}

}  // namespace

PinnedPool::~PinnedPool() {
    for (auto& s : slabs_) cudaFreeHost(s.p);
}

void* PinnedPool::get(size_t bytes) {
    bytes = static_cast<size_t>(round_up(static_cast<int64_t>(std::max<size_t>(bytes, 16)), 64));
    for (; cur_ < slabs_.size(); ++cur_) {
        Slab& s = slabs_[cur_];
        if (s.cap - s.used >= bytes) {
            void* p = s.p + s.used;
            s.used += bytes;
            return p;
        }
    }
    const size_t cap = std::max<size_t>({bytes, slabs_.empty() ? size_t(1) << 20 : 2 * slabs_.back().cap});
    Slab s{nullptr, cap, bytes};
    SOL_CUDA(cudaMallocHost(reinterpret_cast<void**>(&s.p), cap));
    slabs_.push_back(s);
    cur_ = slabs_.size() - 1;
    return s.p;
}

void PinnedPool::reset() {
    for (auto& s : slabs_) s.used = 0;
    cur_ = 0;
}

Queue::Queue(int device, size_t arena_bytes, bool coalesce) : device_(device), coalesce_(coalesce) {
    SOL_CUDA(cudaSetDevice(device));
    SOL_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    slabs_.push_back(std::make_unique<Arena>());
    slabs_.back()->init(arena_bytes ? arena_bytes : (256ull << 20));
    SOL_CUDA(cudaEventCreate(&ev_start_));
    SOL_CUDA(cudaEventCreate(&ev_end_));
}

Queue::~Queue() {
    cudaStreamSynchronize(stream_);
    if (ev_start_) cudaEventDestroy(ev_start_);
    if (ev_end_) cudaEventDestroy(ev_end_);
    if (stream_) cudaStreamDestroy(stream_);
}

void Queue::defer(int code, const std::string& msg) {
    if (err_.code == 0) err_ = {code, msg};
}

void Queue::mark_start() {
    if (!timing_) {
        SOL_CUDA(cudaEventRecord(ev_start_, stream_));
        timing_ = true;
    }
}

uint8_t* Queue::resolve(uint64_t vptr, uint64_t bytes) {
    const uint32_t ref = static_cast<uint32_t>(vptr >> 32);
    const uint64_t off = vptr & 0xffffffffull;
    auto it = allocs_.find(ref);
    if (it == allocs_.end()) {
        if (freed_.count(ref)) defer(SOL_E_USE_AFTER_FREE, "use after free of ref " + std::to_string(ref));
        else defer(SOL_E_UNKNOWN_REF, "unknown ref " + std::to_string(ref));
        return nullptr;
    }
    if (off + bytes > it->second.bytes) {
        defer(SOL_E_OUT_OF_BOUNDS, "access beyond allocation " + std::to_string(ref));
        return nullptr;
    }
    return arena_ptr(it->second.slab, it->second.off) + off;
}

std::pair<int, int64_t> Queue::arena_alloc(size_t bytes) {
    for (size_t i = 0; i < slabs_.size(); ++i) {
        const int64_t off = slabs_[i]->alloc(bytes);
        if (off >= 0) return {static_cast<int>(i), off};
    }
    // grow: a new slab from the stream-ordered allocator (never blocks the launch stream)
    size_t biggest = 0;
    for (auto& a : slabs_) biggest = std::max(biggest, a->capacity());
    slabs_.push_back(std::make_unique<Arena>());
    slabs_.back()->init(std::max(2 * biggest, bytes + kAlign), stream_);
    const int64_t off = slabs_.back()->alloc(bytes);
    if (off < 0) throw CudaError(static_cast<int>(cudaErrorMemoryAllocation), "device arena growth failed");
    return {static_cast<int>(slabs_.size() - 1), off};
}

uint64_t Queue::malloc_async(uint64_t bytes) {
    if (bytes == 0 || bytes > 0xffffffffull) throw std::invalid_argument("malloc_async: bytes must be in (0, 2^32)");
    if (next_ref_ > 0xffffffffull) throw std::overflow_error("virtual pointer refs exhausted");
    const uint32_t ref = static_cast<uint32_t>(next_ref_++);
    const auto [slab, off] = arena_alloc(bytes);
    allocs_[ref] = {slab, off, bytes};
    // fresh allocations read as zeros (the reference's allocs_[ref].resize(bytes), runtime.cpp:187);
    // stream-ordered, so the host never waits
    SOL_CUDA(cudaMemsetAsync(arena_ptr(slab, off), 0, bytes, stream_));
    freed_.erase(ref);
    return static_cast<uint64_t>(ref) << 32;
}

void Queue::free_async(uint64_t vptr) {
    if ((vptr & 0xffffffffull) != 0) throw std::invalid_argument("free_async frees whole allocations (offset must be 0)");
    if (failed()) return;
    const uint32_t ref = static_cast<uint32_t>(vptr >> 32);
    auto it = allocs_.find(ref);
    if (it == allocs_.end()) {
        defer(SOL_E_UNKNOWN_REF, "free of unknown ref " + std::to_string(ref));
        return;
    }
    close_copy_run();  // pending copies into this block must land before reuse
    slabs_[it->second.slab]->free(it->second.off);
    allocs_.erase(it);
    freed_[ref] = true;
}

void* Queue::staging(size_t bytes) { return pinned_.get(bytes); }

void Queue::memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes) {
    if (failed() || bytes == 0) return;
    uint8_t* d = resolve(dst, bytes);
    if (!d) return;
    mark_start();
    stats_.h2d_bytes += bytes;
    stats_.h2d_ops += 1;
    // one packed transfer scatters its copies concurrently: a copy overlapping one already in the
    // open run closes the run first, so the later copy still lands last (program order)
    for (const PendingCopy& c : run_)
        if (d < c.dst + c.bytes && c.dst < d + bytes) {
            close_copy_run();
            break;
        }
    // snapshot now (reference: "H2D snapshots the host range at enqueue time")
    const uint64_t off = round_up(static_cast<int64_t>(run_payload_.size()), 16);
    run_payload_.resize(off + bytes);
    std::memcpy(run_payload_.data() + off, src, bytes);
    run_.push_back({d, off, bytes});
    if (!coalesce_) close_copy_run();
}

void Queue::close_copy_run() {
    if (run_.empty()) return;
    const uint64_t total = run_payload_.size();
    if (coalesce_ && run_.size() > 1 && total >= kPackThreshold) {
        // one packed transfer: [table | payload] -> device staging -> scatter kernel
        const uint64_t tab_bytes = round_up(static_cast<int64_t>(run_.size() * sizeof(ScatterEntry)), 16);
        uint8_t* host = static_cast<uint8_t*>(staging(tab_bytes + total));
        ScatterEntry* tab = reinterpret_cast<ScatterEntry*>(host);
        for (size_t i = 0; i < run_.size(); ++i)
            tab[i] = {reinterpret_cast<uint64_t>(run_[i].dst), tab_bytes + run_[i].off, run_[i].bytes};
        std::memcpy(host + tab_bytes, run_payload_.data(), total);
        const auto [dslab, doff] = arena_alloc(tab_bytes + total);
        uint8_t* dev = arena_ptr(dslab, doff);
        SOL_CUDA(cudaMemcpyAsync(dev, host, tab_bytes + total, cudaMemcpyHostToDevice, stream_));
        const int n = static_cast<int>(run_.size());
        scatter_kernel<<<std::min(n, 1024), 256, 0, stream_>>>(dev, n);
        SOL_CUDA(cudaGetLastError());
        slabs_[dslab]->free(doff);  // stream-ordered: later users run after the scatter
        stats_.packed_transfers += 1;
    } else {
        uint8_t* host = static_cast<uint8_t*>(staging(total));
        std::memcpy(host, run_payload_.data(), total);
        for (auto& c : run_)
            SOL_CUDA(cudaMemcpyAsync(c.dst, host + c.off, c.bytes, cudaMemcpyHostToDevice, stream_));
    }
    run_.clear();
    run_payload_.clear();
}

void Queue::memcpy_d2h(void* dst, uint64_t src, uint64_t bytes) {
    if (failed() || bytes == 0) return;
    uint8_t* s = resolve(src, bytes);
    if (!s) return;
    close_copy_run();
    mark_start();
    void* pinned = staging(bytes);
    SOL_CUDA(cudaMemcpyAsync(pinned, s, bytes, cudaMemcpyDeviceToHost, stream_));
    d2h_.push_back({dst, pinned, bytes});
    stats_.d2h_bytes += bytes;
    stats_.d2h_ops += 1;
}

void Queue::launch(Module* m, const uint64_t* args, int nargs) {
    if (m == nullptr) throw std::invalid_argument("launch: null module");
    if (nargs != m->n_args)
        throw std::invalid_argument("launch: module '" + m->family + "' expects " + std::to_string(m->n_args) +
                                    " args, got " + std::to_string(nargs));
    if (failed()) return;
    close_copy_run();
    std::vector<void*> ptrs(nargs);
    for (int i = 0; i < nargs; ++i) {
        ptrs[i] = resolve(args[i], m->arg_bytes[i]);
        if (!ptrs[i]) return;
    }
    const size_t need = m->scratch_bytes();
    if (need > scratch_bytes_) {
        if (scratch_off_ >= 0) slabs_[scratch_slab_]->free(scratch_off_);
        std::tie(scratch_slab_, scratch_off_) = arena_alloc(need);
        scratch_bytes_ = need;
    }
    mark_start();
    m->run(ptrs.data(), nargs, scratch_off_ >= 0 ? arena_ptr(scratch_slab_, scratch_off_) : nullptr, stream_, false);
    stats_.launches += 1;
}

void Queue::barrier() { close_copy_run(); }

int Queue::synchronize(std::string* msg) {
    close_copy_run();
    if (timing_) SOL_CUDA(cudaEventRecord(ev_end_, stream_));
    const cudaError_t e = cudaStreamSynchronize(stream_);
    if (e != cudaSuccess) defer(SOL_E_CUDA + static_cast<int>(e), cudaGetErrorString(e));
    if (timing_) {
        float ms = 0.f;
        if (cudaEventElapsedTime(&ms, ev_start_, ev_end_) == cudaSuccess) stats_.device_time_us += ms * 1000.0;
        timing_ = false;
    }
    for (auto& d : d2h_) std::memcpy(d.user, d.pinned, d.bytes);
    d2h_.clear();
    pinned_.reset();  // the stream is idle: every staging slab is free again
    if (msg) *msg = err_.msg;
    return err_.code;
}

// ---------------------------------------------------------------------------------------------
// Plan
// ---------------------------------------------------------------------------------------------

namespace {

__global__ void scale_kernel(float* p, uint64_t n, float s) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] *= s;
}

__global__ void scale_bf16_kernel(__nv_bfloat16* p, uint64_t n, float s) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        p[i] = __float2bfloat16_rn(__bfloat162float(p[i]) * s);
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL ") + what + ": " + ncclGetErrorString(r));
}

}  // namespace

Plan::Plan(int device) : device_(device) {
    SOL_CUDA(cudaSetDevice(device));
    SOL_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
}

Plan::~Plan() {
    cudaStreamSynchronize(stream_);
    if (copy_stream_) cudaStreamSynchronize(copy_stream_);
    for (auto& kv : staged_) {
        if (kv.second.dev) cudaFree(kv.second.dev);
        if (kv.second.ready) cudaEventDestroy(kv.second.ready);
        if (kv.second.consumed) cudaEventDestroy(kv.second.consumed);
    }
    for (cudaEvent_t e : fences_)
        if (e) cudaEventDestroy(e);
    if (copy_stream_) cudaStreamDestroy(copy_stream_);
    if (comm_stream_) cudaStreamSynchronize(comm_stream_);
    for (cudaEvent_t e : ar_events_) cudaEventDestroy(e);
    if (comm_stream_) cudaStreamDestroy(comm_stream_);
    if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
    steps_.clear();
    if (base_) cudaFree(base_);
    if (comm_) ncclCommDestroy(static_cast<ncclComm_t>(comm_));
    for (auto& e : events_)
        if (e) cudaEventDestroy(e);
    if (stream_) cudaStreamDestroy(stream_);
}

int Plan::add_buffer(uint64_t bytes, bool persistent) {
    if (finalized_) throw std::invalid_argument("plan already finalized");
    bufs_.push_back({std::max<uint64_t>(bytes, 16), persistent});
    return static_cast<int>(bufs_.size()) - 1;
}

void Plan::add_step(std::unique_ptr<Module> m, const int32_t* ids, int n) {
    if (finalized_) throw std::invalid_argument("plan already finalized");
    if (n != m->n_args) throw std::invalid_argument("plan step: module '" + m->family + "' expects " +
                                                    std::to_string(m->n_args) + " buffers");
    Step s;
    s.module = std::move(m);
    for (int i = 0; i < n; ++i) {
        if (ids[i] < 0 || ids[i] >= static_cast<int>(bufs_.size())) throw std::invalid_argument("bad buffer id");
        if (bufs_[ids[i]].bytes < s.module->arg_bytes[i])
            throw std::invalid_argument("plan step: buffer " + std::to_string(ids[i]) + " smaller than '" +
                                        s.module->family + "' argument " + std::to_string(i));
        s.ids.push_back(ids[i]);
    }
    steps_.push_back(std::move(s));
}

void Plan::add_allreduce(int id, uint64_t count, int dtype, float scale) {
    if (id < 0 || id >= static_cast<int>(bufs_.size())) throw std::invalid_argument("bad buffer id");
    Step s;
    s.ar_id = id;
    s.ar_count = count;
    s.ar_dtype = dtype;
    s.ar_scale = scale;
    s.ids = {id};
    steps_.push_back(std::move(s));
}

void Plan::finalize() {
    if (finalized_) return;
    for (int i = 0; i < static_cast<int>(steps_.size()); ++i)
        for (int id : steps_[i].ids) {
            Buf& b = bufs_[id];
            if (b.first < 0) b.first = i;
            b.last = i;
        }
    uint64_t off = 0;
    for (auto& b : bufs_)
        if (b.persistent || b.first < 0) {
            b.off = off;
            off += round_up(b.bytes, kAlign);
        }
    const uint64_t transient_base = off;
    // greedy interval packing of transient buffers, largest first
    std::vector<int> order;
    for (int i = 0; i < static_cast<int>(bufs_.size()); ++i)
        if (!bufs_[i].persistent && bufs_[i].first >= 0) order.push_back(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return bufs_[a].bytes > bufs_[b].bytes; });
    std::vector<int> placed;
    uint64_t high = 0;
    for (int i : order) {
        Buf& b = bufs_[i];
        const uint64_t sz = round_up(b.bytes, kAlign);
        std::vector<std::pair<uint64_t, uint64_t>> busy;
        for (int j : placed) {
            const Buf& o = bufs_[j];
            if (o.first <= b.last && b.first <= o.last) busy.push_back({o.off, o.off + round_up(o.bytes, kAlign)});
        }
        std::sort(busy.begin(), busy.end());
        uint64_t cand = 0;
        for (auto& [lo, hi] : busy) {
            if (cand + sz <= lo) break;
            cand = std::max(cand, hi);
        }
        b.off = cand;
        high = std::max(high, cand + sz);
        placed.push_back(i);
    }
    for (int i : placed) bufs_[i].off += transient_base;
    scratch_off_ = transient_base + high;
    for (auto& s : steps_)
        if (s.module) scratch_bytes_ = std::max<uint64_t>(scratch_bytes_, s.module->scratch_bytes());
    total_ = scratch_off_ + round_up(scratch_bytes_, kAlign) + kAlign;
    SOL_CUDA(cudaSetDevice(device_));
    SOL_CUDA(cudaMalloc(&base_, total_));
    SOL_CUDA(cudaMemset(base_, 0, total_));
    finalized_ = true;
}

void* Plan::buffer_ptr(int id) const {
    if (!finalized_) throw std::invalid_argument("plan not finalized");
    if (id < 0 || id >= static_cast<int>(bufs_.size())) throw std::invalid_argument("bad buffer id");
    return base_ + bufs_[id].off;
}

void Plan::run_step(Step& s, cudaStream_t st) {
    if (s.module) {
        void* ptrs[64];
        std::vector<void*> big;
        void** p = ptrs;
        if (s.ids.size() > 64) {
            big.resize(s.ids.size());
            p = big.data();
        }
        for (size_t i = 0; i < s.ids.size(); ++i) p[i] = base_ + bufs_[s.ids[i]].off;
        s.module->run(p, static_cast<int>(s.ids.size()), base_ + scratch_off_, st, frozen_);
        return;
    }
    void* buf = base_ + bufs_[s.ar_id].off;
    if (comm_ && nranks_ > 1) {
        nccl_check(ncclAllReduce(buf, buf, s.ar_count, s.ar_dtype == DT_BF16 ? ncclBfloat16 : ncclFloat32, ncclSum,
                                 static_cast<ncclComm_t>(comm_), st),
                   "allreduce");
    }
    if (s.ar_scale != 1.f) {
        const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ceil_div(s.ar_count, 256), 4096));
        if (s.ar_dtype == DT_BF16) scale_bf16_kernel<<<grid, 256, 0, st>>>(static_cast<__nv_bfloat16*>(buf), s.ar_count, s.ar_scale);
        else scale_kernel<<<grid, 256, 0, st>>>(static_cast<float*>(buf), s.ar_count, s.ar_scale);
        SOL_CUDA(cudaGetLastError());
    }
}

void Plan::run_steps(cudaStream_t st) {
    static const bool sync_steps = std::getenv("SOL_SYNC_STEPS") != nullptr;  // hang bisection (eager)
    // all-reduce groups go to the comm stream; the plan stream joins it before the first module step
    // after the last group (the optimizer reads the reduced gradients)
    size_t last_ar = steps_.size();
    for (size_t i = 0; i < steps_.size(); ++i)
        if (!steps_[i].module) last_ar = i;
    const bool overlap = comm_ && last_ar < steps_.size() && !sync_steps;
    int n_groups = 0;
    if (overlap) {
        if (!comm_stream_) SOL_CUDA(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking));
        for (size_t i = 0; i < steps_.size(); ++i)
            if (!steps_[i].module && (i == 0 || steps_[i - 1].module)) ++n_groups;
        while (static_cast<int>(ar_events_.size()) < n_groups + 1) {
            cudaEvent_t e;
            SOL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            ar_events_.push_back(e);
        }
    }
    // every weight packing of this run (training: the master weights SGD updated last run) in one
    // launch ahead of the steps, instead of one small pack launch per conv step
    {
        static const bool no_batch = std::getenv("SOL_NO_PACK_BATCH") != nullptr;
        if (!no_batch) {
            pack_batch_begin();
            try {
                std::vector<void*> big;
                for (auto& s : steps_) {
                    if (!s.module) continue;
                    big.resize(s.ids.size());
                    for (size_t k = 0; k < s.ids.size(); ++k) big[k] = base_ + bufs_[s.ids[k]].off;
                    s.module->prepack(big.data(), st, frozen_);
                }
            } catch (...) {
                pack_batch_end(st);
                throw;
            }
            pack_batch_end(st);
        }
    }
    int group = 0;
    bool joined = !overlap;
    for (size_t i = 0; i < steps_.size();) {
        if (!joined && i > last_ar && steps_[i].module) {
            SOL_CUDA(cudaEventRecord(ar_events_[n_groups], comm_stream_));
            SOL_CUDA(cudaStreamWaitEvent(st, ar_events_[n_groups], 0));
            joined = true;
        }
        if (steps_[i].module || !comm_) {
            if (sync_steps && steps_[i].module) {
                std::fprintf(stderr, "[sol] step %zu %s\n", i, steps_[i].module->family.c_str());
                std::fflush(stderr);
            }
            run_step(steps_[i], st);
            if (sync_steps) SOL_CUDA(cudaStreamSynchronize(st));
            ++i;
            continue;
        }
        // a run of gradient all-reduces: one NCCL group (aggregated launches); the 1/G mean is
        // ncclAvg when the scale is exactly the replica count, else a scale kernel afterwards
        size_t j = i;
        cudaStream_t cs = st;
        if (overlap) {
            SOL_CUDA(cudaEventRecord(ar_events_[group], st));
            SOL_CUDA(cudaStreamWaitEvent(comm_stream_, ar_events_[group], 0));
            cs = comm_stream_;
            ++group;
        }
        nccl_check(ncclGroupStart(), "group");
        for (; j < steps_.size() && !steps_[j].module; ++j) {
            Step& s = steps_[j];
            void* buf = base_ + bufs_[s.ar_id].off;
            const bool avg = s.ar_scale == 1.f / static_cast<float>(nranks_);
            nccl_check(ncclAllReduce(buf, buf, s.ar_count, s.ar_dtype == DT_BF16 ? ncclBfloat16 : ncclFloat32,
                                     avg ? ncclAvg : ncclSum, static_cast<ncclComm_t>(comm_), cs),
                       "allreduce");
        }
        nccl_check(ncclGroupEnd(), "group");
        for (size_t k = i; k < j; ++k) {
            Step& s = steps_[k];
            if (s.ar_scale == 1.f || s.ar_scale == 1.f / static_cast<float>(nranks_)) continue;
            void* buf = base_ + bufs_[s.ar_id].off;
            const unsigned grid = static_cast<unsigned>(std::min<uint64_t>(ceil_div(s.ar_count, 256), 4096));
            if (s.ar_dtype == DT_BF16) scale_bf16_kernel<<<grid, 256, 0, cs>>>(static_cast<__nv_bfloat16*>(buf), s.ar_count, s.ar_scale);
            else scale_kernel<<<grid, 256, 0, cs>>>(static_cast<float*>(buf), s.ar_count, s.ar_scale);
            SOL_CUDA(cudaGetLastError());
        }
        i = j;
    }
    if (!joined) {  // plan ends with an all-reduce group
        SOL_CUDA(cudaEventRecord(ar_events_[n_groups], comm_stream_));
        SOL_CUDA(cudaStreamWaitEvent(st, ar_events_[n_groups], 0));
    }
}

void Plan::stage_h2d(int id, const void* src, uint64_t bytes) {
    if (!finalized_) finalize();
    if (bytes > bufs_.at(id).bytes) throw std::invalid_argument("staged h2d larger than buffer");
    SOL_CUDA(cudaSetDevice(device_));
    if (!copy_stream_) SOL_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    Staged& st = staged_[id];
    if (!st.dev) {
        SOL_CUDA(cudaMalloc(&st.dev, bufs_[id].bytes));
        SOL_CUDA(cudaEventCreateWithFlags(&st.ready, cudaEventDisableTiming));
        SOL_CUDA(cudaEventCreateWithFlags(&st.consumed, cudaEventDisableTiming));
    }
    // re-staging before a run replaces the pending batch: the copies are ordered on copy_stream_
    // the staging area is free once the previous run moved its content into the plan buffer
    if (st.consumed_valid) SOL_CUDA(cudaStreamWaitEvent(copy_stream_, st.consumed, 0));
    SOL_CUDA(cudaMemcpyAsync(st.dev, src, bytes, cudaMemcpyHostToDevice, copy_stream_));
    SOL_CUDA(cudaEventRecord(st.ready, copy_stream_));
    st.bytes = bytes;
    st.pending = true;
}

uint64_t Plan::copy_fence() {
    SOL_CUDA(cudaSetDevice(device_));
    if (!copy_stream_) SOL_CUDA(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking));
    cudaEvent_t& e = fences_[fence_next_ % kFences];
    if (!e) SOL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SOL_CUDA(cudaEventRecord(e, copy_stream_));
    return fence_next_++;
}

void Plan::copy_wait(uint64_t ticket) {
    if (ticket >= fence_next_) throw std::invalid_argument("plan: copy fence ticket was never issued");
    // an overwritten slot holds a LATER fence on the same in-order stream: waiting on it is a
    // superset of the requested wait
    SOL_CUDA(cudaEventSynchronize(fences_[ticket % kFences]));
}

void Plan::consume_staged() {
    for (auto& kv : staged_) {
        Staged& st = kv.second;
        if (!st.pending) continue;
        SOL_CUDA(cudaStreamWaitEvent(stream_, st.ready, 0));
        SOL_CUDA(cudaMemcpyAsync(base_ + bufs_[kv.first].off, st.dev, st.bytes, cudaMemcpyDeviceToDevice, stream_));
        SOL_CUDA(cudaEventRecord(st.consumed, stream_));
        st.consumed_valid = true;
        st.pending = false;
    }
}

void Plan::run(bool use_graph) {
    if (!finalized_) finalize();
    SOL_CUDA(cudaSetDevice(device_));
    consume_staged();
    if (!use_graph) {
        run_steps(stream_);
        has_run_ = true;
        return;
    }
    if (!has_run_) {
        // the first execution is always eager: kernel attributes and frozen-parameter caches are
        // set up outside stream capture (each call is exactly one pass of the plan)
        run_steps(stream_);
        has_run_ = true;
        return;
    }
    if (!graph_exec_) {
        cudaGraph_t g;
        SOL_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
        try {
            run_steps(stream_);
        } catch (...) {
            cudaStreamEndCapture(stream_, &g);
            throw;
        }
        SOL_CUDA(cudaStreamEndCapture(stream_, &g));
        SOL_CUDA(cudaGraphInstantiate(&graph_exec_, g, 0));
        SOL_CUDA(cudaGraphDestroy(g));
    }
    SOL_CUDA(cudaGraphLaunch(graph_exec_, stream_));
}

void Plan::sync() { SOL_CUDA(cudaStreamSynchronize(stream_)); }

void Plan::profile(double* times, int n) {
    if (!finalized_) finalize();
    std::vector<cudaEvent_t> ev(steps_.size() + 1);
    for (auto& e : ev) SOL_CUDA(cudaEventCreate(&e));
    SOL_CUDA(cudaEventRecord(ev[0], stream_));
    for (size_t i = 0; i < steps_.size(); ++i) {
        run_step(steps_[i], stream_);
        SOL_CUDA(cudaEventRecord(ev[i + 1], stream_));
    }
    SOL_CUDA(cudaStreamSynchronize(stream_));
    for (size_t i = 0; i < steps_.size() && static_cast<int>(i) < n; ++i) {
        float ms = 0.f;
        SOL_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
        times[i] = ms * 1000.0;
    }
    for (auto& e : ev) cudaEventDestroy(e);
}

void Plan::h2d(int id, const void* src, uint64_t bytes) {
    if (!finalized_) finalize();
    if (bytes > bufs_.at(id).bytes) throw std::invalid_argument("h2d larger than buffer");
    SOL_CUDA(cudaMemcpyAsync(base_ + bufs_[id].off, src, bytes, cudaMemcpyHostToDevice, stream_));
}

void Plan::d2h(void* dst, int id, uint64_t bytes) {
    if (!finalized_) finalize();
    if (bytes > bufs_.at(id).bytes) throw std::invalid_argument("d2h larger than buffer");
    SOL_CUDA(cudaMemcpyAsync(dst, base_ + bufs_[id].off, bytes, cudaMemcpyDeviceToHost, stream_));
}

void Plan::event_record(int slot) {
    if (slot < 0 || slot >= 16) throw std::invalid_argument("event slot");
    if (!events_[slot]) SOL_CUDA(cudaEventCreate(&events_[slot]));
    SOL_CUDA(cudaEventRecord(events_[slot], stream_));
}

float Plan::event_elapsed(int a, int b) {
    if (a < 0 || a >= 16 || b < 0 || b >= 16 || !events_[a] || !events_[b]) throw std::invalid_argument("event slot");
    float ms = 0.f;
    SOL_CUDA(cudaEventSynchronize(events_[b]));
    SOL_CUDA(cudaEventElapsedTime(&ms, events_[a], events_[b]));
    return ms;
}

void Plan::set_comm(const uint8_t id[128], int rank, int nranks) {
    SOL_CUDA(cudaSetDevice(device_));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    ncclComm_t c;
    nccl_check(ncclCommInitRank(&c, nranks, uid, rank), "init");
    comm_ = c;
    nranks_ = nranks;
}

int Plan::set_lr(float lr) {
    SOL_CUDA(cudaSetDevice(device_));
    int n = 0;
    for (auto& s : steps_)
        if (s.module && s.module->set_lr(lr, stream_)) ++n;
    return n;
}

double Plan::time_step(int i, int reps) {
    if (!finalized_) finalize();
    if (i < 0 || i >= static_cast<int>(steps_.size()) || !steps_[i].module) throw std::invalid_argument("time_step: not a module step");
    SOL_CUDA(cudaSetDevice(device_));
    cudaEvent_t a, b;
    SOL_CUDA(cudaEventCreate(&a));
    SOL_CUDA(cudaEventCreate(&b));
    std::vector<float> t;
    run_step(steps_[i], stream_);  // warm-up (first-run caches)
    for (int r = 0; r < std::max(reps, 1); ++r) {
        SOL_CUDA(cudaEventRecord(a, stream_));
        run_step(steps_[i], stream_);
        SOL_CUDA(cudaEventRecord(b, stream_));
        SOL_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SOL_CUDA(cudaEventElapsedTime(&ms, a, b));
        t.push_back(ms);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    std::sort(t.begin(), t.end());
    return 1000.0 * t[t.size() / 2];
}

bool Plan::step_set_option(int i, int key, int value) {
    if (i < 0 || i >= static_cast<int>(steps_.size()) || !steps_[i].module) throw std::invalid_argument("not a module step");
    const bool ok = steps_[i].module->set_option(key, value);
    if (ok && graph_exec_) {  // a captured graph holds the old launch configuration
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
    }
    return ok;
}

bool Plan::link_bn_stats(int conv_step, int bn_step, int bn_binding) {
    const int n = static_cast<int>(steps_.size());
    if (conv_step < 0 || conv_step >= n || bn_step <= conv_step || bn_step >= n || !steps_[conv_step].module ||
        !steps_[bn_step].module)
        throw std::invalid_argument("link_bn_stats: a conv step followed by a BN step");
    Module* conv = steps_[conv_step].module.get();
    const int blocks = conv->stat_blocks();
    if (blocks <= 0) return false;
    double* partial = nullptr;
    const float* shift = nullptr;
    if (!steps_[bn_step].module->use_producer_stats(bn_binding, blocks, &partial, &shift)) return false;
    conv->set_stat_output(partial, shift);
    if (graph_exec_) {
        cudaGraphExecDestroy(graph_exec_);
        graph_exec_ = nullptr;
    }
    return true;
}

void Plan::comm_info(int* nranks, int* rank, int* cuda_device) const {
    *nranks = 1;
    *rank = 0;
    *cuda_device = device_;
    if (!comm_) return;
    auto c = static_cast<ncclComm_t>(comm_);
    nccl_check(ncclCommCount(c, nranks), "count");
    nccl_check(ncclCommUserRank(c, rank), "rank");
    nccl_check(ncclCommCuDevice(c, cuda_device), "device");
}

}  // namespace solb200
