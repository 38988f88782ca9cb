// Device runtime: stream-ordered arena, the CommandQueue mirror (rt::CommandQueue,
// include/sol/runtime.hpp:95-145) and execution plans (fe::DevicePlan, frontend.hpp:52-61).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "module.hpp"

namespace solb200 {

// First-fit sub-allocator over one device slab. Allocation and free are host-side bookkeeping
// only: every consumer is ordered on the owning stream, so a freed block may be handed out again
// immediately (the cudaMallocAsync contract) and nothing ever blocks the launch stream.
class Arena {
public:
    Arena() = default;
    ~Arena();
    // stream != nullptr: the slab comes from cudaMallocAsync on that stream (stream-ordered growth)
    void init(size_t bytes, cudaStream_t stream = nullptr);
    // returns offset or -1 when full
    int64_t alloc(size_t bytes);
    void free(int64_t off);
    uint8_t* base() const { return base_; }
    size_t capacity() const { return cap_; }
    size_t in_use() const { return used_; }

private:
    uint8_t* base_ = nullptr;
    size_t cap_ = 0, used_ = 0;
    std::map<int64_t, size_t> free_;   // offset -> size
    std::map<int64_t, size_t> live_;   // offset -> size
};

// Reusable page-locked staging for the queue's copies: slabs grow geometrically and are recycled
// after every synchronize (the stream is idle then), so steady-state copies never call
// cudaMallocHost (a slow, implicitly synchronising call).
class PinnedPool {
public:
    ~PinnedPool();
    void* get(size_t bytes);
    void reset();
    uint64_t slabs() const { return slabs_.size(); }

private:
    struct Slab {
        uint8_t* p;
        size_t cap, used;
    };
    std::vector<Slab> slabs_;
    size_t cur_ = 0;
};

struct QueueErr {
    int code;
    std::string msg;
};

class Queue {
public:
    Queue(int device, size_t arena_bytes, bool coalesce);
    ~Queue();

    uint64_t malloc_async(uint64_t bytes);
    void free_async(uint64_t vptr);
    void memcpy_h2d(uint64_t dst, const void* src, uint64_t bytes);
    void memcpy_d2h(void* dst, uint64_t src, uint64_t bytes);
    void launch(Module* m, const uint64_t* args, int nargs);
    void barrier();
    int synchronize(std::string* msg);
    sol_transfer_stats stats() const {
        sol_transfer_stats s = stats_;
        s.pinned_slabs = pinned_.slabs();
        s.device_slabs = slabs_.size();
        return s;
    }
    cudaStream_t stream() const { return stream_; }

private:
    struct Alloc {
        int slab;
        int64_t off;
        uint64_t bytes;
    };
    // first fit over the arena slabs; a full arena grows by a new stream-ordered slab
    std::pair<int, int64_t> arena_alloc(size_t bytes);
    uint8_t* arena_ptr(int slab, int64_t off) const { return slabs_[slab]->base() + off; }
    // resolves to a device pointer; on failure records the deferred error and returns nullptr
    uint8_t* resolve(uint64_t vptr, uint64_t bytes);
    bool failed() const { return err_.code != 0; }
    void defer(int code, const std::string& msg);
    void close_copy_run();
    void* staging(size_t bytes);
    void mark_start();

    int device_;
    cudaStream_t stream_ = nullptr;
    std::vector<std::unique_ptr<Arena>> slabs_;
    PinnedPool pinned_;
    bool coalesce_;
    std::map<uint32_t, Alloc> allocs_;
    std::map<uint32_t, bool> freed_;
    uint64_t next_ref_ = 1;
    QueueErr err_{0, ""};
    sol_transfer_stats stats_{};
    // open H2D copy run (coalescing): payload staged in pinned memory
    struct PendingCopy {
        uint8_t* dst;
        uint64_t off;
        uint64_t bytes;
    };
    std::vector<PendingCopy> run_;
    std::vector<uint8_t> run_payload_;
    struct D2H {
        void* user;
        void* pinned;
        uint64_t bytes;
    };
    std::vector<D2H> d2h_;
    int scratch_slab_ = -1;
    int64_t scratch_off_ = -1;
    size_t scratch_bytes_ = 0;
    cudaEvent_t ev_start_ = nullptr, ev_end_ = nullptr;
    bool timing_ = false;
};

class Plan {
public:
    explicit Plan(int device);
    ~Plan();
    int add_buffer(uint64_t bytes, bool persistent);
    void add_step(std::unique_ptr<Module> m, const int32_t* ids, int n);
    void add_allreduce(int id, uint64_t count, int dtype, float scale);
    void finalize();
    void* buffer_ptr(int id) const;
    void set_frozen(bool f) { frozen_ = f; }
    void run(bool use_graph);
    void sync();
    cudaStream_t stream() const { return stream_; }
    void profile(double* times_us, int n);
    int num_steps() const { return static_cast<int>(steps_.size()); }
    const Module* step_module(int i) const { return steps_[i].module.get(); }
    uint64_t arena_bytes() const { return total_; }
    void set_comm(const uint8_t id[128], int rank, int nranks);
    void comm_info(int* nranks, int* rank, int* cuda_device) const;
    int set_lr(float lr);  // SgdUpdate steps' runtime learning rate; returns how many steps took it
    double time_step(int i, int reps);  // median device time (us) of step i run alone, eagerly
    bool step_set_option(int i, int key, int value);
    // BN statistics from a conv step's epilogue for a later training-BN step (Module::use_producer_stats)
    bool link_bn_stats(int conv_step, int bn_step, int bn_binding);
    void h2d(int id, const void* src, uint64_t bytes);
    void stage_h2d(int id, const void* src, uint64_t bytes);
    // host-side fences on the copy stream: a ticket taken after stage_h2d() calls is complete once
    // those copies have read their pinned sources (the host may then refill them)
    uint64_t copy_fence();
    void copy_wait(uint64_t ticket);
    void d2h(void* dst, int id, uint64_t bytes);
    void event_record(int slot);
    float event_elapsed(int a, int b);

private:
    struct Buf {
        uint64_t bytes;
        bool persistent;
        int first = -1, last = -1;
        uint64_t off = 0;
    };
    struct Step {
        std::unique_ptr<Module> module;
        std::vector<int> ids;
        // all-reduce step
        int ar_id = -1;
        uint64_t ar_count = 0;
        int ar_dtype = 0;
        float ar_scale = 1.f;
    };
    void run_step(Step& s, cudaStream_t st);
    void run_steps(cudaStream_t st);
    void consume_staged();
    struct Staged {
        void* dev = nullptr;
        uint64_t bytes = 0;
        bool pending = false, consumed_valid = false;
        cudaEvent_t ready = nullptr, consumed = nullptr;
    };

    int device_;
    cudaStream_t stream_ = nullptr;
    std::vector<Buf> bufs_;
    std::vector<Step> steps_;
    uint8_t* base_ = nullptr;
    uint64_t total_ = 0, scratch_off_ = 0, scratch_bytes_ = 0;
    bool finalized_ = false, frozen_ = false, has_run_ = false;
    cudaGraphExec_t graph_exec_ = nullptr;
    void* comm_ = nullptr;  // ncclComm_t
    int nranks_ = 1;
    cudaEvent_t events_[16] = {};
    cudaStream_t copy_stream_ = nullptr;
    // gradient all-reduce buckets run on comm_stream_, overlapped with the rest of the backward
    // pass: fork (event on the plan stream) before each bucket, join before the first module step
    // after the last bucket
    cudaStream_t comm_stream_ = nullptr;
    std::vector<cudaEvent_t> ar_events_;
    std::map<int, Staged> staged_;
    static constexpr int kFences = 8;
    cudaEvent_t fences_[kFences] = {};
    uint64_t fence_next_ = 0;
};

}  // namespace solb200
