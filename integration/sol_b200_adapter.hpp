// Reference-side adapter: binds the B200 backend (libsolb200.so, C ABI include/solb200.h) into the
// reference's own C++ interfaces (reference = /root/reference/proj, solmini). This is the code a
// maintainer adds to the reference tree; it is compiled here against the reference headers and
// linked with the reference's own objects by integration/Makefile.
//
//   B200Backend::lower_group / interpret / run_kernel   replace   sol::dfp::lower_group
//       (include/sol/dfp.hpp:43-45), sol::dfp::interpret (dfp.hpp:53, src/dfp_interp.cpp:152-164)
//       and sol::dfp::run_kernel (dfp.hpp:57-58, dfp_interp.cpp:166-198) with the same contract:
//       inputs ordered activations then params exactly as KernelIR::inputs, f32 buffers in the
//       binding metas, arity/length mismatch -> ShapeMismatchError, output written once.
//   B200Provider : sol::dnn::KernelProvider              (include/sol/dnn.hpp:44-64): Conv2d /
//       Linear and their data/weight gradients on tcgen05 tensor cores, served through the
//       reference's candidates / heuristic_choice / autotune / execute_choice (src/dnn.cpp).
//   B200Queue                                            mirrors sol::rt::CommandQueue
//       (include/sol/runtime.hpp:95-145) over sol_b200_queue_*; VirtualPtr values pass unchanged.
//
// Every ABI status maps to the reference's exception types (include/sol/errors.hpp). There is no
// CPU fallback: an op signature the backend has no kernel for is an error at compile time.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "sol/dfp.hpp"
#include "sol/dnn.hpp"
#include "sol/errors.hpp"
#include "sol/kernel_ir.hpp"
#include "sol/model.hpp"
#include "sol/runtime.hpp"
#include "solb200.h"

namespace solb200::ref {

// ABI status -> reference exception (errors.hpp:11-57). `unsupported_as_provider` selects
// NoProviderError (heavy layers, dnn.cpp) over UnsupportedInGroupError (fused groups).
void check(int status, bool unsupported_as_provider = false);

// Device queue: rt::CommandQueue semantics (never-blocking malloc/free over a stream-ordered
// arena, H2D snapshot at enqueue, D2H visible after synchronize, deferred first error).
class B200Queue {
public:
    explicit B200Queue(int device = 0, uint64_t arena_bytes = 1ull << 30, bool coalesce = true);
    ~B200Queue();
    B200Queue(const B200Queue&) = delete;
    B200Queue& operator=(const B200Queue&) = delete;

    sol::rt::VirtualPtr malloc_async(uint64_t bytes);                              // runtime.hpp:104
    void free_async(sol::rt::VirtualPtr p);                                        // :105
    void memcpy_h2d(sol::rt::VirtualPtr dst, const void* src, uint64_t bytes);     // :107
    void memcpy_d2h(void* dst, sol::rt::VirtualPtr src, uint64_t bytes);           // :108
    void launch(sol_b200_module_t m, const std::vector<sol::rt::VirtualPtr>& args);  // :110-113
    void barrier();                                                                // :114
    sol::rt::SyncResult synchronize();                                             // :116
    sol_transfer_stats stats() const;                                              // :118
    sol_b200_queue_t handle() const { return q_; }

private:
    sol_b200_queue_t q_ = nullptr;
};

// One compiled execution unit ("module compile" = lower_group's replacement). `inputs` / `output`
// are exactly the KernelIR bindings lower_group would produce for the same (graph, unit,
// overrides): names, metas, is_param flags, in KernelIR input order.
struct B200Unit {
    sol_b200_module_t module = nullptr;
    std::string name;
    std::vector<sol::TensorBinding> inputs;
    sol::TensorBinding output;
    std::string family;       // kernel family the backend selected
    std::shared_ptr<const void> storage;  // device storage of every argument (adapter-internal)
    ~B200Unit();
};

class B200Backend {
public:
    // dtype: SOL_DT_F32 (f32 storage, TF32 tensor cores) matches the reference's f32 buffers.
    explicit B200Backend(int device = 0, int dtype = SOL_DT_F32, uint64_t arena_bytes = 1ull << 30);

    // lower_group(g, unit, flavor, overrides) -> compiled unit. Accepts fused groups and heavy
    // nodes alike (a heavy unit is a one-op module); unknown op signatures throw.
    std::shared_ptr<B200Unit> lower_group(const sol::ModelGraph& g, const sol::dfp::ExecUnit& unit,
                                          const std::map<std::string, sol::TensorMeta>& overrides = {});
    // dfp::interpret's contract on the device: host f32 buffers in the binding metas.
    void interpret(const B200Unit& k, const std::vector<sol::dfp::BufferRef>& inputs,
                   sol::dfp::BufferRef output);
    // dfp::run_kernel's contract: binds by name, relayouts to the binding metas, returns a tensor.
    sol::Tensor run_kernel(const B200Unit& k, const sol::TensorMap& activations,
                           const std::map<std::string, sol::Tensor>& params);

    B200Queue& queue() { return queue_; }
    int dtype() const { return dtype_; }

private:
    int dtype_;
    B200Queue queue_;
    std::mutex mu_;  // one producer per queue (runtime.hpp:95-100)
};

// Heavy-layer provider "b200" (dnn.hpp:44-64). NHWC activations (ActLayout::ChannelsLast),
// [out,in] weights. execute() returns a new host tensor by value, like the built-in providers;
// the module for each layer shape is compiled once (keyed like the reference's TuneCache).
class B200Provider final : public sol::dnn::KernelProvider {
public:
    explicit B200Provider(std::shared_ptr<B200Backend> backend, double cost = 0.1);
    std::string name() const override { return "b200"; }
    bool supports(sol::OpKind op) const override;
    std::vector<std::string> algorithms(sol::OpKind op) const override;
    std::vector<sol::ActLayout> activation_layouts(sol::OpKind op, const sol::TensorMeta& in_meta) const override;
    std::vector<sol::dnn::WeightOrientation> orientations(sol::OpKind op, sol::DeviceKind dev,
                                                          sol::FlavorId flavor) const override;
    double relative_cost(sol::OpKind op, const std::string& algorithm) const override { return cost_; }
    sol::Tensor execute(const sol::dnn::ImplChoice& choice, const sol::LayerNode& node,
                        const std::vector<const sol::Tensor*>& inputs,
                        const std::vector<const sol::Tensor*>& params) const override;

private:
    std::shared_ptr<B200Backend> backend_;
    double cost_;
    mutable std::mutex mu_;
    mutable std::map<std::string, std::shared_ptr<B200Unit>> modules_;
};

}  // namespace solb200::ref
