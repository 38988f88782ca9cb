// Execution-unit modules: a compiled ExecUnit (dfp::ExecUnit, include/sol/dfp.hpp:21-28) bound
// to one hand-written sm_100a kernel family (DFP groups) or tcgen05 provider (heavy nodes).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "../../include/solb200.h"
#include "common.cuh"

namespace solb200 {

struct UnsupportedError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ShapeError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

class Module {
public:
    virtual ~Module();
    // args: bindings in order, then the output (device pointers)
    virtual void run(void* const* args, int nargs, void* scratch, cudaStream_t s, bool frozen) = 0;
    virtual size_t scratch_bytes() const { return 0; }
    // Extra outputs written by this module on behalf of sibling units (mask bits; see
    // sol_b200_module_set_sibling_outputs). Returns false if the module cannot produce them.
    virtual bool set_sibling_outputs(int mask) { return mask == 0; }
    // Module options (SOL_MODOPT_*); returns false when the option does not apply to the module.
    virtual bool set_option(int key, int value) { return false; }
    // Runtime learning rate of SgdUpdate modules (stream-ordered device write; graph replays read it).
    virtual bool set_lr(float lr, cudaStream_t s) { return false; }
    // Weight packing of this run issued ahead of the plan's steps (inside a pack batch, pack.cuh);
    // false when the module packs nothing this run.
    virtual bool prepack(void* const* args, cudaStream_t s, bool frozen) { return false; }
    // BatchNorm statistics from the producing conv's epilogue (sol_b200_module_link_bn_stats):
    // a conv reports how many partial blocks its epilogue would write (0: cannot) and takes the
    // buffers; a BN unit switches the BN whose input is `binding` to those partials and returns
    // its partial buffer and shift array (nullptr: no such training BN).
    virtual int stat_blocks() const { return 0; }
    virtual void set_stat_output(double* partial, const float* shift) {}
    virtual bool use_producer_stats(int binding, int blocks, double** partial, const float** shift) { return false; }

    std::string family;
    int n_args = 0;
    int launches = 1;
    int launches_frozen = -1;  // per run in a frozen plan (-1: same as launches)
    double algo_bytes = 0.0;
    double algo_flops = 0.0;
    std::vector<size_t> arg_bytes;  // minimum bytes each arg must span (queue bounds checks)

protected:
    // module-owned device constants / caches (freed with the module)
    void* dev_alloc(size_t bytes);
    std::vector<void*> owned_;
};

std::unique_ptr<Module> compile_unit(const sol_unit_desc& d);

}  // namespace solb200
