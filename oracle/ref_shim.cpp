// TEST INFRASTRUCTURE ONLY (oracle). extern "C" shim over the reference solmini library so the
// Python tests, golden-fixture generator and bench.py's reference/cpu_baseline leg can drive the
// reference's own code paths:
//   * the f64 oracle            run_reference        (/root/reference/proj/src/reference.cpp:589-605)
//   * the compiled f32 CPU path run_pipeline -> partition -> lower_group/run_kernel for DFP units
//                               (proj/src/dfp_lower.cpp:70-165, :923-1139; dfp_interp.cpp:166-198)
//                               and heuristic_choice/execute_choice for heavy units
//                               (proj/src/dnn.cpp:99-111, :292-305)
//   * the training graph        build_training_graph (proj/src/autodiff.cpp:230-249)
//   * the partition             dfp::partition       (proj/src/dfp_lower.cpp:70-165)
// Nothing in the product path (paper_2003_10688_b200/) links or loads this library.

#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <json.hpp>

#include "sol/autodiff.hpp"
#include "sol/dfp.hpp"
#include "sol/dnn.hpp"
#include "sol/errors.hpp"
#include "sol/model_io.hpp"
#include "sol/passes.hpp"
#include "sol/reference.hpp"

using namespace sol;

namespace {

thread_local std::string g_err;

struct Session {
    ModelGraph g;                 // shape-inferred graph currently executed
    TensorMap inputs;             // canonical (graph-meta) host inputs
    TensorMap env;                // every tensor produced by the last run
    std::vector<std::pair<std::string, std::string>> param_grads;
};

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

const Tensor* lookup(Session* s, const std::string& name) {
    auto it = s->env.find(name);
    if (it != s->env.end()) return &it->second;
    auto ip = s->g.params.find(name);
    if (ip != s->g.params.end()) return &ip->second;
    auto ii = s->inputs.find(name);
    if (ii != s->inputs.end()) return &ii->second;
    return nullptr;
}

// Canonical meta of a named tensor: graph metas are canonical unless relayouted.
Tensor canonical(const Tensor& t) {
    TensorMeta m = t.meta();
    m.layout = LayoutId{};
    // canonical order: tags sorted N.., C.., P(desc) as produced by the graph builders
    // (meta_nchw lists [N0, C0, P1, P0]); plain params keep their order.
    return t.meta() == m ? t : t.relayout(m);
}

}  // namespace

extern "C" {

const char* solref_last_error() { return g_err.c_str(); }

void* solref_load(const char* model_json, const char* weights, size_t wlen, int64_t batch,
                  int training) {
    Session* s = nullptr;
    int rc = guarded([&] {
        auto sess = std::make_unique<Session>();
        ModelGraph g = parse_model_json(model_json);
        g.params = weights_from_bytes(std::string(weights, wlen));
        g.validate_and_sort();
        g = infer_shapes(g, batch);
        if (training) {
            auto tg = autodiff::build_training_graph(g);
            sess->param_grads = tg.param_grads;
            g = infer_shapes(tg.graph, batch);
        }
        sess->g = std::move(g);
        s = sess.release();
    });
    return rc == 0 ? s : nullptr;
}

void solref_free(void* h) { delete static_cast<Session*>(h); }

// Rewrites the session graph with the reference pass pipeline (passes.cpp:168-178).
int solref_pipeline(void* h) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        s->g = run_pipeline(s->g);
    });
}

int solref_set_input(void* h, const char* name, const float* data, int64_t n) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        const GraphInput* gi = s->g.find_input(name);
        if (!gi) throw ShapeMismatchError(std::string("no graph input ") + name);
        Tensor t(gi->meta);
        if (t.element_count() != n) throw ShapeMismatchError("input size mismatch");
        if (t.meta().dtype == Dtype::F32) std::memcpy(t.f32(), data, n * sizeof(float));
        else for (int64_t i = 0; i < n; ++i) t.set_mem(i, data[i]);
        s->inputs[name] = std::move(t);
    });
}

// Overwrites a parameter (f32 payload in its plain row-major order).
int solref_set_param(void* h, const char* name, const float* data, int64_t n) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        Tensor& t = s->g.params.at(name);
        if (t.element_count() != n) throw ShapeMismatchError("param size mismatch");
        for (int64_t i = 0; i < n; ++i) t.set_mem(i, data[i]);
    });
}

// f64 oracle: every node output (reference.cpp:589-605).
int solref_run_reference(void* h) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        s->env = run_reference(s->g, s->inputs);
    });
}

// autodiff::update_bn_running_stats (autodiff.cpp:356-384) on the session parameters from the last
// run's environment (call solref_run_reference first).
int solref_update_bn_running_stats(void* h) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        autodiff::update_bn_running_stats(s->g, s->g.params, s->env);
    });
}

// The reference's compiled f32 CPU path: partition -> DFP kernels via lower_group/run_kernel,
// heavy layers via the builtin providers' heuristic choice. Runs on the current session graph
// (call solref_pipeline first to apply the reference passes).
int solref_run_compiled(void* h) {
    return guarded([&] {
        auto* s = static_cast<Session*>(h);
        static const dnn::ProviderRegistry reg = dnn::ProviderRegistry::with_builtins();
        DeviceGraph dg = clone_for_device(s->g, DeviceKind::Host, flavor_scalar());
        auto units = dfp::partition(dg);
        TensorMap env = s->inputs;
        for (const auto& u : units) {
            if (u.kind == dfp::ExecUnit::Kind::DfpGroup) {
                KernelIR k = dfp::lower_group(s->g, u, flavor_scalar());
                env[u.output] = dfp::run_kernel(k, env, s->g.params);
            } else {
                const LayerNode* n = s->g.find_node(u.output);
                auto cands = dnn::candidates(reg, s->g, *n, DeviceKind::Host, flavor_scalar());
                auto choice = dnn::heuristic_choice(reg, cands, *n);
                std::vector<const Tensor*> ins, pars;
                for (const auto& in : n->inputs) ins.push_back(&env.at(in));
                for (const auto& p : n->params) pars.push_back(&s->g.params.at(p));
                env[u.output] = dnn::execute_choice(reg, choice, *n, ins, pars);
            }
        }
        s->env = std::move(env);
    });
}

// Element count of a named tensor (env, param or input), -1 if absent.
int64_t solref_numel(void* h, const char* name) {
    auto* s = static_cast<Session*>(h);
    const Tensor* t = lookup(s, name);
    return t ? t->element_count() : -1;
}

// Copies a tensor out in canonical layout as f32.
int64_t solref_get(void* h, const char* name, float* out, int64_t n) {
    int64_t got = -1;
    guarded([&] {
        auto* s = static_cast<Session*>(h);
        const Tensor* t = lookup(s, name);
        if (!t) throw ShapeMismatchError(std::string("no tensor ") + name);
        Tensor c = canonical(*t);
        if (c.element_count() > n) throw ShapeMismatchError("output buffer too small");
        for (int64_t i = 0; i < c.element_count(); ++i) out[i] = static_cast<float>(c.get_mem(i));
        got = c.element_count();
    });
    return got;
}

// JSON documents describing the session: the graph (model_io schema), the partition
// (ExecUnit list) and the parameter->gradient map of a training session.
static int put_string(const std::string& s, char* buf, size_t len) {
    if (s.size() + 1 > len) {
        g_err = "buffer too small: need " + std::to_string(s.size() + 1);
        return static_cast<int>(-(static_cast<long>(s.size()) + 1));
    }
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
}

int solref_graph_json(void* h, char* buf, size_t len) {
    auto* s = static_cast<Session*>(h);
    std::string j;
    if (guarded([&] { j = model_to_json(s->g); }) != 0) return -1;
    return put_string(j, buf, len);
}

int solref_partition_json(void* h, char* buf, size_t len) {
    auto* s = static_cast<Session*>(h);
    std::string out;
    int rc = guarded([&] {
        auto units = dfp::partition(clone_for_device(s->g, DeviceKind::Host, flavor_scalar()));
        nlohmann::json arr = nlohmann::json::array();
        for (const auto& u : units) {
            nlohmann::json ju;
            ju["kind"] = u.kind == dfp::ExecUnit::Kind::DfpGroup ? "dfp" : "dnn";
            ju["node_ids"] = u.node_ids;
            ju["output"] = u.output;
            ju["inputs"] = u.inputs;
            ju["params"] = u.params;
            nlohmann::json ops = nlohmann::json::array();
            for (const auto& id : u.node_ids) ops.push_back(op_name(s->g.find_node(id)->op));
            ju["ops"] = ops;
            arr.push_back(ju);
        }
        out = arr.dump();
    });
    if (rc != 0) return -1;
    return put_string(out, buf, len);
}

int solref_param_grads_json(void* h, char* buf, size_t len) {
    auto* s = static_cast<Session*>(h);
    nlohmann::json arr = nlohmann::json::array();
    for (const auto& [p, gnode] : s->param_grads) arr.push_back({p, gnode});
    return put_string(arr.dump(), buf, len);
}

// Reference metric helpers (tensor.cpp:322-329) over flat canonical buffers.
double solref_oracle_err(const float* a, const float* b, int64_t n) {
    double scale = 0.0;
    for (int64_t i = 0; i < n; ++i) scale = std::max({scale, (double)std::abs(a[i]), (double)std::abs(b[i])});
    double floor = std::max(0.01 * scale, 1e-8), worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double x = a[i], y = b[i];
        worst = std::max(worst, std::abs(x - y) / std::max({std::abs(x), std::abs(y), floor}));
    }
    return worst;
}

}  // extern "C"
