// Drives the reference's OWN compile pipeline (model_io -> infer_shapes -> [autodiff
// build_training_graph] -> run_pipeline -> clone_for_device -> dfp::partition) and its own heavy-layer
// dispatch (ProviderRegistry / candidates / heuristic_choice / execute_choice) with the B200 backend
// plugged in through integration/sol_b200_adapter.*, then checks, against the reference itself:
//   * every fused unit compiled by B200Backend::lower_group carries exactly the KernelIR bindings the
//     reference's lower_group produces, and its device output equals the reference's f64 oracle
//     (reference_node member by member on the same inputs) within 1e-5 -- and, for inference graphs,
//     the reference's own fused-kernel interpreter (dfp::run_kernel) within 1e-5 (the interpreter's
//     training units recompute batch statistics quadratically: minutes per unit, so not run there);
//     movement units bit-exact;
//   * every heavy node dispatched to provider "b200" matches the reference's built-in providers run
//     on the TF32-rounded operands the tensor cores read, within 1e-3 (f32 accumulation order);
//   * the graph outputs match the reference's f64 oracle run_reference within 1e-2 (TF32 through the
//     network); for training graphs the loss within 1e-2 (gradients: per unit, see below);
//   * the contract edges: duplicate registration, interpret arity / length errors, an unservable
//     layer (grouped conv) -> NoProviderError, queue deferred errors.
// Usage: test_adapter <model.json> <weights.solw> <batch> <train 0|1> [seed]
// Prints one JSON line; exit 0 only if every check passed. Test infrastructure (run by
// tests/test_gpu_integration.py on a B200).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <random>
#include <sstream>

#include "sol/autodiff.hpp"
#include "sol/model_io.hpp"
#include "sol/passes.hpp"
#include "sol/reference.hpp"
#include "sol_b200_adapter.hpp"

using namespace sol;

namespace {

int g_fail = 0;
std::vector<std::string> g_notes;

void expect(bool ok, const std::string& what) {
    if (!ok) {
        ++g_fail;
        if (g_notes.size() < 20) g_notes.push_back(what);
    }
}

std::string slurp(const char* path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) throw IoError(std::string("cannot open ") + path);
    std::stringstream ss;
    ss << f.rdbuf();
    return ss.str();
}

bool movement_only(const ModelGraph& g, const dfp::ExecUnit& u) {
    for (const auto& id : u.node_ids) {
        OpKind op = g.find_node(id)->op;
        if (op != OpKind::Flatten && op != OpKind::FlattenBack && op != OpKind::Copy) return false;
    }
    return true;
}

Tensor tf32(const Tensor& t) {
    Tensor r = t;
    float* p = r.f32();
    for (int64_t i = 0; i < r.element_count(); ++i) {
        uint32_t u;
        std::memcpy(&u, p + i, 4);
        u &= 0xFFFFE000u;
        std::memcpy(p + i, &u, 4);
    }
    return r;
}

// max over channels |got - want| / (max over channels of sum |dy|): the rounding bound of a sum
double sum_err(const Tensor& got, const Tensor& want, const Tensor& dy) {
    TensorMeta cf = apply_act_layout(dy.meta(), ActLayout::ChannelsFirst);
    Tensor d = dy.meta() == cf ? dy : dy.relayout(cf);
    const int c_pos = cf.find(DimTag{DimPurpose::Channel, 0});
    const int64_t C = cf.dims[c_pos].extent;
    int64_t inner = 1;
    for (int64_t i = c_pos + 1; i < cf.rank(); ++i) inner *= cf.dims[i].extent;
    std::vector<double> acc(static_cast<size_t>(C), 0.0);
    for (int64_t i = 0; i < d.element_count(); ++i) acc[(i / inner) % C] += std::fabs(d.get_mem(i));
    double scale = 1e-30, diff = 0.0;
    for (double a : acc) scale = std::max(scale, a);
    for (int64_t i = 0; i < got.element_count(); ++i) diff = std::max(diff, std::fabs(got.get_mem(i) - want.get_mem(i)));
    return diff / scale;
}

template <class E, class F>
bool throws(F f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s model.json weights.solw batch train [seed]\n", argv[0]);
        return 2;
    }
    const int64_t batch = std::atoll(argv[3]);
    const bool train = std::atoi(argv[4]) != 0;
    const uint64_t seed = argc > 5 ? std::strtoull(argv[5], nullptr, 10) : 5;
    try {
        ModelGraph g0 = parse_model_json(slurp(argv[1]));
        g0.params = weights_from_bytes(slurp(argv[2]));
        g0.validate_and_sort();
        ModelGraph g = infer_shapes(g0, batch);
        std::vector<std::pair<std::string, std::string>> param_grads;
        if (train) {
            auto tg = autodiff::build_training_graph(g);
            param_grads = tg.param_grads;
            g = infer_shapes(tg.graph, batch);
        }
        g = run_pipeline(g);
        DeviceGraph dg = clone_for_device(g, DeviceKind::Host, flavor_scalar());
        const auto units = dfp::partition(dg);

        // inputs: x ~ U(-1, 1), one-hot labels i % C
        TensorMap inputs;
        std::mt19937_64 rng(seed);
        for (const auto& gi : g.graph_inputs) {
            Tensor t(gi.meta);
            if (gi.name == "t") {
                const int64_t n = gi.meta.dims[0].extent, c = gi.meta.dims[1].extent;
                for (int64_t i = 0; i < n; ++i) t.set({i, i % c}, 1.0);
            } else {
                t.fill_uniform(rng, -1.0, 1.0);
            }
            inputs[gi.name] = std::move(t);
        }

        auto backend = std::make_shared<solb200::ref::B200Backend>(0, SOL_DT_F32);
        dnn::ProviderRegistry reg = dnn::ProviderRegistry::with_builtins();
        const dnn::ProviderRegistry builtins = dnn::ProviderRegistry::with_builtins();
        reg.register_provider(std::make_shared<solb200::ref::B200Provider>(backend));
        expect(throws<DuplicateProviderError>([&] {
                   reg.register_provider(std::make_shared<solb200::ref::B200Provider>(backend));
               }),
               "duplicate provider registration must throw DuplicateProviderError");

        TensorMap env = inputs;
        double worst_dfp = 0.0, worst_heavy = 0.0, worst_interp = 0.0;
        int n_dfp = 0, n_heavy = 0, n_exact = 0;
        bool contract_checked = false;
        auto t0 = std::chrono::steady_clock::now();
        for (const auto& u : units) {
            if (u.kind == dfp::ExecUnit::Kind::DfpGroup) {
                KernelIR k = dfp::lower_group(g, u, flavor_scalar());
                auto b = backend->lower_group(g, u);
                bool same = b->inputs.size() == k.inputs.size() && b->output == k.output;
                for (size_t i = 0; same && i < k.inputs.size(); ++i) same = b->inputs[i] == k.inputs[i];
                expect(same, "bindings of unit " + u.output + " differ from lower_group's KernelIR");
                Tensor got = backend->run_kernel(*b, env, g.params);
                // the reference's f64 oracle on the same inputs, member node by member node
                TensorMap local;
                for (const auto& id : u.node_ids) {
                    const LayerNode* n = g.find_node(id);
                    std::vector<const Tensor*> ins, pars;
                    for (const auto& in : n->inputs) ins.push_back(local.count(in) ? &local.at(in) : &env.at(in));
                    for (const auto& p : n->params) pars.push_back(&g.params.at(p));
                    local[id] = reference_node(*n, ins, pars);
                }
                const Tensor& want = local.at(u.output);
                if (movement_only(g, u)) {
                    bool eq = got.element_count() == want.element_count() && max_rel_err(got, want) == 0.0;
                    expect(eq, "movement unit " + u.output + " not bit-exact");
                    ++n_exact;
                } else {
                    const OpKind op = g.find_node(u.output)->op;
                    // a per-channel sum of dy (bias / beta gradients) can cancel to ~0 (e.g. a conv bias
                    // in front of a BatchNorm): measure it against the magnitude of what was summed
                    const bool reduction = u.node_ids.size() == 1 &&
                                           (op == OpKind::Conv2dBackB || op == OpKind::LinearBackB ||
                                            op == OpKind::BatchNormBackBeta);
                    const double e = reduction ? sum_err(got, want, env.at(g.find_node(u.output)->inputs[0]))
                                               : oracle_err(got, want);
                    worst_dfp = std::max(worst_dfp, e);
                    expect(e <= 1e-5, "fused unit " + u.output + " (" + b->family + ") err " + std::to_string(e));
                }
                if (!train) {  // and the reference's own fused-kernel interpreter (KernelIR semantics)
                    Tensor interp = dfp::run_kernel(k, env, g.params);
                    const double e = oracle_err(got, interp);
                    worst_interp = std::max(worst_interp, e);
                    expect(e <= 1e-5, "fused unit " + u.output + " vs interpret err " + std::to_string(e));
                }
                if (!contract_checked) {  // interpret's argument contract (dfp_interp.cpp:152-161)
                    contract_checked = true;
                    std::vector<dfp::BufferRef> none;
                    std::vector<float> out(static_cast<size_t>(k.output.meta.element_count()));
                    expect(throws<ShapeMismatchError>([&] { backend->interpret(*b, none, {out.data(), 1 << 30}); }),
                           "interpret arity mismatch must throw ShapeMismatchError");
                    std::vector<std::vector<float>> bufs;
                    std::vector<dfp::BufferRef> refs;
                    for (const auto& bi : b->inputs) {
                        bufs.emplace_back(static_cast<size_t>(bi.meta.element_count()), 0.5f);
                        refs.push_back({bufs.back().data(), bi.meta.element_count()});
                    }
                    expect(throws<ShapeMismatchError>([&] { backend->interpret(*b, refs, {out.data(), 1}); }),
                           "short output buffer must throw ShapeMismatchError");
                    if (!refs.empty()) {
                        refs[0].len -= 1;
                        expect(throws<ShapeMismatchError>(
                                   [&] { backend->interpret(*b, refs, {out.data(), static_cast<int64_t>(out.size())}); }),
                               "short input buffer must throw ShapeMismatchError");
                    }
                }
                env[u.output] = std::move(got);
                ++n_dfp;
            } else {
                const LayerNode* n = g.find_node(u.output);
                auto cands = dnn::candidates(reg, g, *n, DeviceKind::Host, flavor_scalar());
                auto choice = dnn::heuristic_choice(reg, cands, *n);
                expect(choice.provider == "b200", "heuristic_choice did not pick b200 for " + n->id);
                std::vector<const Tensor*> ins, pars;
                for (const auto& in : n->inputs) ins.push_back(&env.at(in));
                for (const auto& p : n->params) pars.push_back(&g.params.at(p));
                Tensor got = dnn::execute_choice(reg, choice, *n, ins, pars);
                // the built-in providers on the operands as the tensor cores read them (TF32: low 13
                // mantissa bits dropped); what remains is f32 accumulation order
                std::vector<Tensor> rin, rpar;
                std::vector<const Tensor*> rins, rpars;
                for (const Tensor* t : ins) rin.push_back(tf32(*t));
                for (size_t i = 0; i < pars.size(); ++i) rpar.push_back(pars[i]->meta().rank() >= 2 ? tf32(*pars[i]) : *pars[i]);
                for (auto& t : rin) rins.push_back(&t);
                for (auto& t : rpar) rpars.push_back(&t);
                auto bc = dnn::candidates(builtins, g, *n, DeviceKind::Host, flavor_scalar());
                Tensor want = dnn::execute_choice(builtins, dnn::heuristic_choice(builtins, bc, *n), *n, rins, rpars);
                const double e = oracle_err(got, want);
                worst_heavy = std::max(worst_heavy, e);
                expect(e <= 1e-3, "heavy node " + n->id + " err " + std::to_string(e));
                env[u.output] = std::move(got);
                ++n_heavy;
            }
        }
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

        // end to end against the reference's f64 oracle
        TensorMap ref = run_reference(g, inputs);
        double worst_out = 0.0;
        for (const auto& o : g.outputs) {
            if (train && !param_grads.empty()) break;  // training graphs: gradients below
            const double e = oracle_err(env.at(o), ref.at(o));
            worst_out = std::max(worst_out, e);
            expect(e <= 1e-2, "graph output " + o + " err " + std::to_string(e));
        }
        if (std::getenv("SOL_ADAPTER_TRACE")) {  // first tensors where the device chain leaves the oracle
            int shown = 0;
            for (const auto& u : units) {
                const double e = oracle_err(env.at(u.output), ref.at(u.output));
                if (e > 1e-2 && shown++ < 12) {
                    const Tensor& a = env.at(u.output);
                    const Tensor& b = ref.at(u.output);
                    std::fprintf(stderr, "trace %s op %s err %.3e  got[0..2] %g %g  want %g %g\n", u.output.c_str(),
                                 op_name(g.find_node(u.output)->op), e, a.get_mem(0), a.get_mem(1 % a.element_count()),
                                 b.get_mem(0), b.get_mem(1 % b.element_count()));
                }
            }
        }
        // training: the loss within 1e-2 of the oracle's (the TF32 output bar). Parameter gradients of
        // a random-init BatchNorm net are ill-conditioned (BN backward is a small residual of large terms), so the oracle's own
        // gradients move by O(1) under TF32 rounding of its inputs: they are held to the per-unit bars
        // above (each backward unit on the same inputs) and reported here, not asserted end to end.
        double worst_grad = 0.0, loss_err = 0.0;
        for (const auto& pg : param_grads) worst_grad = std::max(worst_grad, oracle_err(env.at(pg.second), ref.at(pg.second)));
        for (const auto& nd : g.nodes) {
            if (nd.op != OpKind::CrossEntropyLoss) continue;
            const double a = env.at(nd.id).get_mem(0), b = ref.at(nd.id).get_mem(0);
            loss_err = std::max(loss_err, std::fabs(a - b) / std::max(std::fabs(b), 1e-12));
        }
        if (train) expect(loss_err <= 1e-2, "loss err " + std::to_string(loss_err));

        // a layer the backend cannot serve: grouped (non-depthwise) conv -> NoProviderError
        {
            ModelGraph gg;
            gg.graph_inputs.push_back({"x", meta_nchw(1, 8, 6, 6)});
            LayerNode c;
            c.id = "c";
            c.op = OpKind::Conv2d;
            c.attrs.out_channels = 8;
            c.attrs.kh = c.attrs.kw = 3;
            c.attrs.ph = c.attrs.pw = 1;
            c.attrs.groups = 2;
            c.attrs.has_bias = false;
            c.inputs = {"x"};
            c.params = {"c.W"};
            gg.nodes.push_back(c);
            gg.outputs = {"c"};
            gg.params["c.W"] = Tensor(meta_plain({8, 4, 3, 3}));
            gg = infer_shapes(gg, 1);
            Tensor x(meta_nchw(1, 8, 6, 6));
            const dnn::KernelProvider& p = reg.at("b200");
            dnn::ImplChoice ch{"b200", "tcgen05_igemm", ActLayout::ChannelsLast, dnn::WeightOrientation::OutIn};
            expect(throws<NoProviderError>([&] { p.execute(ch, *gg.find_node("c"), {&x}, {&gg.params.at("c.W")}); }),
                   "grouped conv must throw NoProviderError (no CPU fallback)");
        }

        // queue: deferred first error (runtime.cpp:157-256) through the adapter's B200Queue
        {
            solb200::ref::B200Queue q(0, 1 << 24);
            auto a = q.malloc_async(4096);
            q.free_async(a);
            std::vector<uint8_t> host(4096, 1);
            q.memcpy_h2d(a, host.data(), host.size());  // use after free: deferred
            auto r = q.synchronize();
            expect(r.error == rt::QueueError::UseAfterFree, "queue use-after-free must surface at synchronize");
        }

        std::printf(
            "{\"units\": %zu, \"dfp_units\": %d, \"heavy_units\": %d, \"movement_exact\": %d, \"worst_dfp_err\": %.3e, "
            "\"worst_interp_err\": %.3e, \"worst_heavy_err\": %.3e, \"worst_output_err\": %.3e, \"worst_grad_err\": %.3e, \"loss_err\": %.3e, \"device_secs\": %.2f, "
            "\"failures\": %d",
            units.size(), n_dfp, n_heavy, n_exact, worst_dfp, worst_interp, worst_heavy, worst_out, worst_grad, loss_err, secs, g_fail);
        std::printf(", \"notes\": [");
        for (size_t i = 0; i < g_notes.size(); ++i) std::printf("%s\"%s\"", i ? ", " : "", g_notes[i].c_str());
        std::printf("]}\n");
        return g_fail == 0 ? 0 : 1;
    } catch (const std::exception& e) {
        std::printf("{\"error\": \"%s\"}\n", e.what());
        return 3;
    }
}
