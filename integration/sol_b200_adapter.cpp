// Reference-side adapter implementation (see sol_b200_adapter.hpp).
#include "sol_b200_adapter.hpp"

#include <algorithm>
#include <cstring>
#include <stdexcept>

namespace solb200::ref {

using sol::DimPurpose;
using sol::DimTag;
using sol::OpKind;
using sol::Tensor;
using sol::TensorMeta;

void check(int st, bool unsupported_as_provider) {
    if (st == SOL_OK) return;
    const std::string m = sol_b200_last_error();
    switch (st) {
        case SOL_E_SHAPE_MISMATCH: throw sol::ShapeMismatchError(m);
        case SOL_E_UNSUPPORTED:
            if (unsupported_as_provider) throw sol::NoProviderError(m);
            throw sol::UnsupportedInGroupError(m);
        case SOL_E_OVERFLOW: throw sol::ArithmeticOverflowError(m);
        case SOL_E_OUT_OF_REFS: throw sol::OutOfRefsError(m);
        case SOL_E_INVALID_ARGUMENT: throw std::invalid_argument(m);
        default: throw std::runtime_error("solb200 status " + std::to_string(st) + ": " + m);
    }
}

// ---------------------------------------------------------------------------------------------
// queue
// ---------------------------------------------------------------------------------------------

B200Queue::B200Queue(int device, uint64_t arena_bytes, bool coalesce) {
    check(sol_b200_queue_create(device, arena_bytes, coalesce ? 1 : 0, &q_));
}
B200Queue::~B200Queue() {
    if (q_) sol_b200_queue_destroy(q_);
}
sol::rt::VirtualPtr B200Queue::malloc_async(uint64_t bytes) {
    uint64_t v = 0;
    check(sol_b200_malloc_async(q_, bytes, &v));
    return sol::rt::VirtualPtr::from_value(v);
}
void B200Queue::free_async(sol::rt::VirtualPtr p) { check(sol_b200_free_async(q_, p.value())); }
void B200Queue::memcpy_h2d(sol::rt::VirtualPtr d, const void* s, uint64_t n) {
    check(sol_b200_memcpy_h2d(q_, d.value(), s, n));
}
void B200Queue::memcpy_d2h(void* d, sol::rt::VirtualPtr s, uint64_t n) {
    check(sol_b200_memcpy_d2h(q_, d, s.value(), n));
}
void B200Queue::launch(sol_b200_module_t m, const std::vector<sol::rt::VirtualPtr>& args) {
    std::vector<uint64_t> a;
    a.reserve(args.size());
    for (const auto& v : args) a.push_back(v.value());
    check(sol_b200_launch(q_, m, a.data(), static_cast<int32_t>(a.size())));
}
void B200Queue::barrier() { check(sol_b200_barrier(q_)); }
sol::rt::SyncResult B200Queue::synchronize() {
    char msg[1024] = {0};
    const int st = sol_b200_synchronize(q_, msg, sizeof msg);
    sol::rt::SyncResult r;
    r.message = msg;
    switch (st) {
        case SOL_OK: break;
        case SOL_E_USE_AFTER_FREE: r.error = sol::rt::QueueError::UseAfterFree; break;
        case SOL_E_UNKNOWN_REF: r.error = sol::rt::QueueError::UnknownRef; break;
        case SOL_E_OUT_OF_BOUNDS: r.error = sol::rt::QueueError::OutOfBounds; break;
        default: throw std::runtime_error("solb200 device error " + std::to_string(st) + ": " + msg);
    }
    return r;
}
sol_transfer_stats B200Queue::stats() const {
    sol_transfer_stats s{};
    check(sol_b200_stats(q_, &s));
    return s;
}

B200Unit::~B200Unit() {
    if (module) sol_b200_module_destroy(module);
}

// ---------------------------------------------------------------------------------------------
// metas: canonical dims and device storage
// ---------------------------------------------------------------------------------------------

namespace {

constexpr DimTag kN{DimPurpose::None, 0};
constexpr DimTag kC{DimPurpose::Channel, 0};
constexpr DimTag kH{DimPurpose::Pixel, 1};
constexpr DimTag kW{DimPurpose::Pixel, 0};

enum class Kind { Spatial, NC, Scalar, Plain };

Kind kind_of(const TensorMeta& m) {
    if (m.rank() == 0) return Kind::Scalar;
    if (m.find(kH) >= 0 && m.find(kW) >= 0 && m.find(kC) >= 0) return Kind::Spatial;
    if (m.find(kC) >= 0 && m.rank() == 2) return Kind::NC;
    for (const auto& d : m.dims)
        if (d.tag.purpose != DimPurpose::None)
            throw sol::ShapeMismatchError("solb200 adapter: unsupported meta " + m.str());
    return Kind::Plain;
}

// canonical dim tags in order: [N0 C0 P1 P0] / [N0 C0] / [] / [None r-1 .. None 0]
std::vector<DimTag> canon_tags(const TensorMeta& m) {
    switch (kind_of(m)) {
        case Kind::Spatial: return {kN, kC, kH, kW};
        case Kind::NC: return {kN, kC};
        case Kind::Scalar: return {};
        case Kind::Plain: {
            std::vector<DimTag> t;
            for (int i = static_cast<int>(m.rank()) - 1; i >= 0; --i) t.push_back({DimPurpose::None, i});
            return t;
        }
    }
    return {};
}

std::vector<int64_t> canon_dims(const TensorMeta& m) {
    std::vector<int64_t> d;
    for (const auto& t : canon_tags(m)) d.push_back(m.extent_of(t));
    return d;
}

bool f32_output_op(OpKind op) {
    switch (op) {  // stored f32 whatever the plan dtype (frontend/dfp.py F32_OUTPUT_OPS)
        case OpKind::CrossEntropyLoss:
        case OpKind::BatchNormBackGamma:
        case OpKind::BatchNormBackBeta:
        case OpKind::Conv2dBackW:
        case OpKind::Conv2dBackB:
        case OpKind::LinearBackW:
        case OpKind::LinearBackB:
        case OpKind::SgdUpdate:
            return true;
        default:
            return false;
    }
}

int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }

struct Storage {
    Kind kind;
    std::vector<int64_t> dims;  // canonical
    int64_t ld = 0;             // activation row stride (elements)
    int dtype = SOL_DT_F32;
    bool param = false;
    int64_t elems() const {  // stored elements
        if (kind == Kind::Scalar) return 1;
        if (param || kind == Kind::Plain) {
            int64_t n = 1;
            for (auto d : dims) n *= d;
            return n;
        }
        int64_t pix = dims[0];
        if (kind == Kind::Spatial) pix *= dims[2] * dims[3];
        return pix * ld;
    }
    uint64_t bytes() const { return static_cast<uint64_t>(elems()) * (dtype == SOL_DT_BF16 ? 2 : 4); }
};

sol_binding binding_of(const Storage& s) {
    sol_binding b{};
    b.is_param = s.param ? 1 : 0;
    b.dtype = s.dtype;
    b.rank = static_cast<int32_t>(s.dims.size());
    for (size_t i = 0; i < s.dims.size() && i < 4; ++i) b.dims[i] = s.dims[i];
    b.ld = s.ld;
    return b;
}

Storage storage_of(const TensorMeta& m, bool is_param, bool f32_tensor, int plan_dtype) {
    Storage s;
    s.kind = kind_of(m);
    s.dims = canon_dims(m);
    s.param = is_param || s.kind == Kind::Plain;
    s.dtype = (s.param || f32_tensor) ? SOL_DT_F32 : plan_dtype;
    if (!s.param && s.kind != Kind::Scalar) {
        // channels padded to 16 bytes of the PLAN dtype, also for f32-stored tensors (dfp.py storage_ld)
        s.ld = round_up(s.dims[1], plan_dtype == SOL_DT_BF16 ? 8 : 4);
    }
    return s;
}

// memory strides (elements) of the canonical dims in a row-major-tagged meta
std::vector<int64_t> canon_strides(const TensorMeta& m) {
    std::vector<int64_t> stride(m.rank(), 1);
    for (int64_t i = m.rank() - 2; i >= 0; --i) stride[i] = stride[i + 1] * m.dims[i + 1].extent;
    std::vector<int64_t> out;
    for (const auto& t : canon_tags(m)) out.push_back(stride[m.find(t)]);
    return out;
}

// host f32 buffer in `meta` -> stored f32 image (NHWC with ld padding / dense canonical)
void pack(const float* src, const TensorMeta& meta, const Storage& s, std::vector<float>& dst) {
    if (s.dtype != SOL_DT_F32) throw std::invalid_argument("solb200 adapter: host side is f32");
    dst.assign(static_cast<size_t>(s.elems()), 0.0f);
    if (meta.layout.kind != sol::LayoutId::Kind::RowMajorTagged) {
        Tensor t(meta);
        std::memcpy(t.f32(), src, sizeof(float) * meta.element_count());
        TensorMeta rm = sol::apply_act_layout(meta, sol::ActLayout::ChannelsFirst);
        Tensor r = t.relayout(rm);
        pack(r.f32(), rm, s, dst);
        return;
    }
    const auto st = canon_strides(meta);
    switch (s.kind) {
        case Kind::Scalar: dst[0] = src[0]; return;
        case Kind::Plain: {
            const int64_t n = s.elems();
            if (s.dims.size() == 1 || meta == sol::meta_plain(s.dims)) {
                std::memcpy(dst.data(), src, sizeof(float) * n);
                return;
            }
            // any dim order: walk canonical coordinates
            std::vector<int64_t> c(s.dims.size(), 0);
            for (int64_t i = 0; i < n; ++i) {
                int64_t off = 0;
                for (size_t k = 0; k < c.size(); ++k) off += c[k] * st[k];
                dst[i] = src[off];
                for (int64_t k = static_cast<int64_t>(c.size()) - 1; k >= 0; --k) {
                    if (++c[k] < s.dims[k]) break;
                    c[k] = 0;
                }
            }
            return;
        }
        case Kind::NC:
            for (int64_t n = 0; n < s.dims[0]; ++n)
                for (int64_t c = 0; c < s.dims[1]; ++c) dst[n * s.ld + c] = src[n * st[0] + c * st[1]];
            return;
        case Kind::Spatial: {
            const int64_t N = s.dims[0], C = s.dims[1], H = s.dims[2], W = s.dims[3];
            for (int64_t n = 0; n < N; ++n)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t w = 0; w < W; ++w) {
                        float* row = dst.data() + ((n * H + h) * W + w) * s.ld;
                        const float* base = src + n * st[0] + h * st[2] + w * st[3];
                        for (int64_t c = 0; c < C; ++c) row[c] = base[c * st[1]];
                    }
            return;
        }
    }
}

// stored f32 image -> host f32 buffer in `meta`
void unpack(const std::vector<float>& img, const Storage& s, const TensorMeta& meta, float* dst) {
    if (meta.layout.kind != sol::LayoutId::Kind::RowMajorTagged) {
        TensorMeta rm = sol::apply_act_layout(meta, sol::ActLayout::ChannelsFirst);
        Tensor r(rm);
        unpack(img, s, rm, r.f32());
        Tensor t = r.relayout(meta);
        std::memcpy(dst, t.f32(), sizeof(float) * meta.element_count());
        return;
    }
    const auto st = canon_strides(meta);
    switch (s.kind) {
        case Kind::Scalar: dst[0] = img[0]; return;
        case Kind::Plain: {
            const int64_t n = s.elems();
            std::vector<int64_t> c(s.dims.size(), 0);
            for (int64_t i = 0; i < n; ++i) {
                int64_t off = 0;
                for (size_t k = 0; k < c.size(); ++k) off += c[k] * st[k];
                dst[off] = img[i];
                for (int64_t k = static_cast<int64_t>(c.size()) - 1; k >= 0; --k) {
                    if (++c[k] < s.dims[k]) break;
                    c[k] = 0;
                }
            }
            return;
        }
        case Kind::NC:
            for (int64_t n = 0; n < s.dims[0]; ++n)
                for (int64_t c = 0; c < s.dims[1]; ++c) dst[n * st[0] + c * st[1]] = img[n * s.ld + c];
            return;
        case Kind::Spatial: {
            const int64_t N = s.dims[0], C = s.dims[1], H = s.dims[2], W = s.dims[3];
            for (int64_t n = 0; n < N; ++n)
                for (int64_t h = 0; h < H; ++h)
                    for (int64_t w = 0; w < W; ++w) {
                        const float* row = img.data() + ((n * H + h) * W + w) * s.ld;
                        float* base = dst + n * st[0] + h * st[2] + w * st[3];
                        for (int64_t c = 0; c < C; ++c) base[c * st[1]] = row[c];
                    }
            return;
        }
    }
}

sol_attrs attrs_of(const sol::Attrs& a) {
    sol_attrs x{};
    x.out_channels = a.out_channels;
    x.out_features = a.out_features;
    x.kh = a.kh;
    x.kw = a.kw;
    x.sh = a.sh;
    x.sw = a.sw;
    x.ph = a.ph;
    x.pw = a.pw;
    x.groups = a.groups;
    x.has_bias = a.has_bias ? 1 : 0;
    x.min_init = a.min_init;
    x.count_padding = a.count_padding ? 1 : 0;
    x.eps = a.eps;
    x.momentum = a.momentum;
    x.training = a.training ? 1 : 0;
    x.lr = a.lr;
    x.offset = 0;
    return x;
}

int fill_dims(const TensorMeta& m, int64_t* out) {
    const auto d = canon_dims(m);
    for (int i = 0; i < 4; ++i) out[i] = i < static_cast<int>(d.size()) ? d[i] : 0;
    return static_cast<int>(d.size());
}

// Per-unit compile state: the sol_unit_desc and the storage of every argument.
struct Desc {
    std::vector<sol_unit_op> ops;
    std::vector<sol_binding> bindings;
    std::vector<Storage> arg_storage;  // bindings then output
    sol_unit_desc d{};
};

// `meta_of(name)` / `is_param(name)` resolve boundary tensors; `f32_of(name)` tells whether a
// boundary activation is an f32-stored tensor (loss, parameter gradients).
template <class MetaOf, class F32Of>
void build_desc(Desc& D, const sol::ModelGraph& g, const sol::dfp::ExecUnit& u, int dtype, MetaOf meta_of,
                F32Of f32_of) {
    std::vector<std::string> names(u.inputs.begin(), u.inputs.end());
    names.insert(names.end(), u.params.begin(), u.params.end());
    std::map<std::string, int> index;
    for (size_t i = 0; i < names.size(); ++i) index[names[i]] = static_cast<int>(i);
    for (size_t i = 0; i < names.size(); ++i) {
        const bool param = i >= u.inputs.size();
        D.arg_storage.push_back(storage_of(meta_of(names[i]), param, !param && f32_of(names[i]), dtype));
        D.bindings.push_back(binding_of(D.arg_storage.back()));
    }
    std::map<std::string, int> pos;
    for (size_t k = 0; k < u.node_ids.size(); ++k) pos[u.node_ids[k]] = static_cast<int>(k);
    for (const auto& id : u.node_ids) {
        const sol::LayerNode* n = g.find_node(id);
        if (!n) throw sol::ShapeMismatchError("solb200 adapter: unit member '" + id + "' not in graph");
        sol_unit_op o{};
        o.op = static_cast<int32_t>(n->op);  // SOL_OP_* follow sol::OpKind declaration order
        if (n->inputs.size() > SOL_MAX_OP_IN) throw sol::UnsupportedInGroupError("op arity too large: " + id);
        o.n_inputs = static_cast<int32_t>(n->inputs.size());
        for (size_t i = 0; i < n->inputs.size(); ++i) {
            auto p = pos.find(n->inputs[i]);
            o.inputs[i] = p != pos.end() ? -(p->second + 1) : index.at(n->inputs[i]);
        }
        o.n_params = static_cast<int32_t>(n->params.size());
        for (size_t i = 0; i < n->params.size() && i < 4; ++i) o.params[i] = index.at(n->params[i]);
        o.attrs = attrs_of(n->attrs);
        o.saved_rank = n->saved_meta ? fill_dims(*n->saved_meta, o.saved_dims) : 0;
        o.out_rank = n->out_meta ? fill_dims(*n->out_meta, o.out_dims) : 0;
        D.ops.push_back(o);
    }
    const sol::LayerNode* out = g.find_node(u.output);
    D.arg_storage.push_back(storage_of(meta_of(u.output), false, out && f32_output_op(out->op), dtype));
    D.d.kind = u.kind == sol::dfp::ExecUnit::Kind::DfpGroup ? 0 : 1;
    D.d.n_ops = static_cast<int32_t>(D.ops.size());
    D.d.ops = D.ops.data();
    D.d.n_bindings = static_cast<int32_t>(D.bindings.size());
    D.d.bindings = D.bindings.data();
    D.d.output = binding_of(D.arg_storage.back());
    D.d.dtype = dtype;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// backend: module compile + interpret
// ---------------------------------------------------------------------------------------------

B200Backend::B200Backend(int device, int dtype, uint64_t arena_bytes) : dtype_(dtype), queue_(device, arena_bytes) {
    if (dtype != SOL_DT_F32)
        throw std::invalid_argument("solb200 adapter: the reference's buffers are f32 (use SOL_DT_F32)");
}

std::shared_ptr<B200Unit> B200Backend::lower_group(const sol::ModelGraph& g, const sol::dfp::ExecUnit& u,
                                                   const std::map<std::string, TensorMeta>& overrides) {
    // boundary metas exactly as lower_group's Lower::boundary_meta (dfp_lower.cpp:941-957)
    auto meta_of = [&](const std::string& name) -> TensorMeta {
        auto o = overrides.find(name);
        if (o != overrides.end()) return o->second;
        auto p = g.params.find(name);
        if (p != g.params.end()) return p->second.meta();
        return g.meta_of(name);
    };
    auto f32_of = [&](const std::string& name) {
        const sol::LayerNode* n = g.find_node(name);
        return n && f32_output_op(n->op);
    };
    Desc D;
    build_desc(D, g, u, dtype_, meta_of, f32_of);
    auto unit = std::shared_ptr<B200Unit>(new B200Unit());
    unit->name = "kernel";
    for (const auto& nm : u.inputs) unit->inputs.push_back({nm, meta_of(nm), false});
    for (const auto& nm : u.params) unit->inputs.push_back({nm, meta_of(nm), true});
    unit->output = {u.output, meta_of(u.output), false};
    check(sol_b200_module_create(&D.d, &unit->module), u.kind == sol::dfp::ExecUnit::Kind::DnnNode);
    sol_module_info info{};
    check(sol_b200_module_info(unit->module, &info));
    unit->family = info.family;
    if (info.n_args != static_cast<int32_t>(D.arg_storage.size()))
        throw std::logic_error("solb200 adapter: module argument count mismatch");
    unit->storage = std::make_shared<const std::vector<Storage>>(D.arg_storage);
    return unit;
}

void B200Backend::interpret(const B200Unit& k, const std::vector<sol::dfp::BufferRef>& inputs,
                            sol::dfp::BufferRef output) {
    // the reference's argument contract (dfp_interp.cpp:152-161)
    if (inputs.size() != k.inputs.size())
        throw sol::ShapeMismatchError("kernel '" + k.name + "' expects " + std::to_string(k.inputs.size()) +
                                      " inputs, got " + std::to_string(inputs.size()));
    for (size_t i = 0; i < inputs.size(); ++i)
        if (inputs[i].len < k.inputs[i].meta.element_count())
            throw sol::ShapeMismatchError("kernel input '" + k.inputs[i].name + "' too small");
    if (output.len < k.output.meta.element_count()) throw sol::ShapeMismatchError("kernel output buffer too small");
    const auto& st = *static_cast<const std::vector<Storage>*>(k.storage.get());
    std::lock_guard<std::mutex> lk(mu_);
    std::vector<sol::rt::VirtualPtr> args;
    std::vector<float> img;
    for (size_t i = 0; i < inputs.size(); ++i) {
        auto v = queue_.malloc_async(st[i].bytes());
        pack(inputs[i].data, k.inputs[i].meta, st[i], img);
        queue_.memcpy_h2d(v, img.data(), st[i].bytes());  // snapshot at enqueue
        args.push_back(v);
    }
    const Storage& so = st.back();
    auto vo = queue_.malloc_async(so.bytes());
    args.push_back(vo);
    queue_.launch(k.module, args);
    std::vector<float> out(static_cast<size_t>(so.elems()));
    queue_.memcpy_d2h(out.data(), vo, so.bytes());
    for (auto& a : args) queue_.free_async(a);
    auto r = queue_.synchronize();
    if (!r.ok()) throw std::runtime_error("solb200 queue: " + r.message);
    unpack(out, so, k.output.meta, output.data);
}

Tensor B200Backend::run_kernel(const B200Unit& k, const sol::TensorMap& activations,
                               const std::map<std::string, Tensor>& params) {
    // dfp::run_kernel (dfp_interp.cpp:166-198): bind by name, stage to the binding metas
    std::vector<Tensor> staged;
    staged.reserve(k.inputs.size());
    for (const auto& b : k.inputs) {
        const Tensor* src = nullptr;
        if (b.is_param) {
            auto it = params.find(b.name);
            if (it == params.end()) throw sol::ShapeMismatchError("missing kernel param " + b.name);
            src = &it->second;
        } else {
            auto it = activations.find(b.name);
            if (it == activations.end()) throw sol::ShapeMismatchError("missing kernel input " + b.name);
            src = &it->second;
        }
        Tensor t = src->meta().dtype == sol::Dtype::F32 ? *src : src->to_dtype(sol::Dtype::F32);
        if (!(t.meta() == b.meta)) {
            TensorMeta want = b.meta;
            want.dtype = sol::Dtype::F32;
            t = t.relayout(want);
        }
        staged.push_back(std::move(t));
    }
    std::vector<sol::dfp::BufferRef> refs;
    for (auto& t : staged) refs.push_back({t.f32(), t.element_count()});
    TensorMeta om = k.output.meta;
    om.dtype = sol::Dtype::F32;
    Tensor out(om);
    interpret(k, refs, {out.f32(), out.element_count()});
    return out;
}

// ---------------------------------------------------------------------------------------------
// provider
// ---------------------------------------------------------------------------------------------

B200Provider::B200Provider(std::shared_ptr<B200Backend> backend, double cost) : backend_(std::move(backend)), cost_(cost) {}

bool B200Provider::supports(OpKind op) const {
    switch (op) {
        case OpKind::Conv2d:
        case OpKind::Conv2dBackX:
        case OpKind::Conv2dBackW:
        case OpKind::Linear:
        case OpKind::LinearBackX:
        case OpKind::LinearBackW:
            return true;
        default:
            return false;
    }
}

std::vector<std::string> B200Provider::algorithms(OpKind op) const {
    if (op == OpKind::Linear || op == OpKind::LinearBackX || op == OpKind::LinearBackW) return {"tcgen05_gemm"};
    return {"tcgen05_igemm"};
}

std::vector<sol::ActLayout> B200Provider::activation_layouts(OpKind op, const TensorMeta&) const {
    if (op == OpKind::Linear || op == OpKind::LinearBackX || op == OpKind::LinearBackW)
        return {sol::ActLayout::ChannelsFirst};  // [N, C]: both layouts are the same memory order
    return {sol::ActLayout::ChannelsLast};
}

std::vector<sol::dnn::WeightOrientation> B200Provider::orientations(OpKind, sol::DeviceKind, sol::FlavorId) const {
    return {sol::dnn::WeightOrientation::OutIn};
}

Tensor B200Provider::execute(const sol::dnn::ImplChoice& choice, const sol::LayerNode& node,
                             const std::vector<const Tensor*>& ins,
                             const std::vector<const Tensor*>& params) const {
    if (!supports(node.op)) throw sol::NoProviderError(std::string("b200: unsupported op ") + sol::op_name(node.op));
    if (ins.size() != node.inputs.size() || params.size() != node.params.size())
        throw sol::ShapeMismatchError("b200: operand count mismatch for '" + node.id + "'");
    // a one-node graph view carrying the operand metas, compiled once per layer shape
    std::vector<TensorMeta> in_metas;
    std::string key = sol::dnn::TuneCache::key(node, {}, sol::DeviceKind::SimAccel, sol::flavor_scalar());
    for (const Tensor* t : ins) {
        in_metas.push_back(t->meta());
        key += "|" + t->meta().str();  // operands are bound in the layout they arrive in
    }
    key += "|" + std::to_string(node.attrs.has_bias) + "|" + std::to_string(params.size());
    std::shared_ptr<B200Unit> unit;
    {
        std::lock_guard<std::mutex> lk(mu_);
        auto it = modules_.find(key);
        if (it != modules_.end()) unit = it->second;
    }
    sol::ModelGraph g1;
    sol::LayerNode n = node;
    for (size_t i = 0; i < ins.size(); ++i) {
        n.inputs[i] = "in" + std::to_string(i);
        g1.graph_inputs.push_back({n.inputs[i], sol::apply_act_layout(ins[i]->meta(), sol::ActLayout::ChannelsFirst)});
    }
    for (size_t i = 0; i < params.size(); ++i) {
        n.params[i] = "p" + std::to_string(i);
        Tensor w = *params[i];
        if (w.meta().rank() == 2 && sol::dnn::orientation_of(w.meta()) != sol::dnn::WeightOrientation::OutIn)
            w = sol::dnn::orient_weight(w, sol::dnn::WeightOrientation::OutIn);
        g1.params[n.params[i]] = std::move(w);
    }
    n.id = "out";
    g1.nodes.push_back(n);
    g1.outputs = {"out"};
    sol::dfp::ExecUnit u;
    u.kind = sol::dfp::ExecUnit::Kind::DnnNode;
    u.node_ids = {"out"};
    u.output = "out";
    u.inputs = n.inputs;
    u.params = n.params;
    if (!unit) {
        std::map<std::string, TensorMeta> overrides;
        for (size_t i = 0; i < ins.size(); ++i) overrides[n.inputs[i]] = in_metas[i];
        unit = backend_->lower_group(g1, u, overrides);
        std::lock_guard<std::mutex> lk(mu_);
        modules_[key] = unit;
    }
    sol::TensorMap acts;
    for (size_t i = 0; i < ins.size(); ++i) acts[n.inputs[i]] = *ins[i];
    Tensor out = backend_->run_kernel(*unit, acts, g1.params);
    // result in the choice's layout (weight gradients stay in their canonical plain meta)
    if (kind_of(out.meta()) == Kind::Spatial || kind_of(out.meta()) == Kind::NC) {
        TensorMeta want = sol::dnn::materialize(out.meta(), choice.layout);
        if (!(want == out.meta())) out = out.relayout(want);
    }
    return out;
}

}  // namespace solb200::ref
