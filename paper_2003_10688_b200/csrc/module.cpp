// Unit compiler: sol_unit_desc (ops + attrs + boundary bindings, i.e. an ExecUnit with its
// KernelIR bindings) -> one hand-written kernel family. There is no generic fallback: a unit whose
// op signature no family covers fails at compile time with SOL_E_UNSUPPORTED, mirroring the
// reference's "unknown op -> hard error" policy (dfp_lower.cpp UnsupportedInGroupError).
//
// Op semantics followed (reference = /root/reference/proj):
//   BatchNorm2d inference  dfp_lower.cpp:454-472 / reference.cpp:216-237 (gamma*(x-mu)*rstd+beta)
//   BatchNorm2d training   bn_batch_stats dfp_lower.cpp:362-390 (biased batch variance)
//   ReLU / Add / Copy      dfp_lower.cpp:399-404
//   Max/AvgPool2d          dfp_lower.cpp:406-434 (min_init, count_padding)
//   GlobalAvgPool          dfp_lower.cpp:436-452
//   depthwise Conv2d       dfp_lower.cpp:519-540 (groups == Cin == Cout)
//   backward units         dfp_lower.cpp:542-753, :800-868; reference.cpp:294-584
#include "module.hpp"

#include <cmath>
#include <cstring>
#include <map>
#include <set>

#include "dfp.cuh"
#include "igemm.cuh"
#include "pack.cuh"

namespace solb200 {

Module::~Module() {
    for (void* p : owned_) cudaFree(p);
}

void* Module::dev_alloc(size_t bytes) {
    void* p = nullptr;
    SOL_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
    SOL_CUDA(cudaMemset(p, 0, std::max<size_t>(bytes, 16)));
    owned_.push_back(p);
    return p;
}

namespace {

struct Geo {
    int64_t N = 1, C = 1, H = 1, W = 1, ld = 1;
    int rank = 0;
    int64_t numel() const { return N * C * H * W; }
    int64_t pixels() const { return N * H * W; }
};

Geo geo_of_dims(int rank, const int64_t* d, int64_t ld) {
    Geo g;
    g.rank = rank;
    if (rank == 4) {
        g.N = d[0]; g.C = d[1]; g.H = d[2]; g.W = d[3];
    } else if (rank == 2) {
        g.N = d[0]; g.C = d[1];
    } else if (rank == 1) {
        g.C = d[0];
    } else if (rank == 3) {
        g.C = d[0] * d[1] * d[2];
    }
    g.ld = ld > 0 ? ld : g.C;
    return g;
}

Geo geo_b(const sol_binding& b) { return geo_of_dims(b.rank, b.dims, b.ld); }

int64_t param_numel(const sol_binding& b) {
    int64_t n = 1;
    for (int i = 0; i < b.rank; ++i) n *= b.dims[i];
    return n;
}

size_t elem_size(int dtype) { return dtype == DT_BF16 ? 2 : 4; }

bool is_heavy_op(int op) {
    return op == SOL_OP_CONV2D || op == SOL_OP_LINEAR || op == SOL_OP_CONV2DBACKX ||
           op == SOL_OP_CONV2DBACKW || op == SOL_OP_LINEARBACKX || op == SOL_OP_LINEARBACKW;
}

bool is_depthwise(const sol_unit_op& o, int64_t cin) {
    return o.op == SOL_OP_CONV2D && o.attrs.groups > 1 && o.attrs.groups == o.attrs.out_channels &&
           o.attrs.groups == cin;
}

[[noreturn]] void unsupported(const std::string& what) { throw UnsupportedError(what); }

// bytes an activation binding occupies in plan storage
size_t binding_bytes(const sol_binding& b) {
    if (b.is_param) return static_cast<size_t>(param_numel(b)) * 4;
    if (b.rank == 0) return elem_size(b.dtype);
    Geo g = geo_b(b);
    return static_cast<size_t>(g.pixels() * g.ld) * elem_size(b.dtype);
}

void fill_arg_bytes(Module& m, const sol_unit_desc& d) {
    m.arg_bytes.clear();
    for (int i = 0; i < d.n_bindings; ++i) m.arg_bytes.push_back(binding_bytes(d.bindings[i]));
    m.arg_bytes.push_back(binding_bytes(d.output));
    m.n_args = d.n_bindings + 1;
}

// ---------------------------------------------------------------------------------------------
// fused bottleneck tail (inference, plan-level fusion): relu( bn1(conv1x1(h)) + bn2(conv1x1_s(x)) )
// as ONE dual GEMM: both BatchNorm scales folded into the packed weights, shifts into one bias;
// the downsample branch's output never round-trips through HBM. Unit ops:
//   [Conv2d(h), BatchNorm2d, Conv2d(x), BatchNorm2d, Add, (ReLU | ReLU6)]
// ---------------------------------------------------------------------------------------------

class DualConvModule : public Module {
public:
    explicit DualConvModule(const sol_unit_desc& d) : dtype_(d.dtype) {
        fill_arg_bytes(*this, d);
        if (d.n_ops < 5 || d.n_ops > 6) unsupported("dual conv unit: bad op count");
        const sol_unit_op &c1 = d.ops[0], &n1 = d.ops[1], &c2 = d.ops[2], &n2 = d.ops[3], &ad = d.ops[4];
        if (c1.op != SOL_OP_CONV2D || n1.op != SOL_OP_BATCHNORM2D || c2.op != SOL_OP_CONV2D ||
            n2.op != SOL_OP_BATCHNORM2D || ad.op != SOL_OP_ADD)
            unsupported("dual conv unit: op pattern");
        if (n1.inputs[0] != -1 || n2.inputs[0] != -3 || c1.inputs[0] < 0 || c2.inputs[0] < 0)
            unsupported("dual conv unit: operand wiring");
        if (!((ad.inputs[0] == -2 && ad.inputs[1] == -4) || (ad.inputs[0] == -4 && ad.inputs[1] == -2)))
            unsupported("dual conv unit: Add must join both branches");
        if (n1.attrs.training || n2.attrs.training) unsupported("dual conv unit: inference BatchNorm only");
        for (const sol_unit_op* c : {&c1, &c2}) {
            if (c->attrs.kh != 1 || c->attrs.kw != 1 || c->attrs.ph || c->attrs.pw || c->attrs.groups > 1)
                unsupported("dual conv unit: 1x1 convolutions only");
        }
        if (c1.attrs.sh != 1 || c1.attrs.sw != 1 || c2.attrs.sh != c2.attrs.sw) unsupported("dual conv unit: strides");
        act_ = 0;
        if (d.n_ops == 6) {
            const sol_unit_op& r = d.ops[5];
            if (r.inputs[0] != -5 || (r.op != SOL_OP_RELU && r.op != SOL_OP_RELU6)) unsupported("dual conv unit: activation");
            act_ = r.op == SOL_OP_RELU ? 1 : 2;
        }
        if (dtype_ != DT_BF16) unsupported("dual conv unit: bf16 only");
        i1_ = c1.inputs[0];
        i2_ = c2.inputs[0];
        in1_ = geo_b(d.bindings[i1_]);
        in2_ = geo_b(d.bindings[i2_]);
        out_ = geo_b(d.output);
        s2_ = static_cast<int>(c2.attrs.sh ? c2.attrs.sh : 1);
        if (in1_.C % 64 || in2_.C % 64 || in1_.ld != in1_.C || in2_.ld != in2_.C || out_.ld % 8)
            unsupported("dual conv unit: channels must be 128-byte blocks");
        w1_ = c1.params[0];
        cb1_ = (c1.attrs.has_bias && c1.n_params > 1) ? c1.params[1] : -1;
        w2_ = c2.params[0];
        cb2_ = (c2.attrs.has_bias && c2.n_params > 1) ? c2.params[1] : -1;
        for (int k = 0; k < 4; ++k) {
            bn1_[k] = n1.params[k];
            bn2_[k] = n2.params[k];
        }
        eps1_ = n1.attrs.eps;
        eps2_ = n2.attrs.eps;
        cout_ = static_cast<int>(out_.C);
        packed_ = dev_alloc(static_cast<size_t>(cout_) * (in1_.C + in2_.C) * 2);
        bias_ = static_cast<float*>(dev_alloc(static_cast<size_t>(cout_) * 4));
        family = "conv_fprop_fused_tcgen05";
        algo_flops = 2.0 * out_.pixels() * cout_ * (in1_.C + in2_.C);
        algo_bytes = (in1_.pixels() * in1_.ld + double(out_.pixels()) * in2_.ld + out_.pixels() * out_.ld) * 2.0 +
                     double(cout_) * (in1_.C + in2_.C) * 2.0;
        launches = 2;
        launches_frozen = 1;  // the weight fold is cached once the plan is frozen
    }
    void run(void* const* args, int nargs, void*, cudaStream_t s, bool frozen) override {
        if (nargs != n_args) throw std::invalid_argument("dual conv: wrong argument count");
        if (!(frozen && packed_valid_)) {
            auto P = [&](int i) { return i >= 0 ? static_cast<const float*>(args[i]) : nullptr; };
            DualFold f{P(w1_), P(cb1_), P(bn1_[0]), P(bn1_[1]), P(bn1_[2]), P(bn1_[3]),
                       P(w2_), P(cb2_), P(bn2_[0]), P(bn2_[1]), P(bn2_[2]), P(bn2_[3]),
                       eps1_, eps2_, cout_, static_cast<int>(in1_.C), static_cast<int>(in2_.C)};
            pack_dual_weight(f, packed_, bias_, s);
            packed_valid_ = true;
        }
        IgemmArgs g;
        g.mode = IG_FPROP;
        g.dtype = DT_BF16;
        g.out_dtype = DT_BF16;
        g.src = args[i1_];
        g.wt = packed_;
        g.bias = bias_;
        g.out = args[nargs - 1];
        g.N = static_cast<int>(out_.N);
        g.SH = static_cast<int>(in1_.H);
        g.SW = static_cast<int>(in1_.W);
        g.SC = static_cast<int>(in1_.C);
        g.OH = static_cast<int>(out_.H);
        g.OW = static_cast<int>(out_.W);
        g.Nout = cout_;
        g.K_pad = static_cast<int>(in1_.C + in2_.C);
        g.K1 = static_cast<int>(in1_.C);
        g.ldo = static_cast<int>(out_.ld);
        g.act = act_;
        g.src2 = args[i2_];
        g.SH2 = static_cast<int>(in2_.H);
        g.SW2 = static_cast<int>(in2_.W);
        g.SC2 = static_cast<int>(in2_.C);
        g.s2 = s2_;
        g.tile_n = tile_n_;
        igemm_launch(g, s);
    }
    bool set_option(int key, int value) override {
        if (key != SOL_MODOPT_TILE_N || (value != 0 && value != 128 && value != 256)) return false;
        tile_n_ = value;
        return true;
    }

private:
    int tile_n_ = 0;
    int dtype_, act_ = 0, i1_ = -1, i2_ = -1, s2_ = 1, cout_ = 0;
    Geo in1_, in2_, out_;
    int w1_ = -1, cb1_ = -1, w2_ = -1, cb2_ = -1, bn1_[4] = {}, bn2_[4] = {};
    float eps1_ = 1e-5f, eps2_ = 1e-5f;
    void* packed_ = nullptr;
    float* bias_ = nullptr;
    bool packed_valid_ = false;
};

// ---------------------------------------------------------------------------------------------
// heavy layers: tcgen05 implicit GEMM (KernelProvider::execute replacement, dnn.hpp:61-63)
// ---------------------------------------------------------------------------------------------

class HeavyModule : public Module {
public:
    explicit HeavyModule(const sol_unit_desc& d) : dtype_(d.dtype) {
        const sol_unit_op& o = d.ops[0];
        op_ = o.op;
        const sol_attrs& a = o.attrs;
        kh_ = static_cast<int>(a.kh ? a.kh : 1);
        kw_ = static_cast<int>(a.kw ? a.kw : 1);
        sh_ = static_cast<int>(a.sh ? a.sh : 1);
        sw_ = static_cast<int>(a.sw ? a.sw : 1);
        ph_ = static_cast<int>(a.ph);
        pw_ = static_cast<int>(a.pw);
        if (op_ == SOL_OP_LINEAR || op_ == SOL_OP_LINEARBACKX || op_ == SOL_OP_LINEARBACKW) {
            kh_ = kw_ = sh_ = sw_ = 1;
            ph_ = pw_ = 0;
        }
        if (a.groups > 1 && (op_ == SOL_OP_CONV2D || op_ == SOL_OP_CONV2DBACKX || op_ == SOL_OP_CONV2DBACKW))
            unsupported("grouped (non-depthwise) convolution has no B200 provider");
        const int bk = dtype_ == DT_BF16 ? 64 : 32;
        in_ = geo_b(d.bindings[o.inputs[0]]);
        out_ = geo_b(d.output);
        fill_arg_bytes(*this, d);
        switch (op_) {
            case SOL_OP_CONV2D:
            case SOL_OP_LINEAR: {
                family = op_ == SOL_OP_CONV2D ? "conv_fprop_tcgen05" : "linear_tcgen05";
                w_idx_ = o.params[0];
                b_idx_ = (a.has_bias && o.n_params > 1) ? o.params[1] : -1;
                cin_ = in_.C;
                cout_ = out_.C;
                if (op_ == SOL_OP_CONV2D) {  // the conv's own grid (the unit output may be a fused pool's)
                    conv_oh_ = static_cast<int>((in_.H + 2 * ph_ - kh_) / sh_ + 1);
                    conv_ow_ = static_cast<int>((in_.W + 2 * pw_ - kw_) / sw_ + 1);
                }
                kpad_ = static_cast<int>(round_up(static_cast<int64_t>(kh_) * kw_ * in_.ld, bk));
                nchw_in_ = d.bindings[o.inputs[0]].is_param == 2;
                if (nchw_in_ && op_ != SOL_OP_CONV2D) unsupported("canonical NCHW input only for stem convolutions");
                if (op_ == SOL_OP_CONV2D) {
                    // few-channel stem: halo-tile kernel with its own K order (stem.cu)
                    IgemmArgs g = fprop_args(nullptr, nullptr);
                    g.K_pad = stem_kpad(kh_);
                    if (stem_supported(g)) {
                        stem_ = true;
                        kpad_ = g.K_pad;
                        family = "conv_stem_tcgen05";
                    } else if (nchw_in_) {
                        unsupported("canonical NCHW input needs the stem kernel");
                    }
                }
                packed_ = dev_alloc(static_cast<size_t>(cout_) * kpad_ * elem_size(dtype_));
                algo_flops = 2.0 * out_.pixels() * cout_ * kh_ * kw_ * cin_;
                algo_bytes = (in_.pixels() * in_.ld + out_.pixels() * out_.ld) * double(elem_size(dtype_)) +
                             double(cout_) * cin_ * kh_ * kw_ * elem_size(dtype_);
                launches = 2;
                launches_frozen = 1;  // packed weights (and folded BN) cached in a frozen plan
                break;
            }
            case SOL_OP_CONV2DBACKX:
            case SOL_OP_LINEARBACKX: {
                family = op_ == SOL_OP_CONV2DBACKX ? "conv_dgrad_tcgen05" : "linear_dgrad_tcgen05";
                w_idx_ = o.params[0];
                // in_ = delta (Cout), out_ = dx (Cin)
                cin_ = out_.C;
                cout_ = in_.C;
                kpad_ = static_cast<int>(round_up(static_cast<int64_t>(kh_) * kw_ * in_.ld, bk));
                packed_ = dev_alloc(static_cast<size_t>(cin_) * kpad_ * elem_size(dtype_));
                if (op_ == SOL_OP_CONV2DBACKX && (sh_ > 1 || sw_ > 1) && sh_ * sw_ <= 16) plan_subpixel(bk);
                algo_flops = 2.0 * in_.pixels() * cout_ * kh_ * kw_ * cin_;
                algo_bytes = (in_.pixels() * in_.ld + out_.pixels() * out_.ld) * double(elem_size(dtype_)) +
                             double(cout_) * cin_ * kh_ * kw_ * elem_size(dtype_);
                launches = 2;
                break;
            }
            case SOL_OP_CONV2DBACKW:
            case SOL_OP_LINEARBACKW: {
                family = op_ == SOL_OP_CONV2DBACKW ? "conv_wgrad_tcgen05" : "linear_wgrad_tcgen05";
                // inputs: delta, x ; output dW canonical f32
                x_ = geo_b(d.bindings[o.inputs[1]]);
                cout_ = in_.C;
                cin_ = x_.C;
                WgradArgs w = wargs(nullptr, nullptr, nullptr, nullptr);
                ws_floats_ = wgrad_workspace_floats(w);
                packed_floats_ = static_cast<size_t>(cout_) * kh_ * kw_ * x_.ld;
                if (op_ == SOL_OP_CONV2DBACKW && cin_ <= 4 && stem_wgrad_supported(stem_wgrad_args(), static_cast<int>(in_.ld))) {
                    stem_wg_ = true;  // few-channel stem: halo-tile weight gradient (stem.cu)
                    ws_floats_ = stem_wgrad_workspace_floats();
                    packed_floats_ = 0;
                    family = "conv_stem_wgrad_tcgen05";
                }
                algo_flops = 2.0 * in_.pixels() * cout_ * kh_ * kw_ * cin_;
                algo_bytes = (in_.pixels() * in_.ld + x_.pixels() * x_.ld) * double(elem_size(dtype_)) +
                             double(cout_) * cin_ * kh_ * kw_ * 4.0;
                launches = 2;  // wgrad + (split-K reduce | unpack) into the canonical layout
                break;
            }
            default:
                unsupported("not a heavy op");
        }
        parse_epilogue(d);
    }

    size_t scratch_bytes() const override {
        if (!classes_.empty()) return sub_scratch_;
        return op_ == SOL_OP_CONV2DBACKW || op_ == SOL_OP_LINEARBACKW ? (packed_floats_ + ws_floats_) * 4 + 256 : 0;
    }

    // Strided dgrad by sub-pixel decomposition: the dx pixels of parity class (a, b) only receive
    // the taps kh = a + ph (mod sh), kw = b + pw (mod sw), whose dy offsets are contiguous, so each
    // class is a stride-1 convolution of dy (forward-kernel operand paths, no zero taps); the class
    // grids are interleaved into dx afterwards. Replaces the transposed-conv gather, which spends
    // (sh*sw - 1)/(sh*sw) of its MMAs on structural zeros.
    struct SubClass {
        int th = 0, tw = 0, kh0 = 0, kw0 = 0, offh = 0, offw = 0, OHc = 0, OWc = 0, kpad = 0;
        void* packed = nullptr;
        size_t scratch_off = 0;
    };
    void plan_subpixel(int bk) {
        const int H = static_cast<int>(out_.H), W = static_cast<int>(out_.W);
        size_t off = 0;
        classes_.assign(sh_ * sw_, SubClass{});
        for (int a = 0; a < sh_; ++a) {
            for (int b = 0; b < sw_; ++b) {
                SubClass c;
                int omin_h = 1 << 30, omax_h = -(1 << 30), omin_w = 1 << 30, omax_w = -(1 << 30);
                for (int kh = 0; kh < kh_; ++kh) {
                    const int d = a + ph_ - kh;
                    if (((d % sh_) + sh_) % sh_ != 0) continue;
                    omin_h = std::min(omin_h, d / sh_ - (d < 0 && d % sh_ ? 1 : 0));
                    omax_h = std::max(omax_h, d / sh_ - (d < 0 && d % sh_ ? 1 : 0));
                }
                for (int kw = 0; kw < kw_; ++kw) {
                    const int d = b + pw_ - kw;
                    if (((d % sw_) + sw_) % sw_ != 0) continue;
                    omin_w = std::min(omin_w, d / sw_ - (d < 0 && d % sw_ ? 1 : 0));
                    omax_w = std::max(omax_w, d / sw_ - (d < 0 && d % sw_ ? 1 : 0));
                }
                c.OHc = (H - a + sh_ - 1) / sh_;
                c.OWc = (W - b + sw_ - 1) / sw_;
                if (omin_h <= omax_h && omin_w <= omax_w && c.OHc > 0 && c.OWc > 0) {
                    c.th = omax_h - omin_h + 1;
                    c.tw = omax_w - omin_w + 1;
                    c.offh = omin_h;
                    c.offw = omin_w;
                    c.kh0 = a + ph_ - sh_ * omin_h;
                    c.kw0 = b + pw_ - sw_ * omin_w;
                    c.kpad = static_cast<int>(round_up(static_cast<int64_t>(c.th) * c.tw * in_.ld, bk));
                    c.packed = dev_alloc(static_cast<size_t>(cin_) * c.kpad * elem_size(dtype_));
                    c.scratch_off = off;
                    off += round_up(static_cast<int64_t>(in_.N) * c.OHc * c.OWc * out_.ld * elem_size(dtype_), 256);
                }
                classes_[a * sw_ + b] = c;
            }
        }
        sub_scratch_ = off + 256;
        launches = 1;
        for (auto& c : classes_) launches += c.th ? 2 : 0;
        // the class GEMMs run concurrently on side streams (fork / join with events, so a captured
        // plan gets parallel graph branches), each persistent over its share of the SMs
        if (!std::getenv("SOL_SUBPIX_SERIAL")) {
            int with_taps = 0;
            for (const auto& c : classes_) with_taps += c.th ? 1 : 0;
            if (with_taps > 1) {
                side_.resize(classes_.size());
                side_done_.resize(classes_.size());
                for (size_t i = 0; i < classes_.size(); ++i) {
                    SOL_CUDA(cudaStreamCreateWithFlags(&side_[i], cudaStreamNonBlocking));
                    SOL_CUDA(cudaEventCreateWithFlags(&side_done_[i], cudaEventDisableTiming));
                }
                SOL_CUDA(cudaEventCreateWithFlags(&fork_, cudaEventDisableTiming));
            }
        }
    }
    ~HeavyModule() override {
        for (auto st : side_) cudaStreamDestroy(st);
        for (auto ev : side_done_) cudaEventDestroy(ev);
        if (fork_) cudaEventDestroy(fork_);
    }
    std::vector<cudaStream_t> side_;
    std::vector<cudaEvent_t> side_done_;
    cudaEvent_t fork_ = nullptr;

    void run_subpixel(void* const* args, void* out, void* scratch, cudaStream_t s, bool frozen) {
        // in place: every class stores straight into its stride positions of dx (no scratch, no
        // interleave pass) when all of them take the bf16 TMA paths and either every class has
        // taps or only the first does (a 1x1 strided conv: that class zeroes the rest of each cell)
        int with_taps = 0;
        for (const auto& c : classes_) with_taps += c.th ? 1 : 0;
        const bool only_first = with_taps == 1 && classes_[0].th;
        bool inplace = with_taps == static_cast<int>(classes_.size()) || only_first;
        for (size_t ci = 0; ci < classes_.size() && inplace; ++ci)
            if (classes_[ci].th) inplace = igemm_sub_supported(class_args(classes_[ci], args, out));
        InterleaveArgs il;
        il.sh = sh_;
        il.sw = sw_;
        il.N = static_cast<int>(out_.N);
        il.H = static_cast<int>(out_.H);
        il.W = static_cast<int>(out_.W);
        il.ld = static_cast<int>(out_.ld);
        il.out = out;
        // concurrent classes: each runs persistent over its own SM share. A tile of class c costs
        // (its K blocks = taps x 128-byte channel blocks) + E K-block equivalents of epilogue; SMs
        // go one at a time to the class with the latest finish ceil(tiles / SMs) x tile cost (wave
        // quantisation included). E = 24 measured best on ResNet-50's l2.0 / l3.0 / l4.0 strided
        // dgrads (SOL_SUBPIX_EPI_KB overrides)
        const bool par = !side_.empty();
        const int64_t kb_tap = (static_cast<int64_t>(in_.ld) * static_cast<int64_t>(elem_size(dtype_)) + 127) / 128;
        static const int64_t epi_kb = std::getenv("SOL_SUBPIX_EPI_KB") ? std::atoi(std::getenv("SOL_SUBPIX_EPI_KB")) : 24;
        std::vector<int> share(classes_.size(), 0);
        if (par) {
            std::vector<int64_t> tiles(classes_.size(), 0), tcost(classes_.size(), 0);
            int given = 0;
            for (size_t ci = 0; ci < classes_.size(); ++ci) {
                const SubClass& c = classes_[ci];
                if (!c.th) continue;
                tiles[ci] = ceil_div(static_cast<int64_t>(in_.N) * c.OHc * c.OWc, int64_t(128));
                tcost[ci] = static_cast<int64_t>(c.th) * c.tw * kb_tap + epi_kb;
                share[ci] = 1;
                ++given;
            }
            for (; given < num_sms(); ++given) {
                size_t worst = 0;
                int64_t wt = -1;
                for (size_t ci = 0; ci < classes_.size(); ++ci) {
                    if (!share[ci]) continue;
                    const int64_t t = ceil_div(tiles[ci], static_cast<int64_t>(share[ci])) * tcost[ci];
                    if (t > wt) {
                        wt = t;
                        worst = ci;
                    }
                }
                ++share[worst];
            }
        }
        if (par) SOL_CUDA(cudaEventRecord(fork_, s));
        for (size_t ci = 0; ci < classes_.size(); ++ci) {
            SubClass& c = classes_[ci];
            il.ch[ci] = c.OHc;
            il.cw[ci] = c.OWc;
            if (!c.th) continue;
            cudaStream_t cs = s;
            int ctas = 0;
            if (par) {
                cs = side_[ci];
                SOL_CUDA(cudaStreamWaitEvent(cs, fork_, 0));
                ctas = share[ci];
            }
            void* dst = static_cast<uint8_t*>(scratch) + c.scratch_off;
            il.cls[ci] = dst;
            if (!prepacked_ && !(frozen && packed_valid_))
                pack_dgrad_class(static_cast<const float*>(args[w_idx_]), c.packed, dtype_, static_cast<int>(cout_),
                                 static_cast<int>(cin_), kh_, kw_, static_cast<int>(in_.ld), c.kpad, c.th, c.tw, c.kh0,
                                 c.kw0, sh_, sw_, cs);
            IgemmArgs g = class_args(c, args, inplace ? out : dst);
            g.max_ctas = ctas;
            if (inplace) {
                g.sub_sh = sh_;
                g.sub_sw = sw_;
                g.sub_a = static_cast<int>(ci) / sw_;
                g.sub_b = static_cast<int>(ci) % sw_;
                g.sub_H = static_cast<int>(out_.H);
                g.sub_W = static_cast<int>(out_.W);
                g.sub_zero = only_first ? 1 : 0;
            }
            igemm_launch(g, cs);
            if (par) {
                SOL_CUDA(cudaEventRecord(side_done_[ci], cs));
                SOL_CUDA(cudaStreamWaitEvent(s, side_done_[ci], 0));
            }
        }
        packed_valid_ = true;
        if (!inplace) subpixel_interleave(dtype_, il, s);
    }

    // the stride-1 forward conv computing one sub-pixel class of the strided dgrad
    IgemmArgs class_args(const SubClass& c, void* const* args, void* dst) const {
        IgemmArgs g;
        g.mode = IG_FPROP;
        g.dtype = dtype_;
        g.out_dtype = dtype_;
        g.src = args[0];
        g.wt = c.packed;
        g.out = dst;
        g.N = static_cast<int>(in_.N);
        g.SH = static_cast<int>(in_.H);
        g.SW = static_cast<int>(in_.W);
        g.SC = static_cast<int>(in_.ld);
        g.OH = c.OHc;
        g.OW = c.OWc;
        g.kh = c.th; g.kw = c.tw; g.sh = 1; g.sw = 1; g.ph = -c.offh; g.pw = -c.offw;
        g.Nout = static_cast<int>(cin_);
        g.K_pad = c.kpad;
        g.ldo = static_cast<int>(out_.ld);
        g.tile_n = tile_n_;
        return g;
    }

    // Fused epilogue chain after a Conv2d / Linear fprop (inference BatchNorm folding, the
    // "epilogue fusion" of SURVEY §8f row 3): [BN] -> [Add(residual binding)] -> [ReLU | ReLU6].
    // The plan compiler only forms such units when the conv output has no other consumer.
    void parse_epilogue(const sol_unit_desc& d) {
        if (d.n_ops == 1) return;
        if (op_ == SOL_OP_CONV2DBACKX) {
            // training plan fusion (fusion.fuse_dgrad_relu_back), applied in the GEMM epilogue with
            // the mask read from the ReLU output (passes.relu_mask_from_output):
            //   [Conv2dBackX, ReluBack(dx, relu_out)]                 -> relu_out > 0 ? dx : 0
            //   [Conv2dBackX, Add(dx, g), ReluBack(sum, relu_out)]    -> relu_out > 0 ? dx + g : 0
            if (!classes_.empty()) unsupported("strided dgrad (sub-pixel classes) has no fused epilogue");
            auto check_layout = [&](int idx) {
                const Geo m = geo_b(d.bindings[idx]);
                if (m.ld != out_.ld || m.pixels() != out_.pixels()) unsupported("fused dgrad input layout mismatch");
                algo_bytes += double(m.pixels()) * m.ld * elem_size(dtype_);
            };
            const sol_unit_op& r = d.ops[d.n_ops - 1];
            if (r.op != SOL_OP_RELUBACK || r.n_inputs != 2 || r.inputs[0] != -(d.n_ops - 1) || r.inputs[1] < 0)
                unsupported("dgrad epilogue fusion ends in ReluBack(chain, relu output)");
            if (d.n_ops == 2) {
                res_idx_ = r.inputs[1];
                res_mode_ = 1;
                check_layout(res_idx_);
            } else if (d.n_ops == 3 && d.ops[1].op == SOL_OP_ADD) {
                const int x0 = d.ops[1].inputs[0], x1 = d.ops[1].inputs[1];
                if (x0 == -1 && x1 >= 0) res_idx_ = x1;
                else if (x1 == -1 && x0 >= 0) res_idx_ = x0;
                else unsupported("fused Add must combine dx with a unit input");
                mask_idx_ = r.inputs[1];
                check_layout(res_idx_);
                check_layout(mask_idx_);
            } else {
                unsupported("unsupported fused dgrad epilogue");
            }
            family = "conv_dgrad_fused_tcgen05";
            return;
        }
        if (op_ != SOL_OP_CONV2D && op_ != SOL_OP_LINEAR) unsupported("epilogue fusion only after fprop");
        int k = 1;
        auto prev_ref = [&](int kk) { return -kk; };  // output of member op kk-1 is ref -(kk-1)-1 = -kk
        if (k < d.n_ops && d.ops[k].op == SOL_OP_BATCHNORM2D) {
            const sol_unit_op& b = d.ops[k];
            if (b.attrs.training) unsupported("training BatchNorm cannot fold into the conv epilogue");
            if (b.inputs[0] != prev_ref(k) || b.n_params < 4) unsupported("bad fused BatchNorm");
            bn_g_ = b.params[0];
            bn_b_ = b.params[1];
            bn_m_ = b.params[2];
            bn_v_ = b.params[3];
            bn_eps_ = b.attrs.eps;
            ep_coef_ = static_cast<float*>(dev_alloc(5 * static_cast<size_t>(out_.C) * 4));
            ++k;
        }
        if (k < d.n_ops && d.ops[k].op == SOL_OP_ADD) {
            const sol_unit_op& ad = d.ops[k];
            const int x0 = ad.inputs[0], x1 = ad.inputs[1];
            if (x0 == prev_ref(k) && x1 >= 0) res_idx_ = x1;
            else if (x1 == prev_ref(k) && x0 >= 0) res_idx_ = x0;
            else unsupported("fused Add must combine the conv chain with a unit input");
            const Geo r = geo_b(d.bindings[res_idx_]);
            if (r.ld != out_.ld || r.pixels() != out_.pixels()) unsupported("residual layout mismatch");
            algo_bytes += double(r.pixels()) * r.ld * elem_size(dtype_);  // the residual read
            ++k;
        }
        if (k < d.n_ops && (d.ops[k].op == SOL_OP_RELU || d.ops[k].op == SOL_OP_RELU6)) {
            if (d.ops[k].inputs[0] != prev_ref(k)) unsupported("bad fused activation");
            act_ = d.ops[k].op == SOL_OP_RELU ? 1 : 2;
            ++k;
        }
        if (k < d.n_ops && d.ops[k].op == SOL_OP_MAXPOOL2D) {
            // stem + 3x3/2 max pool (plan fusion fuse_stem_pool): the stem kernel pools its own
            // output rows in shared memory, the full-resolution activation never reaches HBM
            const sol_attrs& pa = d.ops[k].attrs;
            if (d.ops[k].inputs[0] != prev_ref(k) || res_idx_ >= 0) unsupported("bad fused max pool");
            if (pa.kh != 3 || pa.kw != 3 || pa.sh != 2 || pa.sw != 2 || pa.ph != 1 || pa.pw != 1)
                unsupported("fused max pool must be 3x3 / stride 2 / pad 1");
            pool_ = true;
            pool_min_init_ = pa.min_init;
            algo_flops *= double(conv_oh_) * conv_ow_ / (double(out_.H) * out_.W);  // MACs are on the conv grid
            if (!stem_ || !stem_row_supported(fprop_args(nullptr, nullptr)))
                unsupported("fused max pool needs the stride-2 row stem kernel");
            ++k;
        }
        if (k != d.n_ops) unsupported("unsupported fused conv epilogue");
        family = op_ == SOL_OP_CONV2D ? (stem_ ? "conv_stem_fused_tcgen05" : "conv_fprop_fused_tcgen05")
                                      : "linear_fused_tcgen05";
    }

    int stat_blocks() const override {
        if (op_ != SOL_OP_CONV2D || stem_ || pool_ || bn_g_ >= 0 || res_idx_ >= 0 || act_ != 0 || nchw_in_) return 0;
        const IgemmArgs g = fprop_args(nullptr, nullptr);
        return igemm_stats_supported(g) ? igemm_stat_blocks(g) : 0;
    }
    void set_stat_output(double* partial, const float* shift) override {
        stat_partial_ = partial;
        stat_shift_ = shift;
        family = "conv_fprop_bnstats_tcgen05";
    }

    IgemmArgs fprop_args(const void* src, void* out) const {
        IgemmArgs g;
        g.mode = IG_FPROP;
        g.dtype = dtype_;
        g.out_dtype = dtype_;
        g.src = src;
        g.wt = packed_;
        g.out = out;
        g.N = static_cast<int>(in_.N);
        g.SH = static_cast<int>(in_.H);
        g.SW = static_cast<int>(in_.W);
        g.SC = static_cast<int>(nchw_in_ ? in_.C : in_.ld);
        g.src_nchw_f32 = nchw_in_ ? 1 : 0;
        g.OH = conv_oh_ > 0 ? conv_oh_ : static_cast<int>(out_.H);
        g.OW = conv_ow_ > 0 ? conv_ow_ : static_cast<int>(out_.W);
        g.kh = kh_; g.kw = kw_; g.sh = sh_; g.sw = sw_; g.ph = ph_; g.pw = pw_;
        g.Nout = static_cast<int>(cout_);
        g.K_pad = kpad_;
        g.ldo = static_cast<int>(out_.ld);
        g.pool3s2 = pool_ ? 1 : 0;
        g.pool_min_init = pool_min_init_;
        return g;
    }

    // the stem conv's forward geometry (x = input, dy = output grid) for the stem wgrad kernel
    IgemmArgs stem_wgrad_args() const {
        IgemmArgs g;
        g.mode = IG_FPROP;
        g.dtype = dtype_;
        g.out_dtype = dtype_;
        g.N = static_cast<int>(x_.N);
        g.SH = static_cast<int>(x_.H);
        g.SW = static_cast<int>(x_.W);
        g.SC = static_cast<int>(x_.ld);
        g.OH = static_cast<int>(in_.H);
        g.OW = static_cast<int>(in_.W);
        g.kh = kh_; g.kw = kw_; g.sh = sh_; g.sw = sw_; g.ph = ph_; g.pw = pw_;
        g.Nout = static_cast<int>(cout_);
        return g;
    }

    WgradArgs wargs(const void* dy, const void* x, float* dw, float* ws) const {
        WgradArgs w;
        w.dtype = dtype_;
        w.dy = dy;
        w.x = x;
        w.dw = dw;
        w.workspace = ws;
        w.N = static_cast<int>(x_.N);
        w.SH = static_cast<int>(x_.H);
        w.SW = static_cast<int>(x_.W);
        w.SC = static_cast<int>(x_.ld);
        w.OH = static_cast<int>(in_.H);
        w.OW = static_cast<int>(in_.W);
        w.Cout = static_cast<int>(cout_);
        w.kh = kh_; w.kw = kw_; w.sh = sh_; w.sw = sw_; w.ph = ph_; w.pw = pw_;
        w.ld_dy = static_cast<int>(in_.ld);
        return w;
    }

    void run(void* const* args, int nargs, void* scratch, cudaStream_t s, bool frozen) override {
        if (nargs != n_args) throw std::invalid_argument("heavy module: wrong argument count");
        void* out = args[nargs - 1];
        struct ClearPrepack {
            bool& f;
            ~ClearPrepack() { f = false; }
        } clear_prepack{prepacked_};
        switch (op_) {
            case SOL_OP_CONV2D:
            case SOL_OP_LINEAR: {
                if (!prepacked_ && !(frozen && packed_valid_)) {
                    if (stem_)
                        pack_stem_weight(static_cast<const float*>(args[w_idx_]), packed_, static_cast<int>(cout_),
                                         static_cast<int>(cin_), kh_, kw_, kpad_, s);
                    else
                        pack_conv_weight(static_cast<const float*>(args[w_idx_]), packed_, dtype_,
                                         static_cast<int>(cout_), static_cast<int>(cin_), kh_, kw_,
                                         static_cast<int>(in_.ld), kpad_, s);
                    packed_valid_ = true;
                }
                IgemmArgs g = fprop_args(args[0], out);
                g.bias = b_idx_ >= 0 ? static_cast<const float*>(args[b_idx_]) : nullptr;
                if (ep_coef_) {
                    if (!(frozen && coef_valid_)) {
                        bn_infer_coef(static_cast<const float*>(args[bn_g_]), static_cast<const float*>(args[bn_b_]),
                                      static_cast<const float*>(args[bn_m_]), static_cast<const float*>(args[bn_v_]),
                                      bn_eps_, ep_coef_, static_cast<int>(cout_), s);
                        coef_valid_ = true;
                    }
                    g.ep_scale = ep_coef_ + 2 * cout_;
                    g.ep_shift = ep_coef_ + 4 * cout_;
                }
                if (res_idx_ >= 0) {
                    g.residual = args[res_idx_];
                    g.ld_res = static_cast<int>(out_.ld);
                }
                g.act = act_;
                g.tile_n = tile_n_;
                g.stat_partial = stat_partial_;
                g.stat_shift = stat_shift_;
                g.stat_blocks = stat_partial_ ? igemm_stat_blocks(g) : 0;
                if (stem_) stem_launch(g, s);
                else igemm_launch(g, s);
                break;
            }
            case SOL_OP_CONV2DBACKX:
            case SOL_OP_LINEARBACKX: {
                if (!classes_.empty()) {
                    run_subpixel(args, out, scratch, s, frozen);
                    break;
                }
                // stride 1: dx = conv(dy, mirrored transposed taps, padding k-1-p), which runs on the
                // forward kernels' TMA (1x1) / TMA-im2col (k x k) operand paths
                const bool as_fprop = sh_ == 1 && sw_ == 1 && ph_ <= kh_ - 1 && pw_ <= kw_ - 1;
                if (!prepacked_ && !(frozen && packed_valid_)) {
                    pack_conv_weight_t(static_cast<const float*>(args[w_idx_]), packed_, dtype_,
                                       static_cast<int>(cout_), static_cast<int>(cin_), kh_, kw_,
                                       static_cast<int>(in_.ld), kpad_, s, as_fprop);
                    packed_valid_ = true;
                }
                IgemmArgs g;
                g.mode = as_fprop ? IG_FPROP : IG_DGRAD;
                g.dtype = dtype_;
                g.out_dtype = dtype_;
                g.src = args[0];
                g.wt = packed_;
                g.out = out;
                g.N = static_cast<int>(in_.N);
                g.SH = static_cast<int>(in_.H);
                g.SW = static_cast<int>(in_.W);
                g.SC = static_cast<int>(in_.ld);
                g.OH = static_cast<int>(out_.H);
                g.OW = static_cast<int>(out_.W);
                g.kh = kh_; g.kw = kw_; g.sh = sh_; g.sw = sw_;
                g.ph = as_fprop ? kh_ - 1 - ph_ : ph_;
                g.pw = as_fprop ? kw_ - 1 - pw_ : pw_;
                g.Nout = static_cast<int>(cin_);
                g.K_pad = kpad_;
                g.ldo = static_cast<int>(out_.ld);
                g.tile_n = tile_n_;
                if (res_idx_ >= 0) {  // fused [Add +] ReluBack: mask = relu output > 0
                    g.residual = args[res_idx_];
                    g.ld_res = static_cast<int>(out_.ld);
                    g.res_mode = res_mode_;
                    if (mask_idx_ >= 0) g.mask = args[mask_idx_];
                }
                igemm_launch(g, s);
                break;
            }
            default: {
                if (stem_wg_) {
                    IgemmArgs g = stem_wgrad_args();
                    g.src = args[1];
                    stem_wgrad_launch(g, args[0], static_cast<int>(cin_), static_cast<float*>(scratch),
                                      static_cast<float*>(out), s);
                    break;
                }
                float* packed = static_cast<float*>(scratch);
                float* ws = ws_floats_ ? packed + round_up(static_cast<int64_t>(packed_floats_), 64) : nullptr;
                WgradArgs w = wargs(args[0], args[1], packed, ws);
                w.dw_canon = static_cast<float*>(out);  // reduce (or unpack) straight to canonical dW
                w.canon_cin = static_cast<int>(cin_);
                wgrad_launch(w, s);
                break;
            }
        }
    }
    // Packs this step's weights now (the plan batches every module's packing of a run into one
    // launch before the first step, pack.cuh); run() then skips its own packing once.
    bool prepack(void* const* args, cudaStream_t s, bool frozen) override {
        if (frozen && packed_valid_) return false;
        if (op_ == SOL_OP_CONV2D || op_ == SOL_OP_LINEAR) {
            if (stem_)
                pack_stem_weight(static_cast<const float*>(args[w_idx_]), packed_, static_cast<int>(cout_),
                                 static_cast<int>(cin_), kh_, kw_, kpad_, s);
            else
                pack_conv_weight(static_cast<const float*>(args[w_idx_]), packed_, dtype_, static_cast<int>(cout_),
                                 static_cast<int>(cin_), kh_, kw_, static_cast<int>(in_.ld), kpad_, s);
        } else if (op_ == SOL_OP_CONV2DBACKX || op_ == SOL_OP_LINEARBACKX) {
            if (!classes_.empty()) {
                for (auto& c : classes_)
                    if (c.th)
                        pack_dgrad_class(static_cast<const float*>(args[w_idx_]), c.packed, dtype_,
                                         static_cast<int>(cout_), static_cast<int>(cin_), kh_, kw_,
                                         static_cast<int>(in_.ld), c.kpad, c.th, c.tw, c.kh0, c.kw0, sh_, sw_, s);
            } else {
                const bool as_fprop = sh_ == 1 && sw_ == 1 && ph_ <= kh_ - 1 && pw_ <= kw_ - 1;
                pack_conv_weight_t(static_cast<const float*>(args[w_idx_]), packed_, dtype_, static_cast<int>(cout_),
                                   static_cast<int>(cin_), kh_, kw_, static_cast<int>(in_.ld), kpad_, s, as_fprop);
            }
        } else {
            return false;
        }
        packed_valid_ = true;
        prepacked_ = true;
        return true;
    }
    bool set_option(int key, int value) override {
        if (key != SOL_MODOPT_TILE_N || stem_ ||
            (op_ != SOL_OP_CONV2D && op_ != SOL_OP_LINEAR && op_ != SOL_OP_CONV2DBACKX && op_ != SOL_OP_LINEARBACKX))
            return false;
        if (value != 0 && value != 64 && value != 65 && value != 128 && value != 256) return false;
        if (value == 65 && dtype_ != DT_BF16) return false;
        tile_n_ = value;
        return true;
    }

private:
    bool prepacked_ = false;  // prepack() ran for the current run
    int tile_n_ = 0;  // autotuned tcgen05 tile (SOL_MODOPT_TILE_N)
    int dtype_;
    int op_;
    int kh_, kw_, sh_, sw_, ph_, pw_;
    Geo in_, out_, x_;
    int64_t cin_ = 0, cout_ = 0;
    int kpad_ = 0;
    bool stem_ = false, stem_wg_ = false, nchw_in_ = false, pool_ = false;
    int conv_oh_ = 0, conv_ow_ = 0;
    float pool_min_init_ = -INFINITY;
    std::vector<SubClass> classes_;
    size_t sub_scratch_ = 0;
    int w_idx_ = -1, b_idx_ = -1;
    void* packed_ = nullptr;
    bool packed_valid_ = false;
    size_t ws_floats_ = 0, packed_floats_ = 0;
    // fused epilogue
    float* ep_coef_ = nullptr;
    bool coef_valid_ = false;
    int bn_g_ = -1, bn_b_ = -1, bn_m_ = -1, bn_v_ = -1;
    float bn_eps_ = 1e-5f;
    double* stat_partial_ = nullptr;  // BN statistics epilogue (link_bn_stats)
    const float* stat_shift_ = nullptr;
    int res_idx_ = -1;
    int res_mode_ = 0;  // 1: the residual binding is a ReLU output used as a backward mask
    int mask_idx_ = -1;  // fused Add + ReluBack: the ReLU output binding (residual = the added gradient)
    int act_ = 0;
};

// ---------------------------------------------------------------------------------------------
// row kernels: Softmax / CrossEntropyLoss / SoftmaxCeBack / CeBack / SoftmaxBack
// ---------------------------------------------------------------------------------------------

class RowModule : public Module {
public:
    explicit RowModule(const sol_unit_desc& d) : dtype_(d.dtype), op_(d.ops[0].op) {
        fill_arg_bytes(*this, d);
        const Geo g = geo_b(d.bindings[d.ops[0].inputs[0]]);
        if (g.H != 1 || g.W != 1) unsupported("row ops over pixel dims are not supported");
        rows_ = static_cast<int>(g.N);
        cols_ = static_cast<int>(g.C);
        ld_ = static_cast<int>(g.ld);
        if (op_ == SOL_OP_CROSSENTROPYLOSS || op_ == SOL_OP_SOFTMAXCEBACK || op_ == SOL_OP_CEBACK ||
            op_ == SOL_OP_SOFTMAXBACK) {
            const Geo t = geo_b(d.bindings[d.ops[0].inputs[1]]);
            if (t.ld != g.ld) throw ShapeError("row op operands differ in row stride");
        }
        family = op_ == SOL_OP_SOFTMAX ? "softmax_rows" : op_ == SOL_OP_CROSSENTROPYLOSS ? "ce_loss" : "ce_back";
        algo_bytes = double(rows_) * ld_ * elem_size(dtype_) * (op_ == SOL_OP_SOFTMAX ? 2 : 3);
    }
    void run(void* const* args, int nargs, void*, cudaStream_t s, bool) override {
        if (nargs != n_args) throw std::invalid_argument("row module: wrong argument count");
        switch (op_) {
            case SOL_OP_SOFTMAX: softmax_rows(dtype_, args[0], args[1], rows_, cols_, ld_, s); break;
            case SOL_OP_CROSSENTROPYLOSS:
                ce_loss(dtype_, args[0], args[1], static_cast<float*>(args[2]), rows_, cols_, ld_, s);
                break;
            case SOL_OP_SOFTMAXCEBACK: ce_back(dtype_, 1, args[0], args[1], args[2], rows_, cols_, ld_, s); break;
            case SOL_OP_CEBACK: ce_back(dtype_, 0, args[0], args[1], args[2], rows_, cols_, ld_, s); break;
            case SOL_OP_SOFTMAXBACK: softmax_back(dtype_, args[0], args[1], args[2], rows_, cols_, ld_, s); break;
            default: unsupported("row op");
        }
    }

private:
    int dtype_, op_;
    int rows_, cols_, ld_;
};

// Flatten / FlattenBack in the reference's canonical order (dfp_lower.cpp:1098-1112).
class FlattenModule : public Module {
public:
    explicit FlattenModule(const sol_unit_desc& d) : dtype_(d.dtype), inverse_(d.ops[0].op == SOL_OP_FLATTENBACK) {
        fill_arg_bytes(*this, d);
        family = inverse_ ? "flatten_back" : "flatten";
        img_ = inverse_ ? geo_b(d.output) : geo_b(d.bindings[d.ops[0].inputs[0]]);
        const Geo flat = inverse_ ? geo_b(d.bindings[d.ops[0].inputs[0]]) : geo_b(d.output);
        if (img_.ld != img_.C || flat.ld != flat.C) unsupported("flatten over padded channel storage");
        algo_bytes = 2.0 * img_.numel() * elem_size(dtype_);
    }
    void run(void* const* args, int nargs, void*, cudaStream_t s, bool) override {
        if (nargs != n_args) throw std::invalid_argument("flatten: wrong argument count");
        flatten_nhwc(dtype_, args[0], args[1], static_cast<int>(img_.N), static_cast<int>(img_.C),
                     static_cast<int>(img_.H), static_cast<int>(img_.W), inverse_, s);
    }

private:
    int dtype_;
    int inverse_;
    Geo img_;
};

// Reorder steps at the plan boundary (fe::Step::Kind::Reorder): canonical f32 host layout
// (NCHW / NC, the reference's meta_nchw order, tensor.cpp:141-151) <-> NHWC plan storage.
class ReorderModule : public Module {
public:
    explicit ReorderModule(const sol_unit_desc& d) : dtype_(d.dtype), inbound_(d.ops[0].op == SOL_OP_REORDER_IN) {
        fill_arg_bytes(*this, d);
        family = inbound_ ? "reorder_in" : "reorder_out";
        stored_ = inbound_ ? geo_b(d.output) : geo_b(d.bindings[0]);
        algo_bytes = stored_.numel() * (4.0 + elem_size(dtype_));
    }
    void run(void* const* args, int nargs, void*, cudaStream_t s, bool) override {
        if (nargs != n_args) throw std::invalid_argument("reorder: wrong argument count");
        const Geo& g = stored_;
        if (g.rank == 0) {
            cast_copy(args[0], inbound_ ? DT_F32 : dtype_, args[1], inbound_ ? dtype_ : DT_F32, 1, s);
        } else if (inbound_) {
            nchw_to_nhwc(static_cast<const float*>(args[0]), args[1], dtype_, static_cast<int>(g.N),
                         static_cast<int>(g.C), static_cast<int>(g.H), static_cast<int>(g.W), static_cast<int>(g.ld), s);
        } else {
            nhwc_to_nchw(args[0], static_cast<float*>(args[1]), dtype_, static_cast<int>(g.N), static_cast<int>(g.C),
                         static_cast<int>(g.H), static_cast<int>(g.W), static_cast<int>(g.ld), s);
        }
    }

private:
    int dtype_;
    bool inbound_;
    Geo stored_;
};

// SgdUpdate: theta' = theta - lr * g (dfp_lower.cpp:780-783; reference.cpp:580-584). f32 master.
class SgdModule : public Module {
public:
    explicit SgdModule(const sol_unit_desc& d) {
        fill_arg_bytes(*this, d);
        family = "sgd_update";
        lr_ = d.ops[0].attrs.lr;
        n_ = param_numel(d.bindings[d.ops[0].inputs[0]]);
        algo_bytes = 12.0 * n_;
        lr_dev_ = static_cast<float*>(dev_alloc(4));
        SOL_CUDA(cudaMemcpy(lr_dev_, &lr_, 4, cudaMemcpyHostToDevice));
    }
    bool set_lr(float lr, cudaStream_t s) override {
        lr_ = lr;
        SOL_CUDA(cudaMemcpyAsync(lr_dev_, &lr_, 4, cudaMemcpyHostToDevice, s));
        return true;
    }
    void run(void* const* args, int nargs, void*, cudaStream_t s, bool) override {
        if (nargs != n_args) throw std::invalid_argument("sgd: wrong argument count");
        float* w = static_cast<float*>(args[0]);
        float* o = static_cast<float*>(args[2]);
        if (o != w) SOL_CUDA(cudaMemcpyAsync(o, w, n_ * 4, cudaMemcpyDeviceToDevice, s));
        sgd_update(o, static_cast<const float*>(args[1]), n_, lr_, nullptr, s, lr_dev_);
    }

private:
    float lr_;
    int64_t n_;
    float* lr_dev_ = nullptr;
};

// Many SgdUpdate ops in one unit (plan-level multi-tensor update): bindings are (param, grad)
// pairs, every parameter is updated in place, the unit output aliases the first parameter.
class SgdMultiModule : public Module {
public:
    explicit SgdMultiModule(const sol_unit_desc& d) {
        fill_arg_bytes(*this, d);
        family = "sgd_update";
        if (d.n_ops > SGD_MULTI_MAX) unsupported("too many parameters for one SGD unit");
        a_.count = d.n_ops;
        a_.lr = d.ops[0].attrs.lr;
        int blocks = 0;
        for (int i = 0; i < d.n_ops; ++i) {
            const sol_unit_op& o = d.ops[i];
            if (o.op != SOL_OP_SGDUPDATE || o.inputs[0] != 2 * i || o.inputs[1] != 2 * i + 1)
                unsupported("multi-SGD unit must list (param, grad) pairs");
            if (o.attrs.lr != a_.lr) unsupported("multi-SGD unit with mixed learning rates");
            a_.n[i] = param_numel(d.bindings[2 * i]);
            a_.block0[i] = blocks;
            blocks += static_cast<int>(ceil_div(a_.n[i], 1024));
            algo_bytes += 12.0 * a_.n[i];
        }
        a_.block0[d.n_ops] = blocks;
        lr_dev_ = static_cast<float*>(dev_alloc(4));
        SOL_CUDA(cudaMemcpy(lr_dev_, &a_.lr, 4, cudaMemcpyHostToDevice));
        a_.lr_dev = lr_dev_;
    }
    bool set_lr(float lr, cudaStream_t s) override {
        a_.lr = lr;
        SOL_CUDA(cudaMemcpyAsync(lr_dev_, &a_.lr, 4, cudaMemcpyHostToDevice, s));
        return true;
    }
    void run(void* const* args, int nargs, void*, cudaStream_t s, bool) override {
        if (nargs != n_args) throw std::invalid_argument("sgd: wrong argument count");
        SgdMultiArgs a = a_;
        for (int i = 0; i < a.count; ++i) {
            a.w[i] = static_cast<float*>(args[2 * i]);
            a.g[i] = static_cast<const float*>(args[2 * i + 1]);
        }
        sgd_multi(a, s);
    }

private:
    SgdMultiArgs a_;
    float* lr_dev_ = nullptr;
};

// ---------------------------------------------------------------------------------------------
// per-channel reductions: BatchNormBack{X,Gamma,Beta} (training), Conv2dBackB, LinearBackB
// ---------------------------------------------------------------------------------------------

Program prog_load(int slot) {
    Program p;
    p.n = 1;
    p.ins[0].op = PW_LD;
    p.ins[0].dst = 0;
    p.ins[0].a = static_cast<uint8_t>(slot);
    return p;
}

void push(Program& p, PwOp op, int dst, int a = 0, int b = 0, int arg = 0, float imm = 0.f) {
    if (p.n >= DFP_MAX_INS) unsupported("fused unit too long for one program");
    PwInstr& i = p.ins[p.n++];
    i.op = op;
    i.dst = static_cast<uint8_t>(dst);
    i.a = static_cast<uint8_t>(a);
    i.b = static_cast<uint8_t>(b);
    i.arg = static_cast<int16_t>(arg);
    i.imm = imm;
}

class ReduceModule : public Module {
public:
    explicit ReduceModule(const sol_unit_desc& d) : dtype_(d.dtype) {
        fill_arg_bytes(*this, d);
        const sol_unit_op& o = d.ops[0];
        op_ = o.op;
        training_ = o.attrs.training != 0;
        eps_ = o.attrs.eps;
        delta_ = geo_b(d.bindings[o.inputs[0]]);
        C_ = static_cast<int>(delta_.ld);       // reduce over the stored (padded) width
        Creal_ = static_cast<int>(delta_.C);
        blocks_ = dfp_reduce_blocks(delta_.pixels(), C_, dtype_);
        const bool needs_x = op_ == SOL_OP_BATCHNORMBACKX || op_ == SOL_OP_BATCHNORMBACKGAMMA;
        if (needs_x && !training_) unsupported("BatchNorm backward in inference mode");
        if (needs_x && C_ != Creal_) unsupported("BatchNorm backward over padded channel storage");
        if (needs_x) {
            x_idx_ = o.inputs[1];
            shift_ = static_cast<float*>(dev_alloc(C_ * 4));
            xhat_ = static_cast<float*>(dev_alloc(3 * C_ * 4));
            coef_ = static_cast<float*>(dev_alloc(3 * C_ * 4));
            gamma_idx_ = o.n_params > 0 ? o.params[0] : -1;
        }
        switch (op_) {
            case SOL_OP_BATCHNORMBACKX: family = "bn_back_x"; launches = 3; break;
            case SOL_OP_BATCHNORMBACKGAMMA: family = "bn_back_gamma"; launches = 2; break;
            case SOL_OP_BATCHNORMBACKBETA: family = "bn_back_beta"; launches = 2; break;
            default: family = "bias_grad"; launches = 2; break;
        }
        const double es = double(elem_size(dtype_));
        algo_bytes = delta_.numel() * es * (needs_x ? 2 : 1) + (op_ == SOL_OP_BATCHNORMBACKX ? delta_.numel() * es : 0);
    }
    size_t scratch_bytes() const override { return static_cast<size_t>(blocks_) * C_ * 4 * 8 + 256; }

    // BatchNormBackX also writes its siblings' outputs (bit 0: BatchNormBackGamma, bit 1:
    // BatchNormBackBeta) from the same reduction pass ("fuse sibling BN-backward units").
    bool set_sibling_outputs(int mask) override {
        if (op_ != SOL_OP_BATCHNORMBACKX || (mask & ~3)) return mask == 0;
        n_args += __builtin_popcount(static_cast<unsigned>(mask)) - __builtin_popcount(static_cast<unsigned>(sib_));
        for (int b = 0; b < 2; ++b)
            if ((mask >> b) & 1) arg_bytes.push_back(static_cast<size_t>(Creal_) * 4);
        sib_ = mask;
        return true;
    }

    DfpArgs base(void* const* args, double* partial) const {
        DfpArgs a;
        a.family = FAM_CHAN_REDUCE;
        a.dtype = dtype_;
        a.N = static_cast<int>(delta_.N);
        a.H = static_cast<int>(delta_.H);
        a.W = static_cast<int>(delta_.W);
        a.C = C_;
        a.n_in = 2;
        a.in[0] = args[0];
        a.in_kind[0] = IN_PIX;
        a.in_ld[0] = C_;
        if (x_idx_ >= 0) {
            a.in[1] = args[x_idx_];
            a.in_kind[1] = IN_PIX;
            a.in_ld[1] = C_;
        }
        a.partial = partial;
        a.reduce_blocks = blocks_;
        return a;
    }

    void run(void* const* args, int nargs, void* scratch, cudaStream_t s, bool) override {
        if (nargs != n_args) throw std::invalid_argument("reduce module: wrong argument count");
        double* partial = static_cast<double*>(scratch);
        const int n_sib = __builtin_popcount(static_cast<unsigned>(sib_));
        float* out = static_cast<float*>(args[nargs - 1 - n_sib]);
        float* sib_gamma = nullptr;
        float* sib_beta = nullptr;
        {
            int k = nargs - n_sib;
            if (sib_ & 1) sib_gamma = static_cast<float*>(args[k++]);
            if (sib_ & 2) sib_beta = static_cast<float*>(args[k++]);
        }
        if (op_ == SOL_OP_BATCHNORMBACKBETA || op_ == SOL_OP_CONV2DBACKB || op_ == SOL_OP_LINEARBACKB) {
            DfpArgs a = base(args, partial);
            a.pre = prog_load(0);
            push(a.pre, PW_MOV, 1, 0);
            FinalizeArgs f;
            f.mode = FIN_SUMS;
            f.C = Creal_;
            f.Cstride = C_;
            f.blocks = blocks_;
            f.partial = partial;
            f.out0 = out;
            dfp_reduce_finalize(a, f, s);
            return;
        }
        // BNBackX / BNBackGamma: one pass over (dy, x) gives the x statistics and both sums
        // shifted sums about x's first pixel, read in place by the reduction and the finalisation
        FinalizeArgs f;
        f.mode = FIN_BN_BACK4;
        f.C = C_;
        f.blocks = blocks_;
        f.partial = partial;
        f.count = static_cast<double>(delta_.pixels());
        f.eps = eps_;
        f.shift = nullptr;
        f.shift_x = args[x_idx_];
        f.shift_dtype = dtype_;
        if (op_ == SOL_OP_BATCHNORMBACKGAMMA) {
            f.out1 = out;
        } else {
            f.gamma = static_cast<const float*>(args[gamma_idx_]);
            f.coef = coef_;
            f.xhat = xhat_;
            f.out1 = sib_gamma;
            f.out0 = sib_beta;
        }
        // one pass over (dy, x) + the finalisation [+ the dx apply over each block's own rows], fused
        // in one cooperative launch when the grid is co-resident
        // Only for small tensors: the one-wave reduction grid applies at lower occupancy than the
        // dedicated apply kernel (everywhere: 14.84 vs 14.30 ms per ResNet-50 training step), but when
        // dy and x fit comfortably in L2 the re-read is cheap and the saved launch + finalize win
        // (dy + x <= 60 MB: -90 us per step; 120 MB: worse)
        // SOL_BNBACK_FUSED_APPLY=1/0 forces it on/off; SOL_BNBACK_FUSED_MB sets the size limit
        static const char* fa_env = std::getenv("SOL_BNBACK_FUSED_APPLY");
        static const double fa_mb = std::getenv("SOL_BNBACK_FUSED_MB") ? std::atof(std::getenv("SOL_BNBACK_FUSED_MB")) : 60.0;
        const double pair_mb = 2.0 * static_cast<double>(delta_.pixels()) * C_ * elem_size(dtype_) / 1e6;
        const bool fuse_apply = fa_env ? fa_env[0] == '1' : pair_mb <= fa_mb;
        void* apply_out = (op_ == SOL_OP_BATCHNORMBACKGAMMA || !fuse_apply) ? nullptr : out;
        const int fused = bn_back_reduce(dtype_, args[0], args[x_idx_], C_, delta_.pixels(), nullptr, partial, blocks_,
                                         s, &f, apply_out);
        if (fused == 0) dfp_finalize(f, s);
        if (op_ == SOL_OP_BATCHNORMBACKGAMMA || fused == 2) return;
        bn_back_apply(dtype_, args[0], args[x_idx_], C_, delta_.pixels(), coef_, xhat_, out, s);
    }

private:
    int dtype_;
    int op_;
    bool training_ = false;
    float eps_ = 1e-5f;
    Geo delta_;
    int C_ = 0, Creal_ = 0;
    int blocks_ = 1;
    int x_idx_ = -1, gamma_idx_ = -1;
    int sib_ = 0;
    float *shift_ = nullptr, *xhat_ = nullptr, *coef_ = nullptr;
};

// ---------------------------------------------------------------------------------------------
// DFP fused groups: pointwise / pool / gap / depthwise / pool-backward families
// ---------------------------------------------------------------------------------------------

class DfpModule : public Module {
public:
    explicit DfpModule(const sol_unit_desc& d);
    void run(void* const* args, int nargs, void* scratch, cudaStream_t s, bool frozen) override;
    size_t scratch_bytes() const override { return stats_scratch_; }
    // bit 2: also write relu(output) (bit 3: relu6) for a sibling ReLU unit reading this output
    bool set_sibling_outputs(int mask) override {
        if (mask == 0) return true;
        if ((mask != 4 && mask != 8) || tmpl_.family != FAM_POINTWISE || act_sib_) return false;
        act_sib_ = mask == 4 ? 1 : 2;
        n_args += 1;
        arg_bytes.push_back(arg_bytes.back());
        return true;
    }
    bool set_option(int key, int value) override {
        if (key != SOL_MODOPT_UPDATE_BN_RUNNING_STATS) return false;
        bool any = false;
        for (const auto& b : bn_) any |= b.training && b.m >= 0 && b.v >= 0;
        if (!any) return false;
        update_running_ = value != 0;
        return true;
    }

private:
    bool update_running_ = false;  // training BN: update running_mean / running_var in place

public:
    bool use_producer_stats(int binding, int blocks, double** partial, const float** shift) override {
        for (auto& b : bn_) {
            if (!b.training || b.x_binding != binding || blocks <= 0) continue;
            if (b.ext_partial == nullptr || b.ext_blocks != blocks) {
                b.ext_partial = static_cast<double*>(dev_alloc(static_cast<size_t>(b.C) * blocks * 2 * sizeof(double)));
                b.ext_blocks = blocks;
            }
            *partial = b.ext_partial;
            *shift = b.stats;  // the previous step's batch mean (zeros before the first step)
            return true;
        }
        return false;
    }

private:
    struct SlotSrc {
        int binding;
    };
    struct BnPrep {
        bool training;
        int x_binding;      // training: the BN input (boundary binding)
        int g, b, m, v;     // param bindings
        float eps;
        float momentum;     // training: running-statistics update (autodiff.cpp:356-384)
        int C;
        float* coef;        // [3C] (mean, scale, beta) -> P[3i], P[3i+1], P[3i+2]
        float* shift;
        float* stats;
        int64_t pixels;
        int x_ld;
        int xN, xH, xW;
        double* ext_partial = nullptr;  // statistics written by the producing conv's epilogue
        int ext_blocks = 0;
    };
    struct DwPrep {
        int w, bias;
        int C, kh, kw;
        float* packed;
    };

    // program building
    int key_op(int k) const { return k; }
    int key_b(int b) const { return 1000 + b; }
    int reg_get(int ref);
    int reg_take(int ref);
    void consume(int ref);
    int alloc_reg();
    int emit_value(int key);
    int slot_for(int binding, int kind, int coff);
    void count_uses(int key, const std::set<int>& members, bool root);

    const sol_unit_desc& d_;  // valid during construction only
    DfpArgs tmpl_;
    std::vector<int> slot_binding_;
    std::vector<int> cat_bindings_;
    std::vector<BnPrep> bn_;
    std::vector<DwPrep> dw_;
    std::map<int, int> bn_of_op_;  // op index -> bn_ index
    int dtype_;
    int anchor_ = -1;
    size_t stats_scratch_ = 0;
    size_t argmax_offset_ = 0;
    int act_sib_ = 0;
    bool coef_ready_ = false;
    float* ones_ = nullptr;
    float* zeros_ = nullptr;

    // builder state
    Program* prog_ = nullptr;
    std::map<int, int> uses_, reg_of_;
    unsigned free_regs_ = 0xF;
    std::set<int> prog_members_;
};

int DfpModule::alloc_reg() {
    for (int r = 0; r < 4; ++r)
        if (free_regs_ & (1u << r)) {
            free_regs_ &= ~(1u << r);
            return r;
        }
    unsupported("fused unit needs more than 4 live values");
}

void DfpModule::consume(int key) {
    auto it = uses_.find(key);
    if (it == uses_.end()) return;
    if (--it->second == 0) {
        auto r = reg_of_.find(key);
        if (r != reg_of_.end()) {
            free_regs_ |= 1u << r->second;
            reg_of_.erase(r);
        }
    }
}

int DfpModule::reg_get(int key) {
    auto it = reg_of_.find(key);
    if (it != reg_of_.end()) return it->second;
    const int r = emit_value(key);
    reg_of_[key] = r;
    return r;
}

int DfpModule::reg_take(int key) {
    const int r = reg_get(key);
    if (uses_[key] > 1) {
        const int r2 = alloc_reg();
        push(*prog_, PW_MOV, r2, r);
        consume(key);
        return r2;
    }
    // last use: steal the register
    uses_[key] = 0;
    reg_of_.erase(key);
    return r;
}

int DfpModule::slot_for(int binding, int kind, int coff) {
    for (size_t i = 0; i < slot_binding_.size(); ++i)
        if (slot_binding_[i] == binding && tmpl_.in_kind[i] == kind && tmpl_.in_coff[i] == coff)
            return static_cast<int>(i);
    const int s = static_cast<int>(slot_binding_.size());
    if (s >= DFP_MAX_IN) unsupported("too many unit inputs");
    slot_binding_.push_back(binding);
    tmpl_.in_kind[s] = kind;
    tmpl_.in_coff[s] = coff;
    tmpl_.in_ld[s] = static_cast<int>(geo_b(d_.bindings[binding]).ld);
    tmpl_.n_in = s + 1;
    return s;
}

void DfpModule::count_uses(int key, const std::set<int>& members, bool root) {
    uses_[key] += 1;
    if (key >= 1000 || key == 2000) return;
    if (!members.count(key)) unsupported("fused value used on two pixel grids");
    if (uses_[key] > 1 && !root) return;  // already expanded
    const sol_unit_op& o = d_.ops[key];
    const int ni = (o.op == SOL_OP_CONCAT) ? 0 : o.n_inputs;
    for (int i = 0; i < ni; ++i) {
        if (key == anchor_) break;
        const int r = o.inputs[i];
        count_uses(r >= 0 ? key_b(r) : key_op(-r - 1), members, false);
    }
}

// Emits code for value `key` into a fresh register; returns the register.
int DfpModule::emit_value(int key) {
    Program& p = *prog_;
    if (key == 2000) unsupported("anchor value requested outside the post program");
    if (key >= 1000) {
        const int b = key - 1000;
        const int r = alloc_reg();
        const int slot = slot_for(b, IN_PIX, 0);
        push(p, PW_LD, r, slot);
        return r;
    }
    if (key == anchor_) {
        // anchor result is preloaded in r0 by the family kernel
        free_regs_ &= ~1u;
        return 0;
    }
    const sol_unit_op& o = d_.ops[key];
    auto in_key = [&](int i) {
        const int r = o.inputs[i];
        return r >= 0 ? key_b(r) : key_op(-r - 1);
    };
    switch (o.op) {
        case SOL_OP_RELU:
        case SOL_OP_RELU6:
        case SOL_OP_COPY: {
            const int r = reg_take(in_key(0));
            if (o.op != SOL_OP_COPY) push(p, o.op == SOL_OP_RELU ? PW_RELU : PW_RELU6, r);
            return r;
        }
        case SOL_OP_BATCHNORM2D: {
            const int r = reg_take(in_key(0));
            const int bi = bn_of_op_.at(key);
            push(p, PW_BN, r, 0, 0, 5 * bi);
            return r;
        }
        case SOL_OP_ADD: {
            const int ra = reg_take(in_key(0));
            const int rb = reg_get(in_key(1));
            push(p, PW_ADD, ra, ra, rb);
            consume(in_key(1));
            return ra;
        }
        case SOL_OP_RELUBACK:
        case SOL_OP_RELU6BACK: {
            const int ra = reg_take(in_key(0));
            const int rb = reg_get(in_key(1));
            push(p, o.op == SOL_OP_RELUBACK ? PW_MASK : PW_MASK6, ra, ra, rb);
            consume(in_key(1));
            return ra;
        }
        case SOL_OP_CONCAT: {
            if (!cat_bindings_.empty()) unsupported("more than one Concat in a unit");
            int off = 0;
            tmpl_.cat_off[0] = 0;
            for (int i = 0; i < o.n_inputs; ++i) {
                if (o.inputs[i] < 0) unsupported("Concat of a fused intermediate");
                if (o.n_inputs > DFP_MAX_CAT) unsupported("Concat arity");
                const Geo g = geo_b(d_.bindings[o.inputs[i]]);
                if (g.ld != g.C) unsupported("Concat over padded storage");
                cat_bindings_.push_back(o.inputs[i]);
                off += static_cast<int>(g.C);
                tmpl_.cat_off[i + 1] = off;
            }
            tmpl_.n_cat = o.n_inputs;
            const int s = static_cast<int>(slot_binding_.size());
            slot_binding_.push_back(-1);
            tmpl_.in_kind[s] = IN_CAT;
            tmpl_.n_in = s + 1;
            const int r = alloc_reg();
            push(p, PW_LD, r, s);
            return r;
        }
        case SOL_OP_CONCATBACK: {
            if (o.inputs[0] < 0) unsupported("ConcatBack of a fused intermediate");
            const int r = alloc_reg();
            push(p, PW_LD, r, slot_for(o.inputs[0], IN_PIX, static_cast<int>(o.attrs.offset)));
            return r;
        }
        case SOL_OP_FLATTENBACK: {
            if (o.inputs[0] < 0) unsupported("FlattenBack of a fused intermediate");
            const int r = alloc_reg();
            const int s = slot_for(o.inputs[0], IN_FLAT, 0);
            tmpl_.in_hw[s] = static_cast<int>(o.saved_dims[2] * o.saved_dims[3]);
            push(p, PW_LD, r, s);
            return r;
        }
        case SOL_OP_GLOBALAVGPOOLBACK: {
            if (o.inputs[0] < 0) unsupported("GlobalAvgPoolBack of a fused intermediate");
            const int r = alloc_reg();
            push(p, PW_LD, r, slot_for(o.inputs[0], IN_NC, 0));
            const double hw = static_cast<double>(o.saved_dims[2] * o.saved_dims[3]);
            push(p, PW_SCALE, r, 0, 0, 0, static_cast<float>(1.0 / hw));
            return r;
        }
        default:
            unsupported(std::string("op ") + std::to_string(o.op) + " cannot be fused into a DFP kernel");
    }
}

DfpModule::DfpModule(const sol_unit_desc& d) : d_(d), dtype_(d.dtype) {
    fill_arg_bytes(*this, d);
    tmpl_.dtype = dtype_;
    const int n = d.n_ops;
    // anchor
    for (int k = 0; k < n; ++k) {
        const sol_unit_op& o = d.ops[k];
        bool anchor = o.op == SOL_OP_MAXPOOL2D || o.op == SOL_OP_AVGPOOL2D || o.op == SOL_OP_GLOBALAVGPOOL ||
                      o.op == SOL_OP_MAXPOOL2DBACK || o.op == SOL_OP_AVGPOOL2DBACK || o.op == SOL_OP_CONV2D;
        if (anchor) {
            if (anchor_ >= 0) unsupported("unit has two window/global reductions");
            anchor_ = k;
        }
    }
    // geometry helpers
    auto geo_ref = [&](int r) -> Geo {
        if (r >= 0) return geo_b(d.bindings[r]);
        const sol_unit_op& o = d.ops[-r - 1];
        return geo_of_dims(o.out_rank, o.out_dims, 0);
    };
    const Geo out = geo_b(d.output);
    // BN preps (one param pair per BatchNorm2d op)
    for (int k = 0; k < n; ++k) {
        const sol_unit_op& o = d.ops[k];
        if (o.op != SOL_OP_BATCHNORM2D) continue;
        BnPrep b{};
        b.training = o.attrs.training != 0;
        b.g = o.params[0];
        b.b = o.params[1];
        b.m = o.n_params > 2 ? o.params[2] : -1;
        b.v = o.n_params > 3 ? o.params[3] : -1;
        b.eps = o.attrs.eps;
        b.momentum = o.attrs.momentum;
        const Geo xg = geo_ref(o.inputs[0]);
        b.C = static_cast<int>(xg.C);
        b.coef = static_cast<float*>(dev_alloc(5 * b.C * 4));
        if (b.training) {
            if (o.inputs[0] < 0) unsupported("training BatchNorm2d over a fused intermediate");
            b.x_binding = o.inputs[0];
            b.shift = static_cast<float*>(dev_alloc(b.C * 4));
            b.stats = static_cast<float*>(dev_alloc(2 * b.C * 4));
            b.pixels = xg.pixels();
            b.x_ld = static_cast<int>(xg.ld);
            b.xN = static_cast<int>(xg.N);
            b.xH = static_cast<int>(xg.H);
            b.xW = static_cast<int>(xg.W);
            if (xg.ld != xg.C) unsupported("training BatchNorm2d over padded storage");
            stats_scratch_ = std::max(stats_scratch_,
                                      static_cast<size_t>(dfp_reduce_blocks(b.pixels, b.C, dtype_)) * b.C * 2 * 8 + 256);
        }
        bn_of_op_[k] = static_cast<int>(bn_.size());
        if (5 * static_cast<int>(bn_.size()) + 4 >= DFP_MAX_P) unsupported("too many BatchNorms in one unit");
        bn_.push_back(b);
    }
    if (std::any_of(bn_.begin(), bn_.end(), [](const BnPrep& b) { return b.training; })) {
        int cmax = 0;
        for (auto& b : bn_) cmax = std::max(cmax, b.C);
        ones_ = static_cast<float*>(dev_alloc(cmax * 4));
        std::vector<float> ones(cmax, 1.f);
        SOL_CUDA(cudaMemcpy(ones_, ones.data(), cmax * 4, cudaMemcpyHostToDevice));
        zeros_ = static_cast<float*>(dev_alloc(cmax * 4));
    }

    // member sets: pre = ancestors of the anchor's primary input; post = everything else
    std::set<int> pre, post;
    if (anchor_ >= 0) {
        std::vector<int> stack;
        const int r0 = d.ops[anchor_].inputs[0];
        if (r0 < 0) stack.push_back(-r0 - 1);
        while (!stack.empty()) {
            int k = stack.back();
            stack.pop_back();
            if (!pre.insert(k).second) continue;
            const sol_unit_op& o = d.ops[k];
            for (int i = 0; i < o.n_inputs; ++i)
                if (o.inputs[i] < 0) stack.push_back(-o.inputs[i] - 1);
        }
    }
    for (int k = 0; k < n; ++k)
        if (!pre.count(k) && k != anchor_) post.insert(k);

    const int root = n - 1;  // unit output = last member
    // anchor-specific family + geometry
    if (anchor_ < 0) {
        tmpl_.family = FAM_POINTWISE;
        tmpl_.N = static_cast<int>(out.N);
        tmpl_.H = tmpl_.OH = static_cast<int>(out.H);
        tmpl_.W = tmpl_.OW = static_cast<int>(out.W);
        tmpl_.C = static_cast<int>(out.C);
        family = "dfp_pointwise";
    } else {
        const sol_unit_op& a = d.ops[anchor_];
        const Geo src = geo_ref(a.inputs[0]);
        const Geo aout = geo_of_dims(a.out_rank, a.out_dims, 0);
        tmpl_.N = static_cast<int>(src.N);
        tmpl_.C = static_cast<int>(src.C);
        tmpl_.kh = static_cast<int>(a.attrs.kh);
        tmpl_.kw = static_cast<int>(a.attrs.kw);
        tmpl_.sh = static_cast<int>(a.attrs.sh);
        tmpl_.sw = static_cast<int>(a.attrs.sw);
        tmpl_.ph = static_cast<int>(a.attrs.ph);
        tmpl_.pw = static_cast<int>(a.attrs.pw);
        tmpl_.min_init = a.attrs.min_init;
        tmpl_.count_padding = a.attrs.count_padding;
        switch (a.op) {
            case SOL_OP_MAXPOOL2D:
            case SOL_OP_AVGPOOL2D:
                tmpl_.family = FAM_POOL;
                tmpl_.pool_max = a.op == SOL_OP_MAXPOOL2D;
                tmpl_.H = static_cast<int>(src.H);
                tmpl_.W = static_cast<int>(src.W);
                tmpl_.OH = static_cast<int>(aout.H);
                tmpl_.OW = static_cast<int>(aout.W);
                family = a.op == SOL_OP_MAXPOOL2D ? "dfp_maxpool" : "dfp_avgpool";
                break;
            case SOL_OP_GLOBALAVGPOOL:
                tmpl_.family = FAM_GAP;
                tmpl_.H = static_cast<int>(src.H);
                tmpl_.W = static_cast<int>(src.W);
                family = "dfp_gap";
                break;
            case SOL_OP_CONV2D: {
                if (!is_depthwise(a, src.C)) unsupported("non-depthwise Conv2d inside a DFP group");
                tmpl_.family = FAM_DWCONV;
                tmpl_.H = static_cast<int>(src.H);
                tmpl_.W = static_cast<int>(src.W);
                tmpl_.OH = static_cast<int>(aout.H);
                tmpl_.OW = static_cast<int>(aout.W);
                DwPrep w{};
                w.w = a.params[0];
                w.bias = (a.attrs.has_bias && a.n_params > 1) ? a.params[1] : -1;
                w.C = static_cast<int>(src.C);
                w.kh = tmpl_.kh;
                w.kw = tmpl_.kw;
                w.packed = static_cast<float*>(dev_alloc(static_cast<size_t>(w.C) * w.kh * w.kw * 4));
                dw_.push_back(w);
                family = "dfp_dwconv";
                algo_flops = 2.0 * aout.pixels() * w.C * w.kh * w.kw;
                break;
            }
            case SOL_OP_MAXPOOL2DBACK:
            case SOL_OP_AVGPOOL2DBACK: {
                // grid = dx (anchor output), windows = delta (anchor input 0)
                tmpl_.family = a.op == SOL_OP_MAXPOOL2DBACK ? FAM_MAXPOOL_BACK : FAM_AVGPOOL_BACK;
                tmpl_.H = static_cast<int>(aout.H);
                tmpl_.W = static_cast<int>(aout.W);
                tmpl_.OH = static_cast<int>(src.H);
                tmpl_.OW = static_cast<int>(src.W);
                if (a.op == SOL_OP_MAXPOOL2DBACK) {
                    if (a.inputs[1] < 0) unsupported("MaxPool2dBack over a fused forward input");
                    tmpl_.pool_x = slot_for(a.inputs[1], IN_PIX, 0);
                    // one argmax byte per (window, channel)
                    argmax_offset_ = (stats_scratch_ + 255) / 256 * 256;
                    stats_scratch_ = argmax_offset_ + static_cast<size_t>(src.pixels()) * tmpl_.C;
                }
                family = a.op == SOL_OP_MAXPOOL2DBACK ? "dfp_maxpool_back" : "dfp_avgpool_back";
                break;
            }
        }
    }

    // pre program (anchor input at source pixels)
    if (anchor_ >= 0) {
        prog_ = &tmpl_.pre;
        uses_.clear();
        reg_of_.clear();
        free_regs_ = 0xF;
        const int r0 = d.ops[anchor_].inputs[0];
        const int key0 = r0 >= 0 ? key_b(r0) : key_op(-r0 - 1);
        count_uses(key0, pre, true);
        const int r = reg_get(key0);
        if (r != 0) push(tmpl_.pre, PW_MOV, 0, r);
    }
    // post program (output pixels; r0 holds the anchor result)
    {
        prog_ = &tmpl_.post;
        uses_.clear();
        reg_of_.clear();
        free_regs_ = 0xF;
        std::set<int> members = post;
        if (anchor_ >= 0) {
            members.insert(anchor_);
            free_regs_ &= ~1u;
            reg_of_[key_op(anchor_)] = 0;
        }
        count_uses(key_op(root), members, true);
        const int r = reg_get(key_op(root));
        if (r != 0) push(tmpl_.post, PW_MOV, 0, r);
    }
    tmpl_.out_ld = static_cast<int>(out.ld);
    if (tmpl_.family == FAM_POINTWISE || tmpl_.family == FAM_GAP) {
        if (out.C != tmpl_.C && tmpl_.family == FAM_POINTWISE) tmpl_.C = static_cast<int>(out.C);
    }
    // parameter arrays: BN coefficient triples at P[3i..3i+2]
    for (size_t i = 0; i < bn_.size(); ++i) {
        for (int k = 0; k < 5; ++k) tmpl_.P[5 * i + k] = bn_[i].coef + k * bn_[i].C;
    }
    // algorithmic bytes: external activation inputs + output
    double bytes = binding_bytes(d.output);
    for (int i = 0; i < d.n_bindings; ++i)
        if (!d.bindings[i].is_param) bytes += binding_bytes(d.bindings[i]);
    algo_bytes = bytes;
    launches = 1;
    launches_frozen = 1;  // frozen: inference BN coefficients and depthwise packs are cached
    for (auto& b : bn_) {
        launches += b.training ? 2 : 1;  // training: row reduction + finalize
        if (b.training) launches_frozen += 2;
    }
    launches += static_cast<int>(dw_.size());
}

void DfpModule::run(void* const* args, int nargs, void* scratch, cudaStream_t s, bool frozen) {
    if (nargs != n_args) throw std::invalid_argument("dfp module: wrong argument count");
    // BN coefficients (inference: from running stats; training: from batch statistics)
    for (auto& b : bn_) {
        if (!b.training) {
            if (!(frozen && coef_ready_))
                bn_infer_coef(static_cast<const float*>(args[b.g]), static_cast<const float*>(args[b.b]),
                              static_cast<const float*>(args[b.m]), static_cast<const float*>(args[b.v]), b.eps,
                              b.coef, b.C, s);
            continue;
        }
        if (b.ext_partial) {
            // statistics from the producing conv's epilogue: sums of (y - previous mean) per
            // (M tile, row quarter) block; the finalisation reads the shift before it overwrites
            // the mean with this step's (same thread per channel)
            FinalizeArgs f;
            f.mode = FIN_BN_STATS;
            f.C = b.C;
            f.blocks = b.ext_blocks;
            f.partial = b.ext_partial;
            f.count = static_cast<double>(b.pixels);
            f.eps = b.eps;
            f.shift = b.stats;
            f.gamma = static_cast<const float*>(args[b.g]);
            f.beta = static_cast<const float*>(args[b.b]);
            f.stats_out = b.stats;
            f.coef = b.coef;
            if (b.m >= 0 && b.v >= 0 && update_running_) {
                f.running_mean = static_cast<float*>(args[b.m]);
                f.running_var = static_cast<float*>(args[b.v]);
                f.momentum = b.momentum;
            }
            dfp_finalize(f, s);
            continue;
        }
        double* partial = static_cast<double*>(scratch);
        // shift = x's first pixel, read in place by the reduction and the finalize (no copy launch)
        DfpArgs a;
        a.family = FAM_CHAN_REDUCE;
        a.dtype = dtype_;
        a.N = b.xN;
        a.H = b.xH;
        a.W = b.xW;
        a.C = b.C;
        a.n_in = 1;
        a.in[0] = args[b.x_binding];
        a.in_ld[0] = b.x_ld;
        a.P[0] = nullptr;  // in-place shift: the fast row reduction reads x's first pixel
        push(a.pre, PW_LD, 0, 0);                 // r0 = x
        push(a.pre, PW_PARAM, 1, 0, 0, 0);        // r1 = shift
        push(a.pre, PW_SCALE, 1, 0, 0, 0, -1.f);  // r1 = -shift
        push(a.pre, PW_ADD, 0, 0, 1);             // r0 = x - shift
        push(a.pre, PW_MOV, 1, 0);                // r1 = r0
        a.partial = partial;
        a.reduce_blocks = dfp_reduce_blocks(b.pixels, b.C, dtype_);
        FinalizeArgs f;
        f.mode = FIN_BN_STATS;
        f.C = b.C;
        f.blocks = a.reduce_blocks;
        f.partial = partial;
        f.count = static_cast<double>(b.pixels);
        f.eps = b.eps;
        f.shift = nullptr;
        f.shift_x = args[b.x_binding];
        f.shift_dtype = dtype_;
        f.gamma = static_cast<const float*>(args[b.g]);
        f.beta = static_cast<const float*>(args[b.b]);
        f.stats_out = b.stats;
        f.coef = b.coef;
        // update_bn_running_stats (autodiff.cpp:356-384): momentum, unbiased variance, in place on
        // the running_mean / running_var parameters, from the same f64 batch statistics
        if (b.m >= 0 && b.v >= 0 && update_running_) {
            f.running_mean = static_cast<float*>(args[b.m]);
            f.running_var = static_cast<float*>(args[b.v]);
            f.momentum = b.momentum;
        }
        dfp_reduce_finalize(a, f, s);  // statistics + finalisation (one cooperative launch when possible)
    }
    for (auto& w : dw_) {
        if (!(frozen && coef_ready_))
            pack_dw_weight(static_cast<const float*>(args[w.w]), w.packed, w.C, w.kh, w.kw, s);
    }
    coef_ready_ = true;
    DfpArgs a = tmpl_;
    for (size_t i = 0; i < slot_binding_.size(); ++i)
        if (slot_binding_[i] >= 0) a.in[i] = args[slot_binding_[i]];
    for (size_t i = 0; i < cat_bindings_.size(); ++i) a.cat_ptr[i] = args[cat_bindings_[i]];
    if (!dw_.empty()) {
        a.dw_w = dw_[0].packed;
        a.dw_b = dw_[0].bias >= 0 ? static_cast<const float*>(args[dw_[0].bias]) : nullptr;
    }
    a.out = args[nargs - 1 - (act_sib_ ? 1 : 0)];
    if (act_sib_) {
        a.out2 = args[nargs - 1];
        a.act2 = act_sib_;
    }
    if (a.family == FAM_MAXPOOL_BACK) a.argmax = static_cast<uint8_t*>(scratch) + argmax_offset_;
    dfp_launch(a, s);
}

}  // namespace

std::unique_ptr<Module> compile_unit(const sol_unit_desc& d) {
    if (d.n_ops <= 0 || d.ops == nullptr) throw std::invalid_argument("empty unit");
    if (d.dtype != DT_F32 && d.dtype != DT_BF16) throw std::invalid_argument("unit dtype");
    for (int k = 0; k < d.n_ops; ++k) {
        const sol_unit_op& o = d.ops[k];
        if (o.n_inputs > SOL_MAX_OP_IN) throw std::invalid_argument("op arity");
        for (int i = 0; i < o.n_inputs; ++i) {
            const int r = o.inputs[i];
            if (r >= d.n_bindings || (r < 0 && -r - 1 >= k)) throw std::invalid_argument("bad operand ref");
        }
    }
    const sol_unit_op& o0 = d.ops[0];
    if (d.kind == 1 && d.n_ops >= 5 && o0.op == SOL_OP_CONV2D && d.ops[2].op == SOL_OP_CONV2D)
        return std::make_unique<DualConvModule>(d);
    if (d.kind == 1 && (d.n_ops == 2 || d.n_ops == 3) && o0.op == SOL_OP_CONV2DBACKX) return std::make_unique<HeavyModule>(d);
    if (d.kind == 1 && d.n_ops > 1 && (o0.op == SOL_OP_CONV2D || o0.op == SOL_OP_LINEAR)) {
        // heavy node + fused epilogue chain (plan-level fusion, see HeavyModule::parse_epilogue)
        const Geo g = geo_b(d.bindings[o0.inputs[0]]);
        if (o0.op == SOL_OP_LINEAR || !is_depthwise(o0, g.C)) return std::make_unique<HeavyModule>(d);
    }
    if (d.n_ops > 1 && o0.op == SOL_OP_SGDUPDATE) return std::make_unique<SgdMultiModule>(d);
    if (d.n_ops == 1) {
        const int op = o0.op;
        if (is_heavy_op(op)) {
            if (op == SOL_OP_CONV2D) {
                const Geo g = geo_b(d.bindings[o0.inputs[0]]);
                if (!is_depthwise(o0, g.C)) return std::make_unique<HeavyModule>(d);
            } else {
                return std::make_unique<HeavyModule>(d);
            }
        }
        switch (op) {
            case SOL_OP_SOFTMAX:
            case SOL_OP_CROSSENTROPYLOSS:
            case SOL_OP_SOFTMAXCEBACK:
            case SOL_OP_CEBACK:
            case SOL_OP_SOFTMAXBACK:
                return std::make_unique<RowModule>(d);
            case SOL_OP_FLATTEN:
            case SOL_OP_FLATTENBACK:
                return std::make_unique<FlattenModule>(d);
            case SOL_OP_SGDUPDATE:
                return std::make_unique<SgdModule>(d);
            case SOL_OP_REORDER_IN:
            case SOL_OP_REORDER_OUT:
                return std::make_unique<ReorderModule>(d);
            case SOL_OP_BATCHNORMBACKX:
            case SOL_OP_BATCHNORMBACKGAMMA:
            case SOL_OP_BATCHNORMBACKBETA:
            case SOL_OP_CONV2DBACKB:
            case SOL_OP_LINEARBACKB:
                return std::make_unique<ReduceModule>(d);
            default:
                break;
        }
    }
    for (int k = 0; k < d.n_ops; ++k) {
        const int op = d.ops[k].op;
        const bool single_only = (is_heavy_op(op) && !(op == SOL_OP_CONV2D)) || op == SOL_OP_SOFTMAX ||
                                 op == SOL_OP_CROSSENTROPYLOSS || op == SOL_OP_SOFTMAXCEBACK || op == SOL_OP_CEBACK ||
                                 op == SOL_OP_SOFTMAXBACK || op == SOL_OP_FLATTEN ||
                                 op == SOL_OP_SGDUPDATE || op == SOL_OP_BATCHNORMBACKX ||
                                 op == SOL_OP_BATCHNORMBACKGAMMA || op == SOL_OP_BATCHNORMBACKBETA ||
                                 op == SOL_OP_CONV2DBACKB || op == SOL_OP_LINEARBACKB;
        if (single_only) unsupported("op " + std::to_string(op) + " must form its own unit on B200");
    }
    return std::make_unique<DfpModule>(d);
}

}  // namespace solb200
