// graph_test.cpp -- C++ test of the routefast_b200 graph layer (include/routefast_b200/graph.hpp),
// written the way the reference's proj/tests/rewrite_test.cpp / graph_test.cpp exercise theirs:
// stacked self-attention fixtures (graph_fixtures.cpp:16-114 re-stated here), pattern finder,
// rewrite structure, idempotence, typed errors, DCE, and -- with a GPU -- original vs rewritten
// graph through interpret() (Rewrite.SemanticPreservationSingleLayer, rewrite_test.cpp:239-263).
//   graph_test --cpu   host logic only (rewriter, IR)       graph_test   everything (needs a B200)
// Tolerance on the device: 2e-2 (bf16 attention kernel vs the f32 un-fused chain).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>

#include "routefast_b200/graph.hpp"

namespace rf = routefast_b200;

static int g_failed = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
            ++g_failed;                                                      \
        }                                                                    \
    } while (0)

template <typename E, typename F>
static bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static rf::Graph fixture(int64_t B, int64_t H, int64_t S, int64_t d, int64_t local_window, const std::vector<rf::LayerKind>& layers) {
    rf::Graph g;
    g.inputs.push_back({"hidden", {B, H, S, d}, rf::DType::f32});
    g.inputs.push_back({"attention_mask", {B, 1, 1, S}, rf::DType::f32});
    g.initializers.push_back({"attn_scale", {1}, rf::DType::f32, {1.0 / std::sqrt(static_cast<double>(d))}});
    g.initializers.push_back({"mask_zero", {1}, rf::DType::f32, {0.0}});
    g.initializers.push_back({"mask_neg", {1}, rf::DType::f32, {-65504.0}});
    bool any_local = false;
    for (auto k : layers) any_local = any_local || k == rf::LayerKind::local;
    if (any_local) {
        rf::Initializer w{"local_window_pattern", {1, 1, S, S}, rf::DType::f32, {}};
        w.data.assign(static_cast<size_t>(S * S), 0.0);
        for (int64_t i = 0; i < S; ++i)
            for (int64_t j = 0; j < S; ++j)
                if (i - j <= local_window / 2 - 1 && j - i <= local_window / 2) w.data[static_cast<size_t>(i * S + j)] = 1.0;
        g.initializers.push_back(std::move(w));
    }
    std::string hidden = "hidden";
    for (size_t l = 0; l < layers.size(); ++l) {
        const std::string p = "layer" + std::to_string(l);
        const bool local = layers[l] == rf::LayerKind::local;
        rf::Node ex{p + "/mask/Expand", rf::OpKind::Expand, {"attention_mask"}, {p + "/mask/expanded"}, {}};
        ex.attrs.emplace("shape", std::vector<int64_t>{B, 1, S, S});
        g.nodes.push_back(ex);
        std::string cond = p + "/mask/expanded";
        if (local) {
            g.nodes.push_back({p + "/mask/window_and", rf::OpKind::Mul, {cond, "local_window_pattern"}, {p + "/mask/window_cond"}, {}});
            cond = p + "/mask/window_cond";
        }
        g.nodes.push_back({p + "/mask/" + (local ? "Where_1" : "Where_2"), rf::OpKind::Where, {cond, "mask_zero", "mask_neg"}, {p + "/mask/bias2d"}, {}});
        g.nodes.push_back({p + "/q_scale", rf::OpKind::Mul, {hidden, "attn_scale"}, {p + "/q_scaled"}, {}});
        rf::Node kt{p + "/k_transpose", rf::OpKind::Transpose, {hidden}, {p + "/k_t"}, {}};
        kt.attrs.emplace("perm", std::vector<int64_t>{0, 1, 3, 2});
        g.nodes.push_back(kt);
        g.nodes.push_back({p + "/qk_matmul", rf::OpKind::MatMul, {p + "/q_scaled", p + "/k_t"}, {p + "/scores"}, {}});
        g.nodes.push_back({p + "/mask_add", rf::OpKind::Add, {p + "/scores", p + "/mask/bias2d"}, {p + "/scores_masked"}, {}});
        rf::Node sm{p + "/softmax", rf::OpKind::Softmax, {p + "/scores_masked"}, {p + "/attn"}, {}};
        sm.attrs.emplace("axis", static_cast<int64_t>(-1));
        g.nodes.push_back(sm);
        g.nodes.push_back({p + "/av_matmul", rf::OpKind::MatMul, {p + "/attn", hidden}, {p + "/out"}, {}});
        hidden = p + "/out";
    }
    g.outputs.push_back(hidden);
    rf::validate_graph(g);
    return g;
}

static void host_logic() {
    using LK = rf::LayerKind;
    // FindPatterns.* (rewrite_test.cpp:27-94)
    rf::Graph tiny = rf::parse_graph(R"({"inputs": [{"name": "x", "shape": [4, 4], "dtype": "f32"}], "outputs": ["y"],
        "nodes": [{"name": "m", "op": "MatMul", "inputs": ["x", "x"], "outputs": ["y"]}]})");
    CHECK(rf::find_sdpa_patterns(tiny).empty());
    auto one = fixture(1, 2, 64, 32, 128, {LK::global});
    auto m = rf::find_sdpa_patterns(one);
    CHECK(m.size() == 1 && m[0].q == "hidden" && m[0].k == "hidden" && m[0].v == "hidden" && !m[0].k_pre_transposed);
    CHECK(m.size() == 1 && m[0].kind == LK::global && std::fabs(m[0].scale - 1.0 / std::sqrt(32.0)) < 1e-12);
    auto four = rf::find_sdpa_patterns(fixture(1, 2, 64, 32, 128, {LK::local, LK::local, LK::global, LK::local}));
    CHECK(four.size() == 4 && four[0].kind == LK::local && four[2].kind == LK::global && four[3].kind == LK::local);
    // Rewrite.* (rewrite_test.cpp:96-176)
    CHECK(rf::serialize_graph(rf::rewrite(tiny, {})) == rf::serialize_graph(tiny));
    rf::RewriteOptions o64;
    o64.head_dim = 64;
    rf::Graph rw = rf::rewrite(fixture(1, 2, 128, 64, 128, {LK::local, LK::global}), o64);
    std::vector<const rf::Node*> fused;
    for (const auto& n : rw.nodes) {
        if (n.op == rf::OpKind::FusedFlashAttention) fused.push_back(&n);
        CHECK(n.op != rf::OpKind::Where && n.op != rf::OpKind::Expand && n.op != rf::OpKind::Softmax);
    }
    CHECK(fused.size() == 2);
    if (fused.size() == 2) {
        CHECK(fused[0]->attr_int("window_left", -99) == 63 && fused[0]->attr_int("window_right", -99) == 64);
        CHECK(fused[1]->attr_int("window_left", -99) == -1 && fused[1]->attr_int("window_right", -99) == -1);
        CHECK(std::fabs(fused[0]->attr_real("scale", 0.0) - 0.125) < 1e-12 && fused[0]->inputs.size() == 4);
    }
    for (const auto& [name, shape] : rf::infer_shapes(rw))
        CHECK(!(shape.size() >= 2 && shape[shape.size() - 1] == 128 && shape[shape.size() - 2] == 128));
    rf::RewriteOptions o32;
    o32.head_dim = 32;
    rf::Graph once = rf::rewrite(fixture(1, 2, 64, 32, 128, {LK::local, LK::global, LK::local}), o32);
    CHECK(rf::serialize_graph(rf::rewrite(once, o32)) == rf::serialize_graph(once));
    rf::RewriteOptions bad = o32;
    bad.head_dim = 48;
    CHECK(throws<rf::UnsupportedHeadDim>([&] { rf::rewrite(one, bad); }));
    CHECK(throws<rf::UnsupportedHeadDim>([&] { rf::rewrite(one, o64); }));
    rf::RewriteOptions renamed = o32;
    renamed.mask_input = "no_such_input";
    CHECK(throws<rf::NoAttentionMaskInput>([&] { rf::rewrite(one, renamed); }));
    // Dce.* (rewrite_test.cpp:178-206), parse round trip, typed IR errors (graph_test.cpp)
    CHECK(rf::serialize_graph(rf::dce(one)) == rf::serialize_graph(one));
    CHECK(rf::serialize_graph(rf::parse_graph(rf::serialize_graph(once))) == rf::serialize_graph(once));
    CHECK(throws<rf::SchemaError>([] { rf::parse_graph("{\"inputs\": ["); }));
    CHECK(throws<rf::ValidationError>([] { rf::parse_graph(R"({"inputs": [], "outputs": ["y"], "nodes": []})"); }));
    CHECK(throws<rf::SchemaError>([] { rf::op_from_name("Conv"); }));
}

static void device_logic() {
    using LK = rf::LayerKind;
    struct Case { int64_t B, H, S, d, w; std::vector<LK> layers; int64_t padded; };
    const Case cases[] = {{1, 2, 96, 32, 128, {LK::local}, 7},                 // SemanticPreservationSingleLayer
                          {1, 4, 512, 64, 128, {LK::local, LK::global}, 40},
                          {2, 2, 257, 64, 64, {LK::global, LK::local, LK::local, LK::global}, 20}};  // SPEC.md:674 shapes
    for (const Case& c : cases) {
        rf::Graph g = fixture(c.B, c.H, c.S, c.d, c.w, c.layers);
        rf::RewriteOptions opt;
        opt.head_dim = c.d;
        opt.local_window = c.w;
        rf::Graph rw = rf::rewrite(g, opt);
        std::mt19937_64 rng(7);
        rf::Tensor hidden({c.B, c.H, c.S, c.d});
        for (auto& v : hidden.data) v = static_cast<float>(2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0);
        rf::Tensor mask = rf::Tensor::full({c.B, 1, 1, c.S}, 1.0f);
        for (int64_t i = 0; i < c.padded; ++i) mask.data[mask.data.size() - 1 - static_cast<size_t>(i)] = 0.0f;
        rf::TensorMap in{{"hidden", hidden}, {"attention_mask", mask}};
        rf::InterpretStats sa, sb;
        auto a = rf::interpret(g, in, 0, &sa);
        auto b = rf::interpret(rw, in, 0, &sb);
        const rf::Tensor& ta = a.at(g.outputs[0]);
        const rf::Tensor& tb = b.at(g.outputs[0]);
        CHECK(ta.shape == tb.shape);
        double worst = 0.0;  // unpadded query rows (see verify_rewrite in paper_2603_12646_b200/graph.py)
        for (int64_t bh = 0; bh < c.B * c.H; ++bh)
            for (int64_t i = 0; i < c.S; ++i) {
                if (bh / c.H == c.B - 1 && i >= c.S - c.padded) continue;
                for (int64_t x = 0; x < c.d; ++x) {
                    const size_t idx = static_cast<size_t>((bh * c.S + i) * c.d + x);
                    worst = std::max(worst, static_cast<double>(std::fabs(ta.data[idx] - tb.data[idx])));
                }
            }
        std::printf("S=%lld d=%lld layers=%zu: max-abs %.3e; largest tensor %zu -> %zu bytes, %.3f -> %.3f ms\n",
                    static_cast<long long>(c.S), static_cast<long long>(c.d), c.layers.size(), worst,
                    sa.largest_tensor_bytes, sb.largest_tensor_bytes, sa.device_ms, sb.device_ms);
        CHECK(worst <= 2e-2);
        CHECK(sa.largest_tensor_bytes == static_cast<size_t>(c.B * c.H * c.S * c.S * 4));
        CHECK(sb.largest_tensor_bytes == static_cast<size_t>(c.B * c.H * c.S * c.d * 4));
    }
    rf::Graph g = fixture(1, 2, 16, 32, 128, {LK::global});
    CHECK(throws<rf::ShapeMismatch>([&] { rf::interpret(g, {}); }));
}

int main(int argc, char** argv) {
    const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu") == 0;
    host_logic();
    if (!cpu_only) device_logic();
    if (g_failed == 0) std::printf("all checks passed%s\n", cpu_only ? " (host logic only)" : "");
    return g_failed == 0 ? 0 : 1;
}
