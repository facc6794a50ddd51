// routefast_b200/attention.hpp -- C++ mirror of the reference operator interface
// (reference: proj/core/include/routefast/attention.hpp:15-61, tensor.hpp:16-40), implemented on
// the B200 through the C ABI of librf_fa.so (include/rf_fa.h).  Header-only; link with -lrf_fa.
//
// Same names, argument meaning and error behaviour as the reference:
//   kMaskValue / kMaskThreshold, Tensor, ShapeMismatch, UnsupportedHeadDim, AttentionSpec,
//   FlashStats, flash_attention(q, k, v, spec, tile = 64, stats = nullptr),
//   mask_memory_bytes, fa_memory_bytes.
// A reference call site compiles against this header by switching the namespace.
// There is no CPU fallback: a missing GPU surfaces as std::runtime_error.
#pragma once

#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../rf_fa.h"

namespace routefast_b200 {

constexpr float kMaskValue = RF_MASK_VALUE;          // attention.hpp:15
constexpr float kMaskThreshold = RF_MASK_THRESHOLD;  // attention.hpp:16

class ShapeMismatch : public std::runtime_error {  // tensor.hpp:16-19
public:
    using std::runtime_error::runtime_error;
};
class UnsupportedHeadDim : public std::runtime_error {  // rewrite.hpp:14-17
public:
    using std::runtime_error::runtime_error;
};

enum class DType { f32, f16 };  // graph.hpp:28

// Dense row-major tensor on the host (tensor.hpp:24-40); f16 is stored as f32 values that went
// through a binary16 round trip.
struct Tensor {
    std::vector<int64_t> shape;
    DType dtype = DType::f32;
    std::vector<float> data;

    Tensor() = default;
    explicit Tensor(std::vector<int64_t> shape_in) : shape(std::move(shape_in)) {
        std::size_t n = 1;
        for (int64_t d : shape) {
            if (d < 0) throw ShapeMismatch("negative dimension");
            n *= static_cast<std::size_t>(d);
        }
        data.assign(n, 0.0f);
    }
    std::size_t numel() const { return data.size(); }
    static Tensor full(std::vector<int64_t> shape, float value) {
        Tensor t(std::move(shape));
        for (auto& v : t.data) v = value;
        return t;
    }
};

struct AttentionSpec {  // attention.hpp:18-25
    double scale = 0.0;        // 0 -> 1/sqrt(head_dim)
    int64_t window_left = -1;  // -1 = unbounded
    int64_t window_right = -1;
    std::optional<Tensor> pad_bias;  // [B,1,1,S], 0 or -65504 per key

    double effective_scale(int64_t head_dim) const {  // attention.cpp:34-36
        return scale != 0.0 ? scale : 1.0 / std::sqrt(static_cast<double>(head_dim));
    }
};

struct FlashStats {  // attention.hpp:36-40 (+ what the device path adds)
    std::size_t tile_scratch_floats = 0;
    std::size_t row_state_floats = 0;
    std::size_t output_floats = 0;
    std::size_t workspace_bytes = 0;     // O(S) device workspace of the call
    std::size_t score_matrix_bytes = 0;  // always 0
    int kernel = 0;                      // rf_kernel
};

// Tiled streaming-softmax attention on the GPU: no S x S materialisation, bit-for-bit
// deterministic (attention.hpp:42-48).  `device` selects the CUDA device.
inline Tensor flash_attention(const Tensor& q, const Tensor& k, const Tensor& v, const AttentionSpec& spec,
                              int64_t tile = 64, FlashStats* stats = nullptr, int device = 0) {
    if (q.shape.size() != 4 || k.shape.size() != 4 || v.shape.size() != 4)  // attention.cpp:14-21
        throw ShapeMismatch("attention inputs must be [B,H,S,d]");
    if (q.shape != k.shape || q.shape != v.shape) throw ShapeMismatch("Q, K, V must have identical shapes");
    const int64_t B = q.shape[0], H = q.shape[1], S = q.shape[2], d = q.shape[3];
    const float* bias = nullptr;
    const int64_t* bias_dims = nullptr;
    if (spec.pad_bias) {
        if (spec.pad_bias->shape.size() != 4) throw ShapeMismatch("pad_bias must be [B,1,1,S]");
        bias = spec.pad_bias->data.data();
        bias_dims = spec.pad_bias->shape.data();
    }
    Tensor out({B, H, S, d});
    rf_fa_stats st{};
    const int rc = rf_fa_fwd_host(q.data.data(), k.data.data(), v.data.data(), out.data.data(), B, H, S, d,
                                  spec.scale, spec.window_left, spec.window_right, bias, bias_dims, tile,
                                  RF_DTYPE_BF16, device, &st);
    if (rc == RF_ERR_SHAPE) throw ShapeMismatch(rf_last_error());
    if (rc == RF_ERR_HEAD_DIM) throw UnsupportedHeadDim(rf_last_error());
    if (rc != RF_OK) throw std::runtime_error(std::string("rf_fa: ") + rf_last_error());
    if (stats) {  // attention.cpp:126-130
        stats->tile_scratch_floats = static_cast<std::size_t>(tile);
        stats->row_state_floats = static_cast<std::size_t>(2 * S);
        stats->output_floats = out.data.size();
        stats->workspace_bytes = st.workspace_bytes;
        stats->score_matrix_bytes = st.score_matrix_bytes;
        stats->kernel = st.kernel;
    }
    return out;
}

inline uint64_t mask_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t bytes_per_element) {
    return rf_mask_memory_bytes(batch, heads, seq_len, bytes_per_element);
}
inline uint64_t fa_memory_bytes(uint64_t batch, uint64_t heads, uint64_t seq_len, uint64_t head_dim, uint64_t tile,
                                uint64_t bytes_per_element) {
    return rf_fa_memory_bytes(batch, heads, seq_len, head_dim, tile, bytes_per_element);
}

}  // namespace routefast_b200
