// graph_executor.cu -- runs the 11-op graph IR on the B200 (the caller of the attention operator).
//
// Role of the reference's interpret() (proj/core/src/interpreter.cpp:190-335): bind inputs and
// initializers, run the nodes in topological order, return the graph outputs.  Here every tensor
// lives in HBM (f32 storage; f16 tensors hold binary16-rounded values, tensor.hpp:21-23) and every
// op is a CUDA kernel of this file, except FusedFlashAttention, which casts Q/K/V to bf16 and
// launches the tcgen05 kernel through rf_fa_fwd -- exactly the dispatch of interpreter.cpp:308-318
// (attrs scale / window_left / window_right with defaults 0.0 / -1 / -1, optional 4th input).
// The un-rewritten SDPA chain materialises its [B,H,S,S] tensors (scores, mask, probabilities);
// the rewritten graph never allocates one: InterpretStats::largest_tensor_bytes shows the gap.
//
// Differences from the reference that the tests state as tolerances: MatMul accumulates in f32
// (reference: f64, interpreter.cpp:97-103), Softmax is computed in f32 (reference: f64, :131-140).
// Tensors are released right after their last reader (stream-ordered pool), which the reference,
// keeping every intermediate alive in a map, does not do.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <unordered_map>

#include "../../../include/rf_fa.h"
#include "../fa_internal.h"
#include "routefast_b200/graph.hpp"

namespace routefast_b200 {

namespace {

constexpr int kMaxRank = 8;
using Shape = std::vector<int64_t>;

std::size_t numel_of(const Shape& s) {
    std::size_t n = 1;
    for (int64_t d : s) n *= static_cast<std::size_t>(std::max<int64_t>(d, 0));
    return n;
}

// ---------------------------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------------------------
// Output-driven gather: every output element reads each operand through per-axis strides (0 on a
// broadcast axis, permuted strides for Transpose).  One kernel shape serves Add/Sub/Mul, Where,
// Expand and Transpose.
struct GatherMap {
    int rank;
    long long dims[kMaxRank];          // output dims
    long long stride[3][kMaxRank];     // element strides of up to three operands
};

enum class Ew { Add, Sub, Mul, Where, Copy };

template <Ew kOp>
__global__ void gather_kernel(GatherMap map, const float* __restrict__ a, const float* __restrict__ b,
                              const float* __restrict__ c, float* __restrict__ out, long long n) {
    for (long long flat = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; flat < n;
         flat += static_cast<long long>(gridDim.x) * blockDim.x) {
        long long rem = flat, ia = 0, ib = 0, ic = 0;
#pragma unroll 1
        for (int ax = map.rank - 1; ax >= 0; --ax) {
            const long long coord = rem % map.dims[ax];
            rem /= map.dims[ax];
            ia += coord * map.stride[0][ax];
            if (kOp != Ew::Copy) ib += coord * map.stride[1][ax];
            if (kOp == Ew::Where) ic += coord * map.stride[2][ax];
        }
        float r;
        if (kOp == Ew::Add) r = a[ia] + b[ib];
        else if (kOp == Ew::Sub) r = a[ia] - b[ib];
        else if (kOp == Ew::Mul) r = a[ia] * b[ib];
        else if (kOp == Ew::Where) r = a[ia] != 0.0f ? b[ib] : c[ic];
        else r = a[ia];
        out[flat] = r;
    }
}

// binary16 round trip, round-to-nearest-even, overflow to inf (tensor.cpp:47-98)
__global__ void quantize_f16_kernel(const float* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x)
        out[i] = __half2float(__float2half_rn(in[i]));
}

// Softmax along one axis: tensor viewed as [outer, len, inner]; one CTA per (outer, inner) line.
__global__ void __launch_bounds__(256) softmax_kernel(const float* __restrict__ x, float* __restrict__ y, long long len,
                                                      long long inner) {
    const long long line = blockIdx.x;
    const long long o = line / inner, in = line % inner;
    const float* src = x + o * len * inner + in;
    float* dst = y + o * len * inner + in;
    __shared__ float red[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    float mx = -INFINITY;
    for (long long i = threadIdx.x; i < len; i += blockDim.x) mx = fmaxf(mx, src[i * inner]);
    for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    if (lane == 0) red[warp] = mx;
    __syncthreads();
    mx = red[0];
    for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
    __syncthreads();

    float sum = 0.f;
    for (long long i = threadIdx.x; i < len; i += blockDim.x) sum += expf(src[i * inner] - mx);
    for (int s = 16; s > 0; s >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, s);
    if (lane == 0) red[warp] = sum;
    __syncthreads();
    sum = 0.f;
    for (int w = 0; w < 8; ++w) sum += red[w];
    const float inv = 1.0f / sum;
    for (long long i = threadIdx.x; i < len; i += blockDim.x) dst[i * inner] = expf(src[i * inner] - mx) * inv;
}

// Batched C[m,n] = A[m,k] * B[k,n], row-major f32, batch dims broadcast (numpy rules).
// 64x64 output tile per CTA, 16-deep k slices in shared memory, 4x4 accumulators per thread.
struct BatchMap {
    int rank;
    long long dims[kMaxRank];
    long long sa[kMaxRank];  // block strides (in matrices) of A and B per batch axis, 0 = broadcast
    long long sb[kMaxRank];
};

__global__ void __launch_bounds__(256) matmul_kernel(BatchMap bm, const float* __restrict__ A, const float* __restrict__ B,
                                                     float* __restrict__ C, int M, int N, int K) {
    constexpr int T = 64, KS = 16;
    __shared__ float As[KS][T + 4];
    __shared__ float Bs[KS][T + 4];
    long long rem = blockIdx.z, ba = 0, bb = 0;
    for (int ax = bm.rank - 1; ax >= 0; --ax) {
        const long long coord = rem % bm.dims[ax];
        rem /= bm.dims[ax];
        ba += coord * bm.sa[ax];
        bb += coord * bm.sb[ax];
    }
    const float* a = A + ba * static_cast<long long>(M) * K;
    const float* b = B + bb * static_cast<long long>(K) * N;
    float* c = C + static_cast<long long>(blockIdx.z) * M * N;
    const int row0 = blockIdx.y * T, col0 = blockIdx.x * T;
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += KS) {
        for (int e = threadIdx.x; e < T * KS; e += 256) {
            const int r = e / KS, kk = e % KS;  // A tile: 64 rows x 16 k, k fastest in memory
            const int gr = row0 + r, gk = k0 + kk;
            As[kk][r] = (gr < M && gk < K) ? a[static_cast<long long>(gr) * K + gk] : 0.f;
        }
        for (int e = threadIdx.x; e < T * KS; e += 256) {
            const int kk = e / T, cc = e % T;   // B tile: 16 k x 64 cols, cols fastest in memory
            const int gk = k0 + kk, gc = col0 + cc;
            Bs[kk][cc] = (gk < K && gc < N) ? b[static_cast<long long>(gk) * N + gc] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < KS; ++kk) {
            float av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gr = row0 + ty * 4 + i;
        if (gr >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gc = col0 + tx * 4 + j;
            if (gc < N) c[static_cast<long long>(gr) * N + gc] = acc[i][j];
        }
    }
}

// ---------------------------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------------------------
struct DevTensor {
    Shape shape;
    DType dtype = DType::f32;
    float* ptr = nullptr;
    std::size_t bytes = 0;
};

[[noreturn]] void cuda_throw(cudaError_t e, const char* what) {
    throw std::runtime_error(std::string("rf_graph: ") + what + ": " + cudaGetErrorString(e));
}
#define RF_CUDA(call, what)                      \
    do {                                         \
        cudaError_t e_ = (call);                 \
        if (e_ != cudaSuccess) cuda_throw(e_, what); \
    } while (0)

class Runner {
public:
    Runner(int device, InterpretStats* stats) : stats_(stats) {
        int count = 0;
        if (cudaGetDeviceCount(&count) != cudaSuccess || device < 0 || device >= count) {
            cudaGetLastError();
            throw std::runtime_error("rf_graph: no CUDA device " + std::to_string(device) +
                                     " (the graph executor has no CPU fallback)");
        }
        RF_CUDA(cudaSetDevice(device), "cudaSetDevice");
        RF_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    ~Runner() {
        for (auto& kv : env_) release(kv.second);
        if (stream_ != nullptr) {
            cudaStreamSynchronize(stream_);
            cudaStreamDestroy(stream_);
        }
    }
    Runner(const Runner&) = delete;
    Runner& operator=(const Runner&) = delete;

    cudaStream_t stream() const { return stream_; }

    DevTensor alloc(Shape shape, DType dtype = DType::f32) {
        DevTensor t;
        t.shape = std::move(shape);
        t.dtype = dtype;
        t.bytes = numel_of(t.shape) * sizeof(float);
        if (t.bytes > 0) {
            RF_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&t.ptr), t.bytes, stream_), "cudaMallocAsync");
            live_bytes_ += t.bytes;
            peak_bytes_ = std::max(peak_bytes_, live_bytes_);
            largest_ = std::max(largest_, t.bytes);
        }
        return t;
    }
    void release(DevTensor& t) {
        if (t.ptr != nullptr) {
            cudaFreeAsync(t.ptr, stream_);
            live_bytes_ -= t.bytes;
            t.ptr = nullptr;
        }
    }
    void* scratch(std::size_t bytes) {  // freed by the caller with cudaFreeAsync on stream()
        void* p = nullptr;
        RF_CUDA(cudaMallocAsync(&p, bytes, stream_), "cudaMallocAsync");
        live_bytes_ += bytes;
        peak_bytes_ = std::max(peak_bytes_, live_bytes_);
        return p;
    }
    void scratch_free(void* p, std::size_t bytes) {
        cudaFreeAsync(p, stream_);
        live_bytes_ -= bytes;
    }
    void count_launch(std::size_t n = 1) { launches_ += n; }

    std::unordered_map<std::string, DevTensor> env_;

    void finish(double ms) {
        if (stats_ == nullptr) return;
        stats_->peak_device_bytes = peak_bytes_;
        stats_->launches = launches_;
        stats_->largest_tensor_bytes = largest_;
        stats_->device_ms = ms;
    }

private:
    cudaStream_t stream_ = nullptr;
    InterpretStats* stats_;
    std::size_t live_bytes_ = 0, peak_bytes_ = 0, largest_ = 0, launches_ = 0;
};

int grid_for(std::size_t n, int block = 256) {
    const std::size_t want = (n + block - 1) / block;
    return static_cast<int>(std::min<std::size_t>(std::max<std::size_t>(want, 1), 148 * 16));
}

Shape broadcast_shape(const Shape& a, const Shape& b, const std::string& node) {
    const std::size_t rank = std::max(a.size(), b.size());
    Shape out(rank, 1);
    for (std::size_t i = 0; i < rank; ++i) {
        const int64_t da = i + a.size() < rank ? 1 : a[i + a.size() - rank];
        const int64_t db = i + b.size() < rank ? 1 : b[i + b.size() - rank];
        if (da != db && da != 1 && db != 1) throw ShapeMismatch("node '" + node + "': operands not broadcastable");
        out[i] = std::max(da, db);
    }
    return out;
}

// strides of `shape` viewed through the (right-aligned) output rank, 0 where it broadcasts
void fill_broadcast_strides(const Shape& shape, std::size_t out_rank, long long* stride) {
    std::vector<long long> dense(shape.size(), 1);
    for (std::size_t i = shape.size(); i-- > 1;) dense[i - 1] = dense[i] * shape[i];
    for (std::size_t ax = 0; ax < out_rank; ++ax) {
        if (ax + shape.size() < out_rank) {
            stride[ax] = 0;
        } else {
            const std::size_t j = ax + shape.size() - out_rank;
            stride[ax] = shape[j] == 1 ? 0 : dense[j];
        }
    }
}

GatherMap gather_map(const Shape& out, const std::string& node) {
    if (out.size() > static_cast<std::size_t>(kMaxRank))
        throw ShapeMismatch("node '" + node + "': rank > " + std::to_string(kMaxRank) + " is not supported");
    GatherMap m{};
    m.rank = static_cast<int>(out.size());
    for (std::size_t i = 0; i < out.size(); ++i) m.dims[i] = out[i];
    return m;
}

template <Ew kOp>
void launch_gather(Runner& rt, const GatherMap& map, const float* a, const float* b, const float* c, DevTensor& out) {
    const std::size_t n = numel_of(out.shape);
    if (n == 0) return;
    gather_kernel<kOp><<<grid_for(n), 256, 0, rt.stream()>>>(map, a, b, c, out.ptr, static_cast<long long>(n));
    RF_CUDA(cudaGetLastError(), "gather launch");
    rt.count_launch();
}

DevTensor run_binary(Runner& rt, OpKind op, const DevTensor& a, const DevTensor& b, const std::string& node) {
    DevTensor out = rt.alloc(broadcast_shape(a.shape, b.shape, node));
    GatherMap map = gather_map(out.shape, node);
    fill_broadcast_strides(a.shape, out.shape.size(), map.stride[0]);
    fill_broadcast_strides(b.shape, out.shape.size(), map.stride[1]);
    if (op == OpKind::Add) launch_gather<Ew::Add>(rt, map, a.ptr, b.ptr, nullptr, out);
    else if (op == OpKind::Sub) launch_gather<Ew::Sub>(rt, map, a.ptr, b.ptr, nullptr, out);
    else launch_gather<Ew::Mul>(rt, map, a.ptr, b.ptr, nullptr, out);
    return out;
}

DevTensor run_where(Runner& rt, const DevTensor& cond, const DevTensor& x, const DevTensor& y, const std::string& node) {
    DevTensor out = rt.alloc(broadcast_shape(broadcast_shape(cond.shape, x.shape, node), y.shape, node));
    GatherMap map = gather_map(out.shape, node);
    fill_broadcast_strides(cond.shape, out.shape.size(), map.stride[0]);
    fill_broadcast_strides(x.shape, out.shape.size(), map.stride[1]);
    fill_broadcast_strides(y.shape, out.shape.size(), map.stride[2]);
    launch_gather<Ew::Where>(rt, map, cond.ptr, x.ptr, y.ptr, out);
    return out;
}

DevTensor run_expand(Runner& rt, const DevTensor& x, const Shape& target, const std::string& node) {
    DevTensor out = rt.alloc(broadcast_shape(x.shape, target, node));
    GatherMap map = gather_map(out.shape, node);
    fill_broadcast_strides(x.shape, out.shape.size(), map.stride[0]);
    launch_gather<Ew::Copy>(rt, map, x.ptr, nullptr, nullptr, out);
    return out;
}

DevTensor run_transpose(Runner& rt, const DevTensor& x, const std::vector<int64_t>& perm, const std::string& node) {
    if (perm.size() != x.shape.size()) throw ShapeMismatch("node '" + node + "': transpose perm rank mismatch");
    std::vector<long long> dense(x.shape.size(), 1);
    for (std::size_t i = x.shape.size(); i-- > 1;) dense[i - 1] = dense[i] * x.shape[i];
    Shape out_shape(perm.size());
    for (std::size_t i = 0; i < perm.size(); ++i) {
        if (perm[i] < 0 || perm[i] >= static_cast<int64_t>(perm.size()))
            throw ShapeMismatch("node '" + node + "': transpose perm out of range");
        out_shape[i] = x.shape[static_cast<std::size_t>(perm[i])];
    }
    DevTensor out = rt.alloc(out_shape);
    GatherMap map = gather_map(out.shape, node);
    for (std::size_t i = 0; i < perm.size(); ++i) map.stride[0][i] = dense[static_cast<std::size_t>(perm[i])];
    launch_gather<Ew::Copy>(rt, map, x.ptr, nullptr, nullptr, out);
    return out;
}

void quantize_in_place(Runner& rt, DevTensor& t) {
    const std::size_t n = numel_of(t.shape);
    if (n == 0) return;
    quantize_f16_kernel<<<grid_for(n), 256, 0, rt.stream()>>>(t.ptr, t.ptr, static_cast<long long>(n));
    RF_CUDA(cudaGetLastError(), "quantize_f16 launch");
    rt.count_launch();
}

DevTensor run_cast(Runner& rt, const DevTensor& x, DType target) {
    DevTensor out = rt.alloc(x.shape, target);
    const std::size_t n = numel_of(x.shape);
    if (n == 0) return out;
    if (target == DType::f16) {
        quantize_f16_kernel<<<grid_for(n), 256, 0, rt.stream()>>>(x.ptr, out.ptr, static_cast<long long>(n));
        RF_CUDA(cudaGetLastError(), "quantize_f16 launch");
        rt.count_launch();
    } else {
        RF_CUDA(cudaMemcpyAsync(out.ptr, x.ptr, out.bytes, cudaMemcpyDeviceToDevice, rt.stream()), "D2D copy");
    }
    return out;
}

DevTensor run_softmax(Runner& rt, const DevTensor& x, int64_t axis, const std::string& node) {
    const int64_t rank = static_cast<int64_t>(x.shape.size());
    if (axis < 0) axis += rank;
    if (axis < 0 || axis >= rank) throw ShapeMismatch("node '" + node + "': bad softmax axis");
    std::size_t outer = 1, inner = 1;
    for (int64_t i = 0; i < axis; ++i) outer *= static_cast<std::size_t>(x.shape[i]);
    for (int64_t i = axis + 1; i < rank; ++i) inner *= static_cast<std::size_t>(x.shape[i]);
    const std::size_t len = static_cast<std::size_t>(x.shape[axis]);
    DevTensor out = rt.alloc(x.shape);
    const std::size_t lines = outer * inner;
    if (lines == 0 || len == 0) return out;
    if (lines > 0x7fffffffull) throw ShapeMismatch("node '" + node + "': too many softmax lines");
    softmax_kernel<<<static_cast<unsigned>(lines), 256, 0, rt.stream()>>>(x.ptr, out.ptr, static_cast<long long>(len),
                                                                           static_cast<long long>(inner));
    RF_CUDA(cudaGetLastError(), "softmax launch");
    rt.count_launch();
    return out;
}

DevTensor run_matmul(Runner& rt, const DevTensor& a, const DevTensor& b, const std::string& node) {
    if (a.shape.size() < 2 || b.shape.size() < 2) throw ShapeMismatch("node '" + node + "': MatMul needs rank >= 2");
    const int64_t m = a.shape[a.shape.size() - 2], ka = a.shape[a.shape.size() - 1];
    const int64_t kb = b.shape[b.shape.size() - 2], n = b.shape[b.shape.size() - 1];
    if (ka != kb) throw ShapeMismatch("node '" + node + "': MatMul inner dims differ");
    const Shape batch_a(a.shape.begin(), a.shape.end() - 2), batch_b(b.shape.begin(), b.shape.end() - 2);
    const Shape batch = broadcast_shape(batch_a, batch_b, node);
    Shape out_shape = batch;
    out_shape.push_back(m);
    out_shape.push_back(n);
    DevTensor out = rt.alloc(out_shape);
    const std::size_t batches = numel_of(batch);
    if (batches == 0 || m == 0 || n == 0) return out;
    if (batch.size() > static_cast<std::size_t>(kMaxRank)) throw ShapeMismatch("node '" + node + "': too many batch dims");
    if (batches > 65535 || m > 0x7fffffff || n > 0x7fffffff || ka > 0x7fffffff)
        throw ShapeMismatch("node '" + node + "': MatMul too large for this executor");
    if (ka == 0) {
        RF_CUDA(cudaMemsetAsync(out.ptr, 0, out.bytes, rt.stream()), "cudaMemsetAsync");
        return out;
    }
    BatchMap bm{};
    bm.rank = static_cast<int>(batch.size());
    for (std::size_t i = 0; i < batch.size(); ++i) bm.dims[i] = batch[i];
    fill_broadcast_strides(batch_a, batch.size(), bm.sa);
    fill_broadcast_strides(batch_b, batch.size(), bm.sb);
    dim3 grid(static_cast<unsigned>((n + 63) / 64), static_cast<unsigned>((m + 63) / 64), static_cast<unsigned>(batches));
    matmul_kernel<<<grid, 256, 0, rt.stream()>>>(bm, a.ptr, b.ptr, out.ptr, static_cast<int>(m), static_cast<int>(n),
                                                 static_cast<int>(ka));
    RF_CUDA(cudaGetLastError(), "matmul launch");
    rt.count_launch();
    return out;
}

// interpreter.cpp:308-318 + attention.cpp:14-21,111-116 (check_qkv, pad_bias shape)
DevTensor run_fused_attention(Runner& rt, const Node& node, const DevTensor& q, const DevTensor& k, const DevTensor& v,
                              const DevTensor* pad_bias) {
    if (q.shape.size() != 4 || k.shape.size() != 4 || v.shape.size() != 4)
        throw ShapeMismatch("attention inputs must be [B,H,S,d]");
    if (q.shape != k.shape || q.shape != v.shape) throw ShapeMismatch("Q, K, V must have identical shapes");
    const int64_t B = q.shape[0], H = q.shape[1], S = q.shape[2], d = q.shape[3];
    if (pad_bias != nullptr && pad_bias->shape != Shape{B, 1, 1, S}) throw ShapeMismatch("pad_bias must be [B,1,1,S]");

    DevTensor out = rt.alloc(q.shape);
    const std::size_t n = numel_of(q.shape);
    if (n == 0) return out;

    rf_fa_params p;
    rf_fa_params_init(&p);
    p.B = B;
    p.H = H;
    p.S = S;
    p.d = d;
    p.scale = node.attr_real("scale", 0.0);
    p.window_left = node.attr_int("window_left", -1);
    p.window_right = node.attr_int("window_right", -1);
    p.dtype = RF_DTYPE_BF16;
    p.out_dtype = RF_DTYPE_F32;
    // scratch buffers are released on every exit path, including a throwing RF_CUDA / rt.scratch
    struct Scratch {
        Runner& rt;
        void* ptr = nullptr;
        std::size_t bytes = 0;
        explicit Scratch(Runner& r) : rt(r) {}
        void* get(std::size_t n_bytes) {
            ptr = rt.scratch(n_bytes);
            bytes = n_bytes;
            return ptr;
        }
        ~Scratch() {
            if (ptr != nullptr) rt.scratch_free(ptr, bytes);
        }
    };
    Scratch qkv_buf(rt), ws_buf(rt);
    uint16_t* qkv16 = static_cast<uint16_t*>(qkv_buf.get(3 * n * 2));
    const float* src[3] = {q.ptr, k.ptr, v.ptr};
    for (int t = 0; t < 3; ++t) {
        RF_CUDA(rf::launch_cast_from_f32(src[t], qkv16 + static_cast<std::size_t>(t) * n, static_cast<long long>(n),
                                         RF_DTYPE_BF16, rt.stream()),
                "cast launch");
        rt.count_launch();
    }
    p.q = qkv16;
    p.k = qkv16 + n;
    p.v = qkv16 + 2 * n;
    p.out = out.ptr;
    p.pad_bias = pad_bias != nullptr ? pad_bias->ptr : nullptr;
    std::size_t ws_bytes = 0;
    int rc = rf_fa_fwd_workspace_bytes(&p, &ws_bytes);
    void* ws = nullptr;
    if (rc == RF_OK && ws_bytes > 0) ws = ws_buf.get(ws_bytes);
    if (rc == RF_OK) rc = rf_fa_fwd(&p, ws, ws_bytes, rt.stream());
    if (rc == RF_ERR_SHAPE) throw ShapeMismatch(rf_last_error());
    if (rc == RF_ERR_HEAD_DIM) throw UnsupportedHeadDim(rf_last_error());
    if (rc != RF_OK) throw std::runtime_error(std::string("rf_fa: ") + rf_last_error());
    rt.count_launch(p.pad_bias != nullptr ? 2 : 1);  // (bias_prepare +) attention kernel
    return out;
}

DevTensor upload(Runner& rt, const Shape& shape, DType dtype, const float* host) {
    DevTensor t = rt.alloc(shape, dtype);
    if (t.bytes > 0) RF_CUDA(cudaMemcpyAsync(t.ptr, host, t.bytes, cudaMemcpyHostToDevice, rt.stream()), "H2D copy");
    return t;
}

}  // namespace

TensorMap interpret(const Graph& graph, const TensorMap& inputs, int device, InterpretStats* stats) {
    // bind before touching the device, so that binding errors do not depend on a GPU
    for (const TensorDecl& decl : graph.inputs) {
        auto it = inputs.find(decl.name);
        if (it == inputs.end()) throw ShapeMismatch("graph input '" + decl.name + "' is not bound");
        if (it->second.shape != decl.shape) throw ShapeMismatch("graph input '" + decl.name + "' has wrong shape");
    }
    const std::vector<std::size_t> order = topological_order(graph);

    // last reader of every tensor (position in `order`); graph outputs stay alive to the end
    std::unordered_map<std::string, std::size_t> last_use;
    for (std::size_t pos = 0; pos < order.size(); ++pos)
        for (const std::string& t : graph.nodes[order[pos]].inputs) last_use[t] = pos;
    for (const std::string& t : graph.outputs) last_use[t] = order.size();

    Runner rt(device, stats);
    auto& env = rt.env_;
    std::vector<float> staging;
    for (const TensorDecl& decl : graph.inputs) {
        const Tensor& host = inputs.at(decl.name);
        if (host.data.size() != numel_of(decl.shape)) throw ShapeMismatch("graph input '" + decl.name + "' has wrong shape");
        env[decl.name] = upload(rt, decl.shape, host.dtype, host.data.data());
    }
    for (const Initializer& init : graph.initializers) {
        staging.resize(init.data.size());
        for (std::size_t i = 0; i < init.data.size(); ++i) staging[i] = static_cast<float>(init.data[i]);
        DevTensor t = upload(rt, init.shape, init.dtype, staging.data());
        RF_CUDA(cudaStreamSynchronize(rt.stream()), "stream sync");  // staging is reused
        if (init.dtype == DType::f16) quantize_in_place(rt, t);
        env[init.name] = std::move(t);
    }

    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    RF_CUDA(cudaEventCreate(&ev0), "cudaEventCreate");
    RF_CUDA(cudaEventCreate(&ev1), "cudaEventCreate");
    struct EventGuard {
        cudaEvent_t a, b;
        ~EventGuard() {
            cudaEventDestroy(a);
            cudaEventDestroy(b);
        }
    } guard{ev0, ev1};
    RF_CUDA(cudaEventRecord(ev0, rt.stream()), "cudaEventRecord");

    for (std::size_t pos = 0; pos < order.size(); ++pos) {
        const Node& node = graph.nodes[order[pos]];
        auto in = [&](std::size_t i) -> const DevTensor& {
            auto it = env.find(node.inputs.at(i));
            if (it == env.end() || (it->second.ptr == nullptr && it->second.bytes > 0))
                throw ShapeMismatch("node '" + node.name + "': missing input tensor");
            return it->second;
        };
        DevTensor result;
        switch (node.op) {
            case OpKind::MatMul:
                result = run_matmul(rt, in(0), in(1), node.name);
                break;
            case OpKind::Add:
            case OpKind::Sub:
            case OpKind::Mul:
                result = run_binary(rt, node.op, in(0), in(1), node.name);
                break;
            case OpKind::Softmax:
                result = run_softmax(rt, in(0), node.attr_int("axis", -1), node.name);
                break;
            case OpKind::Transpose: {
                const std::vector<int64_t>* perm = node.attr_ints("perm");
                if (perm == nullptr) throw ShapeMismatch("node '" + node.name + "': missing perm");
                result = run_transpose(rt, in(0), *perm, node.name);
                break;
            }
            case OpKind::Cast: {
                const std::string* to = node.attr_string("to");
                if (to == nullptr) throw ShapeMismatch("node '" + node.name + "': missing 'to'");
                result = run_cast(rt, in(0), dtype_from_name(*to));
                break;
            }
            case OpKind::Where:
                result = run_where(rt, in(0), in(1), in(2), node.name);
                break;
            case OpKind::Expand: {
                const std::vector<int64_t>* target = node.attr_ints("shape");
                if (target == nullptr) throw ShapeMismatch("node '" + node.name + "': missing shape");
                result = run_expand(rt, in(0), *target, node.name);
                break;
            }
            case OpKind::Constant: {
                const std::vector<int64_t>* shape = node.attr_ints("shape");
                const std::vector<double>* values = node.attr_reals("value");
                const double scalar = node.attr_real("scalar", std::numeric_limits<double>::quiet_NaN());
                if (shape != nullptr && values != nullptr) {
                    if (numel_of(*shape) != values->size())
                        throw ShapeMismatch("node '" + node.name + "': constant size mismatch");
                    staging.resize(values->size());
                    for (std::size_t i = 0; i < values->size(); ++i) staging[i] = static_cast<float>((*values)[i]);
                    result = upload(rt, *shape, DType::f32, staging.data());
                    RF_CUDA(cudaStreamSynchronize(rt.stream()), "stream sync");
                } else if (!std::isnan(scalar)) {
                    const float s = static_cast<float>(scalar);
                    result = upload(rt, Shape{1}, DType::f32, &s);
                    RF_CUDA(cudaStreamSynchronize(rt.stream()), "stream sync");
                } else {
                    throw UnsupportedOp("node '" + node.name + "': Constant needs shape+value or scalar");
                }
                break;
            }
            case OpKind::FusedFlashAttention: {
                if (node.inputs.size() < 3) throw ShapeMismatch("node '" + node.name + "': missing input tensor");
                result = run_fused_attention(rt, node, in(0), in(1), in(2), node.inputs.size() > 3 ? &in(3) : nullptr);
                break;
            }
        }
        if (node.outputs.size() != 1) {
            rt.release(result);
            throw UnsupportedOp("node '" + node.name + "': exactly one output supported");
        }
        env[node.outputs[0]] = std::move(result);
        // stream-ordered release of everything this node read for the last time
        for (const std::string& t : node.inputs) {
            auto lu = last_use.find(t);
            if (lu != last_use.end() && lu->second == pos) {
                auto it = env.find(t);
                if (it != env.end()) rt.release(it->second);
            }
        }
        if (last_use.find(node.outputs[0]) == last_use.end()) rt.release(env[node.outputs[0]]);  // never read
    }
    RF_CUDA(cudaEventRecord(ev1, rt.stream()), "cudaEventRecord");

    TensorMap outputs;
    for (const std::string& name : graph.outputs) {
        auto it = env.find(name);
        if (it == env.end() || (it->second.ptr == nullptr && it->second.bytes > 0))
            throw ShapeMismatch("graph output '" + name + "' was not computed");
        Tensor host(it->second.shape);
        host.dtype = it->second.dtype;
        if (it->second.bytes > 0)
            RF_CUDA(cudaMemcpyAsync(host.data.data(), it->second.ptr, it->second.bytes, cudaMemcpyDeviceToHost, rt.stream()),
                    "D2H copy");
        outputs[name] = std::move(host);
    }
    RF_CUDA(cudaStreamSynchronize(rt.stream()), "stream sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    rt.finish(ms);
    return outputs;
}

}  // namespace routefast_b200
