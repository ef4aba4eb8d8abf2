// cbinfer_b200/cbinfer.hpp -- the reference's C++ API (namespace cbinfer) for
// per-frame change-based network evaluation, served by the B200 engine.
//
// Drop-in: a program written against the reference headers
// (/root/reference/proj/core/include/cbinfer/*.hpp) compiles unchanged with
// `-I<repo>/include` placed before the reference's include directory and links
// `libcbinfer_b200.so` (+ libcbx.so) instead of the reference's hot-path
// objects. include/cbinfer/{error,geometry,tensor,baseline,cbconv,network,io}.hpp
// forward here; the reference's own synth.hpp / calibration.hpp (outer loops,
// fixtures -- not this path) keep working on top because they only call the
// public API below.
//
//   reference declaration                          here
//   error.hpp:9-42        exception classes        same classes (+ cuda_error)
//   geometry.hpp:12-49    ConvGeometry             same struct
//   tensor.hpp:13-90      TensorDims, FrameTensor, LabelMap, linear_index,
//                         max_abs_diff, all_finite  same (host value types)
//   baseline.hpp:13-91    FilterMatrix/PatchMatrix/ResultMatrix, conv_full,
//                         relu, maxpool, argmax_classify, full_frame_macs
//                                                   same; computed on the GPU
//   cbconv.hpp:17-120     ChangeMap, ChangeIndexList, StepTimes, LayerStats,
//                         CBConvState, CBConvTrace, detect_changes,
//                         dilate_changes, worst_case_propagation,
//                         extract_indexes, cbconv_forward
//                                                   same; computed on the GPU
//   network.hpp:12-118    LayerKind ... memory_footprint, load_network,
//                         forward_frame, reset_state
//                                                   same; a Network owns a
//                                                   cbx context (cbx.h) on a B200
//   io.hpp:15-31          frame / PPM / label / weight files
//                                                   same formats
//
// The matrix-form ops im2col_full, gen_x_reduced, fill_patch_column, gemm and
// update_output (baseline.hpp:58-80, cbconv.hpp:108-113) are provided for
// source compatibility (GPU kernels, exact order); the network path never
// materializes the patch matrix X or the result matrix Y -- there the gather,
// the contraction and the scatter are one kernel (K4).
//
// Precision: the network-level API runs the B200 engine in the precision of
// DeviceOptions (default: CBINFER_B200_PRECISION = exact | tf32 | f16 from the
// environment for unmodified programs, else tf32); the op-level functions
// (detect/dilate/extract/conv_full/cbconv_forward/...) always use the exact
// fp32 reference order, so they are bit-identical to the reference.
#pragma once

#include <cstddef>
#include <cstdint>
#include <filesystem>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace cbinfer {

// ------------------------------------------------------------------ errors
class error : public std::runtime_error {
public:
    explicit error(const std::string& what) : std::runtime_error(what) {}
};
class shape_error : public error {
public:
    explicit shape_error(const std::string& what) : error(what) {}
};
class geometry_error : public error {
public:
    explicit geometry_error(const std::string& what) : error(what) {}
};
class bounds_error : public error {
public:
    explicit bounds_error(const std::string& what) : error(what) {}
};
class io_error : public error {
public:
    explicit io_error(const std::string& what) : error(what) {}
};
class spec_error : public error {
public:
    explicit spec_error(const std::string& what) : error(what) {}
};
// B200 extension: the device failed (there is no CPU fallback).
class cuda_error : public error {
public:
    explicit cuda_error(const std::string& what) : error(what) {}
};

// ---------------------------------------------------------------- geometry
struct ConvGeometry {
    int kernelH = 1, kernelW = 1;
    int strideH = 1, strideW = 1;
    int padH = 0, padW = 0;
    int inChannels = 1, outChannels = 1;

    int outHeight(int inHeight) const { return (inHeight + 2 * padH - kernelH) / strideH + 1; }
    int outWidth(int inWidth) const { return (inWidth + 2 * padW - kernelW) / strideW + 1; }
    // throws geometry_error for invalid parameters or an empty output grid
    void check_output(int inHeight, int inWidth) const;
    static ConvGeometry pooling(int window, int stride, int channels) {
        ConvGeometry g;
        g.kernelH = g.kernelW = window;
        g.strideH = g.strideW = stride;
        g.inChannels = g.outChannels = channels;
        return g;
    }
};

// ----------------------------------------------------------------- tensors
struct TensorDims {
    int channels = 0, height = 0, width = 0;
    bool operator==(const TensorDims&) const = default;
    std::size_t count() const { return static_cast<std::size_t>(channels) * height * width; }
};

// offset of (c, j, i) in planar storage; bounds_error outside
std::size_t linear_index(int c, int j, int i, const TensorDims& dims);

// Planar CHW fp32 tensor: (c, j, i) at data[(c*height + j)*width + i].
struct FrameTensor {
    int channels = 0, height = 0, width = 0;
    std::vector<float> data;

    FrameTensor() = default;
    FrameTensor(int c, int h, int w) : channels(c), height(h), width(w), data(static_cast<std::size_t>(c) * h * w, 0.0f) {}

    TensorDims dims() const { return {channels, height, width}; }
    std::size_t size() const { return data.size(); }
    bool same_dims(const FrameTensor& o) const {
        return channels == o.channels && height == o.height && width == o.width;
    }
    float& operator()(int c, int j, int i) { return data[(static_cast<std::size_t>(c) * height + j) * width + i]; }
    float operator()(int c, int j, int i) const { return data[(static_cast<std::size_t>(c) * height + j) * width + i]; }
    float& at(int c, int j, int i) { return data[linear_index(c, j, i, dims())]; }
    float at(int c, int j, int i) const { return data[linear_index(c, j, i, dims())]; }
    const float* plane(int c) const { return data.data() + static_cast<std::size_t>(c) * height * width; }
    float* plane(int c) { return data.data() + static_cast<std::size_t>(c) * height * width; }
};

// Row-major uint16 class map.
struct LabelMap {
    int height = 0, width = 0;
    std::vector<std::uint16_t> labels;

    LabelMap() = default;
    LabelMap(int h, int w) : height(h), width(w), labels(static_cast<std::size_t>(h) * w, 0) {}
    std::size_t size() const { return labels.size(); }
    bool same_dims(const LabelMap& o) const { return height == o.height && width == o.width; }
    std::uint16_t& operator()(int j, int i) { return labels[static_cast<std::size_t>(j) * width + i]; }
    std::uint16_t operator()(int j, int i) const { return labels[static_cast<std::size_t>(j) * width + i]; }
};

float max_abs_diff(const FrameTensor& a, const FrameTensor& b);  // shape_error on mismatch
bool all_finite(const FrameTensor& t);

// ---------------------------------------------------------------- matrices
// Filters in the reference layout: K(o, (c*kernelH + j)*kernelW + i), row-major, + bias.
struct FilterMatrix {
    int rows = 0, cols = 0;
    std::vector<float> data, bias;

    FilterMatrix() = default;
    FilterMatrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0f), bias(r, 0.0f) {}
    const float* row(int o) const { return data.data() + static_cast<std::size_t>(o) * cols; }
    float* row(int o) { return data.data() + static_cast<std::size_t>(o) * cols; }
};

// Patch / result matrices: layout types of the reference's matrix-form ops
// (kept for source compatibility; the B200 path never materializes them).
struct PatchMatrix {
    int rows = 0, cols = 0;
    std::vector<float> data;  // column-major
    PatchMatrix() = default;
    PatchMatrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0f) {}
    const float* col(int n) const { return data.data() + static_cast<std::size_t>(n) * rows; }
    float* col(int n) { return data.data() + static_cast<std::size_t>(n) * rows; }
};
struct ResultMatrix {
    int rows = 0, cols = 0;
    std::vector<float> data;  // row-major
    ResultMatrix() = default;
    ResultMatrix(int r, int c) : rows(r), cols(c), data(static_cast<std::size_t>(r) * c, 0.0f) {}
};

// Dense ops (baseline.cpp), on the GPU in the exact fp32 reference order.
PatchMatrix im2col_full(const FrameTensor& input, const ConvGeometry& geom);
ResultMatrix gemm(const FilterMatrix& K, const PatchMatrix& X);
void fill_patch_column(const FrameTensor& input, const ConvGeometry& geom, int y_o, int x_o, float* col);
FrameTensor conv_full(const FrameTensor& input, const FilterMatrix& K, const ConvGeometry& geom);
FrameTensor relu(const FrameTensor& t);
FrameTensor maxpool(const FrameTensor& t, int window, int stride);
LabelMap argmax_classify(const FrameTensor& t);

inline std::uint64_t full_frame_macs(const ConvGeometry& g, int outH, int outW) {
    return static_cast<std::uint64_t>(g.outChannels) * g.inChannels * g.kernelH * g.kernelW * outH * outW;
}

// --------------------------------------------------------- change-based ops
struct ChangeMap {
    int height = 0, width = 0;
    std::vector<std::uint8_t> bits;

    ChangeMap() = default;
    ChangeMap(int h, int w) : height(h), width(w), bits(static_cast<std::size_t>(h) * w, 0) {}
    std::size_t size() const { return bits.size(); }
    bool test(int j, int i) const { return bits[static_cast<std::size_t>(j) * width + i] != 0; }
    void set(int j, int i) { bits[static_cast<std::size_t>(j) * width + i] = 1; }
    std::int64_t count() const;
};

struct ChangeIndexList {
    std::vector<std::int32_t> indices;  // ascending y*w + x
    std::int64_t count() const { return static_cast<std::int64_t>(indices.size()); }
    bool empty() const { return indices.empty(); }
    static ChangeIndexList full(int pixels);
};

// Step times in ns (device time, CUDA events; see cbx_read_step_times for
// how the fused B200 kernels map onto the five steps).
struct StepTimes {
    std::int64_t detect = 0, extract = 0, generate = 0, multiply = 0, update = 0;
    std::int64_t total() const { return detect + extract + generate + multiply + update; }
};

struct LayerStats {
    std::int64_t changedInputPixels = 0;
    std::int64_t changedOutputPixels = 0;
    std::uint64_t gemmMacs = 0;
    StepTimes stepNanos;
};

namespace detail {
// Where a device-resident tensor of a Network comes from (set by the Network).
struct TensorSource {
    virtual ~TensorSource() = default;
    virtual bool present() const = 0;
    virtual std::uint64_t version() const = 0;  // changes with every frame / reset
    virtual void fetch(FrameTensor& out) const = 0;
};
}  // namespace detail

// The std::optional<FrameTensor> of CBConvState (cbconv.hpp:71-72). In a
// state owned by the caller (cbconv_forward) it holds a host tensor; in a
// Network's layers it is a view of the tensor that lives in HBM, copied to
// the host on first access after each frame.
class TensorSlot {
public:
    TensorSlot() = default;
    TensorSlot(const TensorSlot& o) : host_(o.materialized()) {}
    TensorSlot& operator=(const TensorSlot& o);
    TensorSlot(TensorSlot&&) noexcept = default;
    TensorSlot& operator=(TensorSlot&&) noexcept = default;
    TensorSlot& operator=(const FrameTensor& t);
    TensorSlot& operator=(FrameTensor&& t);

    bool has_value() const;
    explicit operator bool() const { return has_value(); }
    const FrameTensor& value() const;
    const FrameTensor& operator*() const { return value(); }
    const FrameTensor* operator->() const { return &value(); }
    void reset();

    void bind(const detail::TensorSource* src) { src_ = src; }  // (Network internals)

private:
    std::unique_ptr<FrameTensor> materialized() const;
    std::unique_ptr<FrameTensor> host_;
    const detail::TensorSource* src_ = nullptr;
    mutable std::unique_ptr<FrameTensor> cache_;
    mutable std::uint64_t cache_version_ = ~0ull;
};

struct CBConvState {
    ConvGeometry geom;
    FilterMatrix filters;
    float threshold = 0.0f;
    bool fuseRelu = false;
    bool collectTimings = true;
    TensorSlot prevInput;
    TensorSlot prevOutput;

    bool has_history() const { return prevInput.has_value(); }
    void reset() {
        prevInput.reset();
        prevOutput.reset();
    }
};

struct CBConvTrace {
    ChangeMap detected;       // input grid; empty (0x0) on a full evaluation
    ChangeIndexList updated;  // output pixels recomputed
};

ChangeMap detect_changes(const FrameTensor& cur, const FrameTensor& prev, float tau);
ChangeMap dilate_changes(const ChangeMap& m, const ConvGeometry& geom);
ChangeMap worst_case_propagation(const ChangeIndexList& updated, const ConvGeometry& geomNext, int height,
                                 int width);
ChangeIndexList extract_indexes(const ChangeMap& m);
PatchMatrix gen_x_reduced(const FrameTensor& input, const ChangeIndexList& idx, const ConvGeometry& geom);
FrameTensor update_output(const FrameTensor& prevOut, const ResultMatrix& Y, const ChangeIndexList& idx,
                          bool fuseRelu);
// One layer, caller-owned state: first frame full, then detect -> dilate ->
// extract -> gathered conv in place, on the GPU (exact fp32 order).
std::pair<FrameTensor, LayerStats> cbconv_forward(CBConvState& state, const FrameTensor& input,
                                                  CBConvTrace* trace = nullptr);

// ----------------------------------------------------------------- network
enum class LayerKind { CBCONV, CONV, RELU, MAXPOOL, CLASSIFY };
const char* to_string(LayerKind k);
LayerKind layer_kind_from_string(const std::string& s);

struct LayerSpec {
    LayerKind kind = LayerKind::CONV;
    ConvGeometry geom;
    int window = 0, stride = 0;
    float threshold = 0.0f;
    bool fuseRelu = false;
    std::string weightsFile;
    bool is_conv() const { return kind == LayerKind::CBCONV || kind == LayerKind::CONV; }
};

struct NetworkSpec {
    int inputChannels = 0, inputHeight = 0, inputWidth = 0, numClasses = 0;
    std::vector<LayerSpec> layers;
};

NetworkSpec network_spec_from_json(const std::string& text);
NetworkSpec load_network_spec(const std::filesystem::path& file);
std::string network_spec_to_json(const NetworkSpec& spec);

struct LayerShape {
    TensorDims in, out;
};
std::vector<LayerShape> chain_dims(NetworkSpec& spec);

struct Layer {
    LayerSpec spec;
    TensorDims inDims, outDims;
    CBConvState state;  // CBCONV: threshold / collectTimings are read at every
                        // forward_frame; prevInput / prevOutput view HBM
};

enum class Engine { Baseline, CBInfer };

// B200 extension: how load_network places the network.
enum class Precision { Exact, TF32, F16 };  // cbx.h CBX_PREC_*
struct DeviceOptions {
    int device = 0;
    Precision precision = Precision::TF32;
    // default options of load_network(spec, dir): CBINFER_B200_PRECISION /
    // CBINFER_B200_DEVICE from the environment (for unmodified programs)
    static DeviceOptions from_environment();
};

namespace detail {
struct Device;  // the cbx context behind a Network
}

struct Network {
    NetworkSpec spec;
    std::vector<Layer> layers;
    std::vector<int> cbLayers;

    std::vector<float> thresholds() const;
    void set_thresholds(const std::vector<float>& taus);

    Network();
    ~Network();
    Network(Network&&) noexcept;
    Network& operator=(Network&&) noexcept;
    Network(const Network&) = delete;  // the state lives on the device
    Network& operator=(const Network&) = delete;

    detail::Device* device() const { return dev_.get(); }  // (B200 internals)
    std::unique_ptr<detail::Device> dev_;
};

struct ForwardResult {
    LabelMap labels;
    std::vector<LayerStats> stats;
    std::uint64_t macsTotal = 0;
};

struct ForwardTrace {
    std::vector<CBConvTrace> cb;
    FrameTensor finalActivation;
};

Network load_network(const NetworkSpec& spec, const std::filesystem::path& weightsDir);
Network load_network(const NetworkSpec& spec, const std::filesystem::path& weightsDir, const DeviceOptions& opt);
ForwardResult forward_frame(Network& net, const FrameTensor& frame, Engine engine = Engine::CBInfer,
                            ForwardTrace* trace = nullptr);
void reset_state(Network& net);

enum class MemoryMode { BaselineNaive, BaselineShared, CBInfer };
MemoryMode memory_mode_from_string(const std::string& s);
struct MemoryReport {
    std::uint64_t intermediateValues = 0, patchMatrixValues = 0, parameterValues = 0, cbExtraValues = 0,
                  totalValues = 0;
};
MemoryReport memory_footprint(const NetworkSpec& spec, MemoryMode mode);

// ---------------------------------------------------------------------- io
FrameTensor read_frame_f32le(const std::filesystem::path& file, int channels, int height, int width);
void write_frame_f32le(const std::filesystem::path& file, const FrameTensor& t);
FrameTensor read_ppm(const std::filesystem::path& file);
LabelMap read_labels_u16le(const std::filesystem::path& file, int height, int width);
void write_labels_u16le(const std::filesystem::path& file, const LabelMap& m);
FilterMatrix read_weights_f32le(const std::filesystem::path& file, const ConvGeometry& geom);
void write_weights_f32le(const std::filesystem::path& file, const FilterMatrix& filters);

}  // namespace cbinfer
