// cbinfer_b200.cpp -- the reference's C++ API (include/cbinfer_b200/cbinfer.hpp)
// served by the B200 engine through the C-ABI (include/cbx.h).
//
// Host code only: value types, file formats, the netspec parser, and the
// glue that moves the reference's host tensors to and from the device for
// the op-level functions. Every computation on the path runs in libcbx.so
// (sm_100a kernels); nothing here computes a convolution, a change mask or
// an index list on the CPU.
#include "cbinfer_b200/cbinfer.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>

#include "cbx.h"
#include "json.hpp"

namespace cbinfer {

namespace {

// cbx status -> the reference exception hierarchy (error.hpp:9-42)
void check(int rc, const cbx_ctx* ctx = nullptr) {
    if (rc == CBX_OK) return;
    const std::string m = cbx_last_error(ctx);
    switch (rc) {
        case CBX_E_SHAPE: throw shape_error(m);
        case CBX_E_GEOMETRY: throw geometry_error(m);
        case CBX_E_BOUNDS: throw bounds_error(m);
        case CBX_E_IO: throw io_error(m);
        case CBX_E_SPEC: throw spec_error(m);
        case CBX_E_CUDA: throw cuda_error(m);
        default: throw error(m);
    }
}

void cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw cuda_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer for the op-level functions (synchronous, default stream).
template <class T>
struct Dev {
    T* p = nullptr;
    size_t n = 0;
    explicit Dev(size_t count) : n(count) {
        cuda(cudaMalloc(reinterpret_cast<void**>(&p), std::max<size_t>(count, 1) * sizeof(T) + 16), "cudaMalloc");
        cuda(cudaMemset(p, 0, std::max<size_t>(count, 1) * sizeof(T) + 16), "cudaMemset");
        cuda(cudaStreamSynchronize(nullptr), "cudaStreamSynchronize");  // legacy-stream memset vs non-blocking streams
    }
    Dev(const T* host, size_t count) : Dev(count) {
        if (count) cuda(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy H2D");
    }
    ~Dev() { cudaFree(p); }
    Dev(const Dev&) = delete;
    Dev& operator=(const Dev&) = delete;
    void get(T* host) const {
        if (n) cuda(cudaMemcpy(host, p, n * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    }
};

cbx_geom to_cbx(const ConvGeometry& g) {
    return cbx_geom{g.kernelH, g.kernelW, g.strideH, g.strideW, g.padH, g.padW, g.inChannels, g.outChannels};
}

std::vector<char> slurp(const std::filesystem::path& file) {
    std::ifstream in(file, std::ios::binary | std::ios::ate);
    if (!in) throw io_error("cannot open " + file.string());
    const std::streamsize size = in.tellg();
    in.seekg(0);
    std::vector<char> buf(static_cast<size_t>(size));
    if (size > 0 && !in.read(buf.data(), size)) throw io_error("failed reading " + file.string());
    return buf;
}

void spill(const std::filesystem::path& file, const void* data, size_t bytes) {
    std::ofstream out(file, std::ios::binary | std::ios::trunc);
    if (!out) throw io_error("cannot open " + file.string() + " for writing");
    out.write(static_cast<const char*>(data), static_cast<std::streamsize>(bytes));
    if (!out) throw io_error("failed writing " + file.string());
}

void require_finite(const std::vector<float>& v, const std::filesystem::path& file) {
    if (!std::all_of(v.begin(), v.end(), [](float x) { return std::isfinite(x); }))
        throw io_error("non-finite value in " + file.string());
}

// Elapsed device time between two events, ns.
int64_t event_ns(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.0f;
    cuda(cudaEventElapsedTime(&ms, a, b), "cudaEventElapsedTime");
    return static_cast<int64_t>(static_cast<double>(ms) * 1e6);
}

}  // namespace

// ------------------------------------------------------------ geometry/tensor
void ConvGeometry::check_output(int inHeight, int inWidth) const {
    if (kernelH < 1 || kernelW < 1 || strideH < 1 || strideW < 1 || padH < 0 || padW < 0)
        throw geometry_error("invalid convolution geometry");
    if (inHeight + 2 * padH < kernelH || inWidth + 2 * padW < kernelW)
        throw geometry_error("convolution output would be empty: input " + std::to_string(inHeight) + "x" +
                             std::to_string(inWidth) + ", kernel " + std::to_string(kernelH) + "x" +
                             std::to_string(kernelW));
}

std::size_t linear_index(int c, int j, int i, const TensorDims& d) {
    const bool inside = c >= 0 && c < d.channels && j >= 0 && j < d.height && i >= 0 && i < d.width;
    if (!inside)
        throw bounds_error("coordinate (" + std::to_string(c) + "," + std::to_string(j) + "," + std::to_string(i) +
                           ") outside tensor " + std::to_string(d.channels) + "x" + std::to_string(d.height) + "x" +
                           std::to_string(d.width));
    return (static_cast<std::size_t>(c) * d.height + j) * d.width + i;
}

float max_abs_diff(const FrameTensor& a, const FrameTensor& b) {
    if (!a.same_dims(b)) throw shape_error("max_abs_diff: tensor dimensions differ");
    float m = 0.0f;
    for (size_t k = 0; k < a.data.size(); ++k) m = std::max(m, std::fabs(a.data[k] - b.data[k]));
    return m;
}

bool all_finite(const FrameTensor& t) {
    return std::all_of(t.data.begin(), t.data.end(), [](float x) { return std::isfinite(x); });
}

std::int64_t ChangeMap::count() const {
    return static_cast<std::int64_t>(std::count_if(bits.begin(), bits.end(), [](std::uint8_t b) { return b != 0; }));
}

ChangeIndexList ChangeIndexList::full(int pixels) {
    ChangeIndexList l;
    l.indices.resize(static_cast<size_t>(std::max(pixels, 0)));
    for (int p = 0; p < pixels; ++p) l.indices[static_cast<size_t>(p)] = p;
    return l;
}

// ------------------------------------------------------------------ TensorSlot
std::unique_ptr<FrameTensor> TensorSlot::materialized() const {
    if (!has_value()) return nullptr;
    return std::make_unique<FrameTensor>(value());
}

TensorSlot& TensorSlot::operator=(const TensorSlot& o) {
    if (this != &o) {
        if (src_) throw spec_error("the change-based state of a Network lives on the device (use reset_state)");
        host_ = o.materialized();
    }
    return *this;
}

TensorSlot& TensorSlot::operator=(const FrameTensor& t) {
    if (src_) throw spec_error("the change-based state of a Network lives on the device (use reset_state)");
    host_ = std::make_unique<FrameTensor>(t);
    return *this;
}

TensorSlot& TensorSlot::operator=(FrameTensor&& t) {
    if (src_) throw spec_error("the change-based state of a Network lives on the device (use reset_state)");
    host_ = std::make_unique<FrameTensor>(std::move(t));
    return *this;
}

bool TensorSlot::has_value() const { return src_ ? src_->present() : host_ != nullptr; }

const FrameTensor& TensorSlot::value() const {
    if (!src_) {
        if (!host_) throw spec_error("empty change-based state (no previous frame)");
        return *host_;
    }
    if (!src_->present()) throw spec_error("empty change-based state (no previous frame)");
    const std::uint64_t v = src_->version();
    if (!cache_ || cache_version_ != v) {  // HBM -> host once per frame
        if (!cache_) cache_ = std::make_unique<FrameTensor>();
        src_->fetch(*cache_);
        cache_version_ = v;
    }
    return *cache_;
}

void TensorSlot::reset() {
    if (src_) throw spec_error("the change-based state of a Network lives on the device (use reset_state)");
    host_.reset();
}

// -------------------------------------------------------------- dense ops
namespace {
// X for the listed output pixels (all of them when idx is empty and all_px)
PatchMatrix gather_columns(const FrameTensor& input, const ConvGeometry& g, const std::vector<std::int32_t>* idx,
                           int ncols) {
    PatchMatrix X(g.inChannels * g.kernelH * g.kernelW, ncols);
    if (X.data.empty()) return X;
    Dev<float> din(input.data.data(), input.data.size()), dx(X.data.size());
    std::unique_ptr<Dev<std::int32_t>> di;
    if (idx) di = std::make_unique<Dev<std::int32_t>>(idx->data(), idx->size());
    const cbx_geom cg = to_cbx(g);
    check(cbx_op_gen_x(din.p, input.channels, input.height, input.width, &cg, di ? di->p : nullptr, ncols, dx.p,
                       nullptr));
    cuda(cudaDeviceSynchronize(), "gen_x");
    dx.get(X.data.data());
    return X;
}
}  // namespace

PatchMatrix im2col_full(const FrameTensor& input, const ConvGeometry& g) {
    if (input.channels != g.inChannels)
        throw shape_error("im2col_full: input has " + std::to_string(input.channels) + " channels, geometry expects " +
                          std::to_string(g.inChannels));
    g.check_output(input.height, input.width);
    return gather_columns(input, g, nullptr, g.outHeight(input.height) * g.outWidth(input.width));
}

PatchMatrix gen_x_reduced(const FrameTensor& input, const ChangeIndexList& idx, const ConvGeometry& g) {
    if (input.channels != g.inChannels) throw shape_error("gen_x_reduced: channel count mismatch");
    g.check_output(input.height, input.width);
    const int64_t outPix = static_cast<int64_t>(g.outHeight(input.height)) * g.outWidth(input.width);
    for (std::int32_t p : idx.indices)
        if (p < 0 || p >= outPix) throw bounds_error("gen_x_reduced: output index " + std::to_string(p) + " out of range");
    return gather_columns(input, g, &idx.indices, static_cast<int>(idx.count()));
}

void fill_patch_column(const FrameTensor& input, const ConvGeometry& g, int y_o, int x_o, float* col) {
    ChangeIndexList one;
    one.indices.push_back(y_o * g.outWidth(input.width) + x_o);
    const PatchMatrix X = gather_columns(input, g, &one.indices, 1);
    std::memcpy(col, X.data.data(), X.data.size() * sizeof(float));
}

ResultMatrix gemm(const FilterMatrix& K, const PatchMatrix& X) {
    if (K.cols != X.rows)
        throw shape_error("gemm: K has " + std::to_string(K.cols) + " columns, X has " + std::to_string(X.rows) +
                          " rows");
    ResultMatrix Y(K.rows, X.cols);
    if (Y.data.empty()) return Y;
    Dev<float> dk(K.data.data(), K.data.size()), db(K.bias.data(), K.bias.size()), dx(X.data.data(), X.data.size()),
        dy(Y.data.size());
    check(cbx_op_gemm(dk.p, db.p, K.rows, K.cols, dx.p, X.cols, dy.p, nullptr));
    cuda(cudaDeviceSynchronize(), "gemm");
    dy.get(Y.data.data());
    return Y;
}

FrameTensor update_output(const FrameTensor& prevOut, const ResultMatrix& Y, const ChangeIndexList& idx,
                          bool fuseRelu) {
    if (Y.cols != idx.count())
        throw shape_error("update_output: Y has " + std::to_string(Y.cols) + " columns for " +
                          std::to_string(idx.count()) + " indices");
    if (Y.rows != prevOut.channels) throw shape_error("update_output: Y row count does not match output channels");
    const int64_t plane = static_cast<int64_t>(prevOut.height) * prevOut.width;
    for (std::int32_t p : idx.indices)
        if (p < 0 || p >= plane) throw bounds_error("update_output: index out of range");
    FrameTensor out = prevOut;
    if (idx.empty() || out.data.empty()) return out;
    Dev<float> dout(out.data.data(), out.data.size()), dy(Y.data.data(), Y.data.size());
    Dev<std::int32_t> di(idx.indices.data(), idx.indices.size());
    check(cbx_op_scatter(dout.p, out.channels, out.height, out.width, dy.p, di.p, idx.count(), fuseRelu ? 1 : 0,
                         nullptr));
    cuda(cudaDeviceSynchronize(), "update_output");
    dout.get(out.data.data());
    return out;
}

FrameTensor conv_full(const FrameTensor& input, const FilterMatrix& K, const ConvGeometry& g) {
    if (input.channels != g.inChannels) throw shape_error("conv_full: channel count mismatch");
    g.check_output(input.height, input.width);
    if (K.rows != g.outChannels || K.cols != g.inChannels * g.kernelH * g.kernelW || K.bias.size() != size_t(K.rows))
        throw shape_error("conv_full: filter matrix does not match the geometry");
    const int Ho = g.outHeight(input.height), Wo = g.outWidth(input.width);
    FrameTensor out(g.outChannels, Ho, Wo);
    Dev<float> din(input.data.data(), input.data.size()), dk(K.data.data(), K.data.size()),
        db(K.bias.data(), K.bias.size()), dout(out.data.size());
    const cbx_geom cg = to_cbx(g);
    // all output pixels (idx = null), exact fp32 order (bias first, ascending (c,kj,ki))
    check(cbx_op_cbconv_update(din.p, input.channels, input.height, input.width, dk.p, db.p, &cg, nullptr, Ho * Wo, 0,
                               dout.p, nullptr));
    cuda(cudaDeviceSynchronize(), "conv_full");
    dout.get(out.data.data());
    return out;
}

FrameTensor relu(const FrameTensor& t) {
    FrameTensor out(t.channels, t.height, t.width);
    if (t.data.empty()) return out;
    Dev<float> din(t.data.data(), t.data.size()), dout(out.data.size());
    check(cbx_op_relu(din.p, t.channels, t.height, t.width, dout.p, nullptr));
    cuda(cudaDeviceSynchronize(), "relu");
    dout.get(out.data.data());
    return out;
}

FrameTensor maxpool(const FrameTensor& t, int window, int stride) {
    if (window < 1 || stride < 1 || window > t.height || window > t.width)
        throw geometry_error("invalid pooling window");
    FrameTensor out(t.channels, (t.height - window) / stride + 1, (t.width - window) / stride + 1);
    Dev<float> din(t.data.data(), t.data.size()), dout(out.data.size());
    check(cbx_op_maxpool(din.p, t.channels, t.height, t.width, window, stride, dout.p, nullptr));
    cuda(cudaDeviceSynchronize(), "maxpool");
    dout.get(out.data.data());
    return out;
}

LabelMap argmax_classify(const FrameTensor& t) {
    LabelMap m(t.height, t.width);
    if (t.data.empty()) return m;
    Dev<float> din(t.data.data(), t.data.size());
    Dev<std::uint16_t> dl(m.labels.size());
    check(cbx_op_argmax(din.p, t.channels, t.height, t.width, dl.p, nullptr));
    cuda(cudaDeviceSynchronize(), "argmax_classify");
    dl.get(m.labels.data());
    return m;
}

// -------------------------------------------------------- change-based ops
namespace {

// mask (device bytes) of detect_changes; optional changed count
void detect_dev(const float* cur, const float* prev, int C, int H, int W, float tau, std::uint8_t* mask) {
    Dev<unsigned long long> cnt(1);
    check(cbx_op_detect(cur, prev, C, H, W, tau, mask, cnt.p, nullptr));
}

void dilate_dev(const std::uint8_t* m, int H, int W, const ConvGeometry& g, std::uint8_t* out) {
    const cbx_geom cg = to_cbx(g);
    check(cbx_op_dilate(m, H, W, &cg, out, nullptr));
}

// ascending index list of a device byte mask
std::vector<std::int32_t> extract_dev(const std::uint8_t* m, int64_t n, std::int32_t* idx_dev) {
    Dev<int> cnt(1);
    Dev<unsigned char> ws(cbx_op_extract_workspace(n));
    check(cbx_op_extract(m, n, idx_dev, cnt.p, ws.p, nullptr));
    cuda(cudaDeviceSynchronize(), "extract_indexes");
    int count = 0;
    cnt.get(&count);
    std::vector<std::int32_t> out(static_cast<size_t>(count));
    if (count) cuda(cudaMemcpy(out.data(), idx_dev, sizeof(std::int32_t) * count, cudaMemcpyDeviceToHost), "D2H");
    return out;
}

}  // namespace

ChangeMap detect_changes(const FrameTensor& cur, const FrameTensor& prev, float tau) {
    if (!cur.same_dims(prev)) throw shape_error("detect_changes: frame dimensions differ");
    ChangeMap m(cur.height, cur.width);
    if (m.bits.empty() || cur.channels < 1) return m;
    Dev<float> a(cur.data.data(), cur.data.size()), b(prev.data.data(), prev.data.size());
    Dev<std::uint8_t> dm(m.bits.size());
    detect_dev(a.p, b.p, cur.channels, cur.height, cur.width, tau, dm.p);
    cuda(cudaDeviceSynchronize(), "detect_changes");
    dm.get(m.bits.data());
    return m;
}

ChangeMap dilate_changes(const ChangeMap& m, const ConvGeometry& g) {
    g.check_output(m.height, m.width);
    ChangeMap out(g.outHeight(m.height), g.outWidth(m.width));
    Dev<std::uint8_t> dm(m.bits.data(), m.bits.size()), dout(out.bits.size());
    dilate_dev(dm.p, m.height, m.width, g, dout.p);
    cuda(cudaDeviceSynchronize(), "dilate_changes");
    dout.get(out.bits.data());
    return out;
}

ChangeMap worst_case_propagation(const ChangeIndexList& updated, const ConvGeometry& g, int height, int width) {
    g.check_output(height, width);
    const std::int64_t pixels = static_cast<std::int64_t>(height) * width;
    ChangeMap wave(height, width);
    for (std::int32_t p : updated.indices) {
        if (p < 0 || p >= pixels)
            throw bounds_error("worst_case_propagation: index " + std::to_string(p) + " outside " +
                               std::to_string(height) + "x" + std::to_string(width) + " grid");
        wave.bits[static_cast<size_t>(p)] = 1;
    }
    return dilate_changes(wave, g);
}

ChangeIndexList extract_indexes(const ChangeMap& m) {
    ChangeIndexList l;
    if (m.bits.empty()) return l;
    Dev<std::uint8_t> dm(m.bits.data(), m.bits.size());
    Dev<std::int32_t> idx(m.bits.size());
    l.indices = extract_dev(dm.p, static_cast<int64_t>(m.bits.size()), idx.p);
    return l;
}

std::pair<FrameTensor, LayerStats> cbconv_forward(CBConvState& state, const FrameTensor& input, CBConvTrace* trace) {
    const ConvGeometry& g = state.geom;
    if (input.channels != g.inChannels) throw shape_error("cbconv_forward: channel count mismatch");
    g.check_output(input.height, input.width);
    const FilterMatrix& K = state.filters;
    if (K.rows != g.outChannels || K.cols != g.inChannels * g.kernelH * g.kernelW || K.bias.size() != size_t(K.rows))
        throw shape_error("cbconv_forward: filter matrix does not match the geometry");
    const int Ho = g.outHeight(input.height), Wo = g.outWidth(input.width);
    const int64_t outPix = static_cast<int64_t>(Ho) * Wo;
    const bool history = state.has_history();
    if (history && !input.same_dims(*state.prevInput))
        throw shape_error("cbconv_forward: frame dimensions changed between frames");

    LayerStats st;
    FrameTensor out(g.outChannels, Ho, Wo);
    Dev<float> din(input.data.data(), input.data.size()), dk(K.data.data(), K.data.size()),
        db(K.bias.data(), K.bias.size()), dout(out.data.size());
    Dev<std::int32_t> idx(static_cast<size_t>(outPix));
    cudaEvent_t ev[5];
    for (auto& e : ev) cuda(cudaEventCreate(&e), "cudaEventCreate");
    struct EvGuard {
        cudaEvent_t* e;
        ~EvGuard() {
            for (int i = 0; i < 5; ++i) cudaEventDestroy(e[i]);
        }
    } guard{ev};
    const cbx_geom cg = to_cbx(g);
    ChangeMap m;
    ChangeIndexList list;
    if (!history) {  // first frame: every output pixel (cbconv.cpp:170-192)
        cuda(cudaEventRecord(ev[2]), "cudaEventRecord");
        check(cbx_op_cbconv_update(din.p, g.inChannels, input.height, input.width, dk.p, db.p, &cg, nullptr,
                                   static_cast<int>(outPix), state.fuseRelu, dout.p, nullptr));
        cuda(cudaEventRecord(ev[3]), "cudaEventRecord");
        cuda(cudaDeviceSynchronize(), "cbconv_forward");
        if (state.collectTimings) st.stepNanos.multiply = event_ns(ev[2], ev[3]);
        list = ChangeIndexList::full(static_cast<int>(outPix));
        st.changedInputPixels = static_cast<int64_t>(input.height) * input.width;
    } else {  // detect -> dilate -> extract -> gathered conv in place over prevOutput
        const FrameTensor& prevIn = *state.prevInput;
        const FrameTensor& prevOut = *state.prevOutput;
        Dev<float> dprev(prevIn.data.data(), prevIn.data.size());
        Dev<std::uint8_t> dm(static_cast<size_t>(input.height) * input.width), dd(static_cast<size_t>(outPix));
        cuda(cudaEventRecord(ev[0]), "cudaEventRecord");
        detect_dev(din.p, dprev.p, input.channels, input.height, input.width, state.threshold, dm.p);
        dilate_dev(dm.p, input.height, input.width, g, dd.p);
        cuda(cudaEventRecord(ev[1]), "cudaEventRecord");
        list.indices = extract_dev(dd.p, outPix, idx.p);
        cuda(cudaEventRecord(ev[2]), "cudaEventRecord");
        cuda(cudaMemcpy(dout.p, prevOut.data.data(), prevOut.data.size() * sizeof(float), cudaMemcpyHostToDevice),
             "cudaMemcpy H2D");
        cuda(cudaEventRecord(ev[3]), "cudaEventRecord");
        if (!list.indices.empty())
            check(cbx_op_cbconv_update(din.p, g.inChannels, input.height, input.width, dk.p, db.p, &cg, idx.p,
                                       static_cast<int>(list.indices.size()), state.fuseRelu, dout.p, nullptr));
        cuda(cudaEventRecord(ev[4]), "cudaEventRecord");
        cuda(cudaDeviceSynchronize(), "cbconv_forward");
        m = ChangeMap(input.height, input.width);
        dm.get(m.bits.data());
        if (state.collectTimings) {
            st.stepNanos.detect = event_ns(ev[0], ev[1]);   // detect + dilate (cbconv.hpp:42-43)
            st.stepNanos.extract = event_ns(ev[1], ev[2]);
            st.stepNanos.update = event_ns(ev[2], ev[3]);   // the prevOutput copy; the scatter is fused
            st.stepNanos.multiply = event_ns(ev[3], ev[4]); // gather + contraction + scatter, one kernel
        }
        st.changedInputPixels = m.count();
    }
    dout.get(out.data.data());
    st.changedOutputPixels = list.count();
    st.gemmMacs = static_cast<std::uint64_t>(K.rows) * K.cols * static_cast<std::uint64_t>(list.count());
    if (trace) {
        trace->detected = std::move(m);
        trace->updated = std::move(list);
    }
    state.prevInput = input;
    state.prevOutput = out;
    return {std::move(out), st};
}

// ------------------------------------------------------------------ netspec
const char* to_string(LayerKind k) {
    static const char* names[] = {"CBCONV", "CONV", "RELU", "MAXPOOL", "CLASSIFY"};
    const int i = static_cast<int>(k);
    return i >= 0 && i < 5 ? names[i] : "?";
}

LayerKind layer_kind_from_string(const std::string& s) {
    for (int i = 0; i < 5; ++i)
        if (s == to_string(static_cast<LayerKind>(i))) return static_cast<LayerKind>(i);
    throw spec_error("unknown layer kind \"" + s + "\"");
}

MemoryMode memory_mode_from_string(const std::string& s) {
    if (s == "BASELINE_NAIVE") return MemoryMode::BaselineNaive;
    if (s == "BASELINE_SHARED") return MemoryMode::BaselineShared;
    if (s == "CBINFER") return MemoryMode::CBInfer;
    throw spec_error("unknown memory mode \"" + s + "\"");
}

// Same keys, defaults and error classes as the reference parser
// (network.cpp:43-85): nlohmann/json, the reference's own JSON dependency.
NetworkSpec network_spec_from_json(const std::string& text) {
    using nlohmann::json;
    json doc;
    try {
        doc = json::parse(text);
    } catch (const json::exception& e) {
        throw spec_error(std::string("network spec: invalid JSON: ") + e.what());
    }
    try {
        NetworkSpec spec;
        spec.inputChannels = doc.at("inputChannels").get<int>();
        spec.inputHeight = doc.at("inputHeight").get<int>();
        spec.inputWidth = doc.at("inputWidth").get<int>();
        spec.numClasses = doc.at("numClasses").get<int>();
        for (const auto& jl : doc.at("layers")) {
            LayerSpec l;
            l.kind = layer_kind_from_string(jl.at("kind").get<std::string>());
            if (l.is_conv()) {
                ConvGeometry& g = l.geom;
                g.kernelH = jl.at("kernelH").get<int>();
                g.kernelW = jl.at("kernelW").get<int>();
                g.strideH = jl.value("strideH", 1);
                g.strideW = jl.value("strideW", 1);
                g.padH = jl.value("padH", 0);
                g.padW = jl.value("padW", 0);
                g.outChannels = jl.at("outChannels").get<int>();
                l.weightsFile = jl.at("weightsFile").get<std::string>();
            }
            if (l.kind == LayerKind::CBCONV) {
                l.threshold = jl.value("threshold", 0.0f);
                l.fuseRelu = jl.value("fuseRelu", false);
                if (l.threshold < 0.0f) throw spec_error("network spec: negative threshold");
            }
            if (l.kind == LayerKind::MAXPOOL) {
                l.window = jl.at("window").get<int>();
                l.stride = jl.at("stride").get<int>();
            }
            spec.layers.push_back(std::move(l));
        }
        return spec;
    } catch (const json::exception& e) {
        throw spec_error(std::string("network spec: ") + e.what());
    }
}

NetworkSpec load_network_spec(const std::filesystem::path& file) {
    std::ifstream in(file);
    if (!in) throw io_error("cannot open network spec " + file.string());
    std::stringstream ss;
    ss << in.rdbuf();
    return network_spec_from_json(ss.str());
}

std::string network_spec_to_json(const NetworkSpec& spec) {
    using nlohmann::json;
    json layers = json::array();
    for (const auto& l : spec.layers) {
        json jl{{"kind", to_string(l.kind)}};
        if (l.is_conv()) {
            const ConvGeometry& g = l.geom;
            jl.update({{"kernelH", g.kernelH}, {"kernelW", g.kernelW}, {"strideH", g.strideH}, {"strideW", g.strideW},
                       {"padH", g.padH}, {"padW", g.padW}, {"outChannels", g.outChannels},
                       {"weightsFile", l.weightsFile}});
        }
        if (l.kind == LayerKind::CBCONV) jl.update({{"threshold", l.threshold}, {"fuseRelu", l.fuseRelu}});
        if (l.kind == LayerKind::MAXPOOL) jl.update({{"window", l.window}, {"stride", l.stride}});
        layers.push_back(std::move(jl));
    }
    json doc{{"inputChannels", spec.inputChannels},
             {"inputHeight", spec.inputHeight},
             {"inputWidth", spec.inputWidth},
             {"numClasses", spec.numClasses},
             {"layers", std::move(layers)}};
    return doc.dump(2) + "\n";
}

namespace {
std::vector<cbx_layer_desc> descs(const NetworkSpec& spec) {
    std::vector<cbx_layer_desc> d(spec.layers.size());
    for (size_t k = 0; k < spec.layers.size(); ++k) {
        const LayerSpec& l = spec.layers[k];
        d[k].kind = static_cast<int>(l.kind);
        d[k].geom = to_cbx(l.geom);
        d[k].window = l.window;
        d[k].stride = l.stride;
        d[k].threshold = l.threshold;
        d[k].fuseRelu = l.fuseRelu ? 1 : 0;
    }
    return d;
}
cbx_net_desc net_desc(const NetworkSpec& spec, const std::vector<cbx_layer_desc>& d) {
    return cbx_net_desc{spec.inputChannels, spec.inputHeight, spec.inputWidth, spec.numClasses,
                        static_cast<int>(d.size()), d.data()};
}
}  // namespace

std::vector<LayerShape> chain_dims(NetworkSpec& spec) {
    const auto d = descs(spec);
    const auto nd = net_desc(spec, d);
    std::vector<cbx_layer_desc> out(std::max<size_t>(d.size(), 1));
    std::vector<int> dims(6 * std::max<size_t>(d.size(), 1));
    check(cbx_chain_dims(&nd, out.data(), dims.data()));
    std::vector<LayerShape> shapes(d.size());
    for (size_t k = 0; k < d.size(); ++k) {
        spec.layers[k].geom.inChannels = out[k].geom.inChannels;
        shapes[k].in = {dims[6 * k], dims[6 * k + 1], dims[6 * k + 2]};
        shapes[k].out = {dims[6 * k + 3], dims[6 * k + 4], dims[6 * k + 5]};
    }
    return shapes;
}

// Static value accounting of the paper's memory comparison (network.cpp:322-388):
// naive = a buffer per layer output (RELU in place) and an X matrix per conv;
// shared = a ping-pong pair sized for the largest output and one X for the
// largest conv; CBInfer adds per-CBCONV previous input + output and one
// change map, index list (largest grid each) and Y (largest output).
MemoryReport memory_footprint(const NetworkSpec& spec, MemoryMode mode) {
    NetworkSpec s = spec;
    const auto shapes = chain_dims(s);
    MemoryReport r;
    std::uint64_t sumOut = 0, sumX = 0, maxOut = 0, maxX = 0, prev = 0, maxGrid = 0, maxY = 0;
    for (size_t k = 0; k < s.layers.size(); ++k) {
        const LayerSpec& l = s.layers[k];
        const TensorDims& in = shapes[k].in;
        const TensorDims& out = shapes[k].out;
        if (l.kind != LayerKind::RELU) {
            sumOut += out.count();
            maxOut = std::max<std::uint64_t>(maxOut, out.count());
        }
        if (l.is_conv()) {
            const std::uint64_t rowsK = static_cast<std::uint64_t>(l.geom.inChannels) * l.geom.kernelH * l.geom.kernelW;
            const std::uint64_t x = rowsK * out.height * out.width;
            sumX += x;
            maxX = std::max(maxX, x);
            r.parameterValues += rowsK * l.geom.outChannels + l.geom.outChannels;
        }
        if (l.kind == LayerKind::CBCONV) {
            prev += in.count() + out.count();
            maxGrid = std::max({maxGrid, static_cast<std::uint64_t>(in.height) * in.width,
                                static_cast<std::uint64_t>(out.height) * out.width});
            maxY = std::max<std::uint64_t>(maxY, out.count());
        }
    }
    if (mode == MemoryMode::BaselineNaive) {
        r.intermediateValues = sumOut;
        r.patchMatrixValues = sumX;
    } else {
        r.intermediateValues = 2 * maxOut;
        r.patchMatrixValues = maxX;
    }
    if (mode == MemoryMode::CBInfer) r.cbExtraValues = prev + 2 * maxGrid + maxY;
    r.totalValues = r.intermediateValues + r.patchMatrixValues + r.parameterValues + r.cbExtraValues;
    return r;
}

// ------------------------------------------------------------------ network
namespace detail {

struct Device {
    cbx_ctx* ctx = nullptr;
    std::vector<int> cb;          // CBCONV layer indices
    std::vector<LayerShape> shapes;
    int lh = 0, lw = 0, final_layer = -1;
    std::uint64_t version = 0;    // advances with every frame and reset
    bool step_times = false;
    std::vector<float> taus;      // thresholds installed on the device

    struct Source : TensorSource {
        const Device* dev;
        int layer;
        bool input;
        Source(const Device* d, int l, bool in) : dev(d), layer(l), input(in) {}
        bool present() const override { return cbx_has_history(dev->ctx) == 1; }
        std::uint64_t version() const override { return dev->version; }
        void fetch(FrameTensor& out) const override {
            const TensorDims& d = input ? dev->shapes[layer].in : dev->shapes[layer].out;
            out = FrameTensor(d.channels, d.height, d.width);
            if (input)
                check(cbx_get_input(dev->ctx, CBX_ENGINE_CBINFER, layer, 0, out.data.data()), dev->ctx);
            else
                check(cbx_get_activation(dev->ctx, CBX_ENGINE_CBINFER, layer, 0, out.data.data()), dev->ctx);
        }
    };
    std::vector<std::unique_ptr<Source>> sources;

    ~Device() {
        if (ctx) cbx_destroy(ctx);
    }
};

}  // namespace detail

Network::Network() = default;
Network::~Network() = default;
Network::Network(Network&&) noexcept = default;
Network& Network::operator=(Network&&) noexcept = default;

std::vector<float> Network::thresholds() const {
    std::vector<float> t;
    for (int k : cbLayers) t.push_back(layers[static_cast<size_t>(k)].state.threshold);
    return t;
}

void Network::set_thresholds(const std::vector<float>& taus) {
    if (taus.size() != cbLayers.size())
        throw spec_error("expected " + std::to_string(cbLayers.size()) + " thresholds, got " +
                         std::to_string(taus.size()));
    for (float t : taus)
        if (t < 0.0f) throw spec_error("negative threshold");
    for (size_t k = 0; k < taus.size(); ++k) layers[static_cast<size_t>(cbLayers[k])].state.threshold = taus[k];
}

DeviceOptions DeviceOptions::from_environment() {
    DeviceOptions o;
    if (const char* p = std::getenv("CBINFER_B200_PRECISION")) {
        const std::string s = p;
        if (s == "exact") o.precision = Precision::Exact;
        else if (s == "tf32") o.precision = Precision::TF32;
        else if (s == "f16") o.precision = Precision::F16;
        else throw spec_error("CBINFER_B200_PRECISION must be exact, tf32 or f16");
    }
    if (const char* d = std::getenv("CBINFER_B200_DEVICE")) o.device = std::atoi(d);
    return o;
}

Network load_network(const NetworkSpec& spec, const std::filesystem::path& weightsDir) {
    return load_network(spec, weightsDir, DeviceOptions::from_environment());
}

Network load_network(const NetworkSpec& spec, const std::filesystem::path& weightsDir, const DeviceOptions& opt) {
    Network net;
    net.spec = spec;
    const auto shapes = chain_dims(net.spec);
    // weights first (io errors name the layer, network.cpp:218-225), then the device
    for (size_t k = 0; k < net.spec.layers.size(); ++k) {
        const LayerSpec& l = net.spec.layers[k];
        Layer layer;
        layer.spec = l;
        layer.inDims = shapes[k].in;
        layer.outDims = shapes[k].out;
        if (l.is_conv()) {
            try {
                layer.state.filters = read_weights_f32le(weightsDir / l.weightsFile, l.geom);
            } catch (const io_error& e) {
                throw io_error("layer " + std::to_string(k + 1) + " (" + to_string(l.kind) + "): " + e.what());
            }
            layer.state.geom = l.geom;
            layer.state.threshold = l.threshold;
            layer.state.fuseRelu = l.fuseRelu;
        }
        if (l.kind == LayerKind::CBCONV) net.cbLayers.push_back(static_cast<int>(k));
        net.layers.push_back(std::move(layer));
    }
    auto dev = std::make_unique<detail::Device>();
    dev->shapes = shapes;
    dev->cb = net.cbLayers;
    const auto d = descs(net.spec);
    const auto nd = net_desc(net.spec, d);
    check(cbx_create(&nd, opt.device, 1, static_cast<int>(opt.precision), &dev->ctx));
    for (size_t k = 0; k < net.layers.size(); ++k)
        if (net.layers[k].spec.is_conv()) {
            const FilterMatrix& f = net.layers[k].state.filters;
            check(cbx_load_layer(dev->ctx, static_cast<int>(k), f.data.data(), f.bias.data()), dev->ctx);
        }
    dev->taus = net.thresholds();
    const bool cls = net.spec.layers.back().kind == LayerKind::CLASSIFY;
    dev->lh = cls ? shapes.back().in.height : shapes.back().out.height;
    dev->lw = cls ? shapes.back().in.width : shapes.back().out.width;
    dev->final_layer = static_cast<int>(net.spec.layers.size()) - (cls ? 2 : 1);
    for (int k : net.cbLayers) {
        dev->sources.push_back(std::make_unique<detail::Device::Source>(dev.get(), k, true));
        net.layers[static_cast<size_t>(k)].state.prevInput.bind(dev->sources.back().get());
        dev->sources.push_back(std::make_unique<detail::Device::Source>(dev.get(), k, false));
        net.layers[static_cast<size_t>(k)].state.prevOutput.bind(dev->sources.back().get());
    }
    net.dev_ = std::move(dev);
    return net;
}

ForwardResult forward_frame(Network& net, const FrameTensor& frame, Engine engine, ForwardTrace* trace) {
    if (frame.channels != net.spec.inputChannels || frame.height != net.spec.inputHeight ||
        frame.width != net.spec.inputWidth)
        throw shape_error("forward_frame: frame does not match network input dimensions");
    detail::Device& dev = *net.dev_;
    // per-layer state the caller may have edited since the last frame
    const auto taus = net.thresholds();
    if (taus != dev.taus) {
        check(cbx_set_thresholds(dev.ctx, taus.data(), static_cast<int>(taus.size())), dev.ctx);
        dev.taus = taus;
    }
    bool timings = false;
    for (int k : net.cbLayers) timings |= net.layers[static_cast<size_t>(k)].state.collectTimings;
    if (timings != dev.step_times) {
        check(cbx_set_option(dev.ctx, CBX_OPT_STEP_TIMES, timings ? 1 : 0), dev.ctx);
        dev.step_times = timings;
    }
    const size_t nl = net.layers.size();
    ForwardResult r;
    r.labels = LabelMap(dev.lh, dev.lw);
    std::vector<cbx_layer_stats> st(nl);
    std::uint64_t macs = 0;
    const int eng = engine == Engine::CBInfer ? CBX_ENGINE_CBINFER : CBX_ENGINE_BASELINE;
    ++dev.version;  // the device state changes (even when the call fails half-way)
    check(cbx_forward(dev.ctx, eng, frame.data.data(), r.labels.labels.data(), st.data(), &macs), dev.ctx);
    r.stats.resize(nl);
    for (size_t k = 0; k < nl; ++k) {
        r.stats[k].changedInputPixels = st[k].changedInputPixels;
        r.stats[k].changedOutputPixels = st[k].changedOutputPixels;
        r.stats[k].gemmMacs = st[k].gemmMacs;
    }
    r.macsTotal = macs;
    if (timings && engine == Engine::CBInfer) {
        std::vector<int64_t> ns(nl * 5);
        check(cbx_read_step_times(dev.ctx, ns.data()), dev.ctx);
        for (int k : net.cbLayers) {
            if (!net.layers[static_cast<size_t>(k)].state.collectTimings) continue;
            StepTimes& t = r.stats[static_cast<size_t>(k)].stepNanos;
            const int64_t* v = ns.data() + 5 * static_cast<size_t>(k);
            t = StepTimes{v[0], v[1], v[2], v[3], v[4]};
        }
    }
    if (trace) {
        trace->cb.clear();
        for (size_t c = 0; c < net.cbLayers.size(); ++c) {
            trace->cb.emplace_back();
            if (engine != Engine::CBInfer) continue;  // the dense engine leaves CB traces empty
            const LayerShape& sh = dev.shapes[static_cast<size_t>(net.cbLayers[c])];
            CBConvTrace& t = trace->cb.back();
            ChangeMap m(sh.in.height, sh.in.width);
            std::vector<std::int32_t> idx(static_cast<size_t>(sh.out.height) * sh.out.width);
            int64_t n = 0;
            int first = 0;
            check(cbx_get_trace(dev.ctx, static_cast<int>(c), 0, m.bits.data(), idx.data(), &n, &first), dev.ctx);
            if (!first) t.detected = std::move(m);
            idx.resize(static_cast<size_t>(n));
            t.updated.indices = std::move(idx);
        }
        if (dev.final_layer < 0) {
            trace->finalActivation = frame;
        } else {
            const TensorDims& d = dev.shapes[static_cast<size_t>(dev.final_layer)].out;
            trace->finalActivation = FrameTensor(d.channels, d.height, d.width);
            check(cbx_get_activation(dev.ctx, eng, dev.final_layer, 0, trace->finalActivation.data.data()), dev.ctx);
        }
    }
    return r;
}

void reset_state(Network& net) {
    check(cbx_reset(net.dev_->ctx), net.dev_->ctx);
    ++net.dev_->version;
}

// ----------------------------------------------------------------------- io
FrameTensor read_frame_f32le(const std::filesystem::path& file, int channels, int height, int width) {
    const auto buf = slurp(file);
    const size_t want = static_cast<size_t>(channels) * height * width * 4;
    if (buf.size() != want)
        throw io_error(file.string() + ": expected " + std::to_string(want) + " bytes, got " +
                       std::to_string(buf.size()));
    FrameTensor t(channels, height, width);
    std::memcpy(t.data.data(), buf.data(), buf.size());
    require_finite(t.data, file);
    return t;
}

void write_frame_f32le(const std::filesystem::path& file, const FrameTensor& t) {
    spill(file, t.data.data(), t.data.size() * 4);
}

// Binary PPM (P6, maxval 255), '#' comments allowed in the header; planar
// RGB scaled by 1/255 exactly like the reference (px / 255.0f).
FrameTensor read_ppm(const std::filesystem::path& file) {
    const auto buf = slurp(file);
    size_t pos = 0;
    auto token = [&]() {
        for (;;) {
            while (pos < buf.size() && std::isspace(static_cast<unsigned char>(buf[pos]))) ++pos;
            if (pos < buf.size() && buf[pos] == '#') {
                while (pos < buf.size() && buf[pos] != '\n') ++pos;
                continue;
            }
            break;
        }
        const size_t start = pos;
        while (pos < buf.size() && !std::isspace(static_cast<unsigned char>(buf[pos]))) ++pos;
        return std::string(buf.data() + start, pos - start);
    };
    if (token() != "P6") throw io_error(file.string() + ": not a binary PPM (P6) file");
    int dims[3];
    for (int& v : dims) {
        const std::string t = token();
        char* end = nullptr;
        const long x = std::strtol(t.c_str(), &end, 10);
        if (t.empty() || *end) throw io_error(file.string() + ": malformed PPM header");
        v = static_cast<int>(x);
    }
    const int w = dims[0], h = dims[1];
    if (w <= 0 || h <= 0) throw io_error(file.string() + ": invalid PPM dimensions");
    if (dims[2] != 255) throw io_error(file.string() + ": only 8-bit PPM supported");
    ++pos;  // the single whitespace byte before the raster
    const size_t plane = static_cast<size_t>(w) * h;
    if (pos > buf.size() || buf.size() - pos < 3 * plane) throw io_error(file.string() + ": truncated PPM pixel data");
    FrameTensor t(3, h, w);
    const auto* px = reinterpret_cast<const unsigned char*>(buf.data() + pos);
    for (int c = 0; c < 3; ++c) {
        float* dst = t.plane(c);
        for (size_t p = 0; p < plane; ++p) dst[p] = px[3 * p + c] / 255.0f;
    }
    return t;
}

LabelMap read_labels_u16le(const std::filesystem::path& file, int height, int width) {
    const auto buf = slurp(file);
    const size_t want = static_cast<size_t>(height) * width * 2;
    if (buf.size() != want)
        throw io_error(file.string() + ": expected " + std::to_string(want) + " bytes, got " +
                       std::to_string(buf.size()));
    LabelMap m(height, width);
    std::memcpy(m.labels.data(), buf.data(), buf.size());
    return m;
}

void write_labels_u16le(const std::filesystem::path& file, const LabelMap& m) {
    spill(file, m.labels.data(), m.labels.size() * 2);
}

FilterMatrix read_weights_f32le(const std::filesystem::path& file, const ConvGeometry& g) {
    const size_t kv = static_cast<size_t>(g.outChannels) * g.inChannels * g.kernelH * g.kernelW;
    const size_t want = (kv + static_cast<size_t>(g.outChannels)) * 4;
    const auto buf = slurp(file);
    if (buf.size() != want)
        throw io_error(file.string() + ": expected " + std::to_string(want) + " bytes (kernel " +
                       std::to_string(g.outChannels) + "x" + std::to_string(g.inChannels) + "x" +
                       std::to_string(g.kernelH) + "x" + std::to_string(g.kernelW) + " + bias), got " +
                       std::to_string(buf.size()));
    FilterMatrix f(g.outChannels, g.inChannels * g.kernelH * g.kernelW);
    std::memcpy(f.data.data(), buf.data(), kv * 4);
    std::memcpy(f.bias.data(), buf.data() + kv * 4, static_cast<size_t>(g.outChannels) * 4);
    require_finite(f.data, file);
    require_finite(f.bias, file);
    return f;
}

void write_weights_f32le(const std::filesystem::path& file, const FilterMatrix& f) {
    std::vector<float> all(f.data);
    all.insert(all.end(), f.bias.begin(), f.bias.end());
    spill(file, all.data(), all.size() * 4);
}

}  // namespace cbinfer
