// context.cu -- lanes of a cbx_ctx (see context.hpp).
#include <algorithm>
#include <cstring>
#include <map>

#include "context.hpp"

namespace cbx {

Context::Context(const cbx_net_desc& net, int device, int S, int precision, int lanes) : device_(device), S_(S) {
    if (S < 1) throw Error(CBX_E_ARG, "num_streams must be >= 1");
    if (lanes < 1) lanes = 1;
    lanes = std::min(lanes, S);
    CBX_CUDA(cudaSetDevice(device));
    off_.resize(lanes + 1);
    for (int l = 0; l <= lanes; ++l) off_[l] = (int)((int64_t)S * l / lanes);
    try {
        for (int l = 0; l < lanes; ++l)
            lanes_.emplace_back(new Engine(net, device, off_[l + 1] - off_[l], precision));
        CBX_CUDA(cudaStreamCreateWithFlags(&main_, cudaStreamNonBlocking));
        ev_.assign(lanes, nullptr);
        for (auto& e : ev_) CBX_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    } catch (...) {
        for (auto e : ev_)
            if (e) cudaEventDestroy(e);
        if (main_) cudaStreamDestroy(main_);
        throw;
    }
    nl_ = lanes_[0]->num_layers();
    ncb_ = 0;
    for (int k = 0; k < net.numLayers; ++k) ncb_ += net.layers[k].kind == CBX_CBCONV;
    lh_ = lanes_[0]->label_h();
    lw_ = lanes_[0]->label_w();
    frame_elems_ = (size_t)net.inputChannels * net.inputHeight * net.inputWidth;
}

Context::~Context() {
    cudaSetDevice(device_);
    for (auto& l : lanes_) l->sync();
    if (main_) cudaStreamSynchronize(main_);
    lanes_.clear();
    for (auto e : ev_)
        if (e) cudaEventDestroy(e);
    if (main_) cudaStreamDestroy(main_);
}

int Context::lane_of(int s, int& local) const {
    if (s < 0 || s >= S_) throw Error(CBX_E_BOUNDS, "stream index out of range");
    int l = (int)(std::upper_bound(off_.begin(), off_.end(), s) - off_.begin()) - 1;
    local = s - off_[l];
    return l;
}

void Context::join() {
    for (size_t l = 0; l < lanes_.size(); ++l) {
        CBX_CUDA(cudaEventRecord(ev_[l], lanes_[l]->stream()));
        CBX_CUDA(cudaStreamWaitEvent(main_, ev_[l], 0));
    }
}

void Context::load_layer(int layer, const float* K, const float* bias) {
    for (auto& l : lanes_) l->load_layer(layer, K, bias);
}
void Context::set_thresholds(const float* taus, int n) {
    for (auto& l : lanes_) l->set_thresholds(taus, n);
}
void Context::get_thresholds(float* taus, int n) const { lanes_[0]->get_thresholds(taus, n); }
void Context::set_option(int option, int value) {
    for (auto& l : lanes_) l->set_option(option, value);
}
void Context::reset() {
    for (auto& l : lanes_) l->reset();
}

void Context::forward_host(int engine, const float* frames, uint16_t* labels, cbx_layer_stats* stats,
                           uint64_t* macs) {
    if (!frames) throw Error(CBX_E_ARG, "frames is null");
    // enqueue every lane before reading anything back, so the lanes overlap
    for (size_t l = 0; l < lanes_.size(); ++l) lanes_[l]->enqueue_host(engine, frames + frame_elems_ * off_[l]);
    join();
    if (labels) read_labels(engine, labels);
    read_stats(engine, stats, macs);
}

void Context::forward_host_u8(int engine, const uint8_t* frames, uint16_t* labels, cbx_layer_stats* stats,
                              uint64_t* macs) {
    if (!frames) throw Error(CBX_E_ARG, "frames is null");
    for (size_t l = 0; l < lanes_.size(); ++l) lanes_[l]->enqueue_host_u8(engine, frames + frame_elems_ * off_[l]);
    join();
    if (labels) read_labels(engine, labels);
    read_stats(engine, stats, macs);
}

int64_t Context::submit_u8(int engine, const uint8_t* frames, uint16_t* labels) {
    if (!frames || !labels) throw Error(CBX_E_ARG, "null frames or labels");
    Sub& sub = subs_[submitted_ % 3];
    sub.lane_tickets.assign(lanes_.size(), -1);
    for (size_t l = 0; l < lanes_.size(); ++l)
        sub.lane_tickets[l] =
            lanes_[l]->submit_u8(engine, frames + frame_elems_ * off_[l], labels + (size_t)lh_ * lw_ * off_[l]);
    sub.ticket = submitted_;
    return submitted_++;
}

void Context::forward_device(int engine, const float* const* frames_dev) {
    if (!frames_dev) throw Error(CBX_E_ARG, "frames is null");
    for (size_t l = 0; l < lanes_.size(); ++l) lanes_[l]->forward_device(engine, frames_dev + off_[l]);
    join();
}

void Context::forward_device_u8(int engine, const uint8_t* const* frames_dev) {
    if (!frames_dev) throw Error(CBX_E_ARG, "frames is null");
    for (size_t l = 0; l < lanes_.size(); ++l) lanes_[l]->forward_device_u8(engine, frames_dev + off_[l]);
    join();
}

int64_t Context::submit(int engine, const float* frames, uint16_t* labels) {
    if (!frames || !labels) throw Error(CBX_E_ARG, "null frames or labels");
    Sub& sub = subs_[submitted_ % 3];
    sub.lane_tickets.assign(lanes_.size(), -1);
    for (size_t l = 0; l < lanes_.size(); ++l)
        sub.lane_tickets[l] =
            lanes_[l]->submit(engine, frames + frame_elems_ * off_[l], labels + (size_t)lh_ * lw_ * off_[l]);
    sub.ticket = submitted_;
    return submitted_++;
}

void Context::wait(int64_t ticket, cbx_layer_stats* stats, uint64_t* macs) {
    const Sub& sub = subs_[((ticket % 3) + 3) % 3];
    if (ticket < 0 || sub.ticket != ticket)
        throw Error(CBX_E_ARG, "cbx_wait: unknown or expired ticket (at most the last 3 submissions can be waited on)");
    for (size_t l = 0; l < lanes_.size(); ++l)
        lanes_[l]->wait(sub.lane_tickets[l], stats ? stats + (size_t)nl_ * off_[l] : nullptr,
                        macs ? macs + off_[l] : nullptr);
}

void Context::sync() {
    for (auto& l : lanes_) l->sync();
    CBX_CUDA(cudaStreamSynchronize(main_));
}

void Context::read_labels(int engine, uint16_t* labels) {
    if (!labels) throw Error(CBX_E_ARG, "null labels");
    for (size_t l = 0; l < lanes_.size(); ++l) lanes_[l]->read_labels(engine, labels + (size_t)lh_ * lw_ * off_[l]);
}

void Context::read_stats(int engine, cbx_layer_stats* stats, uint64_t* macs) {
    for (size_t l = 0; l < lanes_.size(); ++l)
        lanes_[l]->read_stats(engine, stats ? stats + (size_t)nl_ * off_[l] : nullptr, macs ? macs + off_[l] : nullptr);
}

const uint16_t* Context::labels_device(int engine) {
    if (lanes_.size() != 1)
        throw Error(CBX_E_ARG, "cbx_labels_device: labels of a multi-lane context live in one buffer per lane "
                               "(use cbx_read_labels, or create the context with one lane)");
    return lanes_[0]->labels_device(engine);
}

void Context::get_activation(int engine, int layer, int s, float* out) {
    int local;
    const int l = lane_of(s, local);
    lanes_[l]->get_activation(engine, layer, local, out);
}

void Context::get_trace(int cb, int s, uint8_t* detected, int32_t* updated, int64_t* n, int* first) {
    int local;
    const int l = lane_of(s, local);
    lanes_[l]->get_trace(cb, local, detected, updated, n, first);
}

void Context::get_input(int engine, int layer, int s, float* out) {
    int local;
    const int l = lane_of(s, local);
    lanes_[l]->get_input(engine, layer, local, out);
}

void Context::read_step_times(int64_t* nanos) {
    if (!nanos) throw Error(CBX_E_ARG, "null output");
    std::vector<int64_t> lane((size_t)nl_ * 5);
    for (size_t l = 0; l < lanes_.size(); ++l) {
        lanes_[l]->read_step_times(lane.data());
        for (int s = off_[l]; s < off_[l + 1]; ++s)
            std::memcpy(nanos + (size_t)s * nl_ * 5, lane.data(), sizeof(int64_t) * lane.size());
    }
}

void Context::worst_case_counts(int64_t* worst) {
    if (!worst) throw Error(CBX_E_ARG, "null output");
    const int per = std::max(0, ncb_ - 1);
    for (size_t l = 0; l < lanes_.size(); ++l) lanes_[l]->worst_case_counts(worst + (size_t)per * off_[l]);
}

// Lanes one after the other (no overlap), the times of the same kernel in
// different lanes summed: per-kernel device time over all streams.
void Context::profile(int engine, const float* const* frames_dev, const uint8_t* const* frames_u8,
                      std::vector<cbx_kernel_time>& out) {
    out.clear();
    std::map<std::pair<std::string, int>, size_t> pos;
    for (size_t l = 0; l < lanes_.size(); ++l) {
        std::vector<cbx_kernel_time> v;
        lanes_[l]->profile(engine, frames_dev ? frames_dev + off_[l] : nullptr, frames_u8 ? frames_u8 + off_[l] : nullptr, v);
        for (const auto& t : v) {
            const auto key = std::make_pair(std::string(t.name), t.layer);
            auto it = pos.find(key);
            if (it == pos.end()) {
                pos[key] = out.size();
                out.push_back(t);
            } else {
                out[it->second].ms += t.ms;
            }
        }
    }
}

int Context::last_launch_count() const {
    int n = 0;
    for (const auto& l : lanes_) n += l->last_launch_count();
    return n;
}

}  // namespace cbx
