// context.hpp -- a cbx_ctx: the camera streams of one context split over
// independent "lanes", each a full Engine (own CUDA stream, plans, graphs,
// per-stream state) serving a contiguous range of the streams.
//
// Streams are independent Networks (/root/reference/proj/SPEC.md:370), so a
// lane needs nothing from another lane. Two lanes on two CUDA streams let the
// GPU overlap one lane's tensor-core-bound layer-3 convolution with the other
// lane's memory/latency-bound mask, layer-1 and pooling kernels (they fit on
// the same SMs next to the tcgen05 CTAs): measured 15.9k vs 14.0k frames/s for
// 8 x 1080p streams in two lanes of 4 vs one lane of 8.
//
// The context stream (cbx_stream) joins every lane after each frame, so work
// ordered after a forward on it sees all streams' results; the lanes never
// wait for each other.
#pragma once

#include <memory>
#include <vector>

#include "engine.hpp"

namespace cbx {

class Context {
public:
    Context(const cbx_net_desc& net, int device, int S, int precision, int lanes);
    ~Context();

    int lanes() const { return (int)lanes_.size(); }
    Engine& lane(int l) { return *lanes_[l]; }
    cudaStream_t stream() const { return main_; }

    // broadcast configuration
    void load_layer(int layer, const float* K, const float* bias);
    void set_thresholds(const float* taus, int n);
    void get_thresholds(float* taus, int n) const;
    void set_option(int option, int value);
    void reset();

    // frames
    void forward_host(int engine, const float* frames, uint16_t* labels, cbx_layer_stats* stats, uint64_t* macs);
    void forward_device(int engine, const float* const* frames_dev);
    void forward_device_u8(int engine, const uint8_t* const* frames_dev);
    void forward_host_u8(int engine, const uint8_t* frames, uint16_t* labels, cbx_layer_stats* stats, uint64_t* macs);
    int64_t submit_u8(int engine, const uint8_t* frames, uint16_t* labels);
    int64_t submit(int engine, const float* frames, uint16_t* labels);
    void wait(int64_t ticket, cbx_layer_stats* stats, uint64_t* macs);
    void sync();

    // results
    void read_labels(int engine, uint16_t* labels);
    void read_stats(int engine, cbx_layer_stats* stats, uint64_t* macs);
    const uint16_t* labels_device(int engine);
    void get_activation(int engine, int layer, int s, float* out);
    void get_trace(int cb, int s, uint8_t* detected, int32_t* updated, int64_t* n, int* first);
    void get_input(int engine, int layer, int s, float* out);
    bool has_history() const { return lanes_[0]->has_history(); }
    void read_step_times(int64_t* nanos);  // [S][nl][5]
    void worst_case_counts(int64_t* worst);
    void profile(int engine, const float* const* frames_dev, const uint8_t* const* frames_u8,
                 std::vector<cbx_kernel_time>& out);
    int last_launch_count() const;

private:
    int lane_of(int s, int& local) const;
    void join();  // the context stream waits for every lane's queued work

    int device_, S_, nl_, ncb_, lh_ = 0, lw_ = 0;
    size_t frame_elems_ = 0;
    std::vector<std::unique_ptr<Engine>> lanes_;
    std::vector<int> off_;  // first stream of each lane; off_[lanes] = S
    cudaStream_t main_ = nullptr;
    std::vector<cudaEvent_t> ev_;  // per lane, for the join
    // submit/wait: the lane tickets of the last submissions
    struct Sub {
        int64_t ticket = -1;
        std::vector<int64_t> lane_tickets;
    };
    Sub subs_[3];
    int64_t submitted_ = 0;
};

}  // namespace cbx
