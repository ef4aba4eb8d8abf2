// engine.hpp -- per-network device runtime behind the C-ABI (include/cbx.h).
//
// One Engine = one reference `Network` (network.hpp:54-68) replicated over S
// independent camera streams on one device. It owns the persistent per-layer
// state (channels-last activations with zero halos, change masks, index
// lists), captures the whole frame as a CUDA graph, and reproduces
// forward_frame (network.cpp:252-315) with every CBCONV evaluated by the
// change-based pipeline and every other layer updated incrementally over the
// pixels its input actually changed (exact: unchanged inputs give bitwise
// unchanged outputs, so the full-frame recomputation of the reference is
// reproduced without re-running it).
#pragma once

#include <cuda_runtime.h>

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/cbx.h"
#include "common.cuh"
#include "conv_mpr.hpp"
#include "conv_tc.hpp"

namespace cbx {

// Error carrying a cbx_status (mapped 1:1 to the reference exceptions).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void cuda_check(cudaError_t e, const char* what);
#define CBX_CUDA(x) ::cbx::cuda_check((x), #x)


// chain_dims (network.cpp:128-188)
std::vector<int> chain_dims(const cbx_net_desc& net, std::vector<cbx_layer_desc>& layers);

class Engine {
public:
    Engine(const cbx_net_desc& net, int device, int S, int precision);
    ~Engine();

    void load_layer(int layer, const float* K, const float* bias);
    void set_thresholds(const float* taus, int n);
    void get_thresholds(float* taus, int n) const;
    void reset();

    // frames: host S*C*H*W floats (pinned or pageable)
    void forward_host(int engine, const float* frames, uint16_t* labels, cbx_layer_stats* stats,
                      uint64_t* macs);
    void enqueue_host(int engine, const float* frames);  // forward_host without the read-back
    // 8-bit interleaved host frames (PPM raster), decoded on the device
    void forward_host_u8(int engine, const uint8_t* frames, uint16_t* labels, cbx_layer_stats* stats, uint64_t* macs);
    void enqueue_host_u8(int engine, const uint8_t* frames);
    int64_t submit_u8(int engine, const uint8_t* frames, uint16_t* labels);
    int num_streams() const { return S_; }
    void forward_device(int engine, const float* const* frames_dev);
    // 8-bit interleaved frames already on the device (frames_dev[s] = H x W x C bytes)
    void forward_device_u8(int engine, const uint8_t* const* frames_dev);
    // the 8-bit camera path runs natively (RGB8 detection + kind::i8 layer 1)
    bool u8_native() const;
    // pipelined host-frame path (cbx_submit / cbx_wait)
    int64_t submit(int engine, const float* frames, uint16_t* labels);
    void wait(int64_t ticket, cbx_layer_stats* stats, uint64_t* macs);
    void sync();
    void read_labels(int engine, uint16_t* labels);
    void read_stats(int engine, cbx_layer_stats* stats, uint64_t* macs);
    const uint16_t* labels_device(int engine);
    void get_activation(int engine, int layer, int s, float* out);
    void get_trace(int cb, int s, uint8_t* detected, int32_t* updated, int64_t* n, int* first);
    void worst_case_counts(int64_t* worst);

    void profile(int engine, const float* const* frames_dev, const uint8_t* const* frames_u8,
                 std::vector<cbx_kernel_time>& out);
    void read_step_times(int64_t* out);  // [nl][5] of the last graph launch (CBX_OPT_STEP_TIMES)
    bool has_history() const { return has_history_; }
    void get_input(int engine, int layer, int s, float* out);
    void set_option(int option, int value);

    cudaStream_t stream() const { return stream_; }
    int last_launch_count() const { return last_launches_; }
    int num_layers() const { return (int)layers_.size(); }
    int label_h() const { return lh_; }
    int label_w() const { return lw_; }

private:
    struct Plan;
    Plan& plan(int engine);
    void build_plan(Plan& p, bool baseline);
    void record(Plan& p, bool full);
    void launch(Plan& p, bool full);
    void stage_frame_pointers(int engine, const float* const* cur, const float* const* prev);
    // picks the frame path (8-bit native or fp32), decodes when needed, stages
    // the pointer tables; returns whether the frame is a full evaluation
    bool prepare_frame(int engine, const float* const* f32, const uint8_t* const* u8);
    void frame_done(int engine);  // history bookkeeping after a frame was enqueued
    void finish_stats(Plan& p, bool full, int engine);
    void stats_from(const unsigned long long* hs, bool full, int engine, cbx_layer_stats* out, uint64_t* macs) const;
    bool enqueue(int engine, const float* const* frames_dev, const uint8_t* const* frames_u8,
                 unsigned long long* stats_dst);
    void mark(const char* name, int layer);
    int tail_end(int k) const;
    int final_tensor() const;
    bool fuse_tail_ = true;

public:
    struct ProfMark {
        std::string name;
        int layer;
        cudaEvent_t ev;
    };

private:
    std::vector<ProfMark>* prof_ = nullptr;
    std::vector<ProfMark>* tmarks_ = nullptr;        // capture in progress with step times
    size_t tmarks_used_ = 0;
    const std::vector<ProfMark>* last_tm_ = nullptr;  // marks of the last launched graph
    bool step_times_ = false;

    int device_, S_, precision_;
    cbx_net_desc net_{};
    std::vector<cbx_layer_desc> layers_;
    std::vector<int> dims_;  // 6 per layer
    std::vector<int> cb_layers_;
    int lh_ = 0, lw_ = 0;
    cudaStream_t stream_ = nullptr;

    // weights (reference layout), per layer
    std::vector<float*> dK_, dBias_;
    std::vector<std::vector<float>> hK_, hB_;  // host copies (kernel-parameter filters)
    std::vector<std::unique_ptr<TcLayer, TcLayerDeleter>> tc_;
    std::vector<int> f16_layers_;  // tcgen05 layers with fp16 operands (their input has an fp16 shadow)
    // multi-pixel-row tcgen05 convs (conv_mpr.cu): narrow layers with a
    // 4-channel input, fp16 operands converted while gathering
    std::vector<std::unique_ptr<MprLayer, MprLayerDeleter>> mpr_;
    bool any_f16_ = false;  // some layer has fp16 operands: the plan keeps an overflow flag
    int list_group(int k, bool u8) const;  // group width of layer k's update list (1 = pixel indices)
    int group_width_for(const cbx_geom& g) const;
    bool pack_f16(int k) const;
    void check_f16_overflow(const unsigned long long* hs, int engine);
    bool last_ovf_[2] = {false, false};
    // device counters of one frame: [nl][S][2] + the fp16 overflow flag
    size_t stats_words() const { return (size_t)2 * S_ * layers_.size() + 1; }

public:
    // 0 = exact fp32 (CUDA cores), 1 = tcgen05 tf32, 2 = tcgen05 f16, -1 = not a conv
    int layer_operands(int layer) const;

private:
    std::unique_ptr<Plan> cb_, base_;
    bool has_history_ = false;

    // frame pointer tables (device) and host copies
    const float** d_cur_ = nullptr;
    const float** d_prev_ = nullptr;
    std::vector<const float*> last_cb_frames_;

    // 8-bit camera path (TC precisions, RGB frames with W % 16 == 0, conv
    // first layer): detection on the bytes fused with the RGBX expansion of
    // the frame, layer 1 as a kind::i8 tcgen05 conv over the RGBX bytes.
    std::unique_ptr<TcLayer, TcLayerDeleter> tc8_;
    std::unique_ptr<MprLayer, MprLayerDeleter> mpr8_;  // the same as a multi-pixel-row conv (preferred)
    bool u8_opt_ = true;          // CBX_OPT_U8_NATIVE
    bool rec_u8_ = false;         // the frame being recorded/launched is 8-bit native
    const uint8_t** d_cur8_ = nullptr;
    const uint8_t** d_prev8_ = nullptr;
    std::vector<const uint8_t*> last_cb_frames8_;
    bool hist_u8_ = false;        // the change-based history holds 8-bit frames
    float* prev_dec_ = nullptr;   // decoded 8-bit history for an fp32 frame that follows it
    uint8_t* slots8_[3] = {nullptr, nullptr, nullptr};  // 8-bit host staging (CB ping-pong + baseline)
    std::vector<const float*> cur_f32_;   // pointers of the frame being enqueued (fp32 path)
    std::vector<const uint8_t*> cur_u8_;  // (8-bit native path)
    // host-input staging slots: CB ping-pong + baseline
    float* slots_[3] = {nullptr, nullptr, nullptr};
    int parity_ = 0, parity8_ = 0;

    // submit/wait ring: staging slots, copy stream, per-slot events and counters
    static constexpr int kRing = 3;
    float* ring_[kRing] = {nullptr, nullptr, nullptr};
    uint8_t* ring_u8_[kRing] = {nullptr, nullptr, nullptr};  // 8-bit submissions
    int64_t submit_any(int engine, const float* frames, const uint8_t* frames_u8, uint16_t* labels);
    cudaStream_t copy_st_ = nullptr;
    cudaEvent_t copied_[kRing] = {nullptr, nullptr, nullptr}, done_[kRing] = {nullptr, nullptr, nullptr};
    unsigned long long* h_ring_stats_ = nullptr;  // pinned, [kRing][nl][S][2]
    bool ring_full_[kRing] = {false, false, false};
    int64_t ring_ticket_[kRing] = {-1, -1, -1};
    int64_t submitted_ = 0;

    // host stats of the last forward, per engine
    std::vector<cbx_layer_stats> last_stats_[2];
    std::vector<uint64_t> last_macs_[2];
    unsigned long long* h_stats_ = nullptr;  // pinned mirror, [engine][nl][S][2]
    bool stats_pending_[2] = {false, false};  // device counters not yet read back
    int last_launches_ = 0;
    bool last_full_[2] = {true, true};
};

}  // namespace cbx
