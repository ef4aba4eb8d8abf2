/*
 * cbx.h -- C-ABI of the B200-native CBinfer change-based inference path.
 *
 * This is the drop-in boundary: plain C types, POD descriptors, int status
 * codes, no torch or C++ types. It replaces the per-frame network-evaluation
 * API of the reference (namespace cbinfer, /root/reference/proj):
 *
 *   cbx_create + cbx_load_layer  <- load_network            core/include/cbinfer/network.hpp:88
 *                                   (+ read_weights_f32le   core/include/cbinfer/io.hpp:29)
 *   cbx_forward / _device        <- forward_frame           core/include/cbinfer/network.hpp:93-94
 *   cbx_submit / cbx_wait        <- forward_frame, pipelined (host frames; copy overlaps compute)
 *   cbx_worst_case_counts        <- worst_case_propagation  cbconv.cpp:84-97 (cbench analyze-prop)
 *   cbx_reset                    <- reset_state             core/include/cbinfer/network.hpp:97
 *   cbx_set_thresholds           <- Network::set_thresholds core/include/cbinfer/network.hpp:67
 *   cbx_get_thresholds           <- Network::thresholds     core/include/cbinfer/network.hpp:66
 *   cbx_chain_dims               <- chain_dims              core/include/cbinfer/network.hpp:45
 *   cbx_get_trace / _activation  <- ForwardTrace/CBConvTrace network.hpp:80-83, cbconv.hpp:82-85
 *   cbx_op_*                     <- detect_changes / dilate_changes / extract_indexes /
 *                                   maxpool / argmax_classify (cbconv.hpp:87-106,
 *                                   baseline.hpp:69-79), on device pointers
 *   cbx_random_filters           <- random_filters          core/include/cbinfer/synth.hpp:80
 *   cbx_synth_frame              <- synth_frame             core/include/cbinfer/synth.hpp:46
 *
 * Status codes map 1:1 onto the reference exception hierarchy
 * (core/include/cbinfer/error.hpp:9-42); the message of the last failure on a
 * context is returned by cbx_last_error(ctx) (or cbx_last_error(NULL) for
 * context-free calls, per thread).
 *
 * Threading: a context is one Network (a batch of S independent camera
 * streams) on one device. It is stream-affine and not thread-safe, mirroring
 * "one Network processes one frame at a time"; distinct
 * contexts may run concurrently.
 */
#ifndef CBX_H
#define CBX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CBX_API __attribute__((visibility("default")))

typedef enum {
    CBX_OK = 0,
    CBX_E_SHAPE = 1,    /* shape_error    */
    CBX_E_GEOMETRY = 2, /* geometry_error */
    CBX_E_BOUNDS = 3,   /* bounds_error   */
    CBX_E_IO = 4,       /* io_error       */
    CBX_E_SPEC = 5,     /* spec_error     */
    CBX_E_CUDA = 6,     /* CUDA runtime / device failure (no CPU fallback exists) */
    CBX_E_ARG = 7       /* invalid argument (null pointer, bad enum) */
} cbx_status;

/* LayerKind, network.hpp:12 */
typedef enum { CBX_CBCONV = 0, CBX_CONV = 1, CBX_RELU = 2, CBX_MAXPOOL = 3, CBX_CLASSIFY = 4 } cbx_layer_kind;

/* Engine, network.hpp:70 */
typedef enum { CBX_ENGINE_BASELINE = 0, CBX_ENGINE_CBINFER = 1 } cbx_engine;

/* Arithmetic of the convolution contraction.
 *   EXACT: the reference fp32 accumulation order bit for bit (bias first,
 *     ascending (c,kj,ki), one rounding per multiply and per add), CUDA cores.
 *   TF32: convolutions with channels-last inputs and >= 32 outputs run on
 *     tcgen05 tensor cores, kind::tf32 (operands rounded to 10 mantissa bits,
 *     fp32 accumulate). The planar first layer and narrow 1x1 heads stay EXACT.
 *   F16: as TF32, but a layer with > 128 outputs fed by a MAXPOOL runs
 *     kind::f16 with fp16 operands (the same 10 mantissa bits, round to
 *     nearest, a 5-bit exponent: |x| <= 65504, subnormal below 6.1e-5; fp32
 *     accumulate). Twice the tensor rate and half the operand bytes of tf32.
 *     The MAXPOOL writes an fp16 shadow of its output and flags any value out
 *     of range; that frame and every later one until the next full evaluation
 *     then fail with CBX_E_ARG when their stats are read (cbx_forward,
 *     cbx_wait, cbx_read_stats), and the next frame is evaluated in full.
 *     Weights out of the fp16 range are rejected by cbx_load_layer. */
typedef enum { CBX_PREC_EXACT = 0, CBX_PREC_TF32 = 1, CBX_PREC_F16 = 2 } cbx_precision;

/* ConvGeometry, geometry.hpp:12-49 */
typedef struct {
    int kernelH, kernelW, strideH, strideW, padH, padW, inChannels, outChannels;
} cbx_geom;

/* LayerSpec, network.hpp:17-27 (weights are passed separately) */
typedef struct {
    int kind;       /* cbx_layer_kind */
    cbx_geom geom;  /* conv kinds; inChannels is filled by cbx_chain_dims/cbx_create */
    int window;     /* MAXPOOL */
    int stride;     /* MAXPOOL */
    float threshold;/* CBCONV, >= 0 */
    int fuseRelu;   /* CBCONV */
} cbx_layer_desc;

/* NetworkSpec, network.hpp:29-35 */
typedef struct {
    int inputChannels, inputHeight, inputWidth, numClasses;
    int numLayers;
    const cbx_layer_desc* layers;
} cbx_net_desc;

/* LayerStats, cbconv.hpp:55-60 (timings are measured with CUDA events by the caller) */
typedef struct {
    int64_t changedInputPixels;
    int64_t changedOutputPixels;
    uint64_t gemmMacs;
} cbx_layer_stats;

typedef struct cbx_ctx cbx_ctx;

CBX_API const char* cbx_last_error(const cbx_ctx* ctx);
CBX_API const char* cbx_version(void);

/* chain_dims: validates the chain, fills layers[k].geom.inChannels and writes
 * per-layer in/out dims (dims[6k..6k+5] = inC,inH,inW,outC,outH,outW). */
CBX_API int cbx_chain_dims(const cbx_net_desc* net, cbx_layer_desc* layers_out, int* dims);

/* Create a network context on `device` serving `num_streams` independent
 * camera streams (each with its own change-based state). */
CBX_API int cbx_create(const cbx_net_desc* net, int device, int num_streams, int precision,
                       cbx_ctx** out);
/* cbx_create with an explicit lane count: the streams are split into `lanes`
 * contiguous groups, each evaluated by its own engine on its own CUDA stream
 * so that the groups' kernels overlap on the GPU (one group's tcgen05
 * layer-3 conv next to another group's mask / layer-1 / pooling kernels).
 * lanes <= 0: automatic (2 when num_streams >= 2, else 1); cbx_create uses
 * automatic. Results are identical for any lane count. */
CBX_API int cbx_create_ex(const cbx_net_desc* net, int device, int num_streams, int precision, int lanes,
                          cbx_ctx** out);
CBX_API int cbx_num_lanes(const cbx_ctx* ctx);
/* Operand format of layer `layer`'s convolution: 0 = fp32 on CUDA cores
 * (exact reference order), 1 = tcgen05 kind::tf32, 2 = tcgen05 kind::f16
 * (fp16 operands rounded to nearest, fp32 accumulation; CBX_PREC_F16 only),
 * 3 = tcgen05 kind::i8 on 8-bit camera frames (layer 0 only, see
 * CBX_OPT_U8_NATIVE; fp32 frames still take the exact fp32 path), -1 = not a conv. */
CBX_API int cbx_layer_operands(const cbx_ctx* ctx, int layer);
CBX_API void cbx_destroy(cbx_ctx* ctx);

/* Install the filters of conv layer `layer` (0-based index in the layer
 * list) in the reference layout: K row-major [outC][inC*kH*kW] with columns in
 * (c, kj, ki) order (baseline.hpp:11-12), then outC biases. Host memory. */
CBX_API int cbx_load_layer(cbx_ctx* ctx, int layer, const float* K, const float* bias);

CBX_API int cbx_set_thresholds(cbx_ctx* ctx, const float* taus, int n);
CBX_API int cbx_get_thresholds(const cbx_ctx* ctx, float* taus, int n);

/* Runtime options. CBX_OPT_FUSE_TAIL (default 1): run the per-pixel layers
 * that end the network (1x1 CONV / RELU / CLASSIFY after the last tcgen05
 * conv) inside that conv's epilogue; their intermediate tensors are then not
 * materialized (cbx_get_activation reports CBX_E_SPEC for them). 0 keeps every
 * layer's output, e.g. for per-layer parity checks. Results are identical. */
/* CBX_OPT_TC_PAIR (default -1 = auto = single-CTA tiles): CTA grouping of the
 * tcgen05 convs. 1 pairs the two SMs of a TPC (cta_group::2, M = 256 tiles,
 * each SM holds half the filter bank); 0 forces one CTA per tile. Same tf32
 * error bound either way. */
/* CBX_OPT_STEP_TIMES (default 0): record CUDA event nodes at the kernel
 * boundaries of the frame graph so cbx_read_step_times can return the
 * reference's per-layer StepTimes (cbconv.hpp:44-52) -- the collectTimings
 * switch of CBConvState (cbconv.hpp:70). Off: no timing nodes in the graph. */
/* CBX_OPT_U8_NATIVE (default 1): 8-bit camera frames (cbx_forward_u8,
 * cbx_submit_u8, cbx_forward_device_u8) run natively in the tensor-core
 * precisions when the frame is 3-channel with a width divisible by 16 and the
 * first layer is a conv: change detection on the bytes (decoded exactly as
 * read_ppm, so layer-1 masks and index lists stay bit-exact) fused with an
 * RGBX copy of the frame, and layer 1 as a tcgen05 kind::i8 conv over those
 * bytes (filters as three 8-bit digits of a 22-bit fixed-point weight, exact
 * integer accumulation: layer-1 outputs within ~2^-22 relative of the fp32
 * reference instead of bitwise; cbx_layer_operands(ctx, 0) reports 3). 0 decodes
 * 8-bit frames into fp32 planar frames first (the fp32 path: layer 1 bitwise).
 * Changing it makes the next frame a full evaluation. */
typedef enum { CBX_OPT_FUSE_TAIL = 0, CBX_OPT_TC_PAIR = 1, CBX_OPT_STEP_TIMES = 2, CBX_OPT_U8_NATIVE = 3 } cbx_option;
CBX_API int cbx_set_option(cbx_ctx* ctx, int option, int value);

/* Drops all change-based state of every stream: the next frame is a full
 * evaluation (reset_state, network.cpp:317-320). */
CBX_API int cbx_reset(cbx_ctx* ctx);

/* One frame for each of the S streams, HOST buffers:
 *   frames: S planar CHW fp32 frames back to back (S*C*H*W floats)
 *   labels: S label maps (uint16, row-major), may be NULL
 *   stats : S*numLayers entries (stream-major), may be NULL
 *   macs  : S entries (macsTotal per stream), may be NULL
 * Synchronous: returns after labels/stats are in host memory. The
 * Baseline engine evaluates every layer full-frame and leaves the
 * change-based state untouched (network.cpp:278-285). */
CBX_API int cbx_forward(cbx_ctx* ctx, int engine, const float* frames, uint16_t* labels,
                        cbx_layer_stats* stats, uint64_t* macs);

/* Device-resident variant for clips already in HBM: frames_dev[s] points to
 * stream s's planar frame on the context's device. Asynchronous on the
 * context stream; use cbx_sync / cbx_read_* afterwards. The frame buffers are
 * read by kernels that run after this call returns, and each frame is also
 * the detection reference (prevInput of the first CBCONV) of the NEXT call:
 * a frame buffer must stay valid and unmodified until the work of the call
 * after the one that passed it has completed (cbx_sync, or an event recorded
 * on cbx_stream after that call). */
CBX_API int cbx_forward_device(cbx_ctx* ctx, int engine, const float* const* frames_dev);
/* Pipelined host-frame serving (forward_frame, network.hpp:93-94, split in
 * two): cbx_submit enqueues one frame of every stream -- host -> device copy
 * on a copy stream into a staging ring, the change-based evaluation on the
 * context stream once the copy has landed, labels copied back into `labels`
 * -- and returns at once with a ticket; the copy of the next submission
 * overlaps the kernels of this one. cbx_wait(ticket) blocks until that frame
 * is done; `labels` is then valid and stats/macs (nullable) are filled as by
 * cbx_forward. Frames are consumed in submission order (each is the next
 * frame of every stream). `frames` and `labels` must stay valid until the
 * wait returns; pin them (cudaHostAlloc) for the copies to overlap. Only the
 * last 3 tickets can be waited on. Change-based engine only. */
CBX_API int cbx_submit(cbx_ctx* ctx, int engine, const float* frames, uint16_t* labels, int64_t* ticket);
CBX_API int cbx_wait(cbx_ctx* ctx, int64_t ticket, cbx_layer_stats* stats, uint64_t* macs);
/* 8-bit camera frames (read_ppm, io.cpp:60-104): `frames` holds S frames back
 * to back, each H x W pixels of inputChannels interleaved bytes (the binary
 * PPM raster). Only the bytes cross PCIe (4x fewer than fp32 planar frames);
 * the device decodes them into the planar fp32 frame px / 255.0f exactly as
 * read_ppm does, so results equal cbx_forward / cbx_submit on read_ppm's
 * tensors bit for bit. Same semantics and ticket ring otherwise. */
CBX_API int cbx_forward_u8(cbx_ctx* ctx, int engine, const uint8_t* frames, uint16_t* labels,
                           cbx_layer_stats* stats, uint64_t* macs);
CBX_API int cbx_submit_u8(cbx_ctx* ctx, int engine, const uint8_t* frames, uint16_t* labels, int64_t* ticket);
/* 8-bit frames already on the device: frames_dev[s] = stream s's H x W x C
 * interleaved bytes (16-byte aligned). Same contract as cbx_forward_device
 * (asynchronous; each frame is the next call's detection reference). */
CBX_API int cbx_forward_device_u8(cbx_ctx* ctx, int engine, const uint8_t* const* frames_dev);
/* cbench analyze-prop (tools/cbench.cpp:242-302) for the last change-based
 * frame (not a full one): for every CBCONV k >= 1 (0-based among CBCONVs), the
 * worst-case updated count of layer k -- the updated set of CBCONV k-1 pushed
 * through the layers in between and dilated by layer k's geometry
 * (worst_case_propagation / dilate_changes, cbconv.cpp:73-97) -- per stream:
 * worst[s * (numCB - 1) + k - 1]. Compare with changedOutputPixels of layer k. */
CBX_API int cbx_worst_case_counts(cbx_ctx* ctx, int64_t* worst);
CBX_API int cbx_sync(cbx_ctx* ctx);
CBX_API int cbx_read_labels(cbx_ctx* ctx, int engine, uint16_t* labels);
CBX_API int cbx_read_stats(cbx_ctx* ctx, int engine, cbx_layer_stats* stats, uint64_t* macs);
/* Device labels buffer [S][Hl][Wl] (single-lane contexts only: CBX_E_ARG otherwise). */
CBX_API int cbx_labels_device(cbx_ctx* ctx, int engine, const uint16_t** labels_dev);

/* Context stream as a cudaStream_t (void* here). */
CBX_API void* cbx_stream(cbx_ctx* ctx);
/* Number of kernel launches (graph kernel nodes) issued by the last forward. */
CBX_API int cbx_last_launch_count(const cbx_ctx* ctx);

/* Per-kernel device time of one forward: the frame is run WITHOUT the CUDA
 * graph, every kernel bracketed by CUDA events on the context stream. The
 * state advances exactly as with cbx_forward_device. */
typedef struct {
    char name[32];
    int layer;
    float ms;
} cbx_kernel_time;
CBX_API int cbx_profile_forward(cbx_ctx* ctx, int engine, const float* const* frames_dev,
                                cbx_kernel_time* out, int cap, int* n);
CBX_API int cbx_profile_forward_u8(cbx_ctx* ctx, int engine, const uint8_t* const* frames_dev,
                                   cbx_kernel_time* out, int cap, int* n);

/* Trace access for parity checks (CBConvTrace / ForwardTrace):
 *   cbx_get_activation: output of layer `layer` for stream s, planar CHW, host
 *   cbx_get_trace: CBCONV ordinal `cb`, stream s: detected input-grid mask
 *   (uint8 H*W, zeroed on the first frame) and the ascending updated index list
 *   (int32, capacity Ho*Wo); *n receives the count; *first is set to 1 when
 *   the last frame was a full evaluation (the reference's empty `detected`). */
CBX_API int cbx_get_activation(cbx_ctx* ctx, int engine, int layer, int s, float* out);
CBX_API int cbx_get_trace(cbx_ctx* ctx, int cb, int s, uint8_t* detected, int32_t* updated,
                          int64_t* n, int* first);
/* Input tensor of layer `layer` for stream s after the last frame, planar CHW
 * host floats: the reference's CBConvState::prevInput (cbconv.hpp:71) when the
 * layer is a CBCONV. Layer 0 returns the last frame the change-based engine
 * consumed (CBX_E_SPEC before the first frame / after a reset). */
CBX_API int cbx_get_input(cbx_ctx* ctx, int engine, int layer, int s, float* out);
/* 1 when the change-based state holds a previous frame (CBConvState::
 * has_history, cbconv.hpp:73): the next frame is evaluated incrementally;
 * 0 after creation, cbx_reset or an fp16 range error; -1 on a null context. */
CBX_API int cbx_has_history(const cbx_ctx* ctx);
/* StepTimes of the last frame launched with CBX_OPT_STEP_TIMES on:
 * nanos[(s * numLayers + k) * 5 + {0..4}] = detect, extract, generate,
 * multiply, update of layer k (stepNanos, cbconv.hpp:44-52; 0 for non-CBCONV
 * work that has no step). The B200 kernels fuse steps: detect = the frame
 * detection kernel (first CBCONV; later CBCONVs detect inside their
 * producer's compare-before-write), extract = dilation + compaction,
 * multiply = the gathered convolution including the patch gather (generate)
 * and the in-place scatter (update), which therefore read 0. Streams that
 * share a lane share the lane's kernels and report the same times. Timed
 * with CUDA events on the device; all zero when the option is off. */
CBX_API int cbx_read_step_times(cbx_ctx* ctx, int64_t* nanos);

/* ---- op level, device pointers, asynchronous on `stream` (cudaStream_t) ---- */
CBX_API int cbx_op_detect(const float* cur, const float* prev, int C, int H, int W, float tau,
                          uint8_t* mask, unsigned long long* count_dev, void* stream);
CBX_API int cbx_op_dilate(const uint8_t* mask, int H, int W, const cbx_geom* geom, uint8_t* out,
                          void* stream);
/* Workspace bytes for cbx_op_extract over n mask bytes. */
CBX_API size_t cbx_op_extract_workspace(int64_t n);
CBX_API int cbx_op_extract(const uint8_t* mask, int64_t n, int32_t* idx, int* count_dev,
                           void* workspace, void* stream);
CBX_API int cbx_op_maxpool(const float* in, int C, int H, int W, int window, int stride,
                           float* out, void* stream);
CBX_API int cbx_op_argmax(const float* t, int C, int H, int W, uint16_t* labels, void* stream);
/* Matrix-form reference ops (the network path never materializes X or Y):
 *   cbx_op_gen_x   <- gen_x_reduced / im2col_full / fill_patch_column
 *                     (cbconv.cpp:115-133, baseline.cpp:9-45): X column-major
 *                     [n][C*kh*kw], column j = the (c,kj,ki) receptive field of
 *                     output pixel idx[j] (idx NULL: pixel j), zero padded.
 *                     Indices must lie in [0, Ho*Wo) (checked by the caller).
 *   cbx_op_gemm    <- gemm (baseline.cpp:47-63): Y row-major [rows][n] =
 *                     bias + K X, ascending r, no FMA (bitwise the reference).
 *   cbx_op_scatter <- update_output without its copy (cbconv.cpp:135-155):
 *                     out[c][idx[j]] = Y[c][j] (max(0, .) when relu), in place. */
CBX_API int cbx_op_gen_x(const float* in, int C, int H, int W, const cbx_geom* geom, const int32_t* idx,
                         int64_t n, float* X, void* stream);
CBX_API int cbx_op_gemm(const float* K, const float* bias, int rows, int cols, const float* X, int64_t n,
                        float* Y, void* stream);
CBX_API int cbx_op_scatter(float* out, int C, int H, int W, const float* Y, const int32_t* idx, int64_t n,
                           int relu, void* stream);
/* The decode of cbx_forward_u8 on device buffers: S interleaved 8-bit frames
 * (H x W x C) -> S planar fp32 frames px / 255.0f (read_ppm, io.cpp:60-104). */
CBX_API int cbx_op_decode_u8(const uint8_t* in, int S, int C, int H, int W, float* out, void* stream);
/* relu (baseline.cpp:113-117): out = max(0, in) element-wise, planar CHW. */
CBX_API int cbx_op_relu(const float* in, int C, int H, int W, float* out, void* stream);
/* Reduced conv over an index list (gen_x_reduced + gemm + update_output,
 * cbconv.cpp:115-155), planar CHW in/out, exact fp32 order; out is updated in
 * place at the listed output pixels. */
CBX_API int cbx_op_cbconv_update(const float* in, int C, int H, int W, const float* K,
                                 const float* bias, const cbx_geom* geom, const int32_t* idx,
                                 int n, int fuseRelu, float* out, void* stream);

/* ---- input fixtures (synth.hpp) ---- */
CBX_API int cbx_random_filters(const cbx_geom* geom, uint32_t seed, float* K, float* bias);
typedef struct {
    int size, velocity;
    float intensity;
} cbx_sprite;
typedef struct {
    int channels, height, width, frames;
    int numSprites;
    const cbx_sprite* sprites;
    float noiseAmplitude;
    uint32_t seed;
} cbx_synth_cfg;
/* Host frame (noise supported). */
CBX_API int cbx_synth_frame(const cbx_synth_cfg* cfg, int f, float* out);
/* Device frame (noise-free clips only; noise needs the sequential mt19937). */
CBX_API int cbx_synth_frame_device(const cbx_synth_cfg* cfg, int f, float* out_dev, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CBX_H */
