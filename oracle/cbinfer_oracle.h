/*
 * cbinfer_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C CPU restatement of the reference CBinfer change-based inference
 * path (/root/reference/proj/core). It exists so that tests/, the smoke()
 * check in __graft_entry__.py and bench.py's cpu_baseline leg can check the
 * CUDA product path against the reference algorithm on machines where the
 * reference itself is not built. The product (paper_1704_04313_b200) never
 * links, loads or calls anything in this directory.
 *
 * Parity pin: this restatement is checked bit-for-bit against the reference
 * compiled from its own sources (oracle/_ref, see oracle/Makefile) and against
 * the golden vectors in tests/golden/ (made by tests/golden/make_golden.py from
 * the compiled reference). Compile with -ffp-contract=off, exactly like the
 * reference (core/CMakeLists.txt:18-21), so every float op sequence matches.
 *
 * Error convention: functions returning int return 0 on success and a
 * negative ORC_E_* code mirroring the reference exception hierarchy
 * (core/include/cbinfer/error.hpp:9-42).
 */
#ifndef CBINFER_ORACLE_H
#define CBINFER_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_E_SHAPE = -1,
    ORC_E_GEOMETRY = -2,
    ORC_E_BOUNDS = -3,
    ORC_E_IO = -4,
    ORC_E_SPEC = -5,
};

/* ConvGeometry, core/include/cbinfer/geometry.hpp:12-49 */
typedef struct {
    int kernelH, kernelW, strideH, strideW, padH, padW, inChannels, outChannels;
} orc_geom;

int orc_out_height(const orc_geom* g, int h);
int orc_out_width(const orc_geom* g, int w);
int orc_check_output(const orc_geom* g, int h, int w);

/* std::mt19937 (the engine the reference seeds everywhere) */
typedef struct {
    uint32_t state[624];
    int pos;
} orc_mt19937;
void orc_mt_seed(orc_mt19937* r, uint32_t seed);
uint32_t orc_mt_next(orc_mt19937* r);
float orc_unit_float(orc_mt19937* r);

/* ---- hot-path ops (core/src/cbconv.cpp, core/src/baseline.cpp) ---- */
int64_t orc_detect_changes(const float* cur, const float* prev, int C, int H, int W, float tau,
                           uint8_t* m);
int orc_dilate_changes(const uint8_t* m, int H, int W, const orc_geom* g, uint8_t* out);
int orc_worst_case_propagation(const int32_t* idx, int64_t n, const orc_geom* g, int H, int W,
                               uint8_t* out);
int64_t orc_extract_indexes(const uint8_t* m, int64_t n, int32_t* idx);
void orc_fill_patch_column(const float* in, int C, int H, int W, const orc_geom* g, int yo,
                           int xo, float* col);
int orc_gen_x_reduced(const float* in, int C, int H, int W, const int32_t* idx, int64_t n,
                      const orc_geom* g, float* X);
int orc_im2col_full(const float* in, int C, int H, int W, const orc_geom* g, float* X);
void orc_gemm(const float* K, const float* bias, int rows, int cols, const float* X, int64_t n,
              float* Y);
int orc_update_output(float* out, int O, int Ho, int Wo, const float* Y, const int32_t* idx,
                      int64_t n, int fuseRelu);
int orc_conv_full(const float* in, int C, int H, int W, const float* K, const float* bias,
                  const orc_geom* g, float* out);
void orc_relu(const float* in, int64_t n, float* out);
int orc_maxpool(const float* in, int C, int H, int W, int window, int stride, float* out);
void orc_argmax_classify(const float* t, int C, int H, int W, uint16_t* labels);

/* ---- synthetic input fixtures (core/src/synth.cpp) ---- */
typedef struct {
    int size;
    int velocity;
    float intensity;
} orc_sprite;

typedef struct {
    int channels, height, width, frames;
    int numSprites;
    const orc_sprite* sprites;
    float noiseAmplitude;
    uint32_t seed;
} orc_synth_cfg;

int orc_sprite_rect(const orc_synth_cfg* cfg, int s, int f, int rect[4]);
int orc_synth_frame(const orc_synth_cfg* cfg, int f, float* out);
int orc_synth_labels(const orc_synth_cfg* cfg, int f, uint16_t* out);
void orc_random_filters(const orc_geom* g, uint32_t seed, float* K, float* bias);

/* ---- network driver (core/src/network.cpp) ---- */
enum { ORC_CBCONV = 0, ORC_CONV = 1, ORC_RELU = 2, ORC_MAXPOOL = 3, ORC_CLASSIFY = 4 };
enum { ORC_ENGINE_BASELINE = 0, ORC_ENGINE_CBINFER = 1 };

typedef struct {
    int kind;
    orc_geom geom;
    int window, stride;
    float threshold;
    int fuseRelu;
} orc_layer;

typedef struct {
    int64_t changedInputPixels;
    int64_t changedOutputPixels;
    uint64_t gemmMacs;
} orc_stats;

typedef struct orc_net orc_net;

/* chain_dims (network.cpp:128-188); fills geom.inChannels of `layers` in place. */
int orc_chain_dims(int inC, int inH, int inW, int numClasses, orc_layer* layers, int nl,
                   int* dims /* nl*6: in(c,h,w), out(c,h,w) */);
int orc_net_create(int inC, int inH, int inW, int numClasses, const orc_layer* layers, int nl,
                   orc_net** out);
int orc_net_set_weights(orc_net* net, int layer, const float* K, const float* bias);
int orc_net_set_thresholds(orc_net* net, const float* taus, int n);
void orc_net_reset(orc_net* net);
int orc_forward_frame(orc_net* net, const float* frame, int engine, uint16_t* labels,
                      orc_stats* stats, uint64_t* macsTotal);
int orc_net_layer_output(const orc_net* net, int layer, const float** data, int dims[3]);
int orc_net_final_activation(const orc_net* net, const float** data, int dims[3]);
int orc_net_trace(const orc_net* net, int cbOrdinal, const uint8_t** detected, int dims[2],
                  const int32_t** updated, int64_t* n);
/* Timing warm-up: the state one orc_forward_frame(frame) leaves behind, with
 * the full-frame convolutions split over `nthreads` threads (bitwise equal). */
int orc_net_warm(orc_net* net, const float* frame, int nthreads);
int orc_net_copy_state(orc_net* dst, const orc_net* src);
void orc_net_free(orc_net* net);

#ifdef __cplusplus
}
#endif

#endif
