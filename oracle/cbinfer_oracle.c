/*
 * cbinfer_oracle.c -- TEST INFRASTRUCTURE ONLY (see cbinfer_oracle.h).
 *
 * CPU restatement of the reference algorithm. Every function cites the
 * reference file:line it restates; paths are relative to
 * /root/reference/proj/. Build with -ffp-contract=off (oracle/Makefile).
 */
#include "cbinfer_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* geometry -- core/include/cbinfer/geometry.hpp:22-41                  */

int orc_out_height(const orc_geom* g, int h) { return (h + 2 * g->padH - g->kernelH) / g->strideH + 1; }
int orc_out_width(const orc_geom* g, int w) { return (w + 2 * g->padW - g->kernelW) / g->strideW + 1; }

int orc_check_output(const orc_geom* g, int h, int w) {
    if (g->kernelH < 1 || g->kernelW < 1 || g->strideH < 1 || g->strideW < 1 || g->padH < 0 ||
        g->padW < 0)
        return ORC_E_GEOMETRY;
    if (h + 2 * g->padH < g->kernelH || w + 2 * g->padW < g->kernelW) return ORC_E_GEOMETRY;
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* std::mt19937, the engine behind synth.cpp:18-20 and testutil.hpp:15  */

void orc_mt_seed(orc_mt19937* r, uint32_t seed) {
    r->state[0] = seed;
    for (int i = 1; i < 624; ++i) {
        uint32_t p = r->state[i - 1];
        r->state[i] = 1812433253u * (p ^ (p >> 30)) + (uint32_t)i;
    }
    r->pos = 624;
}

static void mt_refill(orc_mt19937* r) {
    for (int i = 0; i < 624; ++i) {
        uint32_t hi = r->state[i] & 0x80000000u;
        uint32_t lo = r->state[(i + 1) % 624] & 0x7fffffffu;
        uint32_t y = hi | lo;
        uint32_t v = r->state[(i + 397) % 624] ^ (y >> 1);
        if (y & 1u) v ^= 0x9908b0dfu;
        r->state[i] = v;
    }
    r->pos = 0;
}

uint32_t orc_mt_next(orc_mt19937* r) {
    if (r->pos >= 624) mt_refill(r);
    uint32_t y = r->state[r->pos++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}

/* synth.cpp:18-20: 24-bit mantissa mapping to [0,1) */
float orc_unit_float(orc_mt19937* r) { return (float)(orc_mt_next(r) >> 8) * (1.0f / 16777216.0f); }

/* ------------------------------------------------------------------ */
/* change detection -- core/src/cbconv.cpp:57-71                        */
/* Strict inequality on both signs of the fp32 difference; any channel. */

int64_t orc_detect_changes(const float* cur, const float* prev, int C, int H, int W, float tau,
                           uint8_t* m) {
    const int64_t plane = (int64_t)H * W;
    memset(m, 0, (size_t)plane);
    for (int c = 0; c < C; ++c) {
        const float* a = cur + c * plane;
        const float* b = prev + c * plane;
        for (int64_t p = 0; p < plane; ++p) {
            const float d = a[p] - b[p];
            if (d > tau || -d > tau) m[p] = 1;
        }
    }
    int64_t n = 0;
    for (int64_t p = 0; p < plane; ++p) n += m[p];
    return n;
}

/* ------------------------------------------------------------------ */
/* dilation -- core/src/cbconv.cpp:19-41 (floor/ceil div, scatter_support)
 * and :73-82 (dilate_changes). Restated as the scatter of every set input
 * pixel onto the output pixels whose zero-padded receptive field holds it. */

static int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
static int cdiv(int a, int b) { return fdiv(a + b - 1, b); }

static void mark_support(uint8_t* out, int Ho, int Wo, const orc_geom* g, int j, int i) {
    int y0 = cdiv(j + g->padH - g->kernelH + 1, g->strideH);
    int y1 = fdiv(j + g->padH, g->strideH);
    int x0 = cdiv(i + g->padW - g->kernelW + 1, g->strideW);
    int x1 = fdiv(i + g->padW, g->strideW);
    if (y0 < 0) y0 = 0;
    if (x0 < 0) x0 = 0;
    if (y1 > Ho - 1) y1 = Ho - 1;
    if (x1 > Wo - 1) x1 = Wo - 1;
    for (int y = y0; y <= y1; ++y)
        for (int x = x0; x <= x1; ++x) out[(int64_t)y * Wo + x] = 1;
}

int orc_dilate_changes(const uint8_t* m, int H, int W, const orc_geom* g, uint8_t* out) {
    int rc = orc_check_output(g, H, W);
    if (rc) return rc;
    const int Ho = orc_out_height(g, H), Wo = orc_out_width(g, W);
    memset(out, 0, (size_t)Ho * Wo);
    for (int j = 0; j < H; ++j)
        for (int i = 0; i < W; ++i)
            if (m[(int64_t)j * W + i]) mark_support(out, Ho, Wo, g, j, i);
    return ORC_OK;
}

/* core/src/cbconv.cpp:84-97 */
int orc_worst_case_propagation(const int32_t* idx, int64_t n, const orc_geom* g, int H, int W,
                               uint8_t* out) {
    int rc = orc_check_output(g, H, W);
    if (rc) return rc;
    const int Ho = orc_out_height(g, H), Wo = orc_out_width(g, W);
    memset(out, 0, (size_t)Ho * Wo);
    const int64_t pixels = (int64_t)H * W;
    for (int64_t k = 0; k < n; ++k) {
        if (idx[k] < 0 || idx[k] >= pixels) return ORC_E_BOUNDS;
        mark_support(out, Ho, Wo, g, idx[k] / W, idx[k] % W);
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* index extraction -- core/src/cbconv.cpp:99-113. The reference scans 256-
 * pixel blocks and concatenates them; only the resulting global ascending
 * order is observable, which a serial scan reproduces. */

int64_t orc_extract_indexes(const uint8_t* m, int64_t n, int32_t* idx) {
    int64_t k = 0;
    for (int64_t p = 0; p < n; ++p)
        if (m[p]) idx[k++] = (int32_t)p;
    return k;
}

/* ------------------------------------------------------------------ */
/* im2col column -- core/src/baseline.cpp:9-31: rows in (c, kj, ki) order,
 * explicit zeros outside the frame. */

void orc_fill_patch_column(const float* in, int C, int H, int W, const orc_geom* g, int yo,
                           int xo, float* col) {
    const int by = yo * g->strideH - g->padH;
    const int bx = xo * g->strideW - g->padW;
    for (int c = 0; c < C; ++c) {
        const float* plane = in + (int64_t)c * H * W;
        for (int kj = 0; kj < g->kernelH; ++kj) {
            const int y = by + kj;
            for (int ki = 0; ki < g->kernelW; ++ki) {
                const int x = bx + ki;
                *col++ = (y >= 0 && y < H && x >= 0 && x < W) ? plane[(int64_t)y * W + x] : 0.0f;
            }
        }
    }
}

/* core/src/cbconv.cpp:115-133 */
int orc_gen_x_reduced(const float* in, int C, int H, int W, const int32_t* idx, int64_t n,
                      const orc_geom* g, float* X) {
    if (C != g->inChannels) return ORC_E_SHAPE;
    int rc = orc_check_output(g, H, W);
    if (rc) return rc;
    const int Wo = orc_out_width(g, W);
    const int64_t outPixels = (int64_t)orc_out_height(g, H) * Wo;
    const int rows = g->inChannels * g->kernelH * g->kernelW;
    for (int64_t k = 0; k < n; ++k) {
        if (idx[k] < 0 || idx[k] >= outPixels) return ORC_E_BOUNDS;
        orc_fill_patch_column(in, C, H, W, g, idx[k] / Wo, idx[k] % Wo, X + k * rows);
    }
    return ORC_OK;
}

/* core/src/baseline.cpp:33-45 */
int orc_im2col_full(const float* in, int C, int H, int W, const orc_geom* g, float* X) {
    if (C != g->inChannels) return ORC_E_SHAPE;
    int rc = orc_check_output(g, H, W);
    if (rc) return rc;
    const int Ho = orc_out_height(g, H), Wo = orc_out_width(g, W);
    const int rows = g->inChannels * g->kernelH * g->kernelW;
    for (int y = 0; y < Ho; ++y)
        for (int x = 0; x < Wo; ++x)
            orc_fill_patch_column(in, C, H, W, g, y, x, X + ((int64_t)y * Wo + x) * rows);
    return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* GEMM -- core/src/baseline.cpp:47-63: accumulator starts at the bias and
 * adds K(o,r)*X(r,n) in ascending r, one rounding per multiply and add. */

void orc_gemm(const float* K, const float* bias, int rows, int cols, const float* X, int64_t n,
              float* Y) {
    for (int64_t j = 0; j < n; ++j) {
        const float* x = X + j * cols;
        for (int o = 0; o < rows; ++o) {
            const float* k = K + (int64_t)o * cols;
            float acc = bias[o];
            for (int r = 0; r < cols; ++r) acc += k[r] * x[r];
            Y[(int64_t)o * n + j] = acc;
        }
    }
}

/* std::max(0.0f, v) == (0.0f < v) ? v : 0.0f (baseline.cpp:115, cbconv.cpp:151) */
static float relu1(float v) { return (0.0f < v) ? v : 0.0f; }

/* core/src/cbconv.cpp:135-155, in place on a caller-made copy of prevOut */
int orc_update_output(float* out, int O, int Ho, int Wo, const float* Y, const int32_t* idx,
                      int64_t n, int fuseRelu) {
    const int64_t plane = (int64_t)Ho * Wo;
    for (int o = 0; o < O; ++o) {
        float* p = out + o * plane;
        const float* yr = Y + (int64_t)o * n;
        for (int64_t k = 0; k < n; ++k) {
            if (idx[k] < 0 || idx[k] >= plane) return ORC_E_BOUNDS;
            p[idx[k]] = fuseRelu ? relu1(yr[k]) : yr[k];
        }
    }
    return ORC_OK;
}

/* core/src/baseline.cpp:65-111: direct convolution with explicit zero
 * products, same accumulation order as gemm over im2col columns. */
int orc_conv_full(const float* in, int C, int H, int W, const float* K, const float* bias,
                  const orc_geom* g, float* out) {
    if (C != g->inChannels) return ORC_E_SHAPE;
    int rc = orc_check_output(g, H, W);
    if (rc) return rc;
    const int Ho = orc_out_height(g, H), Wo = orc_out_width(g, W);
    const int cols = C * g->kernelH * g->kernelW;
    for (int o = 0; o < g->outChannels; ++o) {
        for (int yo = 0; yo < Ho; ++yo)
            for (int xo = 0; xo < Wo; ++xo) {
                const int by = yo * g->strideH - g->padH, bx = xo * g->strideW - g->padW;
                const float* kv = K + (int64_t)o * cols;
                float acc = bias[o];
                for (int c = 0; c < C; ++c)
                    for (int kj = 0; kj < g->kernelH; ++kj)
                        for (int ki = 0; ki < g->kernelW; ++ki) {
                            const int y = by + kj, x = bx + ki;
                            const float v = (y >= 0 && y < H && x >= 0 && x < W)
                                                ? in[((int64_t)c * H + y) * W + x]
                                                : 0.0f;
                            acc += *kv++ * v;
                        }
                out[((int64_t)o * Ho + yo) * Wo + xo] = acc;
            }
    }
    return ORC_OK;
}

/* core/src/baseline.cpp:113-117 */
void orc_relu(const float* in, int64_t n, float* out) {
    for (int64_t k = 0; k < n; ++k) out[k] = relu1(in[k]);
}

/* core/src/baseline.cpp:119-145: floor semantics, first element seeds the
 * max, std::max(m, v) == (m < v) ? v : m. */
int orc_maxpool(const float* in, int C, int H, int W, int window, int stride, float* out) {
    if (window < 1 || stride < 1 || window > H || window > W) return ORC_E_GEOMETRY;
    const int Ho = (H - window) / stride + 1, Wo = (W - window) / stride + 1;
    for (int c = 0; c < C; ++c) {
        const float* p = in + (int64_t)c * H * W;
        for (int y = 0; y < Ho; ++y)
            for (int x = 0; x < Wo; ++x) {
                float m = p[(int64_t)(y * stride) * W + x * stride];
                for (int kj = 0; kj < window; ++kj)
                    for (int ki = 0; ki < window; ++ki) {
                        const float v = p[(int64_t)(y * stride + kj) * W + x * stride + ki];
                        m = (m < v) ? v : m;
                    }
                out[((int64_t)c * Ho + y) * Wo + x] = m;
            }
    }
    return ORC_OK;
}

/* core/src/baseline.cpp:147-163: strict >, ties keep the lowest channel */
void orc_argmax_classify(const float* t, int C, int H, int W, uint16_t* labels) {
    const int64_t plane = (int64_t)H * W;
    for (int64_t p = 0; p < plane; ++p) {
        int best = 0;
        float bv = t[p];
        for (int c = 1; c < C; ++c) {
            const float v = t[(int64_t)c * plane + p];
            if (v > bv) {
                bv = v;
                best = c;
            }
        }
        labels[p] = (uint16_t)best;
    }
}

/* ------------------------------------------------------------------ */
/* synthetic clips -- core/src/synth.cpp                                */

static const int kDirs[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};

/* synth.cpp:33-58 */
int orc_sprite_rect(const orc_synth_cfg* cfg, int s, int f, int rect[4]) {
    const orc_sprite* sp = &cfg->sprites[s];
    if (sp->size > cfg->height || sp->size > cfg->width) return ORC_E_SPEC;
    orc_mt19937 r;
    orc_mt_seed(&r, cfg->seed ^ (0x9e3779b9u * (uint32_t)(s + 1)));
    const int sy = (int)(orc_mt_next(&r) % (uint32_t)(cfg->height - sp->size + 1));
    const int sx = (int)(orc_mt_next(&r) % (uint32_t)(cfg->width - sp->size + 1));
    const int* d = kDirs[orc_mt_next(&r) % 8];
    const int travel = sp->velocity * f;
    int y = sy + d[0] * travel, x = sx + d[1] * travel;
    const int ymax = cfg->height - sp->size, xmax = cfg->width - sp->size;
    y = y < 0 ? 0 : (y > ymax ? ymax : y);
    x = x < 0 ? 0 : (x > xmax ? xmax : x);
    rect[0] = y;
    rect[1] = x;
    rect[2] = y + sp->size;
    rect[3] = x + sp->size;
    return ORC_OK;
}

/* synth.cpp:60-64 */
static float background(int c, int j, int i) {
    const unsigned v = (unsigned)(i * 31 + j * 17 + c * 47) % 101u;
    return 0.2f + 0.25f * ((float)v / 100.0f);
}

/* synth.cpp:66-91 */
int orc_synth_frame(const orc_synth_cfg* cfg, int f, float* out) {
    const int C = cfg->channels, H = cfg->height, W = cfg->width;
    for (int c = 0; c < C; ++c)
        for (int j = 0; j < H; ++j)
            for (int i = 0; i < W; ++i) out[((int64_t)c * H + j) * W + i] = background(c, j, i);
    for (int s = 0; s < cfg->numSprites; ++s) {
        int r[4];
        int rc = orc_sprite_rect(cfg, s, f, r);
        if (rc) return rc;
        const float v = cfg->sprites[s].intensity;
        for (int c = 0; c < C; ++c)
            for (int j = r[0]; j < r[2]; ++j)
                for (int i = r[1]; i < r[3]; ++i) out[((int64_t)c * H + j) * W + i] = v;
    }
    if (cfg->noiseAmplitude > 0.0f) {
        orc_mt19937 r;
        orc_mt_seed(&r, cfg->seed * 2654435761u + (uint32_t)f + 1u);
        const int64_t n = (int64_t)C * H * W;
        for (int64_t k = 0; k < n; ++k)
            out[k] += cfg->noiseAmplitude * (2.0f * orc_unit_float(&r) - 1.0f);
    }
    return ORC_OK;
}

/* synth.cpp:93-101 */
int orc_synth_labels(const orc_synth_cfg* cfg, int f, uint16_t* out) {
    memset(out, 0, sizeof(uint16_t) * (size_t)cfg->height * cfg->width);
    for (int s = 0; s < cfg->numSprites; ++s) {
        int r[4];
        int rc = orc_sprite_rect(cfg, s, f, r);
        if (rc) return rc;
        for (int j = r[0]; j < r[2]; ++j)
            for (int i = r[1]; i < r[3]; ++i) out[(int64_t)j * cfg->width + i] = 1;
    }
    return ORC_OK;
}

/* synth.cpp:188-196 */
void orc_random_filters(const orc_geom* g, uint32_t seed, float* K, float* bias) {
    orc_mt19937 r;
    orc_mt_seed(&r, seed);
    const int fanIn = g->inChannels * g->kernelH * g->kernelW;
    const float scale = 1.0f / sqrtf((float)fanIn);
    const int64_t n = (int64_t)g->outChannels * fanIn;
    for (int64_t k = 0; k < n; ++k) K[k] = scale * (2.0f * orc_unit_float(&r) - 1.0f);
    for (int o = 0; o < g->outChannels; ++o) bias[o] = 0.1f * (2.0f * orc_unit_float(&r) - 1.0f);
}

/* ------------------------------------------------------------------ */
/* network driver -- core/src/network.cpp                               */

typedef struct {
    orc_layer spec;
    int in[3], out[3];
    float* K;
    float* bias;
    /* CBCONV state, cbconv.hpp:65-79 */
    int hasHistory;
    float* prevInput;
    float* prevOutput;
    /* trace, cbconv.hpp:82-85 */
    uint8_t* detected;
    int detectedValid;
    int32_t* updated;
    int64_t nUpdated;
    /* last activation produced by this layer (for parity checks) */
    float* act;
} orc_layer_rt;

struct orc_net {
    int inC, inH, inW, numClasses;
    int nl;
    orc_layer_rt* L;
    float* finalAct;
    int finalDims[3];
};

static int64_t dims_count(const int d[3]) { return (int64_t)d[0] * d[1] * d[2]; }

/* network.cpp:128-188 */
int orc_chain_dims(int inC, int inH, int inW, int numClasses, orc_layer* layers, int nl,
                   int* dims) {
    if (nl < 1) return ORC_E_SPEC;
    if (inC < 1 || inH < 1 || inW < 1) return ORC_E_SPEC;
    if (numClasses < 1) return ORC_E_SPEC;
    int cur[3] = {inC, inH, inW};
    for (int k = 0; k < nl; ++k) {
        orc_layer* l = &layers[k];
        int o[3];
        dims[k * 6 + 0] = cur[0];
        dims[k * 6 + 1] = cur[1];
        dims[k * 6 + 2] = cur[2];
        switch (l->kind) {
            case ORC_CBCONV:
            case ORC_CONV:
                l->geom.inChannels = cur[0];
                if (orc_check_output(&l->geom, cur[1], cur[2])) return ORC_E_GEOMETRY;
                o[0] = l->geom.outChannels;
                o[1] = orc_out_height(&l->geom, cur[1]);
                o[2] = orc_out_width(&l->geom, cur[2]);
                break;
            case ORC_RELU:
                o[0] = cur[0];
                o[1] = cur[1];
                o[2] = cur[2];
                break;
            case ORC_MAXPOOL:
                if (l->window < 1 || l->stride < 1 || l->window > cur[1] || l->window > cur[2])
                    return ORC_E_GEOMETRY;
                o[0] = cur[0];
                o[1] = (cur[1] - l->window) / l->stride + 1;
                o[2] = (cur[2] - l->window) / l->stride + 1;
                break;
            case ORC_CLASSIFY:
                if (k + 1 != nl) return ORC_E_SPEC;
                if (cur[0] != numClasses) return ORC_E_SPEC;
                o[0] = 1;
                o[1] = cur[1];
                o[2] = cur[2];
                break;
            default:
                return ORC_E_SPEC;
        }
        dims[k * 6 + 3] = o[0];
        dims[k * 6 + 4] = o[1];
        dims[k * 6 + 5] = o[2];
        cur[0] = o[0];
        cur[1] = o[1];
        cur[2] = o[2];
    }
    const int hasClassify = layers[nl - 1].kind == ORC_CLASSIFY;
    const int finalC = hasClassify ? dims[(nl - 1) * 6 + 0] : dims[(nl - 1) * 6 + 3];
    if (finalC != numClasses) return ORC_E_SPEC;
    return ORC_OK;
}

/* network.cpp:207-235 (weights are installed by orc_net_set_weights) */
int orc_net_create(int inC, int inH, int inW, int numClasses, const orc_layer* layers, int nl,
                   orc_net** out) {
    *out = NULL;
    if (nl < 1) return ORC_E_SPEC;
    orc_layer* ls = (orc_layer*)malloc(sizeof(orc_layer) * (size_t)nl);
    int* dims = (int*)malloc(sizeof(int) * 6 * (size_t)nl);
    memcpy(ls, layers, sizeof(orc_layer) * (size_t)nl);
    int rc = orc_chain_dims(inC, inH, inW, numClasses, ls, nl, dims);
    if (rc) {
        free(ls);
        free(dims);
        return rc;
    }
    orc_net* net = (orc_net*)calloc(1, sizeof(orc_net));
    net->inC = inC;
    net->inH = inH;
    net->inW = inW;
    net->numClasses = numClasses;
    net->nl = nl;
    net->L = (orc_layer_rt*)calloc((size_t)nl, sizeof(orc_layer_rt));
    for (int k = 0; k < nl; ++k) {
        orc_layer_rt* L = &net->L[k];
        L->spec = ls[k];
        memcpy(L->in, dims + k * 6, sizeof(int) * 3);
        memcpy(L->out, dims + k * 6 + 3, sizeof(int) * 3);
        if (L->spec.kind == ORC_CBCONV || L->spec.kind == ORC_CONV) {
            const int64_t cols = (int64_t)L->spec.geom.inChannels * L->spec.geom.kernelH *
                                 L->spec.geom.kernelW;
            L->K = (float*)calloc((size_t)(L->spec.geom.outChannels * cols), sizeof(float));
            L->bias = (float*)calloc((size_t)L->spec.geom.outChannels, sizeof(float));
        }
        if (L->spec.kind == ORC_CBCONV) {
            L->prevInput = (float*)malloc(sizeof(float) * (size_t)dims_count(L->in));
            L->prevOutput = (float*)malloc(sizeof(float) * (size_t)dims_count(L->out));
            L->detected = (uint8_t*)malloc((size_t)L->in[1] * L->in[2]);
            L->updated = (int32_t*)malloc(sizeof(int32_t) * (size_t)L->out[1] * L->out[2]);
        }
        L->act = (float*)malloc(sizeof(float) * (size_t)dims_count(L->out));
    }
    free(ls);
    free(dims);
    *out = net;
    return ORC_OK;
}

int orc_net_set_weights(orc_net* net, int layer, const float* K, const float* bias) {
    if (layer < 0 || layer >= net->nl) return ORC_E_SPEC;
    orc_layer_rt* L = &net->L[layer];
    if (!L->K) return ORC_E_SPEC;
    const int64_t cols = (int64_t)L->spec.geom.inChannels * L->spec.geom.kernelH *
                         L->spec.geom.kernelW;
    memcpy(L->K, K, sizeof(float) * (size_t)(L->spec.geom.outChannels * cols));
    memcpy(L->bias, bias, sizeof(float) * (size_t)L->spec.geom.outChannels);
    return ORC_OK;
}

/* network.cpp:197-205 */
int orc_net_set_thresholds(orc_net* net, const float* taus, int n) {
    int cb = 0;
    for (int k = 0; k < net->nl; ++k) cb += net->L[k].spec.kind == ORC_CBCONV;
    if (n != cb) return ORC_E_SPEC;
    for (int k = 0; k < n; ++k)
        if (taus[k] < 0.0f) return ORC_E_SPEC;
    int j = 0;
    for (int k = 0; k < net->nl; ++k)
        if (net->L[k].spec.kind == ORC_CBCONV) net->L[k].spec.threshold = taus[j++];
    return ORC_OK;
}

/* network.cpp:317-320 */
void orc_net_reset(orc_net* net) {
    for (int k = 0; k < net->nl; ++k) net->L[k].hasHistory = 0;
}

/* Full-frame conv via im2col + gemm + update_output (network.cpp:241-248) */
static int conv_layer_full(orc_layer_rt* L, const float* in, int fuseRelu, float* out) {
    const orc_geom* g = &L->spec.geom;
    const int rows = g->outChannels, cols = g->inChannels * g->kernelH * g->kernelW;
    const int64_t n = (int64_t)L->out[1] * L->out[2];
    float* X = (float*)malloc(sizeof(float) * (size_t)(cols * n));
    float* Y = (float*)malloc(sizeof(float) * (size_t)(rows * n));
    int rc = orc_im2col_full(in, L->in[0], L->in[1], L->in[2], g, X);
    if (!rc) {
        orc_gemm(L->K, L->bias, rows, cols, X, n, Y);
        for (int o = 0; o < rows; ++o)
            for (int64_t j = 0; j < n; ++j) {
                const float v = Y[o * n + j];
                out[o * n + j] = fuseRelu ? relu1(v) : v;
            }
    }
    free(X);
    free(Y);
    return rc;
}

/* cbconv_forward, core/src/cbconv.cpp:157-228 */
static int cbconv_forward(orc_layer_rt* L, const float* in, float* out, orc_stats* st) {
    const orc_geom* g = &L->spec.geom;
    const int H = L->in[1], W = L->in[2], Ho = L->out[1], Wo = L->out[2];
    const int rows = g->outChannels, cols = g->inChannels * g->kernelH * g->kernelW;
    const int64_t outPix = (int64_t)Ho * Wo;
    int64_t n;
    if (!L->hasHistory) {
        /* first frame: full evaluation (:170-192) */
        n = outPix;
        for (int64_t k = 0; k < n; ++k) L->updated[k] = (int32_t)k;
        memset(out, 0, sizeof(float) * (size_t)(rows * outPix));
        st->changedInputPixels = (int64_t)H * W;
        L->detectedValid = 0;
    } else {
        /* steady state (:193-223) */
        uint8_t* dil = (uint8_t*)malloc((size_t)outPix);
        st->changedInputPixels =
            orc_detect_changes(in, L->prevInput, L->in[0], H, W, L->spec.threshold, L->detected);
        L->detectedValid = 1;
        orc_dilate_changes(L->detected, H, W, g, dil);
        n = orc_extract_indexes(dil, outPix, L->updated);
        free(dil);
        memcpy(out, L->prevOutput, sizeof(float) * (size_t)(rows * outPix));
    }
    float* X = (float*)malloc(sizeof(float) * (size_t)(cols * (n > 0 ? n : 1)));
    float* Y = (float*)malloc(sizeof(float) * (size_t)(rows * (n > 0 ? n : 1)));
    int rc = orc_gen_x_reduced(in, L->in[0], H, W, L->updated, n, g, X);
    if (!rc) {
        orc_gemm(L->K, L->bias, rows, cols, X, n, Y);
        rc = orc_update_output(out, rows, Ho, Wo, Y, L->updated, n, L->spec.fuseRelu);
    }
    free(X);
    free(Y);
    L->nUpdated = n;
    st->changedOutputPixels = n;
    st->gemmMacs = (uint64_t)rows * (uint64_t)cols * (uint64_t)n;
    /* state copies (:225-226) */
    memcpy(L->prevInput, in, sizeof(float) * (size_t)dims_count(L->in));
    memcpy(L->prevOutput, out, sizeof(float) * (size_t)(rows * outPix));
    L->hasHistory = 1;
    return rc;
}

/* forward_frame, core/src/network.cpp:252-315 */
int orc_forward_frame(orc_net* net, const float* frame, int engine, uint16_t* labels,
                      orc_stats* stats, uint64_t* macsTotal) {
    const float* cur = frame;
    int curDims[3] = {net->inC, net->inH, net->inW};
    int classified = 0;
    memset(stats, 0, sizeof(orc_stats) * (size_t)net->nl);
    for (int k = 0; k < net->nl; ++k) {
        orc_layer_rt* L = &net->L[k];
        orc_stats* st = &stats[k];
        int rc = ORC_OK;
        switch (L->spec.kind) {
            case ORC_CBCONV:
                if (engine == ORC_ENGINE_CBINFER) {
                    rc = cbconv_forward(L, cur, L->act, st);
                } else {
                    rc = conv_layer_full(L, cur, L->spec.fuseRelu, L->act);
                    st->changedOutputPixels = (int64_t)L->out[1] * L->out[2];
                    st->gemmMacs = (uint64_t)L->spec.geom.outChannels * L->spec.geom.inChannels *
                                   L->spec.geom.kernelH * L->spec.geom.kernelW * L->out[1] *
                                   L->out[2];
                }
                break;
            case ORC_CONV:
                rc = conv_layer_full(L, cur, 0, L->act);
                st->changedOutputPixels = (int64_t)L->out[1] * L->out[2];
                st->gemmMacs = (uint64_t)L->spec.geom.outChannels * L->spec.geom.inChannels *
                               L->spec.geom.kernelH * L->spec.geom.kernelW * L->out[1] * L->out[2];
                break;
            case ORC_RELU:
                orc_relu(cur, dims_count(L->out), L->act);
                break;
            case ORC_MAXPOOL:
                rc = orc_maxpool(cur, L->in[0], L->in[1], L->in[2], L->spec.window,
                                 L->spec.stride, L->act);
                break;
            case ORC_CLASSIFY:
                net->finalAct = (float*)cur;
                memcpy(net->finalDims, curDims, sizeof(curDims));
                orc_argmax_classify(cur, curDims[0], curDims[1], curDims[2], labels);
                classified = 1;
                break;
        }
        if (rc) return rc;
        if (L->spec.kind != ORC_CLASSIFY) {
            cur = L->act;
            memcpy(curDims, L->out, sizeof(curDims));
        }
    }
    if (!classified) {
        net->finalAct = (float*)cur;
        memcpy(net->finalDims, curDims, sizeof(curDims));
        orc_argmax_classify(cur, curDims[0], curDims[1], curDims[2], labels);
    }
    uint64_t total = 0;
    for (int k = 0; k < net->nl; ++k) total += stats[k].gemmMacs;
    *macsTotal = total;
    return ORC_OK;
}

int orc_net_layer_output(const orc_net* net, int layer, const float** data, int dims[3]) {
    if (layer < 0 || layer >= net->nl) return ORC_E_SPEC;
    *data = net->L[layer].act;
    memcpy(dims, net->L[layer].out, sizeof(int) * 3);
    return ORC_OK;
}

int orc_net_final_activation(const orc_net* net, const float** data, int dims[3]) {
    *data = net->finalAct;
    memcpy(dims, net->finalDims, sizeof(int) * 3);
    return net->finalAct ? ORC_OK : ORC_E_SPEC;
}

int orc_net_trace(const orc_net* net, int cbOrdinal, const uint8_t** detected, int dims[2],
                  const int32_t** updated, int64_t* n) {
    int j = 0;
    for (int k = 0; k < net->nl; ++k) {
        const orc_layer_rt* L = &net->L[k];
        if (L->spec.kind != ORC_CBCONV) continue;
        if (j++ != cbOrdinal) continue;
        *detected = L->detectedValid ? L->detected : NULL;
        dims[0] = L->in[1];
        dims[1] = L->in[2];
        *updated = L->updated;
        *n = L->nUpdated;
        return ORC_OK;
    }
    return ORC_E_SPEC;
}

void orc_net_free(orc_net* net) {
    if (!net) return;
    for (int k = 0; k < net->nl; ++k) {
        orc_layer_rt* L = &net->L[k];
        free(L->K);
        free(L->bias);
        free(L->prevInput);
        free(L->prevOutput);
        free(L->detected);
        free(L->updated);
        free(L->act);
    }
    free(net->L);
    free(net);
}

/* ------------------------------------------------------------------ */
/* timing warm-up (see header)                                         */

typedef struct {
    orc_layer_rt* L;
    const float* in;
    float* out;
    int64_t p0, p1;
    int relu;
} warm_job;

static void* warm_worker(void* arg) {
    warm_job* j = (warm_job*)arg;
    const orc_geom* g = &j->L->spec.geom;
    const int H = j->L->in[1], W = j->L->in[2], Wo = j->L->out[2];
    const int rows = g->outChannels, cols = g->inChannels * g->kernelH * g->kernelW;
    const int64_t plane = (int64_t)j->L->out[1] * Wo;
    float* col = (float*)malloc(sizeof(float) * (size_t)cols);
    for (int64_t p = j->p0; p < j->p1; ++p) {
        orc_fill_patch_column(j->in, j->L->in[0], H, W, g, (int)(p / Wo), (int)(p % Wo), col);
        for (int o = 0; o < rows; ++o) {
            const float* k = j->L->K + (int64_t)o * cols;
            float acc = j->L->bias[o];
            for (int r = 0; r < cols; ++r) acc += k[r] * col[r];
            j->out[o * plane + p] = j->relu ? relu1(acc) : acc;
        }
    }
    free(col);
    return NULL;
}

int orc_net_warm(orc_net* net, const float* frame, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    const float* cur = frame;
    for (int k = 0; k < net->nl; ++k) {
        orc_layer_rt* L = &net->L[k];
        switch (L->spec.kind) {
            case ORC_CBCONV:
            case ORC_CONV: {
                const int64_t pixels = (int64_t)L->out[1] * L->out[2];
                const int64_t chunk = (pixels + nthreads - 1) / nthreads;
                pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
                warm_job* jobs = (warm_job*)malloc(sizeof(warm_job) * (size_t)nthreads);
                int started = 0;
                for (int t = 0; t < nthreads; ++t) {
                    const int64_t a = t * chunk, b = a + chunk < pixels ? a + chunk : pixels;
                    if (a >= b) break;
                    jobs[t] = (warm_job){L, cur, L->act, a, b, L->spec.kind == ORC_CBCONV && L->spec.fuseRelu};
                    pthread_create(&th[t], NULL, warm_worker, &jobs[t]);
                    ++started;
                }
                for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
                free(th);
                free(jobs);
                if (L->spec.kind == ORC_CBCONV) {
                    memcpy(L->prevInput, cur, sizeof(float) * (size_t)dims_count(L->in));
                    memcpy(L->prevOutput, L->act, sizeof(float) * (size_t)dims_count(L->out));
                    L->hasHistory = 1;
                }
                break;
            }
            case ORC_RELU:
                orc_relu(cur, dims_count(L->out), L->act);
                break;
            case ORC_MAXPOOL:
                orc_maxpool(cur, L->in[0], L->in[1], L->in[2], L->spec.window, L->spec.stride, L->act);
                break;
            default:
                break;
        }
        if (L->spec.kind != ORC_CLASSIFY) cur = L->act;
    }
    return ORC_OK;
}

/* Copies the change-based state of src into dst (same spec). */
int orc_net_copy_state(orc_net* dst, const orc_net* src) {
    if (dst->nl != src->nl) return ORC_E_SPEC;
    for (int k = 0; k < src->nl; ++k) {
        const orc_layer_rt* a = &src->L[k];
        orc_layer_rt* b = &dst->L[k];
        b->hasHistory = a->hasHistory;
        if (a->prevInput) memcpy(b->prevInput, a->prevInput, sizeof(float) * (size_t)dims_count(a->in));
        if (a->prevOutput) memcpy(b->prevOutput, a->prevOutput, sizeof(float) * (size_t)dims_count(a->out));
    }
    return ORC_OK;
}
