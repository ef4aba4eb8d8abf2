// conv_tc.cu -- placeholder until the tcgen05 kernel lands.
#include "conv_tc.hpp"
#include "engine.hpp"

namespace cbx {

struct TcLayer {
    cbx_geom g;
};
void TcLayerDeleter::operator()(TcLayer* p) const { delete p; }
bool tc_supported(const cbx_geom&) { return false; }
std::unique_ptr<TcLayer, TcLayerDeleter> make_tc_layer(const cbx_geom& g) {
    return std::unique_ptr<TcLayer, TcLayerDeleter>(new TcLayer{g});
}
void tc_load_weights(TcLayer&, const float*, cudaStream_t) {}
void launch_conv_tc(const TcLayer&, TensorView, TensorView, const float*, const int32_t*, const int*,
                    int64_t, bool, MaskView, float, unsigned long long*, int, int, cudaStream_t) {
    throw Error(CBX_E_CUDA, "tcgen05 path not built");
}

}  // namespace cbx
