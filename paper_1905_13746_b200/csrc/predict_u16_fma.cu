// K-PRED instantiation: uint16_t rows, fma mode (kernels in predict_kernels.cuh).
#include "predict_kernels.cuh"

namespace gnb {
template cudaError_t launch_typed<uint16_t, true>(const PredictMaps*, const PredictParams&, int,
                                          cudaStream_t);
}  // namespace gnb
