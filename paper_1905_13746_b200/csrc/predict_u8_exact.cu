// K-PRED instantiation: uint8_t rows, exact mode (kernels in predict_kernels.cuh).
#include "predict_kernels.cuh"

namespace gnb {
template cudaError_t launch_typed<uint8_t, false>(const PredictMaps*, const PredictParams&, int,
                                          cudaStream_t);
}  // namespace gnb
