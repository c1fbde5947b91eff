// K-PRED instantiation: uint16_t rows, exact mode (kernels in predict_kernels.cuh).
#include "predict_kernels.cuh"

namespace gnb {
template cudaError_t launch_typed<uint16_t, false>(const PredictMaps*, const PredictParams&, int,
                                          cudaStream_t);
}  // namespace gnb
