// K-PRED instantiation: int32_t rows, exact mode (kernels in predict_kernels.cuh).
#include "predict_kernels.cuh"

namespace gnb {
template cudaError_t launch_typed<int32_t, false>(const PredictMaps*, const PredictParams&, int,
                                          cudaStream_t);
}  // namespace gnb
