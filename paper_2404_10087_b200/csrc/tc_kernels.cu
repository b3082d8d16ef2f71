// Tensor-core (tcgen05) Hogwild sweeps -- placeholder until the sm_100a
// kernels land; tc_supported() == false routes every call to the CUDA-core
// kernels in hog_kernels.cu.
#include "engine.cuh"

namespace ftkcu {

bool tc_supported(const KView&) { return false; }

cudaError_t launch_tc_factor(const KView&, int64_t, int64_t, float, float, int, cudaStream_t) {
  return cudaErrorNotSupported;
}

cudaError_t launch_tc_core(const KView&, int64_t, int64_t, float*, int, float*, size_t,
                           cudaStream_t) {
  return cudaErrorNotSupported;
}

}  // namespace ftkcu
