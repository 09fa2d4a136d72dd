// tcgen05 GEMM placeholder (replaced by the TMA/TMEM kernel).
#include "dense_kernels.cuh"
#include "sd_common.h"

namespace sd {
bool gemm_sm100_supported(const GemmArgs&) { return false; }
void launch_gemm_sm100(const GemmArgs&, cudaStream_t) { fail(SD_ERR_CONFIG, "tcgen05 GEMM not built"); }
}  // namespace sd
