// fek_status.h -- shared CUDA error recording for every translation unit of
// libfek.so: the message is kept per host thread and returned by
// fek_last_cuda_error() (include/fek.h).
#pragma once

#include <cuda_runtime.h>

namespace fek {
// records "<what>: <cuda error string>" and returns FEK_ERR_CUDA
int record_cuda_error(cudaError_t e, const char *what);
}  // namespace fek
