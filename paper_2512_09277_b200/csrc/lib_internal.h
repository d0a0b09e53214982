// lib_internal.h -- symbols shared between the translation units of
// libmetro_b200.so (hidden: the library is built with -fvisibility=hidden).
#pragma once
#include <cuda_runtime.h>

namespace metro {
// records e as the thread's last CUDA error (metro_last_cuda_error) and
// returns METRO_ECUDA
int cuda_fail(cudaError_t e);
}  // namespace metro
