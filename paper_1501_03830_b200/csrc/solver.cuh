// Pipeline-level declarations shared by the C ABI.
#pragma once
#include <cuda_runtime.h>
#include "dense.cuh"

namespace bse {

double launch_peak(int which, int blocks, int iters, double* sink, cudaStream_t s);

}  // namespace bse
