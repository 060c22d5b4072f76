// FP64 tensor-core (DMMA) element-tensor kernels for high-degree simplices.
#pragma once
#include "common.cuh"
#define FE_DMMA_VARIANTS
