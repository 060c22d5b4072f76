// Sum-factorised kernels for quadrilaterals / hexahedra (filled in below).
#pragma once
#include "common.cuh"
#define FE_TENSOR_VARIANTS
