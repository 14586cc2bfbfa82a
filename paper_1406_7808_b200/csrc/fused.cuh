// Fused multi-sweep kernels (see fused.cu).
#pragma once
#include "kernels.cuh"
