// Fused multi-stage stencil passes (filled in by later milestones).
#include "fused.cuh"
