// fused sm_100a kernels (added in a later step)
#include "kernels.cuh"
