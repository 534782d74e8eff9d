// pass_m4.cu -- the loss+gradient scheduler and its kernels for HR order m = 4 (Eq. 2).
#include "pass_impl.cuh"

HRKAN_DEFINE_DISPATCH(4)
