// kernels_generic.cu -- the run-time-k, run-time-degree kernel
// (boys_eval_generic_kernel, boys_device.cuh) for orders above the templated
// kernels' 32 and for the equivalence tests.
#include "boys_launch.h"

namespace boysfn_dev {

const void* kernel_generic() { return reinterpret_cast<const void*>(&boys_eval_generic_kernel<>); }

}  // namespace boysfn_dev
