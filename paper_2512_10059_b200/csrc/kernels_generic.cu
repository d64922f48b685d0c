// kernels_generic.cu -- the run-time-k, run-time-degree kernels
// (boys_eval_generic_tma_kernel, and boys_eval_generic_kernel where no tensor
// map applies or a region is forced; boys_device.cuh) for orders above the
// templated kernels' 32 and for the equivalence tests.
#include "boys_launch.h"

namespace boysfn_dev {

const void* kernel_generic() { return reinterpret_cast<const void*>(&boys_eval_generic_kernel<>); }
const void* kernel_generic_tma(bool soa) {
  return soa ? reinterpret_cast<const void*>(&boys_eval_generic_tma_kernel<true>)
             : reinterpret_cast<const void*>(&boys_eval_generic_tma_kernel<false>);
}

}  // namespace boysfn_dev
