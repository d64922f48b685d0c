// kernels_generic.cu -- the run-time-k, run-time-degree kernels
// (boys_eval_generic_tma_kernel, and boys_eval_generic_kernel where no tensor
// map applies or a region is forced; boys_device.cuh) for orders above the
// templated kernels' 32 and for the equivalence tests.
#include "boys_launch.h"

namespace boysfn_dev {

const void* kernel_generic() { return reinterpret_cast<const void*>(&boys_eval_generic_kernel<>); }
// the staged form (KM = 0)
const void* kernel_generic_stage(bool soa) {
  return soa ? reinterpret_cast<const void*>(&boys_eval_generic_tma_kernel<0, true>)
             : reinterpret_cast<const void*>(&boys_eval_generic_tma_kernel<0, false>);
}
// k <= 32, 36, 40, 48, 56, 64: the register array's bound
const void* kernel_generic_tma(int k, bool soa) {
#define BOYSFN_GT(KM)                                                                 \
  if (k <= KM)                                                                        \
    return soa ? reinterpret_cast<const void*>(&boys_eval_generic_tma_kernel<KM, true>) \
               : reinterpret_cast<const void*>(&boys_eval_generic_tma_kernel<KM, false>);
  BOYSFN_GT(32)
  BOYSFN_GT(36)
  BOYSFN_GT(40)
  BOYSFN_GT(48)
  BOYSFN_GT(56)
  BOYSFN_GT(64)
#undef BOYSFN_GT
  return nullptr;
}

}  // namespace boysfn_dev
