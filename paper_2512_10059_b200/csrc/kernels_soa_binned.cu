// kernels_soa_binned.cu -- per-warp region-binned groups, SoA (kStoreSoABinned), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_binned_kernel<K, NA, MA, NB, MB, kStoreSoABinned>
#define BOYSFN_GETTER kernel_soa_binned
#include "kernel_table.inc"
