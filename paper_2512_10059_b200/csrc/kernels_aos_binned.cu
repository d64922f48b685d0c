// kernels_aos_binned.cu -- per-warp region-binned groups, AoS (kStoreAoSBinned), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_binned_kernel<K, NA, MA, NB, MB, kStoreAoSBinned>
#define BOYSFN_GETTER kernel_aos_binned
#include "kernel_table.inc"
