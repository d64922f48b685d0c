// kernels_aos_xpose.cu -- per-warp tiles, AoS via a padded smem transpose (kStoreAoSXpose), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_kernel<K, NA, MA, NB, MB, kStoreAoSXpose>
#define BOYSFN_GETTER kernel_aos_xpose
#include "kernel_table.inc"
