// kernels_region.cu -- the one-x forced-region kernel of boys_batch_region, k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_region_kernel<K, NA, MA, NB, MB>
#define BOYSFN_GETTER kernel_region
#include "kernel_table.inc"
