// kernels_soa.cu -- per-warp tiles, SoA rows (kStoreSoA), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_kernel<K, NA, MA, NB, MB, kStoreSoA>
#define BOYSFN_GETTER kernel_soa
#include "kernel_table.inc"
