// kernels_soa_block.cu -- block tiles, SoA 1 KB row segments by LSU (kStoreSoABlock), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_block_kernel<K, NA, MA, NB, MB, kStoreSoABlock>
#define BOYSFN_GETTER kernel_soa_block
#include "kernel_table.inc"
