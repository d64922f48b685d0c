// kernels_aos_block_tma.cu -- block tiles, AoS by TMA 1D bulk stores (kStoreAoSBlockTma), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreAoSBlockTma, kAoSTmaTileX>
#define BOYSFN_GETTER kernel_aos_block_tma
#include "kernel_table.inc"
