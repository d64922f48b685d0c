// kernels_soa_block_tma.cu -- block tiles, SoA by TMA 2D tensor stores (kStoreSoABlockTma), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockTma, kSoATmaTileX>
#define BOYSFN_GETTER kernel_soa_block_tma
#include "kernel_table.inc"
