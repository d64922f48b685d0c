// kernels_soa_block_bulk.cu -- block tiles, SoA rows by per-row 1D bulk copies (kStoreSoABlockBulk): any ld, any 8-B alignment, k = 0..32.
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockBulk, kSoATmaTileX>
#define BOYSFN_GETTER kernel_soa_block_bulk
#include "kernel_table.inc"
