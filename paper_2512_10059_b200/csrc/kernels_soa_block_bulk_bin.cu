// kernels_soa_block_bulk_bin.cu -- kStoreSoABlockBulk with the tile's x region-sorted first (kStoreSoABlockBulkBin), k = 0..32.
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockBulkBin, kBinTmaTileX>
#define BOYSFN_GETTER kernel_soa_block_bulk_bin
#include "kernel_table.inc"
