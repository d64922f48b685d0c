// kernels_soa_block_bulk_w3.cu -- the per-row bulk-copy SoA store with 384-x tiles (kStoreSoABlockBulkW3), k = 0..32 (used above kSoAWideKmax for rows off a 32-B sector boundary).
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockBulkW3, kSoAWide3TileX>
#define BOYSFN_GETTER kernel_soa_block_bulk_w3
#include "kernel_table.inc"
