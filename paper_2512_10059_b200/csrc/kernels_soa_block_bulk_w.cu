// kernels_soa_block_bulk_w.cu -- the per-row bulk-copy SoA store with 512-x tiles (kStoreSoABlockBulkW), k = 0..kSoAWideKmax (used at k >= kSoAWideKmin for rows off 1-KB boundaries).
#define BOYSFN_TABLE_KMAX BOYSFN_SOA_WIDE_KMAX
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockBulkW, kSoAWideTileX>
#define BOYSFN_GETTER kernel_soa_block_bulk_w
#include "kernel_table.inc"
