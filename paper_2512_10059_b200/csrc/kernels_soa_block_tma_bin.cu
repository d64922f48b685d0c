// kernels_soa_block_tma_bin.cu -- region-sorted block tiles, SoA by TMA 2D tensor stores (kStoreSoABlockTmaBin), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockTmaBin, kBinTmaTileX>
#define BOYSFN_GETTER kernel_soa_block_tma_bin
#include "kernel_table.inc"
