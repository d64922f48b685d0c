// kernels_aos_block_tma_bin.cu -- region-sorted block tiles, AoS by TMA 1D bulk stores (kStoreAoSBlockTmaBin), k = 0..32, embedded-degree and padded-degree variants.
#define BOYSFN_KERNEL boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreAoSBlockTmaBin, kBinTmaTileX>
#define BOYSFN_GETTER kernel_aos_block_tma_bin
#include "kernel_table.inc"
