// kernels_aos_sorted.cu -- per-warp region-sorted groups with TMA in and out, AoS (kStoreAoSSorted), k = 0..kSortedKmax.
#define BOYSFN_KERNEL boys_eval_sorted_kernel<K, NA, MA, NB, MB, kStoreAoSSorted>
#define BOYSFN_GETTER kernel_aos_sorted
#define BOYSFN_TABLE_KMAX kSortedKmax
#include "kernel_table.inc"
