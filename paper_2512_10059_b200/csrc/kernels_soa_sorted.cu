// kernels_soa_sorted.cu -- per-warp region-sorted groups with TMA in and out, SoA (kStoreSoASorted), k = 0..kSortedKmax.
#define BOYSFN_KERNEL boys_eval_sorted_kernel<K, NA, MA, NB, MB, kStoreSoASorted>
#define BOYSFN_GETTER kernel_soa_sorted
#define BOYSFN_TABLE_KMAX kSortedKmax
#include "kernel_table.inc"
