// boys_launch.h -- host-side internals shared by the kernel instantiation units
// and the C ABI (capi.cu).  Not installed; the public surface is
// include/boysfn_b200.h.
#pragma once

#include "boys_device.cuh"

namespace boysfn_dev {

// Degree variants of the kernel for one order k.
//   kVariantEmbedded: the exact (n, m) of the paper's tables for that k
//                     (r_A[k] per Appendix C, r_B = (5, 6)); used whenever a
//                     table set has that degree profile.
//   kVariantPadded:   every rational padded to kMaxCoef-1 (any custom set).
//   kVariantCompact:  r_A padded to (9, 13) and r_B to (6, 7): every degree of
//                     Appendix C and of this repo's generator output fits, so
//                     a generated or hand-edited set does not pay for 23/23
//                     Horner (the padded kernels ran k = 32 at 5.2 TB/s).
enum Variant : int { kVariantEmbedded = 0, kVariantPadded = 1, kVariantCompact = 2 };
constexpr int kCompactNA = 9, kCompactMA = 13, kCompactNB = 6, kCompactMB = 7;

constexpr int kKernelKmax = 32;

// x per block-TMA tile (= threads per block) of the plain SoA and AoS stores:
// 256 x gives 2 KB SoA row segments and 2x longer AoS spans; 0.2-0.4% (SoA)
// and 0.4-1.2% (AoS) over 128 x at k >= 10 (profiles/r01_tma_tile256.txt).
#ifndef BOYSFN_SOA_TMA_BX
#define BOYSFN_SOA_TMA_BX 256
#endif
constexpr int kSoATmaTileX = BOYSFN_SOA_TMA_BX;
// The bulk store with 512-x tiles (4-KB row segments) for SoA strides whose
// rows do not start on a 1-KB boundary, at k = 10..26: a tile's row segment
// then touches 5 KB-units for 4 KB written instead of 3 for 2, and the rate
// at such strides rises 2-5% (k = 16, ld = n + 1: 2.40 -> 2.31 ms; k = 24:
// 3.53 -> 3.37 ms).  Above k = 26 a 512-x stage leaves one resident block;
// k = 25, 26 are compiled for two (block_tma_min_blocks;
// profiles/r02_soa_wide_tiles.txt).
#ifndef BOYSFN_SOA_WIDE_BX  // A/B builds
#define BOYSFN_SOA_WIDE_BX 512
#define BOYSFN_SOA_WIDE_KMIN 10
#define BOYSFN_SOA_WIDE_KMAX 26
#endif
constexpr int kSoAWideTileX = BOYSFN_SOA_WIDE_BX;
constexpr int kSoAWideKmin = BOYSFN_SOA_WIDE_KMIN, kSoAWideKmax = BOYSFN_SOA_WIDE_KMAX;
// Above that, rows off a 32-B sector boundary (the plain bulk store's case)
// take 384-x tiles (3-KB segments; a 384-thread block with its stage fits
// twice per SM up to k = 32): 2-3% at k = 27..32 (k = 32, ld = n + 1: 4.66 ->
// 4.51 ms).  Sector-aligned rows keep the 256-x tensor store there, which the
// 384-x tiles did not beat (profiles/r02_soa_wide_tiles.txt).
constexpr int kSoAWide3TileX = 384;
constexpr int kAoSTmaTileX = 256;
#ifndef BOYSFN_BIN_TMA_BX
#define BOYSFN_BIN_TMA_BX 128
#endif
constexpr int kBinTmaTileX = BOYSFN_BIN_TMA_BX;  // region-sorted block-TMA stores (SoA and AoS)

// Tile width (= threads per block) of a block-TMA store kind; kBlockX otherwise.
constexpr int block_tma_tile_x(int store) {
  return store == kStoreSoABlockTma      ? kSoATmaTileX
         : store == kStoreSoABlockBulk   ? kSoATmaTileX
         : store == kStoreSoABlockBulkW  ? kSoAWideTileX
         : store == kStoreSoABlockBulkW3 ? kSoAWide3TileX
         : store == kStoreAoSBlockTma    ? kAoSTmaTileX
         : store == kStoreSoABlockTmaBin ? kBinTmaTileX
         : store == kStoreAoSBlockTmaBin ? kBinTmaTileX
                                         : kBlockX;
}

// Kernel entry points, one translation unit per store path.
const void* kernel_soa(int k, int variant);
const void* kernel_aos_xpose(int k, int variant);
const void* kernel_soa_block(int k, int variant);
const void* kernel_soa_binned(int k, int variant);
const void* kernel_aos_binned(int k, int variant);
const void* kernel_soa_block_tma(int k, int variant);
const void* kernel_aos_block_tma(int k, int variant);
const void* kernel_soa_block_tma_bin(int k, int variant);
const void* kernel_soa_block_bulk_w(int k, int variant);  // k <= kSoAWideKmax
const void* kernel_soa_block_bulk_w3(int k, int variant);
const void* kernel_soa_block_bulk(int k, int variant);
const void* kernel_aos_block_tma_bin(int k, int variant);
const void* kernel_region(int k, int variant);
const void* kernel_generic();
const void* kernel_generic_tma(int k, bool soa);  // nullptr above 64
const void* kernel_generic_stage(bool soa);

// Exact degrees of the embedded kernels (from embedded_tables.inc).
void embedded_degrees(int k, int* na, int* ma, int* nb, int* mb);

}  // namespace boysfn_dev
