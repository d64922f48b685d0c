// kernels_aos_block_tma_swz.cu -- the swizzled-stage AoS block-TMA kernels
// (kStoreAoSBlockTmaSwz), which exist for k + 1 in {16, 32} only (k = 15, 31),
// in the three degree variants.  Other orders get nullptr.
#include "variant_degrees.h"

namespace boysfn_dev {
namespace {

template <int K, int V>
const void* entry() {
  using D = VariantDegrees<K, V>;
  return reinterpret_cast<const void*>(&boys_eval_block_tma_kernel<K, D::NA, D::MA, D::NB, D::MB, kStoreAoSBlockTmaSwz, kSwzTmaTileX>);
}

template <int K>
const void* pick(int variant) {
  switch (variant) {
    case kVariantEmbedded: return entry<K, kVariantEmbedded>();
    case kVariantPadded: return entry<K, kVariantPadded>();
    default: return entry<K, kVariantCompact>();
  }
}

}  // namespace

const void* kernel_aos_block_tma_swz(int k, int variant) {
  if (variant < 0 || variant > 2) return nullptr;
  if (k == 15) return pick<15>(variant);
  if (k == 31) return pick<31>(variant);
  return nullptr;
}

}  // namespace boysfn_dev
