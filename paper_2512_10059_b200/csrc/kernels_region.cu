// kernels_region.cu -- instantiates boys_region_kernel, the forced-region seam
// of boys_batch_region (eval.cpp:59-81), k = 0..32, embedded-degree and
// padded-degree variants.
#include <utility>

#include "boys_launch.h"
#include "embedded_tables.inc"

namespace boysfn_dev {
namespace {

template <int K, int V>
const void* entry() {
  constexpr int NA = V == kVariantEmbedded ? kEmbDegA[K][0] : kMaxCoef - 1;
  constexpr int MA = V == kVariantEmbedded ? kEmbDegA[K][1] : kMaxCoef - 1;
  constexpr int NB = V == kVariantEmbedded ? kEmbDegB[0] : kMaxCoef - 1;
  constexpr int MB = V == kVariantEmbedded ? kEmbDegB[1] : kMaxCoef - 1;
  return reinterpret_cast<const void*>(&boys_region_kernel<K, NA, MA, NB, MB>);
}

template <size_t... Ks>
const void* lookup(int k, int v, std::index_sequence<Ks...>) {
  static const void* const table[2][sizeof...(Ks)] = {
      {entry<static_cast<int>(Ks), kVariantEmbedded>()...},
      {entry<static_cast<int>(Ks), kVariantPadded>()...}};
  return table[v][k];
}

}  // namespace

const void* kernel_region(int k, int variant) {
  if (k < 0 || k > kKernelKmax || variant < 0 || variant > 1) return nullptr;
  return lookup(k, variant, std::make_index_sequence<kKernelKmax + 1>{});
}

}  // namespace boysfn_dev
