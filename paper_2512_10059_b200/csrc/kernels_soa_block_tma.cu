// kernels_soa_block_tma.cu -- instantiates boys_eval_block_tma_kernel for the kStoreSoABlockTma output
// path, k = 0..32, embedded-degree and padded-degree variants (66 kernels).
// Split per store path so nvcc compiles the three units in parallel.
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
  return reinterpret_cast<const void*>(&boys_eval_block_tma_kernel<K, NA, MA, NB, MB, kStoreSoABlockTma>);
}

template <size_t... Ks>
const void* lookup(int k, int v, std::index_sequence<Ks...>) {
  static const void* const table[2][sizeof...(Ks)] = {
      {entry<static_cast<int>(Ks), kVariantEmbedded>()...},
      {entry<static_cast<int>(Ks), kVariantPadded>()...}};
  return table[v][k];
}

}  // namespace

const void* kernel_soa_block_tma(int k, int variant) {
  if (k < 0 || k > kKernelKmax || variant < 0 || variant > 1) return nullptr;
  return lookup(k, variant, std::make_index_sequence<kKernelKmax + 1>{});
}

}  // namespace boysfn_dev
