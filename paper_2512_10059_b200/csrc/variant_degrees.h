// variant_degrees.h -- compile-time degrees of a (K, variant) kernel
// instantiation (boys_launch.h: Variant), for the instantiation units.
#pragma once

#include "boys_launch.h"
#include "embedded_tables.inc"

namespace boysfn_dev {

template <int K, int V>
struct VariantDegrees {
  static constexpr int NA = V == kVariantEmbedded ? kEmbDegA[K][0] : V == kVariantCompact ? kCompactNA : kMaxCoef - 1;
  static constexpr int MA = V == kVariantEmbedded ? kEmbDegA[K][1] : V == kVariantCompact ? kCompactMA : kMaxCoef - 1;
  static constexpr int NB = V == kVariantEmbedded ? kEmbDegB[0] : V == kVariantCompact ? kCompactNB : kMaxCoef - 1;
  static constexpr int MB = V == kVariantEmbedded ? kEmbDegB[1] : V == kVariantCompact ? kCompactMB : kMaxCoef - 1;
};

}  // namespace boysfn_dev
