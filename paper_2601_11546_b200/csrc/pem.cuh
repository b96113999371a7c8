// pem.cuh -- PEM model constants and the correctly-rounded linear cost term.
#pragma once
#include <stdint.h>

#include "block.cuh"

namespace rsd {

struct PemModel {
  double ap, bp, ad, bd;
  long long cap, mns, mnbt;
};

__device__ __forceinline__ double lin(double a, double x, double b) {
  return __dadd_rn(__dmul_rn(a, x), b);
}

}  // namespace rsd
