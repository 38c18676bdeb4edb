// Compile-time decoders (K2, Horner back end) for every canonical erasure
// pattern of ReedSolomon(6,2); coefficients = coding.hpp:535-566 folded by the compiler.
#include "gs_special.cuh"

namespace gsb {

int special_decoders_kreedsolomon_6_2(SpecialEntry* out) {
  int c = 0;
  add_decoders<kReedSolomon, 6, 2>(out, c);
  return c;
}

}  // namespace gsb
