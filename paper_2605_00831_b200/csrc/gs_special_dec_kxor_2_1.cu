// Compile-time decoders (K2, Horner back end) for every canonical erasure
// pattern of Xor(2,1); coefficients = coding.hpp:535-566 folded by the compiler.
#include "gs_special.cuh"

namespace gsb {

int special_decoders_kxor_2_1(SpecialEntry* out) {
  int c = 0;
  add_decoders<kXor, 2, 1>(out, c);
  return c;
}

}  // namespace gsb
