// Compile-time decoders (K2, Horner back end) for the canonical erasure
// patterns losing 1 data shard(s) of ReedSolomon(6,2); coefficients = coding.hpp:535-566 folded by the compiler.
#include "gs_special.cuh"

namespace gsb {

int special_decoders_kreedsolomon_6_2_e1(SpecialEntry* out) {
  int c = 0;
  add_decoders<kReedSolomon, 6, 2, 1>(out, c);
  return c;
}

}  // namespace gsb
