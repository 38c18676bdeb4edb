// Compile-time decoders (K2, Horner back end) for the canonical erasure
// patterns losing 2 data shard(s) of ReedSolomon(8,2); coefficients = coding.hpp:535-566 folded by the compiler.
#include "gs_special.cuh"

namespace gsb {

int special_decoders_kreedsolomon_8_2_e2(SpecialEntry* out) {
  int c = 0;
  add_decoders<kReedSolomon, 8, 2, 2>(out, c);
  return c;
}

}  // namespace gsb
