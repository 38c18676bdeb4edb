// Compile-time encoders (K1, Horner back end) for the common schemes.
// RS(n,k) coefficients are the reference's Cauchy matrix (coding.hpp:108-114).
#include "gs_special.cuh"

namespace gsb {

int special_encoders(SpecialEntry* out) {
  int c = 0;
  add_encoder<kXor, 2, 1>(out, c);
  add_encoder<kXor, 3, 1>(out, c);
  add_encoder<kXor, 4, 1>(out, c);
  add_encoder<kXor, 5, 1>(out, c);
  add_encoder<kXor, 6, 1>(out, c);
  add_encoder<kXor, 7, 1>(out, c);
  add_encoder<kXor, 8, 1>(out, c);
  add_encoder<kReedSolomon, 2, 1>(out, c);
  add_encoder<kReedSolomon, 2, 2>(out, c);
  add_encoder<kReedSolomon, 3, 1>(out, c);
  add_encoder<kReedSolomon, 3, 2>(out, c);
  add_encoder<kReedSolomon, 4, 1>(out, c);
  add_encoder<kReedSolomon, 4, 2>(out, c);
  add_encoder<kReedSolomon, 4, 3>(out, c);
  add_encoder<kReedSolomon, 4, 4>(out, c);
  add_encoder<kReedSolomon, 5, 2>(out, c);
  add_encoder<kReedSolomon, 6, 1>(out, c);
  add_encoder<kReedSolomon, 6, 2>(out, c);
  add_encoder<kReedSolomon, 6, 3>(out, c);
  add_encoder<kReedSolomon, 8, 1>(out, c);
  add_encoder<kReedSolomon, 8, 2>(out, c);
  add_encoder<kReedSolomon, 8, 3>(out, c);
  add_encoder<kReedSolomon, 8, 4>(out, c);
  add_encoder<kReedSolomon, 10, 2>(out, c);
  add_encoder<kReedSolomon, 10, 4>(out, c);
  add_encoder<kReedSolomon, 12, 3>(out, c);
  add_encoder<kReedSolomon, 12, 4>(out, c);
  add_encoder<kReedSolomon, 16, 4>(out, c);
  return c;
}

}  // namespace gsb
