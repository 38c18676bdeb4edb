// Redirect shim (see coding.hpp here): the reference's gf256_test.cpp,
// compiled unmodified, exercises the B200 library's GF(2^8) arithmetic (the
// C ABI's gs_gf_mul / gs_gf_inv / gs_gf_div, the field the kernels' tables
// and Horner constants are built from). Test infrastructure only.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>

#include "../../../../include/gs_capi.h"

namespace ghostserve::gf256 {

inline constexpr unsigned kPoly = 0x11D;  // the field the library implements (gf256.hpp:14)

inline std::uint8_t add(std::uint8_t a, std::uint8_t b) { return static_cast<std::uint8_t>(a ^ b); }
inline std::uint8_t mul(std::uint8_t a, std::uint8_t b) { return gs_gf_mul(a, b); }
inline std::uint8_t inv(std::uint8_t a) {
  std::uint8_t r = 0;
  if (gs_gf_inv(a, &r) != GS_OK) throw std::domain_error("gf256::inv(0)");
  return r;
}
inline std::uint8_t div(std::uint8_t a, std::uint8_t b) {
  std::uint8_t r = 0;
  if (gs_gf_div(a, b, &r) != GS_OK) throw std::domain_error("gf256::div by 0");
  return r;
}
inline const std::uint8_t* mul_row(std::uint8_t c) {
  static const auto table = [] {
    std::array<std::array<std::uint8_t, 256>, 256> t{};
    for (unsigned x = 0; x < 256; ++x)
      for (unsigned y = 0; y < 256; ++y) t[x][y] = gs_gf_mul(static_cast<std::uint8_t>(x), static_cast<std::uint8_t>(y));
    return t;
  }();
  return table[c].data();
}

}  // namespace ghostserve::gf256
