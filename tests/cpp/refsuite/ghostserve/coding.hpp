// Redirect shim for running the REFERENCE's own unit suite against the B200
// library: proj/tests/coding_test.cpp (compiled unmodified, in place, from
// /root/reference) includes "ghostserve/coding.hpp" and uses namespace
// ghostserve; with this directory first on the include path that name is the
// drop-in facade (include/ghostserve_gpu/coding.hpp), so every encode /
// reconstruct the suite makes runs the sm_100a kernels through the C ABI.
// Test infrastructure only.
#pragma once

#include <cstdint>
#include <vector>

#include "ghostserve_gpu/coding.hpp"

namespace ghostserve_gpu::detail {
// The suite's MDS check calls the reference's Gauss-Jordan rank test
// (coding.hpp:187-223); restated over the library's own GF(2^8) (gs_gf_mul,
// gs_gf_inv). Returns false if singular.
inline bool gf_invert_matrix(std::vector<std::uint8_t>& m, int dim, std::vector<std::uint8_t>& inv) {
  inv.assign(static_cast<std::size_t>(dim) * dim, 0);
  for (int i = 0; i < dim; ++i) inv[static_cast<std::size_t>(i) * dim + i] = 1;
  auto at = [dim](std::vector<std::uint8_t>& v, int r, int c) -> std::uint8_t& {
    return v[static_cast<std::size_t>(r) * dim + c];
  };
  for (int col = 0; col < dim; ++col) {
    int piv = -1;
    for (int r = col; r < dim && piv < 0; ++r)
      if (at(m, r, col)) piv = r;
    if (piv < 0) return false;
    if (piv != col)
      for (int c = 0; c < dim; ++c) {
        std::swap(at(m, piv, c), at(m, col, c));
        std::swap(at(inv, piv, c), at(inv, col, c));
      }
    std::uint8_t pi = 0;
    if (gs_gf_inv(at(m, col, col), &pi) != GS_OK) return false;
    for (int c = 0; c < dim; ++c) {
      at(m, col, c) = gs_gf_mul(at(m, col, c), pi);
      at(inv, col, c) = gs_gf_mul(at(inv, col, c), pi);
    }
    for (int r = 0; r < dim; ++r) {
      if (r == col) continue;
      const std::uint8_t f = at(m, r, col);
      if (!f) continue;
      for (int c = 0; c < dim; ++c) {
        at(m, r, c) ^= gs_gf_mul(f, at(m, col, c));
        at(inv, r, c) ^= gs_gf_mul(f, at(inv, col, c));
      }
    }
  }
  return true;
}
}  // namespace ghostserve_gpu::detail

// A real namespace (not an alias) so the reference's own headers can reopen
// `namespace ghostserve { ... }`; everything of the facade is visible in it.
namespace ghostserve {
using namespace ghostserve_gpu;
}
