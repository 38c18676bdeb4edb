// RDP(p = 11) two-column recovery, lost pairs (2, j > 2) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i2(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 2>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 2>{});
}
}  // namespace gsb
