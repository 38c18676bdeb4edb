// RDP(p = 11) two-column recovery, lost pairs (6, j > 6) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i6(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 6>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 6>{});
}
}  // namespace gsb
