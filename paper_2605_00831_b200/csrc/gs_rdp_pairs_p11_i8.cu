// RDP(p = 11) two-column recovery, lost pairs (8, j > 8) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i8(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 8>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 8>{});
}
}  // namespace gsb
