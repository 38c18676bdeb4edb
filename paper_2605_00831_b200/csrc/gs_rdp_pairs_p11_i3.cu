// RDP(p = 11) two-column recovery, lost pairs (3, j > 3) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i3(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 3>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 3>{});
}
}  // namespace gsb
