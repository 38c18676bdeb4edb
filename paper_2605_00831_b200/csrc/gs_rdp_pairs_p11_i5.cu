// RDP(p = 11) two-column recovery, lost pairs (5, j > 5) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i5(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 5>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 5>{});
}
}  // namespace gsb
