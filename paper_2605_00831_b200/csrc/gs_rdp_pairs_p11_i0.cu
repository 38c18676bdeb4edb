// RDP(p = 11) two-column recovery, lost pairs (0, j > 0) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i0(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 0>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 0>{});
}
}  // namespace gsb
