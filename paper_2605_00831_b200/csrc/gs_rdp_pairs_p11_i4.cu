// RDP(p = 11) two-column recovery, lost pairs (4, j > 4) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i4(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 4>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 4>{});
}
}  // namespace gsb
