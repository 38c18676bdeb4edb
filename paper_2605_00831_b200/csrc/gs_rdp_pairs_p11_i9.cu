// RDP(p = 11) two-column recovery, lost pairs (9, j > 9) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i9(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 9>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 9>{});
}
}  // namespace gsb
