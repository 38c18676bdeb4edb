// RDP(p = 11) two-column recovery, lost pairs (7, j > 7) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i7(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 7>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 7>{});
}
}  // namespace gsb
