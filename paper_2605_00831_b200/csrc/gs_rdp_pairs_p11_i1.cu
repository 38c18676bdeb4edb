// RDP(p = 11) two-column recovery, lost pairs (1, j > 1) -- see gs_rdp_pairs.cuh.
#include "gs_rdp_pairs.cuh"

namespace gsb {
void rdp_pairs_p11_i1(RdpPair* t) {
  rdp_pairs_register<kRdpPairP, 1>(t, std::make_integer_sequence<int, kRdpPairP - 1 - 1>{});
}
}  // namespace gsb
