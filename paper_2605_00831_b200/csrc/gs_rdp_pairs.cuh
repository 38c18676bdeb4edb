// gs_rdp_pairs.cuh -- RDP two-column recovery kernels with the lost pair as
// a compile-time constant (k_rdp_recover_bulk<CAP, P, LI, LJ>): the zig-zag
// chains of coding.hpp:384-413 fully unroll and run in registers. Compiled
// for p = 11 (n = 8..10, the configs' shard counts), one translation unit per
// first lost column (gs_rdp_pairs_p11_i*.cu) so the build parallelises; other
// primes use the runtime-pair kernel.
#pragma once

#include <utility>

#include "gs_rdp.cuh"
#include "gs_special.cuh"

namespace gsb {

constexpr int kRdpPairP = 11;

using RdpPairLaunch = cudaError_t (*)(int grid, int threads, size_t smem, cudaStream_t st,
                                      const PtrTable<kPtrCap>& tab, const RdpGeom& g, int stages, int n_out,
                                      int out0);
struct RdpPair {
  const void* kernel = nullptr;
  RdpPairLaunch launch = nullptr;
};

template <int P, int I, int J>
cudaError_t rdp_pair_launch(int grid, int threads, size_t smem, cudaStream_t st, const PtrTable<kPtrCap>& tab,
                            const RdpGeom& g, int stages, int n_out, int out0) {
  k_rdp_recover_bulk<kPtrCap, P, I, J><<<grid, threads, smem, st>>>(tab, g, stages, n_out, out0);
  return cudaGetLastError();
}

template <int P, int I, int... Js>
void rdp_pairs_register(RdpPair* t, std::integer_sequence<int, Js...>) {
  ((t[I * P + (I + 1 + Js)] = RdpPair{reinterpret_cast<const void*>(&k_rdp_recover_bulk<kPtrCap, P, I, I + 1 + Js>),
                                      &rdp_pair_launch<P, I, I + 1 + Js>}),
   ...);
}

// one per first column I (gs_rdp_pairs_p11_i<I>.cu): fills t[I*P + J], J > I
void rdp_pairs_p11_i0(RdpPair* t);
void rdp_pairs_p11_i1(RdpPair* t);
void rdp_pairs_p11_i2(RdpPair* t);
void rdp_pairs_p11_i3(RdpPair* t);
void rdp_pairs_p11_i4(RdpPair* t);
void rdp_pairs_p11_i5(RdpPair* t);
void rdp_pairs_p11_i6(RdpPair* t);
void rdp_pairs_p11_i7(RdpPair* t);
void rdp_pairs_p11_i8(RdpPair* t);
void rdp_pairs_p11_i9(RdpPair* t);

}  // namespace gsb
