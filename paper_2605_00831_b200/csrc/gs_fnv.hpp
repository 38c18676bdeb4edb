// gs_fnv.hpp -- FNV-1a 64 (parity_store.hpp:19-25), bit-exact, for the
// host-side parity seal and verification. The scalar chain is a serial
// xor -> 64-bit multiply per byte (latency-bound, ~0.6-0.9 GB/s per core);
// independent chunks are advanced in lockstep (four, or up to eight), so the
// multiplier pipelines across chains. Hosts with AVX-512 VBMI/VNNI + GFNI +
// VPCLMULQDQ take the bit-sliced chain of gs_fnv_simd.cpp instead (~6 GB/s
// per chain on one core): fnv1a64_chains picks.
#pragma once

#include <cstddef>
#include <cstdint>

namespace gsb {

constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;

inline uint64_t fnv1a64_one(const uint8_t* p, size_t len, uint64_t h) {
  for (size_t i = 0; i < len; ++i) h = (h ^ p[i]) * kFnvPrime;
  return h;
}

// h[q] = FNV-1a of p[q][0..len) continued from h[q], for q < m (m <= 4).
inline void fnv1a64_x4(const uint8_t* const* p, int m, size_t len, uint64_t* h) {
  if (m == 1) {
    h[0] = fnv1a64_one(p[0], len, h[0]);
    return;
  }
  const uint8_t* p0 = p[0];
  const uint8_t* p1 = m > 1 ? p[1] : p[0];
  const uint8_t* p2 = m > 2 ? p[2] : p[0];
  const uint8_t* p3 = m > 3 ? p[3] : p[0];
  uint64_t a = h[0], b = m > 1 ? h[1] : 0, c = m > 2 ? h[2] : 0, d = m > 3 ? h[3] : 0;
  for (size_t i = 0; i < len; ++i) {
    a = (a ^ p0[i]) * kFnvPrime;
    b = (b ^ p1[i]) * kFnvPrime;
    c = (c ^ p2[i]) * kFnvPrime;
    d = (d ^ p3[i]) * kFnvPrime;
  }
  h[0] = a;
  if (m > 1) h[1] = b;
  if (m > 2) h[2] = c;
  if (m > 3) h[3] = d;
}

// Same for up to eight chains (m <= 8, exactly m multiplies per byte): used
// when the chains outnumber the threads by a non-multiple of four, so every
// thread takes ONE group and the wall time is one chain's length, not two.
template <int M>
inline void fnv1a64_lanes(const uint8_t* const* p, size_t len, uint64_t* h) {
  const uint8_t* q[M];
  uint64_t v[M];
  for (int c = 0; c < M; ++c) {
    q[c] = p[c];
    v[c] = h[c];
  }
  for (size_t i = 0; i < len; ++i) {
#pragma GCC unroll 8
    for (int c = 0; c < M; ++c) v[c] = (v[c] ^ q[c][i]) * kFnvPrime;
  }
  for (int c = 0; c < M; ++c) h[c] = v[c];
}

inline void fnv1a64_x8(const uint8_t* const* p, int m, size_t len, uint64_t* h) {
  switch (m) {
    case 5: return fnv1a64_lanes<5>(p, len, h);
    case 6: return fnv1a64_lanes<6>(p, len, h);
    case 7: return fnv1a64_lanes<7>(p, len, h);
    case 8: return fnv1a64_lanes<8>(p, len, h);
    default: return fnv1a64_x4(p, m, len, h);
  }
}

// gs_fnv_simd.cpp: the bit-sliced chain (same result as fnv1a64_one).
bool fnv_simd_available();          // hardware support and not switched off
bool fnv_simd_set(bool on);         // gs_fnv_host_set_simd (A/B, tests); returns the new state
uint64_t fnv1a64_fast(const uint8_t* p, size_t len, uint64_t h);
constexpr size_t kFnvSimdMin = 2048;  // shorter runs stay scalar
// Split form (bit-sliced when available, scalar otherwise): for any state h
// whose low byte is l, FNV-1a over p[0..len) from h ends in
// h * fnv_pow(len) + fnv_partial(p, len, l, &l_out), with low byte l_out --
// the upper 56 bits of h enter only through the final multiply-add.
uint64_t fnv_pow(uint64_t n);
uint64_t fnv_partial(const uint8_t* p, size_t len, uint32_t l, uint32_t* l_out);

// h[q] = FNV-1a of p[q][0..len) continued from h[q], for q < m (m <= 8).
inline void fnv1a64_chains(const uint8_t* const* p, int m, size_t len, uint64_t* h) {
  if (len >= kFnvSimdMin && fnv_simd_available()) {
    for (int q = 0; q < m; ++q) h[q] = fnv1a64_fast(p[q], len, h[q]);
    return;
  }
  fnv1a64_x8(p, m, len, h);
}

}  // namespace gsb
