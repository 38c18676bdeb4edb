// gs_field.hpp -- GF(2^8) arithmetic and the code's coefficient matrices,
// usable at compile time (for the specialised kernels), on the host (codec
// construction) and on the device.
//
// Field: primitive polynomial x^8+x^4+x^3+x^2+1 (0x11D), generator 2 -- the
// same field as the reference (gf256.hpp:11-36), so every product, inverse and
// Cauchy coefficient is identical byte for byte.
#pragma once

#if defined(__CUDACC_RTC__)
// runtime (NVRTC) compilation of specialised kernels: no host headers
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned long long uintptr_t;
#else
#include <cstddef>
#include <cstdint>
#endif

#ifdef __CUDACC__
#define GS_HD __host__ __device__
#else
#define GS_HD
#endif

namespace gsb {

constexpr unsigned kPoly = 0x11D;

struct FieldTables {
  uint8_t exp[512];
  uint8_t log[256];
};

// gf256.hpp:21-34 builds the same exp/log pair (exp doubled to avoid a mod).
GS_HD constexpr FieldTables make_field_tables() {
  FieldTables t{};
  unsigned x = 1;
  for (unsigned i = 0; i < 255; ++i) {
    t.exp[i] = static_cast<uint8_t>(x);
    t.exp[i + 255] = static_cast<uint8_t>(x);
    t.log[x] = static_cast<uint8_t>(i);
    x <<= 1;
    if (x & 0x100u) x ^= kPoly;
  }
  t.exp[510] = t.exp[0];
  t.exp[511] = t.exp[1];
  return t;
}

// Shift-and-reduce product: needs no tables, so it is cheap to evaluate in
// constant expressions of any depth.
GS_HD constexpr uint8_t gf_mul(uint8_t a, uint8_t b) {
  unsigned acc = 0, x = a;
  for (int i = 0; i < 8; ++i) {
    if (b & (1u << i)) acc ^= x;
    x <<= 1;
    if (x & 0x100u) x ^= kPoly;
  }
  return static_cast<uint8_t>(acc);
}

// a^254 = a^-1 for a != 0 (the multiplicative group has order 255).
GS_HD constexpr uint8_t gf_inv(uint8_t a) {
  uint8_t r = 1, p = a;
  unsigned e = 254;
  while (e) {
    if (e & 1u) r = gf_mul(r, p);
    p = gf_mul(p, p);
    e >>= 1;
  }
  return a ? r : 0;
}

// 2^e in the field (gf256.hpp:59-61), e >= 0.
GS_HD constexpr uint8_t exp2_of(int e) {
  uint8_t r = 1;
  for (int i = 0; i < e % 255; ++i) r = gf_mul(r, 2);
  return r;
}

// Smallest prime >= x (coding.hpp:174-184): the RDP array's p for n data
// columns is smallest_prime_ge(n + 1).
GS_HD constexpr int smallest_prime_ge(int x) {
  int v = x < 2 ? 2 : x;
  for (;; ++v) {
    bool prime = true;
    for (int d = 2; d * d <= v; ++d)
      if (v % d == 0) prime = false;
    if (prime) return v;
  }
}

// Systematic Cauchy coefficient of parity row i, data column j for RS(n, k):
// 1 / (x_i ^ y_j) with x_i = i, y_j = k + j (coding.hpp:108-114).
GS_HD constexpr uint8_t cauchy(int k, int i, int j) {
  return gf_inv(static_cast<uint8_t>(i ^ (k + j)));
}

enum CodeKind : int { kXor = 0, kRdp = 1, kReedSolomon = 2 };

constexpr int kMaxSpecial = 16;  // largest n (and n+k) with compile-time kernels

// Row-major coefficient matrix of fixed capacity: rows are outputs, columns
// are sources (data shards then parity shards, index-aligned with the
// reference's shard numbering: data 0..n-1, parity n..n+k-1).
struct CoefMatrix {
  int rows = 0, cols = 0;
  uint8_t c[kMaxSpecial][2 * kMaxSpecial] = {};
  int out_index[kMaxSpecial] = {};  // which shard each output row rebuilds
};

// Encode matrix for (kind, n, k) as a source->output map: outputs are the k
// parity shards, sources the n data shards.
GS_HD constexpr CoefMatrix encode_matrix(int kind, int n, int k) {
  CoefMatrix m{};
  m.rows = k;
  m.cols = n;
  for (int i = 0; i < k; ++i) {
    m.out_index[i] = n + i;
    for (int j = 0; j < n; ++j) m.c[i][j] = kind == kReedSolomon ? cauchy(k, i, j) : 1;
  }
  return m;
}

// Decode matrix for an erasure pattern given as a bitmask over shard indices
// (bit s set = shard s lost). Follows coding.hpp:535-566 exactly: rows are
// the first e surviving parity rows, the e x e system is inverted by
// Gauss-Jordan, and the inverse is folded into one coefficient per source.
// XOR: the single lost data shard is the XOR of every survivor (:496-502).
// ok=false when the pattern is not decodable (caller reports the error).
struct DecodePlan {
  CoefMatrix m;
  bool ok = false;
};

GS_HD constexpr DecodePlan decode_plan_mask(int kind, int n, int k, uint64_t lost_mask) {
  DecodePlan p{};
  int ld[kMaxSpecial] = {};
  int e = 0;
  for (int s = 0; s < n; ++s)
    if ((lost_mask >> s) & 1u) ld[e++] = s;
  p.m.rows = e;
  p.m.cols = n + k;
  for (int b = 0; b < e; ++b) p.m.out_index[b] = ld[b];
  if (e == 0) {
    p.ok = true;
    return p;
  }
  if (kind != kReedSolomon) {
    for (int s = 0; s < n + k; ++s)
      if (!((lost_mask >> s) & 1u)) p.m.c[0][s] = 1;
    p.ok = e == 1;
    return p;
  }
  int rows[kMaxSpecial] = {};
  int nr = 0;
  for (int i = 0; i < k && nr < e; ++i)
    if (!((lost_mask >> (n + i)) & 1u)) rows[nr++] = i;
  if (nr < e) return p;
  uint8_t sys[kMaxSpecial][kMaxSpecial] = {};
  uint8_t inv[kMaxSpecial][kMaxSpecial] = {};
  for (int a = 0; a < e; ++a) {
    inv[a][a] = 1;
    for (int b = 0; b < e; ++b) sys[a][b] = cauchy(k, rows[a], ld[b]);
  }
  for (int col = 0; col < e; ++col) {
    int piv = -1;
    for (int r = col; r < e; ++r)
      if (sys[r][col] && piv < 0) piv = r;
    if (piv < 0) return p;
    for (int c = 0; c < e; ++c) {
      uint8_t t = sys[piv][c];
      sys[piv][c] = sys[col][c];
      sys[col][c] = t;
      t = inv[piv][c];
      inv[piv][c] = inv[col][c];
      inv[col][c] = t;
    }
    const uint8_t pi = gf_inv(sys[col][col]);
    for (int c = 0; c < e; ++c) {
      sys[col][c] = gf_mul(sys[col][c], pi);
      inv[col][c] = gf_mul(inv[col][c], pi);
    }
    for (int r = 0; r < e; ++r) {
      if (r == col) continue;
      const uint8_t f = sys[r][col];
      for (int c = 0; c < e; ++c) {
        sys[r][c] ^= gf_mul(f, sys[col][c]);
        inv[r][c] ^= gf_mul(f, inv[col][c]);
      }
    }
  }
  for (int b = 0; b < e; ++b) {
    for (int j = 0; j < n; ++j) {
      if ((lost_mask >> j) & 1u) continue;
      uint8_t c = 0;
      for (int a = 0; a < e; ++a) c ^= gf_mul(inv[b][a], cauchy(k, rows[a], j));
      p.m.c[b][j] = c;
    }
    for (int a = 0; a < e; ++a) p.m.c[b][n + rows[a]] = inv[b][a];
  }
  p.ok = true;
  return p;
}

}  // namespace gsb
