// gs_fnv_simd.cpp -- FNV-1a 64 (parity_store.hpp:19-25) on one host core at
// several GB/s per chain, bit-exact, for the host half of the parity seal and
// of the recovery verification (gs_fnv.hpp is the scalar chain it replaces).
//
// The scalar chain h <- (h ^ b) * P costs one 64-bit multiply of latency per
// byte (~0.6 GB/s per chain). Two facts take the multiply off the serial path:
//
//  (1) XOR with a byte touches only the low byte: h ^ b = h + d with
//      d = (l ^ b) - l = b - 2 (b & l), l = h & 0xFF. Unrolled,
//          h_N = h_0 * P^N + sum_i d_i * P^(N-i)              (mod 2^64),
//      a dot product of 9-bit numbers with constant powers of P.
//  (2) The low byte runs on its own chain, l' = ((l ^ b) * 0xB3) & 0xFF
//      (P mod 256 = 0xB3). 0xB3 is odd, so bit j of x * 0xB3 is x_j XOR
//      (the column-j bits of the partial products of x's LOWER bits plus
//      their carries): bit plane j of the chain is a prefix XOR of
//      b_j ^ G_j once planes 0..j-1 are known.
//
// Per 512-byte block (8 zmm): the bytes are bit-transposed into eight
// 512-bit planes (VPSHUFB + GF2P8AFFINEQB + VPERMB per zmm, then an 8 x 8
// qword transpose); the eight planes of the low-byte chain are solved in
// order, each with a carry-save column of the bit-sliced product x * 0xB3
// (VPTERNLOG full adders, 512 bytes per instruction) and a 512-bit prefix
// XOR (VPCLMULQDQ with all-ones inside qwords, carries across qwords on a
// k-mask); b & l is transposed back to bytes and the dot product with
// P^(512-i) runs on VPDPWSSD over four balanced 16-bit limbs of the powers.
// Consecutive blocks overlap: block b+1's plane j needs only block b's exit
// bit j. Needs AVX-512 F/BW/DQ/VBMI/VNNI + GFNI + VPCLMULQDQ (checked at run
// time; fnv1a64_fast falls back to the scalar chain).
#include <immintrin.h>

#include <atomic>
#include <cstddef>
#include <cstdint>

#include "gs_fnv.hpp"

#define GS_SIMD_TARGET \
  __attribute__((target("avx512f,avx512bw,avx512dq,avx512vbmi,avx512vnni,gfni,vpclmulqdq")))

namespace gsb {

namespace {

constexpr int kBlock = 512;                    // bytes per low-byte-chain block (8 zmm)
constexpr int kPerSuper = 4;                    // blocks per dot-product super-block
constexpr int kSuper = kBlock * kPerSuper;      // 2 KiB: weights P^(2048-i), one reduction

struct Tables {
  // c[m][i]: balanced base-2^16 digit m of P^(kSuper-i):
  // sum_m c[m][i] 2^(16m) == P^(kSuper-i) (mod 2^64)
  alignas(64) int16_t c[4][kSuper];
  uint64_t p_super;  // P^kSuper
  Tables() {
    uint64_t w[kSuper];
    uint64_t x = kFnvPrime;
    for (int i = kSuper - 1; i >= 0; --i) {
      w[i] = x;
      x *= kFnvPrime;
    }
    p_super = w[0];
    for (int i = 0; i < kSuper; ++i) {
      uint64_t v = w[i];
      for (int m = 0; m < 4; ++m) {
        int32_t d = static_cast<int32_t>(v & 0xFFFF);
        if (d >= 0x8000) d -= 0x10000;
        c[m][i] = static_cast<int16_t>(d);
        v = (v - static_cast<uint64_t>(static_cast<int64_t>(d))) >> 16;  // exact: v - d is a multiple of 2^16
      }
    }
  }
};

const Tables& tables() {
  static const Tables t;
  return t;
}

struct Consts {
  __m512i rev8;    // reverse the bytes of every qword (VPSHUFB indices, per 16-byte lane)
  __m512i sel;     // byte p of every qword = 1 << p (GF2P8AFFINEQB selector)
  __m512i gather;  // byte 8j + g <- byte 8g + j (8 x 8 byte transpose inside the zmm)
  __m512i ones;
  __m512i last;    // qword index 7 in every lane (broadcast of the last qword)
};

GS_SIMD_TARGET inline Consts make_consts() {
  alignas(64) uint8_t r[64], s[64], g[64];
  for (int i = 0; i < 64; ++i) {
    r[i] = static_cast<uint8_t>((i & 8) + 7 - (i & 7));
    s[i] = static_cast<uint8_t>(1u << (i & 7));
    g[i] = static_cast<uint8_t>(8 * (i & 7) + (i >> 3));
  }
  Consts k;
  k.rev8 = _mm512_load_si512(r);
  k.sel = _mm512_load_si512(s);
  k.gather = _mm512_load_si512(g);
  k.ones = _mm512_set1_epi64(-1);
  k.last = _mm512_set1_epi64(7);
  return k;
}

// 64 bytes -> qword j = bit plane j (bit i = bit j of byte i). GF2P8AFFINEQB
// with the data qword as the matrix and x = 1 << p gives byte p = bit p of
// the eight bytes (row order reversed, hence the byte reversal first).
GS_SIMD_TARGET inline __m512i to_planes64(__m512i z, const Consts& k) {
  z = _mm512_shuffle_epi8(z, k.rev8);
  z = _mm512_gf2p8affine_epi64_epi8(k.sel, z, 0);
  return _mm512_permutexvar_epi8(k.gather, z);
}
GS_SIMD_TARGET inline __m512i from_planes64(__m512i z, const Consts& k) {
  z = _mm512_permutexvar_epi8(k.gather, z);
  z = _mm512_shuffle_epi8(z, k.rev8);
  return _mm512_gf2p8affine_epi64_epi8(k.sel, z, 0);
}

// 8 x 8 transpose of qwords across eight zmm (an involution).
GS_SIMD_TARGET inline void transpose8x8q(__m512i (&r)[8]) {
  __m512i t[8], u[8];
  for (int a = 0; a < 8; a += 2) {
    t[a] = _mm512_unpacklo_epi64(r[a], r[a + 1]);
    t[a + 1] = _mm512_unpackhi_epi64(r[a], r[a + 1]);
  }
  for (int a = 0; a < 8; a += 4) {
    u[a] = _mm512_shuffle_i64x2(t[a], t[a + 2], 0x88);
    u[a + 2] = _mm512_shuffle_i64x2(t[a], t[a + 2], 0xDD);
    u[a + 1] = _mm512_shuffle_i64x2(t[a + 1], t[a + 3], 0x88);
    u[a + 3] = _mm512_shuffle_i64x2(t[a + 1], t[a + 3], 0xDD);
  }
  r[0] = _mm512_shuffle_i64x2(u[0], u[4], 0x88);
  r[4] = _mm512_shuffle_i64x2(u[0], u[4], 0xDD);
  r[2] = _mm512_shuffle_i64x2(u[2], u[6], 0x88);
  r[6] = _mm512_shuffle_i64x2(u[2], u[6], 0xDD);
  r[1] = _mm512_shuffle_i64x2(u[1], u[5], 0x88);
  r[5] = _mm512_shuffle_i64x2(u[1], u[5], 0xDD);
  r[3] = _mm512_shuffle_i64x2(u[3], u[7], 0x88);
  r[7] = _mm512_shuffle_i64x2(u[3], u[7], 0xDD);
}

GS_SIMD_TARGET inline __m512i xor3(__m512i a, __m512i b, __m512i c) { return _mm512_ternarylogic_epi64(a, b, c, 0x96); }
GS_SIMD_TARGET inline __m512i maj3(__m512i a, __m512i b, __m512i c) { return _mm512_ternarylogic_epi64(a, b, c, 0xE8); }

// Exclusive prefix XOR over the 512 bits of e (qword 0 bit 0 first) from the
// entry bit broadcast in `in` (all-ones / zero qwords); `in` becomes the exit
// bit (entry ^ parity of e), broadcast. Everything stays in vector registers:
// within qwords a carry-less product with all-ones, across qwords a 3-step
// shift-XOR scan of the qword parities.
GS_SIMD_TARGET inline __m512i prefix_plane(__m512i e, __m512i& in, const Consts& k) {
  const __m512i ev = _mm512_clmulepi64_epi128(e, k.ones, 0x00);
  const __m512i od = _mm512_clmulepi64_epi128(e, k.ones, 0x01);
  const __m512i incl = _mm512_unpacklo_epi64(ev, od);      // inclusive prefix inside every qword
  const __m512i par = _mm512_srai_epi64(incl, 63);         // qword parity, all-ones / zero
  const __m512i z = _mm512_setzero_si512();
  // exclusive prefix of the parities: lane q <- par[q-1] ^ ... ^ par[0]
  const __m512i y = _mm512_xor_si512(par, _mm512_alignr_epi64(par, z, 7));               // par[q] ^ par[q-1]
  __m512i c = _mm512_xor_si512(_mm512_alignr_epi64(y, z, 7), _mm512_alignr_epi64(y, z, 5));  // par[q-1..q-4]
  c = _mm512_xor_si512(c, _mm512_alignr_epi64(c, z, 4));                                 // par[q-1..q-8]
  const __m512i L = _mm512_ternarylogic_epi64(_mm512_slli_epi64(incl, 1), c, in, 0x96);
  in = _mm512_xor_si512(in, _mm512_permutexvar_epi64(k.last, _mm512_xor_si512(c, par)));
  return L;
}

// The low-byte chain of one 512-byte block, column by column. B = the 8
// planes of its bytes; column<J>() solves plane J from the entry bit
// bits[J] (updated to the block's exit bit) and leaves the planes of b & l
// in U. Column j of y = x + 2x + 16x + 32x + 128x (x = l ^ b) holds x_j,
// x_{j-1}, x_{j-4}, x_{j-5}, x_{j-7} and the carries of the lower columns;
// G_j = XOR of all of them but x_j. Known bits are pre-reduced (full adders)
// to one per column so only a single AND / majority follows each new plane.
struct BlockChain {
  __m512i B[8], X[8], U[8];
  __m512i c12, c23, c34, s4, c45a, c45b, s5, c56a, c56b, c56c, s6, c67a, c67b, c67c, c67d;

  GS_SIMD_TARGET inline void plane(int j, __m512i g, __m512i& in, const Consts& k) {
    const __m512i L = prefix_plane(_mm512_xor_si512(B[j], g), in, k);
    X[j] = _mm512_xor_si512(L, B[j]);
    U[j] = _mm512_and_si512(L, B[j]);
  }
  template <int J>
  GS_SIMD_TARGET inline void column(__m512i& in, const Consts& k) {
    if constexpr (J == 0) {
      plane(0, _mm512_setzero_si512(), in, k);  // column 0 = {x0}
    } else if constexpr (J == 1) {
      plane(1, X[0], in, k);  // column 1 = {x1, x0}
      c12 = _mm512_and_si512(X[1], X[0]);
    } else if constexpr (J == 2) {
      plane(2, _mm512_xor_si512(X[1], c12), in, k);  // column 2 = {x2, x1, c12}
      c23 = maj3(X[2], X[1], c12);
    } else if constexpr (J == 3) {
      plane(3, _mm512_xor_si512(X[2], c23), in, k);  // column 3 = {x3, x2, c23}
      c34 = maj3(X[3], X[2], c23);
    } else if constexpr (J == 4) {
      // column 4 = {x4, x3, x0, c34}
      s4 = xor3(X[3], X[0], c34);
      c45a = maj3(X[3], X[0], c34);
      plane(4, s4, in, k);
      c45b = _mm512_and_si512(X[4], s4);
    } else if constexpr (J == 5) {
      // column 5 = {x5, x4, x1, x0, c45a, c45b}
      const __m512i s5a = xor3(X[1], X[0], c45a);
      c56a = maj3(X[1], X[0], c45a);
      s5 = xor3(s5a, X[4], c45b);
      c56b = maj3(s5a, X[4], c45b);
      plane(5, s5, in, k);
      c56c = _mm512_and_si512(X[5], s5);
    } else if constexpr (J == 6) {
      // column 6 = {x6, x5, x2, x1, c56a, c56b, c56c}
      const __m512i s6a = xor3(X[2], X[1], c56a);
      c67a = maj3(X[2], X[1], c56a);
      const __m512i s6b = xor3(s6a, c56b, c56c);
      c67b = maj3(s6a, c56b, c56c);
      s6 = _mm512_xor_si512(s6b, X[5]);
      c67c = _mm512_and_si512(s6b, X[5]);
      plane(6, s6, in, k);
      c67d = _mm512_and_si512(X[6], s6);
    } else {
      // column 7 = {x7, x6, x3, x2, x0, c67a..c67d}: only its parity is needed
      plane(7, _mm512_xor_si512(xor3(X[6], X[3], X[2]), xor3(X[0], c67a, xor3(c67b, c67c, c67d))), in, k);
    }
  }
};

// Two consecutive blocks, skewed by one column: block 1's column J needs
// block 0's exit bit J, not its later columns, so the two eight-step chains
// overlap into nine steps.
template <int J>
GS_SIMD_TARGET inline void columns2(BlockChain& a, BlockChain& b, __m512i (&bits)[8], const Consts& k) {
  a.column<J>(bits[J], k);
  b.column<J>(bits[J], k);
  if constexpr (J < 7) columns2<J + 1>(a, b, bits, k);
}
GS_SIMD_TARGET inline void load_planes(BlockChain& c, const uint8_t* p, const Consts& k) {
  for (int q = 0; q < 8; ++q) c.B[q] = to_planes64(_mm512_loadu_si512(p + 64 * q), k);
  transpose8x8q(c.B);  // B[j] = plane j of the 512 bytes
}

// Sum of the 16 int32 lanes in int64.
GS_SIMD_TARGET inline uint64_t hsum64(__m512i a) {
  const __m512i s = _mm512_add_epi64(_mm512_cvtepi32_epi64(_mm512_castsi512_si256(a)),
                                     _mm512_cvtepi32_epi64(_mm512_extracti64x4_epi64(a, 1)));
  return static_cast<uint64_t>(_mm512_reduce_add_epi64(s));
}


// sum_i d_i * P^(kSuper-i) contributions of one 512-byte block (index blk in
// its super-block) into the four limb accumulators; d = b - 2 (b & l).
GS_SIMD_TARGET inline void dot_block(const uint8_t* p, const __m512i (&U)[8], int blk, const Tables& tb,
                                     const Consts& k, __m512i (&a)[4]) {
  for (int q = 0; q < 8; ++q) {
    const __m512i b = _mm512_loadu_si512(p + 64 * q);
    const __m512i u = from_planes64(U[q], k);
    for (int half = 0; half < 2; ++half) {
      const __m256i bh = half ? _mm512_extracti64x4_epi64(b, 1) : _mm512_castsi512_si256(b);
      const __m256i uh = half ? _mm512_extracti64x4_epi64(u, 1) : _mm512_castsi512_si256(u);
      const __m512i u16 = _mm512_cvtepu8_epi16(uh);
      const __m512i d = _mm512_sub_epi16(_mm512_sub_epi16(_mm512_cvtepu8_epi16(bh), u16), u16);
      const int o = kBlock * blk + 64 * q + 32 * half;
      for (int m = 0; m < 4; ++m) a[m] = _mm512_dpwssd_epi32(a[m], d, _mm512_load_si512(tb.c[m] + o));
    }
  }
}

GS_SIMD_TARGET inline uint64_t reduce_limbs(__m512i (&a)[4]) {
  // |lane| <= 4 * 16 * 2 * 255 * 2^15 < 2^30: exact in int32. Limbs 0 and 1 are
  // needed mod 2^64 / 2^48 (summed in int64), limbs 2 and 3 only mod 2^32 / 2^16.
  const uint64_t t = hsum64(a[0]) + (hsum64(a[1]) << 16) +
                     (static_cast<uint64_t>(static_cast<uint32_t>(_mm512_reduce_add_epi32(a[2]))) << 32) +
                     (static_cast<uint64_t>(static_cast<uint32_t>(_mm512_reduce_add_epi32(a[3]))) << 48);
  for (int m = 0; m < 4; ++m) a[m] = _mm512_setzero_si512();
  return t;
}

// The 2 KiB super-blocks of p[0 .. nsup * kSuper): advances the low byte `l`
// and returns S = sum_i d_i P^(len-i) over them (a state h with low byte l
// becomes h * P^(nsup * kSuper) + S).
GS_SIMD_TARGET static uint64_t simd_blocks(const uint8_t* p, size_t nsup, uint32_t& l) {
  const Tables& tb = tables();
  const Consts k = make_consts();
  __m512i bits[8];  // entry bit j of the next block, broadcast
  for (int j = 0; j < 8; ++j) bits[j] = _mm512_set1_epi64(((l >> j) & 1u) ? -1 : 0);
  uint64_t acc = 0;
  __m512i a[4];
  for (int m = 0; m < 4; ++m) a[m] = _mm512_setzero_si512();
  BlockChain c0, c1;
  for (size_t s = 0; s < nsup; ++s) {
    const uint8_t* ps = p + s * kSuper;
    for (int blk = 0; blk < kPerSuper; blk += 2) {
      const uint8_t* pb = ps + static_cast<size_t>(blk) * kBlock;
      load_planes(c0, pb, k);
      load_planes(c1, pb + kBlock, k);
      columns2<0>(c0, c1, bits, k);
      transpose8x8q(c0.U);
      transpose8x8q(c1.U);
      dot_block(pb, c0.U, blk, tb, k, a);
      dot_block(pb + kBlock, c1.U, blk + 1, tb, k, a);
    }
    acc = acc * tb.p_super + reduce_limbs(a);
  }
  l = 0;
  for (int j = 0; j < 8; ++j) l |= static_cast<uint32_t>(_mm_cvtsi128_si32(_mm512_castsi512_si128(bits[j])) & 1) << j;
  return acc;
}

inline uint32_t low_step(uint32_t l, uint8_t b) { return ((l ^ b) * 0xB3u) & 0xFFu; }

bool simd_hw() {
  static const bool ok = [] {
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512bw") &&
           __builtin_cpu_supports("avx512dq") && __builtin_cpu_supports("avx512vbmi") &&
           __builtin_cpu_supports("avx512vnni") && __builtin_cpu_supports("gfni") &&
           __builtin_cpu_supports("vpclmulqdq");
  }();
  return ok;
}
std::atomic<bool> g_simd_on{true};
}  // namespace

bool fnv_simd_available() { return simd_hw() && g_simd_on.load(std::memory_order_relaxed); }

bool fnv_simd_set(bool on) {
  g_simd_on.store(on, std::memory_order_relaxed);
  return fnv_simd_available();
}

uint64_t fnv_pow(uint64_t n) {
  uint64_t r = 1, x = kFnvPrime;
  for (; n; n >>= 1, x *= x)
    if (n & 1) r *= x;
  return r;
}

uint64_t fnv_partial(const uint8_t* p, size_t len, uint32_t l, uint32_t* l_out) {
  uint64_t sum = 0;
  size_t i = 0;
  if (len >= kSuper && fnv_simd_available()) {
    const size_t nsup = len / kSuper;
    sum = simd_blocks(p, nsup, l);
    i = nsup * kSuper;
  }
  for (; i < len; ++i) {  // h' = (h + d) P with d = (l ^ b) - l
    const int64_t d = static_cast<int64_t>(l ^ p[i]) - static_cast<int64_t>(l);
    sum = (sum + static_cast<uint64_t>(d)) * kFnvPrime;
    l = low_step(l, p[i]);
  }
  if (l_out) *l_out = l;
  return sum;
}

uint64_t fnv1a64_fast(const uint8_t* p, size_t len, uint64_t h) {
  if (len < kSuper || !fnv_simd_available()) return fnv1a64_one(p, len, h);
  return h * fnv_pow(len) + fnv_partial(p, len, static_cast<uint32_t>(h & 0xFF), nullptr);
}

}  // namespace gsb
