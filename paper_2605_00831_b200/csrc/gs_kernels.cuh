// gs_kernels.cuh -- sm_100a kernels for the shadow-checkpointing byte path.
//
//   K1 encode  : parity_i = sum_j C[i][j] * data_j          (coding.hpp:263-275)
//   K2 rebuild : lost_b   = sum_s D[b][s] * shard_s          (coding.hpp:496-502, 554-566)
//
// Both are one operation -- "apply a GF(2^8) coefficient matrix to a set of
// source shards, byte position by byte position" -- so one kernel family
// serves both. Sources may live in local HBM or in a peer GPU's HBM (NVLink
// P2P loads through a mapped pointer); outputs may be local staging (then
// D2H'd on a copy stream) or a peer's KV buffer (P2P stores).
//
// Two arithmetic back ends, both HBM-streaming with 128-bit loads/stores:
//
//  * Specialised (compile-time coefficients, `k_apply_special`): Horner over
//    the coefficient bits,  p = (((S7)*2 ^ S6)*2 ^ ...)*2 ^ S0,  where S_b is
//    the XOR of the sources whose coefficient has bit b set. A Horner step
//    (x * acc ^ S_b on four packed bytes, xtime4_xor) is 2 ALU + 3 FMA-pipe
//    ops, the ALU merge absorbing one XOR term. Cost per source word ~
//    rows*(35/ns + 2) ops -- about 13 for RS(8,2) encode, ~7 of them ALU.
//
//  * Generic (runtime coefficients, `k_apply_generic`): split-table lookups
//    with PRMT. Byte b = lo3 | bit3 | hi3<<4 | bit7, so
//      c*b = L_c[lo3] ^ H_c[hi3] ^ (bit3 ? c*8 : 0) ^ (bit7 ? c*128 : 0)
//    with 8-entry tables L_c, H_c held in two registers each. Two data words
//    are processed as a pair so each PRMT selector packs 4 nibbles without
//    extra compaction; results accumulate in a byte-permuted domain that is
//    undone once per output word.
#pragma once

#if !defined(__CUDACC_RTC__)
#include <cstdint>
#endif

#include "gs_field.hpp"

namespace gsb {

constexpr int kThreads = 256;
constexpr int kVec = 16;                  // bytes per thread per source per tile
constexpr int kTile = kThreads * kVec;    // 4 KiB of every shard per tile
constexpr int kMaxGenericRows = 4;

template <int CAP>
struct PtrTable {
  const uint8_t* p[CAP];
};

// ---- primitive ops -------------------------------------------------------

// prmt.b32 in its default mode: selector nibble bit 3 = replicate the sign
// of the selected byte (used to build per-byte bit masks in one op).
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

// Multiply four packed field elements by 2 (x): shift, then fold x^8 back in
// as 0x1D where the top bit was set. The fold uses the high half of a 32x32
// product: (a & 0x80808080) * (0x1D << 25) >> 32 places 0x1D in exactly the
// bytes whose msb was set, with no carries between bytes.
__device__ __forceinline__ uint32_t xtime4(uint32_t a) {
  const uint32_t fold = __umulhi(a & 0x80808080u, 0x3A000000u);
  return ((a + a) & 0xFEFEFEFEu) ^ fold;
}

// x * a ^ s, the Horner step, balanced across the integer pipes: the ALU
// (LOP3) does the low-bit mask and one 3-input merge that also absorbs the
// next XOR term s; the FMA pipe (IMAD) does the top-bit split (a - t, exact:
// t = a & 0x7F7F7F7F is a submask of a), the shift and the fold. 2 ALU + 3
// FMA ops instead of 3 ALU + 2 FMA with a separate XOR.
__device__ __forceinline__ uint32_t xtime4_xor(uint32_t a, uint32_t s) {
  const uint32_t t = a & 0x7F7F7F7Fu;
  uint32_t h, t2;
  asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(h) : "r"(t), "r"(0xFFFFFFFFu), "r"(a));  // a - t = a & 0x80808080
  asm("mul.lo.u32 %0, %1, 2;" : "=r"(t2) : "r"(t));
  const uint32_t fold = __umulhi(h, 0x3A000000u);
  return t2 ^ fold ^ s;
}

__device__ __forceinline__ uint4 ld_stream(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void st_stream(uint8_t* p, const uint4& v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint32_t& word(uint4& v, int w) {
  return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
}

// Byte-granular load/store of up to 16 bytes (tail of a shard, or shards
// whose base pointers are not 16-B aligned).
// Fully unrolled with guards so the words stay in registers.
__device__ __forceinline__ uint4 ld_partial(const uint8_t* p, int nbytes) {
  uint32_t w[4] = {0, 0, 0, 0};
#pragma unroll
  for (int b = 0; b < 16; ++b)
    if (b < nbytes) w[b >> 2] |= static_cast<uint32_t>(p[b]) << (8 * (b & 3));
  return make_uint4(w[0], w[1], w[2], w[3]);
}

__device__ __forceinline__ void st_partial(uint8_t* p, const uint4& v, int nbytes) {
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int b = 0; b < 16; ++b)
    if (b < nbytes) p[b] = static_cast<uint8_t>(w[b >> 2] >> (8 * (b & 3)));
}

// ---- tile walk shared by both back ends ------------------------------------
//
// Work = n_stripes x ceil(len / 4 KiB) tiles, walked grid-stride so that
// consecutive CTAs stream consecutive 4 KiB pieces of the same shards.

// Paged KV addressing. A slice in the reference byte order
// [K,V][layer][token][elems] (kv_layout.hpp:59-68) is 2*layers segments of
// page_bytes = chunk tokens x token_bytes; segment (t, l) lives in a paged KV
// cache at  base + l*layer_stride + t*kv_stride  (+ the block). Two modes:
//  * single block (table == nullptr): the chunk is one cache block and the
//    per-stripe base already includes the block's offset;
//  * block table: the chunk spans page_bytes / block_bytes cache blocks;
//    block i of stripe s is table[s * table_stride + i] (the same ids in every
//    layer and for K and V, as in vLLM-style caches), at block * block_bytes.
// Tokens >= valid_tokens of each segment read as zero (pad_partial,
// kv_layout.hpp:73-84) and are never written. page_bytes == 0: contiguous.
struct PageMap {
  uint32_t page_bytes;
  uint32_t layers;
  uint32_t token_bytes;
  uint32_t valid_tokens;
  uint64_t layer_stride;
  uint64_t kv_stride;
  const int32_t* table;
  uint32_t block_bytes;
  uint32_t table_stride;
  // fastdiv_magic() of page_bytes / layers / block_bytes (0: divide)
  uint64_t page_m, layers_m, block_m;
};

// Division by a launch-invariant divisor without the ~20-instruction integer
// divide: q = floor(n * M / 2^64) with M = floor(2^64 / d) + 1 (or 2^64 / d
// for powers of two) is exact for every 32-bit n when 2 <= d < 2^32 (the
// rounding error n * (M - 2^64/d) / 2^64 < 2^-32 < 1/d never crosses an
// integer). M = 0 means "no magic": plain division (d == 1 returns n).
__host__ __device__ constexpr uint64_t fastdiv_magic(uint32_t d) { return d > 1 ? ~0ull / d + 1 : 0; }

__device__ __forceinline__ uint32_t fdiv(uint32_t n, uint32_t d, uint64_t m) {
  if (m == 0) return d == 1 ? n : n / d;
  const uint64_t r = static_cast<uint64_t>(n) * static_cast<uint32_t>(m >> 32) + __umulhi(n, static_cast<uint32_t>(m));
  return static_cast<uint32_t>(r >> 32);
}

struct TileGeom {
  uint64_t len;        // bytes per shard (this launch's range)
  uint32_t tps;        // tiles per stripe
  uint32_t total;      // tiles overall
  int stride;          // pointers per stripe in the table
  int out0;            // first output pointer within a stripe's entries
  int aligned;         // all pointers 16-B aligned -> vector path allowed
  uint32_t paged_slots;  // bit j: source pointer j is a paged base (mapped with src)
  uint64_t logical0;     // slice offset of this launch's byte 0 (for the page mapping)
  PageMap src;           // mapping of paged source slots
  PageMap dst;           // mapping of the outputs (dst.page_bytes == 0: contiguous)
  uint64_t tps_m;        // fastdiv_magic(tps)
  // Optional kernel-internal timing (gs_pipeline_set_timing): {first CTA
  // start, last warp end} in %globaltimer ns, combined with atomics across
  // every launch of one codec call. nullptr = off.
  unsigned long long* tstamp;
  // Paged launches walk tiles page-major (tile t -> stripe t % nstripes,
  // page-tile t / nstripes): consecutive CTAs then read the same (layer, K/V)
  // page of consecutive cache blocks, i.e. contiguous cache memory, instead
  // of 64 pages 2 MiB apart. 0 = stripe-major (contiguous slices).
  uint32_t nstripes;
  uint64_t nstripes_m;  // fastdiv_magic(nstripes)
  // Page-per-tile source mapping (set by the host for paged K1 when every
  // used source is a paged cache, pages -- and cache blocks, with a block
  // table -- are whole multiples of a tile, every token is valid, logical0 is
  // tile-aligned and the outputs are contiguous: the decode-block and prefill
  // chunk checkpoints): a tile is one piece of one page of one block, so its
  // cache offset comes from the tile index (and one table entry) alone, with
  // no per-thread page arithmetic or masking.
  uint32_t tile_pages;
};

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void stamp_start(const TileGeom& g) {
  if (g.tstamp && threadIdx.x == 0) atomicMin(&g.tstamp[0], globaltimer_ns());
}
// Called by every warp when it has issued its last store.
__device__ __forceinline__ void stamp_end(const TileGeom& g) {
  if (g.tstamp) {
    __threadfence();  // this warp's stores performed
    if ((threadIdx.x & 31) == 0) atomicMax(&g.tstamp[1], globaltimer_ns());
  }
}

__device__ __forceinline__ uint32_t tile_stripe(uint32_t t, const TileGeom& g) { return fdiv(t, g.tps, g.tps_m); }

// Offset of logical slice byte `logical` of stripe `s` inside a paged slot;
// `masked` = beyond the valid tokens of its segment.
__device__ __forceinline__ uint64_t paged_offset(const PageMap& m, uint32_t s, uint64_t logical, bool& masked) {
  const uint32_t o = static_cast<uint32_t>(logical);
  const uint32_t q = fdiv(o, m.page_bytes, m.page_m);
  const uint32_t in = o - q * m.page_bytes;
  const uint32_t t = fdiv(q, m.layers, m.layers_m);
  const uint32_t l = q - t * m.layers;
  masked = in >= m.valid_tokens * m.token_bytes;
  uint64_t r = static_cast<uint64_t>(l) * m.layer_stride + static_cast<uint64_t>(t) * m.kv_stride;
  if (m.table) {
    const uint32_t pi = fdiv(in, m.block_bytes, m.block_m);
    const int32_t blk = masked ? 0 : m.table[static_cast<uint64_t>(s) * m.table_stride + pi];
    r += static_cast<uint64_t>(blk) * m.block_bytes + (in - pi * m.block_bytes);
  } else {
    r += in;
  }
  return r;
}

// Same for byte `tile_logical + lane_off` of a CTA tile: when the whole 4 KiB
// tile sits inside one segment (and one cache block), the page arithmetic and
// the block-table lookup depend only on the tile (`paged_tile_base`, inputs
// uniform across the CTA, so the compiler keeps them on the uniform datapath);
// only an add + compare remain per thread. Every paged geometry of the
// configs (4 KiB blocks) takes this path.
struct PagedTile {
  uint64_t base;    // cache offset of the tile's first byte
  uint32_t in0;     // its offset inside the segment
  bool fast;        // the tile stays inside one segment and one block
};

__device__ __forceinline__ PagedTile paged_tile_base(const PageMap& m, uint32_t s, uint64_t tile_logical) {
  PagedTile pt{0, 0, false};
  const uint32_t u = static_cast<uint32_t>(tile_logical);
  const uint32_t q = fdiv(u, m.page_bytes, m.page_m);
  const uint32_t in0 = u - q * m.page_bytes;
  const uint32_t bb = m.table ? m.block_bytes : m.page_bytes;
  const uint32_t pi = m.table ? fdiv(in0, m.block_bytes, m.block_m) : 0;
  const uint32_t ib0 = in0 - pi * bb;
  if (in0 + static_cast<uint32_t>(kTile) <= m.page_bytes && ib0 + static_cast<uint32_t>(kTile) <= bb) {
    const uint32_t t = fdiv(q, m.layers, m.layers_m);
    const uint32_t l = q - t * m.layers;
    uint64_t r = static_cast<uint64_t>(l) * m.layer_stride + static_cast<uint64_t>(t) * m.kv_stride + ib0;
    if (m.table) {
      const bool tile_masked = in0 >= m.valid_tokens * m.token_bytes;  // whole tile beyond valid
      const int32_t blk = tile_masked ? 0 : m.table[static_cast<uint64_t>(s) * m.table_stride + pi];
      r += static_cast<uint64_t>(blk) * m.block_bytes;
    }
    pt.base = r;
    pt.in0 = in0;
    pt.fast = true;
  }
  return pt;
}

__device__ __forceinline__ uint64_t paged_offset_tile(const PageMap& m, uint32_t s, uint64_t tile_logical,
                                                      uint32_t lane_off, bool& masked) {
  const PagedTile pt = paged_tile_base(m, s, tile_logical);
  if (pt.fast) {
    masked = pt.in0 + lane_off >= m.valid_tokens * m.token_bytes;
    return pt.base + lane_off;
  }
  return paged_offset(m, s, tile_logical + lane_off, masked);
}

// ---- specialised back end --------------------------------------------------

// Spec provides: static constexpr CoefMatrix matrix(); NS (#columns), NO (#rows).
template <class Spec>
__device__ __forceinline__ void horner_apply(const uint4 (&src)[Spec::NS], uint4 (&out)[Spec::NO]) {
  constexpr CoefMatrix m = Spec::matrix();
#pragma unroll
  for (int i = 0; i < Spec::NO; ++i) {
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      uint32_t acc = 0;
      bool live = false;
#pragma unroll
      for (int b = 7; b >= 0; --b) {
        uint32_t s = 0;
        bool any = false;
#pragma unroll
        for (int j = 0; j < Spec::NS; ++j)
          if ((m.c[i][j] >> b) & 1u) {
            s ^= word(const_cast<uint4&>(src[j]), w);
            any = true;
          }
        if (live) {
          acc = xtime4_xor(acc, s);
        } else if (any) {
          acc = s;
          live = true;
        }
      }
      word(out[i], w) = acc;
    }
  }
}

template <class Spec>
__device__ constexpr bool column_used(int j) {
  constexpr CoefMatrix m = Spec::matrix();
  for (int i = 0; i < Spec::NO; ++i)
    if (m.c[i][j]) return true;
  return false;
}

template <class Spec>
__device__ constexpr uint32_t used_mask() {
  uint32_t m = 0;
  for (int j = 0; j < Spec::NS && j < 32; ++j)
    if (column_used<Spec>(j)) m |= 1u << j;
  return m;
}

// Each CTA tile covers kThreads * 16 * U bytes of every shard; thread t owns
// the 16-byte groups t, t + kThreads, ... so every warp access is 512
// contiguous bytes, and all loads of a tile are issued before any
// arithmetic. The host guarantees 16-B aligned pointers and len % 16 == 0
// (a ragged tail or misaligned shards go to the generic kernel instead), so
// this kernel carries no byte-granular code at all.
template <class Spec, int CAP, int U, bool PAGED>
__global__ void __launch_bounds__(kThreads) k_apply_special(const PtrTable<CAP> tab, const TileGeom g) {
  static_assert(U == 1, "one 16-byte group per thread per tile");
  stamp_start(g);
  for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
    uint32_t s, tin;
    if (PAGED && g.nstripes) {
      tin = fdiv(t, g.nstripes, g.nstripes_m);
      s = t - tin * g.nstripes;
    } else {
      s = tile_stripe(t, g);
      tin = t - s * g.tps;
    }
    const uint64_t off = static_cast<uint64_t>(tin) * kTile + threadIdx.x * kVec;
    if (off >= g.len) continue;
    const int base = static_cast<int>(s) * g.stride;
    uint4 src[Spec::NS];
    uint4 out[Spec::NO];
    if constexpr (!PAGED) {
#pragma unroll
      for (int j = 0; j < Spec::NS; ++j)
        src[j] = column_used<Spec>(j) ? ld_stream(tab.p[base + j] + off) : make_uint4(0, 0, 0, 0);
      horner_apply<Spec>(src, out);
#pragma unroll
      for (int i = 0; i < Spec::NO; ++i) st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + off, out[i]);
    } else if (g.tile_pages) {
      const uint32_t u = static_cast<uint32_t>(g.logical0) + tin * static_cast<uint32_t>(kTile);
      const uint32_t pg = fdiv(u, g.src.page_bytes, g.src.page_m);
      const uint32_t kv = fdiv(pg, g.src.layers, g.src.layers_m);
      const uint32_t in0 = u - pg * g.src.page_bytes;
      uint64_t soff = static_cast<uint64_t>(pg - kv * g.src.layers) * g.src.layer_stride +
                      static_cast<uint64_t>(kv) * g.src.kv_stride + threadIdx.x * kVec;
      if (g.src.table) {  // multi-block chunk: the tile's block from the table (whole tiles per block)
        const uint32_t pi = fdiv(in0, g.src.block_bytes, g.src.block_m);
        const int32_t blk = g.src.table[static_cast<uint64_t>(s) * g.src.table_stride + pi];
        soff += static_cast<uint64_t>(blk) * g.src.block_bytes + (in0 - pi * g.src.block_bytes);
      } else {
        soff += in0;
      }
#pragma unroll
      for (int j = 0; j < Spec::NS; ++j)
        src[j] = column_used<Spec>(j) ? ld_stream(tab.p[base + j] + soff) : make_uint4(0, 0, 0, 0);
      horner_apply<Spec>(src, out);
#pragma unroll
      for (int i = 0; i < Spec::NO; ++i) st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + off, out[i]);
    } else {
      bool smask = false, dmask = false;
      uint64_t soff = off, doff = off;
      const uint64_t tile_logical = g.logical0 + static_cast<uint64_t>(tin) * kTile;
      const uint32_t lane_off = threadIdx.x * kVec;
      if (g.paged_slots) soff = paged_offset_tile(g.src, s, tile_logical, lane_off, smask);
      if (g.dst.page_bytes) doff = paged_offset_tile(g.dst, s, tile_logical, lane_off, dmask);
      constexpr uint32_t used = used_mask<Spec>();
      if ((g.paged_slots & used) == used) {
        // every used source is a paged cache with the same geometry (K1 over
        // a paged KV cache): one address for all of them, and a masked token
        // (>= valid) is zero in every source, so its parity is zero -- no
        // loads, no per-source selects.
        if (!smask) {
#pragma unroll
          for (int j = 0; j < Spec::NS; ++j)
            src[j] = column_used<Spec>(j) ? ld_stream(tab.p[base + j] + soff) : make_uint4(0, 0, 0, 0);
          horner_apply<Spec>(src, out);
        } else {
#pragma unroll
          for (int i = 0; i < Spec::NO; ++i) out[i] = make_uint4(0, 0, 0, 0);
        }
      } else {
#pragma unroll
        for (int j = 0; j < Spec::NS; ++j) {
          src[j] = make_uint4(0, 0, 0, 0);
          if (column_used<Spec>(j)) {
            const bool paged = (g.paged_slots >> j) & 1u;
            if (!(paged && smask)) src[j] = ld_stream(tab.p[base + j] + (paged ? soff : off));
          }
        }
        horner_apply<Spec>(src, out);
      }
      if (!dmask) {
#pragma unroll
        for (int i = 0; i < Spec::NO; ++i)
          st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + doff, out[i]);
      }
    }
  }
  stamp_end(g);
}

// ---- generic back end ------------------------------------------------------

// Per (row, source) coefficient c: {L0, L1, H0, H1, C8, C128, 0, 0} where
// L = c*{0..7}, H = c*{0,16,..,112} (byte v of the 8-byte pair = entry v),
// C8 = c*8 and C128 = c*128 replicated into all four bytes.
struct CoefWords {
  uint32_t l0, l1, h0, h1, c8, c128, pad0, pad1;
};

GS_HD inline CoefWords make_coef_words(uint8_t c) {
  CoefWords w{};
  uint32_t l[2] = {0, 0}, h[2] = {0, 0};
  for (int v = 0; v < 8; ++v) {
    l[v >> 2] |= static_cast<uint32_t>(gf_mul(c, static_cast<uint8_t>(v))) << (8 * (v & 3));
    h[v >> 2] |= static_cast<uint32_t>(gf_mul(c, static_cast<uint8_t>(v << 4))) << (8 * (v & 3));
  }
  w.l0 = l[0];
  w.l1 = l[1];
  w.h0 = h[0];
  w.h1 = h[1];
  w.c8 = 0x01010101u * gf_mul(c, 8);
  w.c128 = 0x01010101u * gf_mul(c, 128);
  return w;
}

struct PairSel {
  uint32_t loP, hiP, loQ, hiQ, m3P, m3Q, m7P, m7Q;
};

// Selectors for the pair of data words (x, y). Domain P holds byte order
// [x0, y0, x1, y1], domain Q holds [x2, y2, x3, y3].
__device__ __forceinline__ PairSel pair_setup(uint32_t x, uint32_t y) {
  PairSel s;
  const uint32_t lo = (x & 0x07070707u) | ((y & 0x07070707u) << 4);
  const uint32_t hi = ((x >> 4) & 0x07070707u) | (y & 0x70707070u);
  s.loP = lo;
  s.loQ = lo >> 16;
  s.hiP = hi;
  s.hiQ = hi >> 16;
  s.m7P = prmt(x, y, 0xD9C8u);
  s.m7Q = prmt(x, y, 0xFBEAu);
  const uint32_t x4 = x << 4, y4 = y << 4;
  s.m3P = prmt(x4, y4, 0xD9C8u);
  s.m3Q = prmt(x4, y4, 0xFBEAu);
  return s;
}

__device__ __forceinline__ void pair_mac(uint32_t& accP, uint32_t& accQ, const PairSel& s,
                                         const CoefWords& c) {
  accP ^= prmt(c.l0, c.l1, s.loP) ^ prmt(c.h0, c.h1, s.hiP);
  accP ^= s.m3P & c.c8;
  accP ^= s.m7P & c.c128;
  accQ ^= prmt(c.l0, c.l1, s.loQ) ^ prmt(c.h0, c.h1, s.hiQ);
  accQ ^= s.m3Q & c.c8;
  accQ ^= s.m7Q & c.c128;
}

// Undo the pair permutation: x = [P0, P2, Q0, Q2], y = [P1, P3, Q1, Q3].
__device__ __forceinline__ void pair_finish(uint32_t accP, uint32_t accQ, uint32_t& x, uint32_t& y) {
  x = prmt(accP, accQ, 0x6420u);
  y = prmt(accP, accQ, 0x7531u);
}

// One 16-byte group of every source -> KB outputs. FULL: 16-B vector
// loads/stores; otherwise byte-granular (ragged tail / misaligned shards).
template <int KB, int CAP, bool FULL>
__device__ __forceinline__ void generic_group(const PtrTable<CAP>& tab, int base, int out0, uint64_t off,
                                              int nb, const CoefWords* sc, int ns, const TileGeom& g,
                                              uint32_t stripe) {
  bool smask = false, dmask = false;
  uint64_t soff = off, doff = off;
  if (FULL && g.paged_slots) soff = paged_offset(g.src, stripe, g.logical0 + off, smask);
  if (FULL && g.dst.page_bytes) doff = paged_offset(g.dst, stripe, g.logical0 + off, dmask);
  uint32_t acc[KB][4];
#pragma unroll
  for (int r = 0; r < KB; ++r)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[r][q] = 0;
  int j = 0;
  for (; j + 4 <= ns; j += 4) {
    uint4 d[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool paged = FULL && ((g.paged_slots >> (j + u)) & 1u);
      const uint8_t* p = tab.p[base + j + u] + (paged ? soff : off);
      d[u] = (paged && smask) ? make_uint4(0, 0, 0, 0) : (FULL ? ld_stream(p) : ld_partial(p, nb));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const PairSel s0 = pair_setup(d[u].x, d[u].y);
      const PairSel s1 = pair_setup(d[u].z, d[u].w);
#pragma unroll
      for (int r = 0; r < KB; ++r) {
        const CoefWords c = sc[r * ns + j + u];
        pair_mac(acc[r][0], acc[r][1], s0, c);
        pair_mac(acc[r][2], acc[r][3], s1, c);
      }
    }
  }
  for (; j < ns; ++j) {
    const bool paged = FULL && ((g.paged_slots >> j) & 1u);
    const uint8_t* p = tab.p[base + j] + (paged ? soff : off);
    const uint4 d = (paged && smask) ? make_uint4(0, 0, 0, 0) : (FULL ? ld_stream(p) : ld_partial(p, nb));
    const PairSel s0 = pair_setup(d.x, d.y);
    const PairSel s1 = pair_setup(d.z, d.w);
#pragma unroll
    for (int r = 0; r < KB; ++r) {
      const CoefWords c = sc[r * ns + j];
      pair_mac(acc[r][0], acc[r][1], s0, c);
      pair_mac(acc[r][2], acc[r][3], s1, c);
    }
  }
#pragma unroll
  for (int r = 0; r < KB; ++r) {
    uint4 o;
    pair_finish(acc[r][0], acc[r][1], o.x, o.y);
    pair_finish(acc[r][2], acc[r][3], o.z, o.w);
    uint8_t* p = const_cast<uint8_t*>(tab.p[base + out0 + r]) + doff;
    if (FULL) {
      if (!dmask) st_stream(p, o);
    } else {
      st_partial(p, o, nb);
    }
  }
}

// coef: rows x ns CoefWords for this launch's row group (row-major), staged
// in shared memory (broadcast reads: every thread uses the same entry).
template <int KB, int CAP>
__global__ void __launch_bounds__(kThreads) k_apply_generic(const PtrTable<CAP> tab, const TileGeom g,
                                                            const CoefWords* __restrict__ coef,
                                                            int ns) {
  extern __shared__ uint4 smem_coef[];
  CoefWords* sc = reinterpret_cast<CoefWords*>(smem_coef);
  stamp_start(g);
  for (int i = threadIdx.x; i < KB * ns; i += blockDim.x) sc[i] = coef[i];
  __syncthreads();

  for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
    const uint32_t s = tile_stripe(t, g);
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * kTile + threadIdx.x * kVec;
    if (off >= g.len) continue;
    const int base = static_cast<int>(s) * g.stride;
    if (g.aligned && off + kVec <= g.len) {
      generic_group<KB, CAP, true>(tab, base, g.out0, off, kVec, sc, ns, g, s);
    } else {
      const uint64_t rem = g.len - off;
      generic_group<KB, CAP, false>(tab, base, g.out0, off, static_cast<int>(rem < kVec ? rem : kVec), sc, ns, g,
                                    s);
    }
  }
  stamp_end(g);
}

// ============================================================================
// Bulk-copy pipelined specialised kernel (K1/K2 "bulk" variant).
//
// One persistent CTA per SM: warp 0 is a producer that streams each tile of
// every used source into a ring of shared-memory stages with
// cp.async.bulk (the TMA engine's 1-D bulk path, completion on an mbarrier);
// CW consumer warps wait on the stage's full barrier, read their 16-byte
// groups with LDS.128, run the Horner arithmetic and store the outputs with
// STG.128, then release the stage. Memory-level parallelism is set by the
// ring depth (stages x sources x tile bytes, ~200 KB per SM), independent of
// registers and occupancy; the arithmetic of tile i overlaps the loads of
// tiles i+1..i+S-1.
// ============================================================================
namespace bulk {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ uint4 lds128(const uint8_t* p) {
  uint4 r;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "r"(smem_u32(p)));
  return r;
}

constexpr int kMaxStages = 8;

template <class Spec>
struct UsedCols {
  int n = 0;
  int col[2 * kMaxSpecial] = {};
};

template <class Spec>
__host__ __device__ constexpr UsedCols<Spec> used_cols() {
  constexpr CoefMatrix m = Spec::matrix();
  UsedCols<Spec> u{};
  for (int j = 0; j < Spec::NS; ++j) {
    bool any = false;
    for (int i = 0; i < Spec::NO; ++i) any = any || m.c[i][j] != 0;
    if (any) u.col[u.n++] = j;
  }
  return u;
}

}  // namespace bulk

// CW consumer warps; every consumer thread owns U 16-byte groups per tile,
// so a tile is CW*32*16*U bytes of every used source.
template <class Spec, int CAP, int CW, int U>
__global__ void __launch_bounds__((CW + 1) * 32, 1)
    k_apply_special_bulk(const PtrTable<CAP> tab, const TileGeom g, int stages) {
  constexpr bulk::UsedCols<Spec> uc = bulk::used_cols<Spec>();
  constexpr int NU = uc.n;
  constexpr uint32_t T = CW * 32 * kVec * U;  // tile bytes per source
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);
  uint64_t* empty = full + bulk::kMaxStages;
  uint8_t* ring = smem + 2 * bulk::kMaxStages * sizeof(uint64_t) + 112;  // 128-B aligned data

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      bulk::mbar_init(&full[s], 1);
      bulk::mbar_init(&empty[s], CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  stamp_start(g);

  if (warp == CW) {  // ---- producer warp (one elected lane issues) ----
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
        const uint32_t s = tile_stripe(t, g);
        const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * T;
        const uint32_t size = static_cast<uint32_t>(g.len - off < T ? g.len - off : T);
        const int base = static_cast<int>(s) * g.stride;
        bulk::mbar_wait(&empty[stage], phase ^ 1u);
        bulk::mbar_expect_tx(&full[stage], size * NU);
#pragma unroll
        for (int u = 0; u < NU; ++u)
          bulk::bulk_g2s(ring + (static_cast<size_t>(stage) * NU + u) * T, tab.p[base + uc.col[u]] + off, size,
                         &full[stage]);
        if (++stage == stages) {
          stage = 0;
          phase ^= 1u;
        }
      }
    }
    return;
  }

  // ---- consumer warps ----
  int stage = 0;
  uint32_t phase = 0;
  const uint32_t tid = threadIdx.x;  // 0 .. CW*32-1
  for (uint32_t t = blockIdx.x; t < g.total; t += gridDim.x) {
    const uint32_t s = tile_stripe(t, g);
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * T;
    const uint32_t size = static_cast<uint32_t>(g.len - off < T ? g.len - off : T);
    const int base = static_cast<int>(s) * g.stride;
    bulk::mbar_wait(&full[stage], phase);
    const uint8_t* st = ring + static_cast<size_t>(stage) * NU * T;
    uint4 src[U][Spec::NS];
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const uint32_t idx = (v * CW * 32 + tid) * kVec;
#pragma unroll
      for (int j = 0; j < Spec::NS; ++j) src[v][j] = make_uint4(0, 0, 0, 0);
      if (idx < size) {
#pragma unroll
        for (int u = 0; u < NU; ++u) src[v][uc.col[u]] = bulk::lds128(st + u * T + idx);
      }
    }
    __syncwarp();
    if (lane == 0) bulk::mbar_arrive(&empty[stage]);
#pragma unroll
    for (int v = 0; v < U; ++v) {
      const uint32_t idx = (v * CW * 32 + tid) * kVec;
      if (idx < size) {
        uint4 out[Spec::NO];
        horner_apply<Spec>(src[v], out);
#pragma unroll
        for (int i = 0; i < Spec::NO; ++i)
          st_stream(const_cast<uint8_t*>(tab.p[base + g.out0 + i]) + off + idx, out[i]);
      }
    }
    if (++stage == stages) {
      stage = 0;
      phase ^= 1u;
    }
  }
  stamp_end(g);
}

}  // namespace gsb
