// gs_rdp.cuh -- shortened RDP (row-diagonal parity) on sm_100a.
//
// Reference: coding.hpp:225-251 (layout), :277-307 (encode), :343-449
// (two-column recovery), :503-534 (dispatch). The array is (p-1) rows x
// (p+1) columns for the smallest prime p >= n+1; a "dstripe" is p-1
// consecutive bytes of every column. Data columns 0..n-1 (n..p-2 virtual
// zero), row parity = column p-1 (= byte-wise XOR of the data), diagonal
// d = (r + c) mod p stored at row d of the diagonal buffer for d <= p-2.
// Bytes past the last whole dstripe are protected by P (row parity) and
// Q = sum_c 2^c * data_c over GF(2^8).
//
// RDP is position-dependent, so unlike XOR/RS it cannot stream 16-byte
// groups straight through registers: each CTA stages a tile of 256
// dstripes of every column in shared memory with coalesced loads, one
// thread per dstripe evaluates the diagonals (or walks the two recovery
// chains) out of shared memory, and the results leave through shared memory
// with coalesced stores. Single-column recoveries are plain XORs and run on
// the XOR kernels instead.
#pragma once

#include <cstdint>

#include "gs_kernels.cuh"

namespace gsb {

constexpr int kRdpThreads = 256;  // one dstripe per thread per tile
constexpr int kRdpMaxCols = 24;   // p <= 23 -> n <= 22 on this path

// Primes with kernels (p = smallest prime >= n+1 for n = 1..22).
#define GS_RDP_PRIMES(X) X(2) X(3) X(5) X(7) X(11) X(13) X(17) X(19) X(23)

struct RdpGeom {
  int n, p, rows;
  uint64_t len;       // bytes of this launch's range (per column)
  uint64_t logical0;  // absolute offset of byte 0 of the range (multiple of rows)
  uint64_t full;      // absolute end of the whole dstripes
  uint64_t total;     // absolute column length
  uint32_t tps, ntiles;
  int stride;         // pointers per codec stripe in the table
  int aligned;
  // recovery: the two lost array columns (i < j; j == p-1 => row parity lost)
  int li, lj;
  // recovery tail (coding.hpp:415-448): gj = 2^j, inv = 1 / 2^i (j == p-1)
  // or 1 / (2^i ^ 2^j)
  uint8_t gj, inv;
  // pipelined kernels: P/Q tail bytes after the whole-dstripe body `len`
  // (only in a column's last range), handled by the last tile's CTA
  uint32_t tail;
};

// P/Q tail arithmetic: Q = sum_c 2^c d_c is evaluated by Horner (one
// multiply-by-x per column); the two remaining general products of the
// recovery use launch-uniform coefficients computed on the host (RdpGeom
// gj, inv), so no tail byte runs an inversion.
__device__ __forceinline__ uint8_t xtime1(uint8_t a) {
  return static_cast<uint8_t>((a << 1) ^ ((a & 0x80u) ? 0x1Du : 0u));
}

// (a mod p) for a in (-p, 2p): one compare-and-add instead of an integer
// division (all the array index arithmetic stays in that range).
__device__ __forceinline__ int pmod(int a, int p) {
  a = a < 0 ? a + p : a;
  return a >= p ? a - p : a;
}

// All columns of a tile at once: `cols` sources (nullptr = a zero column)
// into smem tiles dst + c*T. On the aligned path each thread issues its
// 16-byte loads of EVERY column before storing any, so the column loads
// overlap instead of paying one memory latency per column.
template <int MAXC>
__device__ __forceinline__ void rdp_load_cols(uint8_t* dst, uint32_t T, const uint8_t* const* src, int cols,
                                              uint32_t bytes, bool aligned) {
  if (!aligned) {
    for (int c = 0; c < cols; ++c) {
      uint8_t* d = dst + static_cast<size_t>(c) * T;
      for (uint32_t b = threadIdx.x; b < T; b += blockDim.x) d[b] = (src[c] && b < bytes) ? src[c][b] : 0;
    }
    return;
  }
  const uint32_t vec = bytes / 16, rem = bytes % 16, nv = T / 16;
  for (uint32_t v0 = 0; v0 < nv; v0 += blockDim.x) {
    const uint32_t v = v0 + threadIdx.x;
    uint4 r[MAXC];
#pragma unroll
    for (int c = 0; c < MAXC; ++c) {
      r[c] = make_uint4(0, 0, 0, 0);
      if (c < cols && src[c] && v < nv) {
        if (v < vec)
          r[c] = ld_stream(src[c] + static_cast<size_t>(v) * 16);
        else if (v == vec && rem)
          r[c] = ld_partial(src[c] + static_cast<size_t>(v) * 16, static_cast<int>(rem));
      }
    }
    if (v < nv) {
#pragma unroll
      for (int c = 0; c < MAXC; ++c)
        if (c < cols) reinterpret_cast<uint4*>(dst + static_cast<size_t>(c) * T)[v] = r[c];
    }
  }
}

__device__ __forceinline__ void rdp_store(uint8_t* dst, const uint8_t* src, uint32_t bytes, bool aligned) {
  if (aligned) {
    const uint32_t vec = bytes / 16;
    for (uint32_t v = threadIdx.x; v < vec; v += blockDim.x)
      st_stream(dst + v * 16, reinterpret_cast<const uint4*>(src)[v]);
    for (uint32_t b = vec * 16 + threadIdx.x; b < bytes; b += blockDim.x) dst[b] = src[b];
  } else {
    for (uint32_t b = threadIdx.x; b < bytes; b += blockDim.x) dst[b] = src[b];
  }
}

// Encode: out0 = row parity (whole range), out1 = diagonal parity (whole
// dstripes) + Q (tail). smem: p-1 column tiles (virtual columns n..p-2 are
// zero, so the diagonal loop is the same for every n) + row + diag tiles.
// P is a template parameter: every index in the diagonal loop is a
// compile-time constant and the 90-odd byte XORs per dstripe fully unroll.
template <int CAP, int P>
__global__ void __launch_bounds__(kRdpThreads) k_rdp_encode(const PtrTable<CAP> tab, const RdpGeom g) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int R = P - 1;
  constexpr uint32_t T = static_cast<uint32_t>(R) * kRdpThreads;
  const int n = g.n;
  uint8_t* data = sm;
  uint8_t* rowp = sm + static_cast<size_t>(R) * T;
  uint8_t* diag = rowp + T;
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * T;
    const uint32_t bytes = static_cast<uint32_t>(g.len - off < T ? g.len - off : T);
    const int base = static_cast<int>(s) * g.stride;
    __syncthreads();  // previous tile's smem fully consumed
    {
      const uint8_t* srcs[R];
#pragma unroll
      for (int c = 0; c < R; ++c) srcs[c] = c < n ? tab.p[base + c] + off : nullptr;  // n..p-2: virtual zero
      rdp_load_cols<R>(data, T, srcs, R, bytes, g.aligned);
    }
    __syncthreads();
    for (uint32_t v16 = threadIdx.x; v16 < T / 16; v16 += blockDim.x) {  // T = rows * 256: 16-B multiple
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int c = 0; c < n; ++c) {
        const uint4 x = reinterpret_cast<const uint4*>(data + static_cast<size_t>(c) * T)[v16];
        v.x ^= x.x;
        v.y ^= x.y;
        v.z ^= x.z;
        v.w ^= x.w;
      }
      reinterpret_cast<uint4*>(rowp)[v16] = v;
    }
    __syncthreads();
    // one whole dstripe per thread
    const uint64_t abs0 = g.logical0 + off;
    const uint32_t sb = threadIdx.x * R;
    if (sb < bytes && abs0 + sb + R <= g.full) {
      uint8_t dv[R];
#pragma unroll
      for (int d = 0; d < R; ++d) {
        uint8_t v = 0;
#pragma unroll
        for (int c = 0; c < R; ++c) {
          const int r = (d - c + P) % P;
          if (r != P - 1) v ^= data[static_cast<size_t>(c) * T + sb + r];
        }
        const int r = (d + 1) % P;  // row-parity column p-1
        if (r != P - 1) v ^= rowp[sb + r];
        dv[d] = v;
      }
#pragma unroll
      for (int d = 0; d < R; ++d) diag[sb + d] = dv[d];
    }
    // tail bytes past the last whole dstripe (only in a column's last tile):
    // Q = sum_c 2^c * data_c, one byte per thread
    const uint64_t tail0 = g.full > abs0 ? g.full - abs0 : 0;
    for (uint64_t x = tail0 + threadIdx.x; x < bytes; x += blockDim.x) {
      uint8_t v = 0;
      for (int c = n - 1; c >= 0; --c) v = xtime1(v) ^ data[static_cast<size_t>(c) * T + x];
      diag[x] = v;
    }
    __syncthreads();
    rdp_store(const_cast<uint8_t*>(tab.p[base + n]) + off, rowp, bytes, g.aligned);
    rdp_store(const_cast<uint8_t*>(tab.p[base + n + 1]) + off, diag, bytes, g.aligned);
  }
}

// Two-column recovery with the diagonal parity present. Slots per codec
// stripe: data 0..n-1 (NULL if lost), row parity (NULL if lost), diagonal;
// outputs: the lost data columns (ascending). smem: p column tiles (array
// order, lost ones are the outputs being built, virtual ones zero) + diag.
template <int CAP, int P>
__global__ void __launch_bounds__(kRdpThreads) k_rdp_recover(const PtrTable<CAP> tab, const RdpGeom g, int n_out,
                                                             int out0) {
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr int p = P, rows = P - 1;
  constexpr uint32_t T = static_cast<uint32_t>(rows) * kRdpThreads;
  const int n = g.n;
  uint8_t* col = sm;                                   // p tiles
  uint8_t* diag = sm + static_cast<size_t>(p) * T;
  const int i = g.li, j = g.lj;
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * T;
    const uint32_t bytes = static_cast<uint32_t>(g.len - off < T ? g.len - off : T);
    const int base = static_cast<int>(s) * g.stride;
    __syncthreads();
    {
      // p array columns (lost ones are the outputs being built, virtual ones
      // zero) followed by the diagonal buffer: p + 1 consecutive smem tiles
      const uint8_t* srcs[P + 1];
#pragma unroll
      for (int c = 0; c < P; ++c) {
        const uint8_t* src = c < n ? tab.p[base + c] : (c == P - 1 ? tab.p[base + n] : nullptr);
        srcs[c] = (c == i || c == j || src == nullptr) ? nullptr : src + off;
      }
      srcs[P] = tab.p[base + n + 1] + off;
      rdp_load_cols<P + 1>(col, T, srcs, P + 1, bytes, g.aligned);
    }
    __syncthreads();
    const uint64_t abs0 = g.logical0 + off;
    const uint32_t sb = threadIdx.x * rows;
    if (sb < bytes && abs0 + sb + rows <= g.full) {
      uint8_t* ci = col + static_cast<size_t>(i) * T + sb;
      uint8_t* cj = col + static_cast<size_t>(j) * T + sb;
      // coding.hpp:384-413: chain (primary i, partner j) then (j, i).
      for (int pass = 0; pass < 2; ++pass) {
        const int prim = pass == 0 ? i : j, part = pass == 0 ? j : i;
        uint8_t* po = pass == 0 ? ci : cj;
        uint8_t* qo = pass == 0 ? cj : ci;
        int d = pmod(part - 1, p);
        const int step = pmod(part - prim, p);
        while (d != p - 1) {
          const int r = pmod(d - prim, p);
          uint8_t v = diag[sb + d];
#pragma unroll
          for (int c = 0; c < p; ++c) {
            if (c == prim) continue;
            const int rc = pmod(d - c, p);
            if (rc != p - 1) v ^= col[static_cast<size_t>(c) * T + sb + rc];
          }
          po[r] = v;
          uint8_t w = 0;
#pragma unroll
          for (int c = 0; c < p; ++c)
            if (c != part) w ^= col[static_cast<size_t>(c) * T + sb + r];
          qo[r] = w;
          d = pmod(d + step, p);
        }
      }
    }
    // coding.hpp:415-448: P/Q algebra on the tail bytes, one byte per thread.
    const uint64_t tail0 = g.full > abs0 ? g.full - abs0 : 0;
    for (uint64_t x = tail0 + threadIdx.x; x < bytes; x += blockDim.x) {
      uint8_t ps = 0, h = 0;
      for (int c = n - 1; c >= 0; --c) {
        const uint8_t v = (c == i || c == j) ? 0 : col[static_cast<size_t>(c) * T + x];
        ps ^= v;
        h = xtime1(h) ^ v;
      }
      const uint8_t qs = diag[x] ^ h;
      uint8_t* ci = col + static_cast<size_t>(i) * T;
      uint8_t* cj = col + static_cast<size_t>(j) * T;
      if (j == p - 1) {
        const uint8_t di = gf_mul(qs, g.inv);
        ci[x] = di;
        cj[x] = static_cast<uint8_t>(ps ^ di);
      } else {
        ps ^= col[static_cast<size_t>(p - 1) * T + x];
        const uint8_t di = gf_mul(static_cast<uint8_t>(qs ^ gf_mul(g.gj, ps)), g.inv);
        ci[x] = di;
        cj[x] = static_cast<uint8_t>(ps ^ di);
      }
    }
    __syncthreads();
    int o = 0;
    if (i < n) rdp_store(const_cast<uint8_t*>(tab.p[base + out0 + o++]) + off, col + static_cast<size_t>(i) * T, bytes,
                         g.aligned);
    if (j < n && o < n_out)
      rdp_store(const_cast<uint8_t*>(tab.p[base + out0 + o]) + off, col + static_cast<size_t>(j) * T, bytes,
                g.aligned);
  }
}


// ============================================================================
// Pipelined RDP kernels (whole-dstripe body of a launch range).
//
// Same producer/consumer shape as k_apply_special_bulk: one persistent CTA
// per SM, a producer warp streams COLUMN tiles (1024 dstripes = 1024*(p-1)
// bytes of one column) into a shared-memory ring with cp.async.bulk, CW
// consumer warps take them in column order. Each consumer thread owns 4
// consecutive dstripes: it loads their 4*(p-1) bytes of a column (LDS.64) and
// transposes them in registers into p-1 "row words" -- word r = byte r of
// each of the 4 dstripes (3 PRMT per word). In that domain a diagonal
// (r + c) mod p is a compile-time register index for every (r, c), so the
// row parity and all diagonals are plain 32-bit XORs over 4 dstripes at once
// (the column loop is unrolled over 0..p-2; columns >= n are the virtual
// zero columns and are skipped). Results are transposed back, staged in
// shared memory and written with cp.async.bulk (TMA bulk store).
// ============================================================================
namespace rdpb {

constexpr int kCW = 8;                                  // consumer warps
constexpr int kNT = kCW * 32;                           // consumer threads
constexpr int kDsPerThread = 4;                         // dstripes per thread per tile
constexpr int kTileDs = kNT * kDsPerThread;             // dstripes per tile (1024)
constexpr int kMaxStages = 16;
constexpr size_t kSmemBudget = 220 * 1024;
constexpr size_t kHeader = 1024;                        // barriers, 128-B aligned data after

__host__ __device__ constexpr uint32_t tile_bytes(int p) { return static_cast<uint32_t>(p - 1) * kTileDs; }
// chain scratch of the recovery kernel: sr[R], sd[R], ai[R+1], aj[R+1] words per thread
__host__ __device__ constexpr size_t chain_bytes(int p) { return static_cast<size_t>(4 * (p - 1) + 2) * kNT * 4; }
__host__ __device__ constexpr size_t out_bytes(int p) { return 2u * 2u * tile_bytes(p); }  // 2 buffers x 2 outputs

// byte q of the thread's 4*R-byte natural block (words w[q >> 2])
template <int R>
__device__ __forceinline__ uint32_t nat_byte_sel(int q) { return static_cast<uint32_t>(q & 3); }

// rows[r] = {byte r of dstripe 0, of dstripe 1, of dstripe 2, of dstripe 3}
template <int R>
__device__ __forceinline__ void to_rows(const uint32_t (&w)[R], uint32_t (&rows)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int q0 = r, q1 = R + r, q2 = 2 * R + r, q3 = 3 * R + r;
    const uint32_t lo = __byte_perm(w[q0 >> 2], w[q1 >> 2], (q0 & 3) | ((4 + (q1 & 3)) << 4));
    const uint32_t hi = __byte_perm(w[q2 >> 2], w[q3 >> 2], (q2 & 3) | ((4 + (q3 & 3)) << 4));
    rows[r] = __byte_perm(lo, hi, 0x5410);
  }
}

// inverse: natural word v = bytes q = 4v..4v+3, byte q = byte (q / R) of rows[q % R]
template <int R>
__device__ __forceinline__ void from_rows(const uint32_t (&rows)[R], uint32_t (&w)[R]) {
#pragma unroll
  for (int v = 0; v < R; ++v) {
    const int q0 = 4 * v, q1 = q0 + 1, q2 = q0 + 2, q3 = q0 + 3;
    const uint32_t lo = __byte_perm(rows[q0 % R], rows[q1 % R], (q0 / R) | ((4 + q1 / R) << 4));
    const uint32_t hi = __byte_perm(rows[q2 % R], rows[q3 % R], (q2 / R) | ((4 + q3 / R) << 4));
    w[v] = __byte_perm(lo, hi, 0x5410);
  }
}

template <int R>
__device__ __forceinline__ void lds_block(const uint8_t* p, uint32_t (&w)[R]) {
  if constexpr (R % 2 == 0) {
#pragma unroll
    for (int v = 0; v < R / 2; ++v) {
      uint32_t a, b;
      asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(bulk::smem_u32(p + 8 * v)));
      w[2 * v] = a;
      w[2 * v + 1] = b;
    }
  } else {
#pragma unroll
    for (int v = 0; v < R; ++v)
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w[v]) : "r"(bulk::smem_u32(p + 4 * v)));
  }
}

template <int R>
__device__ __forceinline__ void sts_block(uint8_t* p, const uint32_t (&w)[R]) {
  if constexpr (R % 2 == 0) {
#pragma unroll
    for (int v = 0; v < R / 2; ++v)
      asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(bulk::smem_u32(p + 8 * v)), "r"(w[2 * v]),
                   "r"(w[2 * v + 1])
                   : "memory");
  } else {
#pragma unroll
    for (int v = 0; v < R; ++v)
      asm volatile("st.shared.u32 [%0], %1;" ::"r"(bulk::smem_u32(p + 4 * v)), "r"(w[v]) : "memory");
  }
}

__device__ __forceinline__ void bulk_s2g(void* gdst, const void* ssrc, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst),
               "r"(bulk::smem_u32(ssrc)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kNT) : "memory"); }

struct Ring {
  uint64_t* full;
  uint64_t* empty;
  uint8_t* data;
  int stages;
  uint32_t tb;
  int stage = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void advance() {
    if (++stage == stages) {
      stage = 0;
      phase ^= 1u;
    }
  }
};

// Producer: for every tile, stream the listed column slots in order.
template <int CAP>
__device__ __forceinline__ void rdp_produce(const PtrTable<CAP>& tab, const RdpGeom& g, Ring ring,
                                            const int* cols, int ncols) {
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * ring.tb;
    const int base = static_cast<int>(s) * g.stride;
    // the last tile of a range may be partial (whole dstripes, any count):
    // the 16-byte-multiple part goes through the bulk engine, the < 16-byte
    // rest is copied by this lane before the arrive that publishes it
    const uint32_t size = static_cast<uint32_t>(g.len - off < ring.tb ? g.len - off : ring.tb);
    const uint32_t bsz = size & ~15u;
    for (int u = 0; u < ncols; ++u) {
      bulk::mbar_wait(&ring.empty[ring.stage], ring.phase ^ 1u);
      uint8_t* dst = ring.data + static_cast<size_t>(ring.stage) * ring.tb;
      const uint8_t* src = tab.p[base + cols[u]] + off;
      for (uint32_t b = bsz; b < size; ++b) dst[b] = src[b];
      bulk::mbar_expect_tx(&ring.full[ring.stage], bsz);
      if (bsz) bulk::bulk_g2s(dst, src, bsz, &ring.full[ring.stage]);
      ring.advance();
    }
  }
}

// Consumer: take the next column stage, return the thread's row words.
template <int R>
__device__ __forceinline__ void take_rows(Ring& ring, uint32_t (&rows)[R]) {
  bulk::mbar_wait(&ring.full[ring.stage], ring.phase);
  uint32_t w[R];
  lds_block<R>(ring.data + static_cast<size_t>(ring.stage) * ring.tb + threadIdx.x * (4 * R), w);
  __syncwarp();
  if ((threadIdx.x & 31) == 0) bulk::mbar_arrive(&ring.empty[ring.stage]);
  ring.advance();
  to_rows<R>(w, rows);
}

__device__ __forceinline__ void init_ring(uint8_t* smem, int stages, Ring& ring, uint32_t tb) {
  ring.full = reinterpret_cast<uint64_t*>(smem);
  ring.empty = ring.full + kMaxStages;
  ring.data = smem + kHeader;
  ring.stages = stages;
  ring.tb = tb;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      bulk::mbar_init(&ring.full[s], 1);
      bulk::mbar_init(&ring.empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// Stage the thread's natural words of output `o` of buffer `buf`, then (one
// thread) bulk-store the tile. Buffer reuse is guarded by wait_group.read 1.
template <int R>
__device__ __forceinline__ void out_stage(uint8_t* outbuf, int buf, int o, uint32_t tb, const uint32_t (&rows)[R]) {
  uint32_t w[R];
  from_rows<R>(rows, w);
  sts_block<R>(outbuf + (static_cast<size_t>(buf) * 2 + o) * tb + threadIdx.x * (4 * R), w);
}

// One thread: write `size` bytes of a staged output tile (bulk engine for the
// 16-byte multiple, plain stores for the rest).
__device__ __forceinline__ void store_tile(uint8_t* gdst, const uint8_t* ssrc, uint32_t size) {
  const uint32_t bsz = size & ~15u;
  if (bsz) bulk_s2g(gdst, ssrc, bsz);
  for (uint32_t b = bsz; b < size; ++b) gdst[b] = ssrc[b];
}

}  // namespace rdpb

// P/Q tail of a column (coding.hpp:237-241, 300-306): bytes [x0, x0 + cnt) past
// the last whole dstripe, one byte per lane, straight from global memory.
template <int CAP>
__device__ __forceinline__ void rdp_encode_tail(const PtrTable<CAP>& tab, int base, int n, uint64_t x0,
                                                uint32_t cnt) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane >= cnt) return;
  const uint64_t x = x0 + lane;
  uint8_t pp = 0, h = 0;
  for (int c = n - 1; c >= 0; --c) {
    const uint8_t v = tab.p[base + c][x];
    pp ^= v;
    h = xtime1(h) ^ v;
  }
  const_cast<uint8_t*>(tab.p[base + n])[x] = pp;
  const_cast<uint8_t*>(tab.p[base + n + 1])[x] = h;
}

// coding.hpp:415-448 on the tail bytes (slots: data 0..n-1, row parity n,
// diagonal n+1; outputs out0.. = lost data columns ascending).
template <int CAP, int P>
__device__ __forceinline__ void rdp_recover_tail(const PtrTable<CAP>& tab, const RdpGeom& g, int base, int out0,
                                                 int n_out, uint64_t x0, uint32_t cnt) {
  const uint32_t lane = threadIdx.x & 31;
  if (lane >= cnt) return;
  const uint64_t x = x0 + lane;
  const int n = g.n, i = g.li, j = g.lj;
  uint8_t ps = 0, h = 0;
  for (int c = n - 1; c >= 0; --c) {
    const uint8_t v = (c == i || c == j) ? 0 : tab.p[base + c][x];
    ps ^= v;
    h = xtime1(h) ^ v;
  }
  const uint8_t qs = tab.p[base + n + 1][x] ^ h;
  uint8_t di, dj;
  if (j == P - 1) {
    di = gf_mul(qs, g.inv);
    dj = 0;
  } else {
    ps ^= tab.p[base + n][x];
    di = gf_mul(static_cast<uint8_t>(qs ^ gf_mul(g.gj, ps)), g.inv);
    dj = static_cast<uint8_t>(ps ^ di);
  }
  const_cast<uint8_t*>(tab.p[base + out0])[x] = di;
  if (n_out > 1 && j < n) const_cast<uint8_t*>(tab.p[base + out0 + 1])[x] = dj;
}

template <int CAP, int P>
__global__ void __launch_bounds__((rdpb::kCW + 1) * 32, 1)
    k_rdp_encode_bulk(const PtrTable<CAP> tab, const RdpGeom g, int stages) {
  using namespace rdpb;
  constexpr int R = P - 1;
  constexpr uint32_t TB = tile_bytes(P);
  extern __shared__ __align__(128) uint8_t smem[];
  Ring ring;
  init_ring(smem, stages, ring, TB);
  uint8_t* outbuf = ring.data + static_cast<size_t>(stages) * TB;
  const int n = g.n;
  if (threadIdx.x >= kNT) {  // producer warp
    if ((threadIdx.x & 31) == 0) {
      int cols[kRdpMaxCols];
      for (int c = 0; c < n; ++c) cols[c] = c;
      rdp_produce(tab, g, ring, cols, n);
    }
    return;
  }
  int buf = 0;
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * TB;
    const int base = static_cast<int>(s) * g.stride;
    uint32_t rowp[R], diag[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rowp[r] = diag[r] = 0;
#pragma unroll
    for (int c = 0; c < R; ++c) {  // data columns 0..n-1 of the p-1 array columns
      if (c < n) {
        uint32_t a[R];
        take_rows<R>(ring, a);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          rowp[r] ^= a[r];
          if ((r + c) % P != P - 1) diag[(r + c) % P] ^= a[r];
        }
      }
    }
    // row-parity column p-1 on diagonal (r + p - 1) mod p = r - 1
#pragma unroll
    for (int r = 1; r < R; ++r) diag[r - 1] ^= rowp[r];
    // outputs: row parity -> slot n, diagonal parity -> slot n + 1
    if (threadIdx.x == 0) bulk_wait_read<1>();  // buffer `buf` (two tiles ago) drained
    consumers_sync();
    out_stage<R>(outbuf, buf, 0, TB, rowp);
    out_stage<R>(outbuf, buf, 1, TB, diag);
    fence_async_smem();
    consumers_sync();
    const uint32_t size = static_cast<uint32_t>(g.len - off < TB ? g.len - off : TB);
    if (threadIdx.x == 0) {
      store_tile(const_cast<uint8_t*>(tab.p[base + n]) + off, outbuf + (static_cast<size_t>(buf) * 2) * TB, size);
      store_tile(const_cast<uint8_t*>(tab.p[base + n + 1]) + off, outbuf + (static_cast<size_t>(buf) * 2 + 1) * TB,
                 size);
      bulk_commit();
    }
    if (g.tail && threadIdx.x < 32 && t - s * g.tps == g.tps - 1) rdp_encode_tail(tab, base, n, g.len, g.tail);
    buf ^= 1;
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

// Two-column recovery (coding.hpp:384-413) on the whole-dstripe body. Lost
// array columns i < j (j == p-1: row parity lost). Syndromes are accumulated
// in row words while the surviving columns stream past:
//   sr[r] = XOR_{c != i,j} A_c[r]            (= A_i[r] ^ A_j[r])
//   sd[d] = Q[d] ^ XOR_{c != i,j} A_c[(d-c) mod p]
// then the reference's two zig-zag chains run on the syndromes out of shared
// memory (their indices depend on the launch-uniform i, j).
// Compile-time form of one chain pass (LI/LJ template arguments): with the
// loop fully unrolled every d and r constant-folds, so the syndromes and both
// recovered columns stay in registers (no shared-memory chain scratch).
__host__ __device__ constexpr int pmod_c(int a, int p) { return ((a % p) + p) % p; }

template <int P, int PRIM, int PART>
__device__ __forceinline__ void rdp_chain_pass(const uint32_t (&rsyn)[P - 1], const uint32_t (&dsyn)[P - 1],
                                               uint32_t (&ap)[P], uint32_t (&aq)[P]) {
  constexpr int step = pmod_c(PART - PRIM, P);
  int d = pmod_c(PART - 1, P);
#pragma unroll
  for (int it = 0; it < P - 1; ++it) {
    if (d != P - 1) {
      const int r = pmod_c(d - PRIM, P);
      const uint32_t v = dsyn[d] ^ aq[pmod_c(d - PART, P)];
      ap[r] = v;
      aq[r] = rsyn[r] ^ v;
      d = pmod_c(d + step, P);
    }
  }
}

// LI/LJ >= 0: the lost pair is a compile-time constant (compiled for the
// primes in GS_RDP_PAIR_PRIMES, gs_rdp_pairs.cu); -1: runtime pair, chain
// walked in shared memory.
template <int CAP, int P, int LI = -1, int LJ = -1>
__global__ void __launch_bounds__((rdpb::kCW + 1) * 32, 1)
    k_rdp_recover_bulk(const PtrTable<CAP> tab, const RdpGeom g, int stages, int n_out, int out0) {
  using namespace rdpb;
  constexpr int R = P - 1;
  constexpr uint32_t TB = tile_bytes(P);
  constexpr bool kPair = LI >= 0;
  extern __shared__ __align__(128) uint8_t smem[];
  Ring ring;
  init_ring(smem, stages, ring, TB);
  uint8_t* outbuf = ring.data + static_cast<size_t>(stages) * TB;
  uint32_t* chain = reinterpret_cast<uint32_t*>(outbuf + out_bytes(P));
  const int n = g.n, i = kPair ? LI : g.li, j = kPair ? LJ : g.lj;
  if (threadIdx.x >= kNT) {  // producer: surviving array columns ascending, then the diagonal
    if ((threadIdx.x & 31) == 0) {
      int cols[kRdpMaxCols + 1];
      int nc = 0;
      for (int c = 0; c < n; ++c)
        if (c != i && c != j) cols[nc++] = c;
      if (j != P - 1) cols[nc++] = n;  // row parity slot
      cols[nc++] = n + 1;              // diagonal slot
      rdp_produce(tab, g, ring, cols, nc);
    }
    return;
  }
  const int tid = threadIdx.x;
  uint32_t* sr = chain;
  uint32_t* sd = chain + R * kNT;
  uint32_t* ai = chain + 2 * R * kNT;
  uint32_t* aj = chain + (3 * R + 1) * kNT;
  auto at = [tid](uint32_t* a, int idx) -> uint32_t& { return a[idx * kNT + tid]; };
  int buf = 0;
  for (uint32_t t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    const uint32_t s = t / g.tps;
    const uint64_t off = static_cast<uint64_t>(t - s * g.tps) * TB;
    const int base = static_cast<int>(s) * g.stride;
    uint32_t rsyn[R], dsyn[R];
#pragma unroll
    for (int r = 0; r < R; ++r) rsyn[r] = dsyn[r] = 0;
#pragma unroll
    for (int c = 0; c < P; ++c) {  // array columns; virtual ones (n <= c < p-1) are zero
      const bool present = (c < n || c == P - 1) && c != i && c != j;
      if (present) {
        uint32_t a[R];
        take_rows<R>(ring, a);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          rsyn[r] ^= a[r];
          if ((r + c) % P != P - 1) dsyn[(r + c) % P] ^= a[r];
        }
      }
    }
    {
      uint32_t q[R];
      take_rows<R>(ring, q);
#pragma unroll
      for (int d = 0; d < R; ++d) dsyn[d] ^= q[d];
    }
    uint32_t ri[R], rj[R];
    if constexpr (kPair) {
      uint32_t ai[P], aj[P];
#pragma unroll
      for (int r = 0; r < P; ++r) ai[r] = aj[r] = 0;
      rdp_chain_pass<P, LI, LJ>(rsyn, dsyn, ai, aj);
      rdp_chain_pass<P, LJ, LI>(rsyn, dsyn, aj, ai);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ri[r] = ai[r];
        rj[r] = aj[r];
      }
    } else {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      at(sr, r) = rsyn[r];
      at(sd, r) = dsyn[r];
      at(ai, r) = 0;
      at(aj, r) = 0;
    }
    at(ai, R) = 0;
    at(aj, R) = 0;
    for (int pass = 0; pass < 2; ++pass) {
      const int prim = pass == 0 ? i : j, part = pass == 0 ? j : i;
      uint32_t* ap = pass == 0 ? ai : aj;
      uint32_t* aq = pass == 0 ? aj : ai;
      int d = pmod(part - 1, P);
      const int step = pmod(part - prim, P);
      while (d != P - 1) {
        const int r = pmod(d - prim, P);
        const uint32_t v = at(sd, d) ^ at(aq, pmod(d - part, P));
        at(ap, r) = v;
        at(aq, r) = at(sr, r) ^ v;
        d = pmod(d + step, P);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ri[r] = at(ai, r);
      rj[r] = at(aj, r);
    }
    }
    if (threadIdx.x == 0) bulk_wait_read<1>();
    consumers_sync();
    out_stage<R>(outbuf, buf, 0, TB, ri);
    if (n_out > 1) out_stage<R>(outbuf, buf, 1, TB, rj);
    fence_async_smem();
    consumers_sync();
    const uint32_t size = static_cast<uint32_t>(g.len - off < TB ? g.len - off : TB);
    if (threadIdx.x == 0) {
      store_tile(const_cast<uint8_t*>(tab.p[base + out0]) + off, outbuf + (static_cast<size_t>(buf) * 2) * TB, size);
      if (n_out > 1)
        store_tile(const_cast<uint8_t*>(tab.p[base + out0 + 1]) + off,
                   outbuf + (static_cast<size_t>(buf) * 2 + 1) * TB, size);
      bulk_commit();
    }
    if (g.tail && threadIdx.x < 32 && t - s * g.tps == g.tps - 1)
      rdp_recover_tail<CAP, P>(tab, g, base, out0, n_out, g.len, g.tail);
    buf ^= 1;
  }
  if (threadIdx.x == 0) bulk_wait_all();
}

}  // namespace gsb
