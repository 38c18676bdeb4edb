// gs_fnv_gpu.cu -- FNV-1a 64 (parity_store.hpp:19-25) of long byte chains on
// the GPU, bit-exact with the serial definition
//
//     h_{i+1} = (h_i ^ b_i) * P  (mod 2^64),  P = 0x100000001b3.
//
// One chain is inherently serial on a CPU (a multiply per byte, ~1 GB/s per
// core); the GPU splits it with two observations.
//
// 1. XOR with a byte only touches the low byte of h, so h ^ b = h + d with
//    d = (s ^ b) - s, s = h mod 256. Given the sequence of low bytes s_i the
//    recurrence is LINEAR:  h_N = h_0 * P^N + sum_i d_i * P^(N - i).
//    That sum is an ordinary parallel reduction (k_fnv_final).
//
// 2. The low bytes follow an 8-bit machine  s' = ((s ^ b) * 0xB3) mod 256
//    (P mod 256 = 0xB3), and bit k of s' depends only on bits <= k:
//        s'_k = s_k ^ b_k ^ bit_k(((s ^ b) mod 2^k) * 0xB3)
//    (0xB3 is odd, so x_k * 2^k * 0xB3 adds exactly x_k at bit k). Once bits
//    < k of every s_i are known, bit k is an XOR prefix scan of
//    e_i = b_k ^ bit_k(...). Four passes of "map + XOR scan", two bits each
//    (k_fnv_pair + k_fnv_scan2), recover every s_i without a serial chain.
//
// Layout: a chain is the concatenation of k buffers of `len` bytes (the
// parity buffers of one chunk, chained in order as ParityChunk::
// compute_checksum does, parity_store.hpp:46-50). Blocks of 16 KiB (256
// threads x 64 contiguous bytes). Between passes the low bytes are kept in a
// scratch byte array, RELATIVE to each block's entry state (so a pass never
// waits for the global scan of its own bits), plus a 1-bit plane for the
// second bit's other hypothesis; the per-block entry bytes come from
// k_fnv_scan2, one CTA per chain.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>

#include "../../include/gs_capi.h"

namespace gsb {
void set_last_error(const char* msg);  // gs_capi.cu
// gs_capi.cu: host-link copies merged into 1-D runs / constant-pitch 2-D copies
int batch_copies(void* const* dst, const void* const* src, int n, size_t bytes, int kind_d2h, cudaStream_t st);
}

namespace {

constexpr int kFT = 256;                       // threads per CTA
constexpr int kFPer = 64;                      // contiguous bytes per thread
constexpr uint32_t kFB = kFT * kFPer;          // 16 KiB per block
constexpr int kFCap = 480;                     // buffer pointers per job
constexpr uint64_t kFnvP = 0x100000001b3ull;
constexpr uint64_t kScratchBudget = 2ull << 30;  // bytes of low-byte scratch per job

int ffail(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  gsb::set_last_error(buf);
  return status;
}

struct FnvJob {
  const uint8_t* p[kFCap];  // chain c, buffer i -> p[c * k + i]
  int k;
  uint64_t len;             // bytes per buffer (multiple of 16)
  uint64_t n;               // bytes per chain = k * len
  uint32_t bpc;             // blocks per chain
  uint32_t nblocks;         // chains * bpc
};

__device__ __forceinline__ uint64_t pow64(uint64_t b, uint64_t e) {
  uint64_t r = 1;
  while (e) {
    if (e & 1) r *= b;
    b *= b;
    e >>= 1;
  }
  return r;
}

// The thread's four 16-byte groups of block `blk`; groups at or past the end
// of the chain are zero and not `valid`.
__device__ __forceinline__ int load_groups(const FnvJob& j, uint32_t c, uint64_t pos0, uint4 (&d)[4]) {
  int nvalid = 0;
  if (pos0 >= j.n) {
#pragma unroll
    for (int q = 0; q < 4; ++q) d[q] = make_uint4(0, 0, 0, 0);
    return 0;
  }
  uint64_t bi = pos0 / j.len;
  uint64_t off = pos0 - bi * j.len;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint64_t p = pos0 + 16u * q;
    if (p < j.n) {
      while (off >= j.len) {
        off -= j.len;
        ++bi;
      }
      d[q] = __ldcs(reinterpret_cast<const uint4*>(j.p[c * j.k + bi] + off));
      ++nvalid;
    } else {
      d[q] = make_uint4(0, 0, 0, 0);
    }
    off += 16;
  }
  return nvalid;
}

__device__ __forceinline__ uint32_t& wd(uint4& v, int w) { return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w; }

// e bits of bit K for the 4 positions of one word (byte j -> nibble bit j):
// e = b_K ^ bit_K(((s ^ b) mod 2^K) * 0xB3), s_true holding the true bits < K.
template <int K>
__device__ __forceinline__ uint32_t e_nibble(uint32_t s_true, uint32_t bw) {
  constexpr uint32_t kMask = ((1u << K) - 1u) * 0x01010101u;
  const uint32_t x = (s_true ^ bw) & kMask;
  uint32_t e;
  if constexpr (K <= 3) {
    // bit K of x*0xB3 only needs x * (0xB3 mod 2^(K+1)) < 2^(2K+1) <= 2^7: the
    // four byte lanes multiply in ONE IMAD without spilling into each other
    constexpr uint32_t c = 0xB3u & ((2u << K) - 1u);
    e = ((x * c) ^ bw) >> K & 0x01010101u;
  } else {
    const uint32_t lo = (x & 0x00FF00FFu) * 0xB3u;         // bytes 0, 2 in 16-bit lanes
    const uint32_t hi = ((x >> 8) & 0x00FF00FFu) * 0xB3u;  // bytes 1, 3
    const uint32_t t = ((lo >> K) & 0x00010001u) | (((hi >> K) & 0x00010001u) << 8);
    e = t ^ ((bw >> K) & 0x01010101u);
  }
  return (e * 0x01020408u) >> 24;  // byte j's bit -> bit j (no other term lands in bits 28..31)
}
__device__ __forceinline__ uint32_t spread_nibble(uint32_t nib) { return (nib * 0x00204081u) & 0x01010101u; }

// exclusive XOR prefix of a thread's 64 e-bits (position order)
__device__ __forceinline__ uint64_t exclusive_xor(uint64_t e, uint32_t& parity) {
  e ^= e << 1;
  e ^= e << 2;
  e ^= e << 4;
  e ^= e << 8;
  e ^= e << 16;
  e ^= e << 32;
  parity = static_cast<uint32_t>(e >> 63);
  return e << 1;
}

// Rounds K and K+1 (K even) in one pass. Bit K as before (relative to the
// block's entry bit K). Bit K+1 depends on the TRUE bit K = rel_K ^ entry_K,
// and entry_K is only known after the global scan -- so it is evaluated for
// both values of entry_K: the h = 0 trajectory goes into the scratch byte
// (bit K+1), its XOR with the h = 1 trajectory into a 1-bit-per-position
// plane D, and both block aggregates into agg (bits 1, 2). The next pass (or
// the final one) selects with entry_K and folds D back in. Halves the data
// passes of the one-bit-per-round form.
template <int K>
__global__ void __launch_bounds__(kFT) k_fnv_pair(const FnvJob j, uint8_t* __restrict__ scratch,
                                                  uint64_t* __restrict__ dplane, uint8_t* __restrict__ agg,
                                                  const uint8_t* __restrict__ entry) {
  __shared__ uint32_t wpar[3][kFT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  for (uint32_t blk = blockIdx.x; blk < j.nblocks; blk += gridDim.x) {
    const uint32_t c = blk / j.bpc, b = blk - c * j.bpc;
    const uint64_t pos0 = static_cast<uint64_t>(b) * kFB + static_cast<uint64_t>(tid) * kFPer;
    uint4 d[4];
    const int nvalid = load_groups(j, c, pos0, d);
    uint4 s[4];
    uint4* sp = reinterpret_cast<uint4*>(scratch + static_cast<uint64_t>(blk) * kFB + tid * kFPer);
    uint64_t* dp = dplane + static_cast<uint64_t>(blk) * kFT + tid;
    const uint32_t ent = K > 0 ? entry[blk] : 0u;
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] = K > 0 ? sp[q] : make_uint4(0, 0, 0, 0);
    if (K > 0 && ((ent >> (K - 2)) & 1u)) {  // previous pair's bit K-1: take the entry_{K-2} = 1 trajectory
      const uint64_t dd = *dp;
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int w = 0; w < 4; ++w)
          wd(s[q], w) ^= spread_nibble(static_cast<uint32_t>(dd >> (16 * q + 4 * w)) & 0xFu) << (K - 1);
    }
    const uint32_t rep = ent * 0x01010101u;  // entry bits < K
    // ---- bit K ----
    uint64_t eK = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int w = 0; w < 4; ++w)
        if (q < nvalid) eK |= static_cast<uint64_t>(e_nibble<K>(wd(s[q], w) ^ rep, wd(d[q], w))) << (16 * q + 4 * w);
    uint32_t parK;
    uint64_t relK = exclusive_xor(eK, parK);
    uint32_t bal = __ballot_sync(0xFFFFFFFFu, parK);
    uint32_t carry = __popc(bal & lt) & 1u;
    if (lane == 0) wpar[0][warp] = __popc(bal) & 1u;
    __syncthreads();
    uint32_t totK = 0;
#pragma unroll
    for (int w = 0; w < kFT / 32; ++w) {
      if (w < warp) carry ^= wpar[0][w];
      totK ^= wpar[0][w];
    }
    if (carry) relK = ~relK;
    // ---- bit K+1 under entry_K = 0 and entry_K = 1 ----
    uint64_t e0 = 0, e1 = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t sh = 16 * q + 4 * w;
        const uint32_t rk = spread_nibble(static_cast<uint32_t>(relK >> sh) & 0xFu) << K;
        const uint32_t base = wd(s[q], w) ^ rep;
        if (q < nvalid) {
          e0 |= static_cast<uint64_t>(e_nibble<K + 1>(base | rk, wd(d[q], w))) << sh;
          e1 |= static_cast<uint64_t>(e_nibble<K + 1>(base | (rk ^ (0x01010101u << K)), wd(d[q], w))) << sh;
        }
      }
    uint32_t par0, par1;
    uint64_t r0 = exclusive_xor(e0, par0), r1 = exclusive_xor(e1, par1);
    const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, par0), b1 = __ballot_sync(0xFFFFFFFFu, par1);
    uint32_t c0 = __popc(b0 & lt) & 1u, c1 = __popc(b1 & lt) & 1u;
    if (lane == 0) {
      wpar[1][warp] = __popc(b0) & 1u;
      wpar[2][warp] = __popc(b1) & 1u;
    }
    __syncthreads();
    uint32_t t0 = 0, t1 = 0;
#pragma unroll
    for (int w = 0; w < kFT / 32; ++w) {
      if (w < warp) {
        c0 ^= wpar[1][w];
        c1 ^= wpar[2][w];
      }
      t0 ^= wpar[1][w];
      t1 ^= wpar[2][w];
    }
    if (c0) r0 = ~r0;
    if (c1) r1 = ~r1;
    if (tid == 0) agg[blk] = static_cast<uint8_t>(totK | (t0 << 1) | (t1 << 2));
#pragma unroll
    for (int q = 0; q < 4; ++q) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint32_t sh = 16 * q + 4 * w;
        wd(s[q], w) |= (spread_nibble(static_cast<uint32_t>(relK >> sh) & 0xFu) << K) |
                       (spread_nibble(static_cast<uint32_t>(r0 >> sh) & 0xFu) << (K + 1));
      }
      sp[q] = s[q];
    }
    *dp = r0 ^ r1;
    __syncthreads();  // wpar reuse
  }
}

// entry bits K and K+1 of every block of chain blockIdx.x: bit K = bit K of
// h0 ^ XOR of earlier blocks' aggregates; bit K+1 likewise over the
// aggregates of the trajectory each block's entry bit K selects.
template <int K>
__global__ void __launch_bounds__(1024) k_fnv_scan2(const uint8_t* __restrict__ agg, uint8_t* __restrict__ entry,
                                                    uint32_t bpc, uint64_t h0) {
  __shared__ uint32_t wpar[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * bpc;
  const uint32_t per = (bpc + blockDim.x - 1) / blockDim.x;
  const uint32_t b0 = min(bpc, tid * per), b1 = min(bpc, b0 + per);
  auto block_exclusive = [&](uint32_t par) -> uint32_t {
    const uint32_t bal = __ballot_sync(0xFFFFFFFFu, par);
    uint32_t pre = __popc(bal & ((1u << lane) - 1u)) & 1u;
    if (lane == 0) wpar[warp] = __popc(bal) & 1u;
    __syncthreads();
    for (int w = 0; w < warp; ++w) pre ^= wpar[w];
    __syncthreads();
    return pre;
  };
  uint32_t par = 0;
  for (uint32_t b = b0; b < b1; ++b) par ^= agg[base + b] & 1u;
  uint32_t preK = block_exclusive(par) ^ (static_cast<uint32_t>(h0 >> K) & 1u);
  // bit K+1 aggregates under each block's now-known entry bit K
  uint32_t p1 = 0, ek = preK;
  for (uint32_t b = b0; b < b1; ++b) {
    const uint32_t a = agg[base + b];
    p1 ^= (a >> (ek ? 2 : 1)) & 1u;
    ek ^= a & 1u;
  }
  uint32_t preK1 = block_exclusive(p1) ^ (static_cast<uint32_t>(h0 >> (K + 1)) & 1u);
  ek = preK;
  for (uint32_t b = b0; b < b1; ++b) {
    const uint32_t a = agg[base + b];
    const uint8_t bits = static_cast<uint8_t>((ek << K) | (preK1 << (K + 1)));
    entry[base + b] = K == 0 ? bits : static_cast<uint8_t>(entry[base + b] | bits);
    preK1 ^= (a >> (ek ? 2 : 1)) & 1u;
    ek ^= a & 1u;
  }
}

__global__ void k_fnv_init(uint64_t* out, int n_chains, uint64_t h0, uint64_t n, const uint64_t* h0s) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < n_chains) out[c] = (h0s ? h0s[c] : h0) * pow64(kFnvP, n);
}

// out[c] += sum over the chain's bytes of d_i * P^(N - i), d_i = (s_i ^ b_i) - s_i.
__global__ void __launch_bounds__(kFT) k_fnv_final(const FnvJob j, const uint8_t* __restrict__ scratch,
                                                   const uint64_t* __restrict__ dplane,
                                                   const uint8_t* __restrict__ entry,
                                                   unsigned long long* __restrict__ out) {
  __shared__ uint64_t pw[kFT];  // P^(64 t)
  __shared__ uint64_t pblk;
  __shared__ uint64_t wsum[kFT / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  pw[tid] = pow64(kFnvP, static_cast<uint64_t>(kFPer) * tid);
  __syncthreads();
  for (uint32_t blk = blockIdx.x; blk < j.nblocks; blk += gridDim.x) {
    const uint32_t c = blk / j.bpc, b = blk - c * j.bpc;
    const uint64_t bstart = static_cast<uint64_t>(b) * kFB;
    const uint64_t bend = bstart + kFB;
    const uint64_t pos0 = bstart + static_cast<uint64_t>(tid) * kFPer;
    if (tid == 0) pblk = bend <= j.n ? pow64(kFnvP, j.n - bend) : 0;
    uint4 d[4];
    const int nvalid = load_groups(j, c, pos0, d);
    const uint4* sp = reinterpret_cast<const uint4*>(scratch + static_cast<uint64_t>(blk) * kFB + tid * kFPer);
    const uint32_t ent = entry[blk];
    const uint32_t rep = ent * 0x01010101u;
    const uint64_t dd = (ent >> 6) & 1u ? dplane[static_cast<uint64_t>(blk) * kFT + tid] : 0;  // bit 7's trajectory
    // four independent 16-byte Horner chains (ILP), joined with P^16
    uint64_t accq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < nvalid) {
        uint4 s = sp[q];
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const uint32_t sw = wd(s, w) ^ rep ^ (spread_nibble(static_cast<uint32_t>(dd >> (16 * q + 4 * w)) & 0xFu) << 7),
                         xw = sw ^ wd(d[q], w);
#pragma unroll
          for (int by = 0; by < 4; ++by) {
            const int64_t di = static_cast<int64_t>((xw >> (8 * by)) & 0xFFu) -
                               static_cast<int64_t>((sw >> (8 * by)) & 0xFFu);
            accq[q] = (accq[q] + static_cast<uint64_t>(di)) * kFnvP;
          }
        }
      }
    }
    constexpr uint64_t kP16 = [] {
      uint64_t r = 1;
      for (int i = 0; i < 16; ++i) r *= kFnvP;
      return r;
    }();
    uint64_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nvalid) acc = acc * kP16 + accq[q];
    __syncthreads();  // pblk visible
    uint64_t contrib = 0;
    if (nvalid > 0) {
      const uint64_t tend = pos0 + 16u * nvalid;
      contrib = acc * (bend <= j.n ? pblk * pw[kFT - 1 - tid] : pow64(kFnvP, j.n - tend));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
    if (lane == 0) wsum[warp] = contrib;
    __syncthreads();
    if (tid == 0) {
      uint64_t sum = 0;
#pragma unroll
      for (int w = 0; w < kFT / 32; ++w) sum += wsum[w];
      atomicAdd(out + c, static_cast<unsigned long long>(sum));
    }
    __syncthreads();  // pblk / wsum reuse
  }
}

template <int K>
cudaError_t pair_and_scan(const FnvJob& j, int grid, int n_chains, uint8_t* scratch, uint64_t* dplane, uint8_t* agg,
                          uint8_t* entry, uint64_t h0, cudaStream_t st) {
  k_fnv_pair<K><<<grid, kFT, 0, st>>>(j, scratch, dplane, agg, entry);
  k_fnv_scan2<K><<<n_chains, 1024, 0, st>>>(agg, entry, j.bpc, h0);
  return cudaGetLastError();
}


// ===========================================================================
// Single-pass windowed FNV (the default; GS_FNV_LEGACY=1 selects the
// multi-pass kernels above for A/B).
//
// The multi-pass form streams the chain five times and a low-byte scratch
// array eight times: ~14 B of HBM per chain byte. Here every chain byte is
// read ONCE: a cluster of kWCS CTAs holds a window of kWCS x 32 KiB in
// registers (64 B of data + 64 B of low-byte state per thread) and resolves
// all eight low-byte bits on chip, one bit per round:
//   * round K: e-bits of bit K from the TRUE bits < K (e_nibble<K>), XOR
//     prefix per thread / warp (ballot) / CTA (smem) / cluster (DSMEM slots +
//     barrier.cluster) -- the window's own bit-K aggregate;
//   * the window's ENTRY bit K comes from its predecessors by a decoupled
//     look-back over a per-window flag word in global memory (bit-K totals
//     and exit bits, published with st.release as soon as they are known),
//     so the windows of one chain are resolved by many clusters at once;
//   * then the final linear sum  sum_i d_i P^(n-i)  of the window, atomically
//     added to the chain's hash (h0 P^n added by k_fnv_init).
// Windows are handed out in order (window-major across the chains) by an
// atomic counter, so a window's predecessors are always owned by running
// clusters (no residency deadlock).
// ===========================================================================
constexpr int kWT = 512;                         // threads per CTA
constexpr uint32_t kWB = kWT * kFPer;            // 32 KiB per CTA per window
constexpr int kWCS = 8;                          // CTAs per cluster (portable size)
constexpr uint64_t kWin = static_cast<uint64_t>(kWB) * kWCS;  // 256 KiB per window

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Store a u32 into the same smem variable of CTA `rank` of this cluster.
__device__ __forceinline__ void st_cluster_u32(uint32_t* local, uint32_t rank, uint32_t v) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// Window flag word (one per window, zeroed per call):
//   bits 0-7 : bit-K totals of the window's e-bits   bits 16-23: totals valid
//   bits 8-15: exit bits (entry ^ total)             bits 24-31: exit valid
// Entry bit K of window w of a chain (w > 0) = exit bit K of window w-1
// = h0_K ^ XOR of the totals of windows 0..w-1. Warp 0 looks back over up to
// 32 predecessors per step: the nearest one with its exit bit published ends
// the walk, nearer ones contribute their totals (spin while any is missing).
template <int K>
__device__ __forceinline__ uint32_t lookback_entry(const uint32_t* flags, uint32_t gw, uint32_t w, uint32_t nc,
                                                   uint64_t h0) {
  const int lane = threadIdx.x & 31;
  uint32_t acc = 0;
  uint32_t back = 0;  // predecessors already folded into acc
  for (;;) {
    // lane l inspects predecessor w - 1 - back - l (if it exists)
    const uint32_t dist = back + lane + 1;
    const bool exists = dist <= w;
    uint32_t v = 0;
    bool have_exit = false, have_total = false;
    if (exists) {
      v = ld_acquire_u32(flags + (gw - dist * nc));
      have_exit = (v >> (24 + K)) & 1u;
      have_total = (v >> (16 + K)) & 1u;
    }
    // the chain start acts as a predecessor whose exit bits are h0's
    const bool start = !exists && dist == w + 1;
    const uint32_t stop_bal = __ballot_sync(0xFFFFFFFFu, have_exit || start);
    const int first = stop_bal ? __ffs(stop_bal) - 1 : 32;
    // every lane nearer than `first` must contribute its total
    const uint32_t need = first >= 32 ? 0xFFFFFFFFu : ((1u << first) - 1u);
    const uint32_t ok_bal = __ballot_sync(0xFFFFFFFFu, have_total);
    if ((ok_bal & need) != need) continue;  // a nearer total is not published yet: spin
    const uint32_t tot = __ballot_sync(0xFFFFFFFFu, have_total && ((v >> K) & 1u)) & need;
    acc ^= __popc(tot) & 1u;
    if (first < 32) {
      const uint32_t ex = __shfl_sync(0xFFFFFFFFu, start ? static_cast<uint32_t>(h0 >> K) : (v >> (8 + K)), first);
      return acc ^ (ex & 1u);
    }
    back += 32;
  }
}

struct WinShared {
  uint64_t pw[kWT];              // P^(64 t)
  uint32_t warp_par[kWT / 32];
  uint32_t cta_tot[8][kWCS];     // [round][cluster rank], written by every CTA of the cluster
  uint32_t gw;                   // window index, written by rank 0
  uint32_t entry;                // entry bit of the current round
  unsigned long long wsum[kWT / 32];
  uint64_t pblk;
};

template <int K>
__device__ __forceinline__ void win_round(WinShared& sh, const FnvJob& j, uint32_t* flags, uint32_t gw, uint32_t w,
                                          uint32_t nc, uint64_t h0, uint32_t rank, int nvalid, const uint4 (&d)[4], uint4 (&s)[4],
                                          uint32_t& flag_word) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // e-bits of bit K from the true bits < K held in s. Positions past the
  // chain's end (zero data) need no masking: their e-bits only feed the
  // prefixes of later positions, which are past the end as well.
  uint64_t eK = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int x = 0; x < 4; ++x)
      eK |= static_cast<uint64_t>(e_nibble<K>(wd(s[q], x), wd(const_cast<uint4&>(d[q]), x))) << (16 * q + 4 * x);
  uint32_t par;
  uint64_t rel = exclusive_xor(eK, par);
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, par);
  uint32_t carry = __popc(bal & ((1u << lane) - 1u)) & 1u;
  if (lane == 0) sh.warp_par[warp] = __popc(bal) & 1u;
  __syncthreads();
  uint32_t cta_tot = 0;
#pragma unroll
  for (int x = 0; x < kWT / 32; ++x) {
    if (x < warp) carry ^= sh.warp_par[x];
    cta_tot ^= sh.warp_par[x];
  }
  if (tid < kWCS) st_cluster_u32(&sh.cta_tot[K][rank], static_cast<uint32_t>(tid), cta_tot);
  cluster_sync_all();
  uint32_t win_tot = 0;
#pragma unroll
  for (int r = 0; r < kWCS; ++r) {
    const uint32_t t = sh.cta_tot[K][r];
    if (static_cast<uint32_t>(r) < rank) carry ^= t;
    win_tot ^= t;
  }
  if (warp == 0) {
    // publish this window's bit-K total first (successors can fold it in),
    // then find the entry bit and publish the exit bit
    if (rank == 0 && lane == 0) {
      flag_word |= (win_tot << K) | (1u << (16 + K));
      st_release_u32(flags + gw, flag_word);
    }
    uint32_t entry = w == 0 ? static_cast<uint32_t>(h0 >> K) & 1u : lookback_entry<K>(flags, gw, w, nc, h0);
    if (lane == 0) {
      sh.entry = entry;
      if (rank == 0) {
        flag_word |= ((entry ^ win_tot) << (8 + K)) | (1u << (24 + K));
        st_release_u32(flags + gw, flag_word);
      }
    }
  }
  __syncthreads();
  carry ^= sh.entry;
  if (carry) rel = ~rel;
#pragma unroll
  for (int q = 0; q < 4; ++q)
#pragma unroll
    for (int x = 0; x < 4; ++x)
      wd(s[q], x) |= spread_nibble(static_cast<uint32_t>(rel >> (16 * q + 4 * x)) & 0xFu) << K;
  __syncthreads();  // sh.entry / warp_par reuse by the next round
}

__global__ void __cluster_dims__(kWCS, 1, 1) __launch_bounds__(kWT, 2)
    k_fnv_window(const FnvJob j, uint64_t h0, const uint64_t* __restrict__ h0s, uint32_t nc, uint32_t total_windows,
                 uint32_t* counter, uint32_t* flags, unsigned long long* __restrict__ out) {
  __shared__ WinShared sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  sh.pw[tid] = pow64(kFnvP, static_cast<uint64_t>(kFPer) * tid);
  // every CTA of the cluster has started (and initialised its shared memory)
  // before rank 0 writes the first window index into their shared memory
  cluster_sync_all();
  for (;;) {
    if (rank == 0 && tid == 0) {
      const uint32_t g = atomicAdd(counter, 1u);
      for (int r = 0; r < kWCS; ++r) st_cluster_u32(&sh.gw, static_cast<uint32_t>(r), g);
    }
    cluster_sync_all();  // sh.gw visible in every CTA (also orders windows)
    const uint32_t gw = sh.gw;
    if (gw >= total_windows) break;
    // window-major order: the windows in flight at once belong to different
    // chains as far as there are chains, so a window's predecessor (same
    // chain, gw - nc) has usually finished and the look-back is one read
    const uint32_t w = gw / nc, c = gw - w * nc;
    const uint64_t hc = h0s ? h0s[c] : h0;  // the chain's seed (per-chain seeds continue earlier chains)
    const uint64_t cta0 = static_cast<uint64_t>(w) * kWin + static_cast<uint64_t>(rank) * kWB;
    const uint64_t pos0 = cta0 + static_cast<uint64_t>(tid) * kFPer;
    uint4 d[4];
    const int nvalid = load_groups(j, c, pos0, d);
    uint4 s[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) s[q] = make_uint4(0, 0, 0, 0);
    uint32_t fw = 0;
    win_round<0>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<1>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<2>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<3>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<4>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<5>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<6>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    win_round<7>(sh, j, flags, gw, w, nc, hc, rank, nvalid, d, s, fw);
    // sum over the thread's bytes of d_i P^(tend - i), four 16-byte Horner chains
    uint64_t accq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < nvalid) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const uint32_t sw = wd(s[q], x), xw = sw ^ wd(d[q], x);
#pragma unroll
          for (int by = 0; by < 4; ++by) {
            const int64_t di = static_cast<int64_t>((xw >> (8 * by)) & 0xFFu) -
                               static_cast<int64_t>((sw >> (8 * by)) & 0xFFu);
            accq[q] = (accq[q] + static_cast<uint64_t>(di)) * kFnvP;
          }
        }
      }
    }
    constexpr uint64_t kP16 = [] {
      uint64_t r = 1;
      for (int i = 0; i < 16; ++i) r *= kFnvP;
      return r;
    }();
    uint64_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nvalid) acc = acc * kP16 + accq[q];
    const uint64_t cend = cta0 + kWB;
    if (tid == 0) sh.pblk = cend <= j.n ? pow64(kFnvP, j.n - cend) : 0;
    __syncthreads();
    uint64_t contrib = 0;
    if (nvalid > 0) {
      const uint64_t tend = pos0 + 16u * nvalid;
      contrib = acc * (cend <= j.n ? sh.pblk * sh.pw[kWT - 1 - tid] : pow64(kFnvP, j.n - tend));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
    if (lane == 0) sh.wsum[warp] = contrib;
    __syncthreads();
    if (tid == 0) {
      uint64_t sum = 0;
#pragma unroll
      for (int x = 0; x < kWT / 32; ++x) sum += sh.wsum[x];
      atomicAdd(out + c, static_cast<unsigned long long>(sum));
    }
    // the next window's cluster barrier (sh.gw) also separates sh.pblk / wsum reuse
  }
}

// ===========================================================================
// Bit-sliced cluster windows (the default; GS_FNV_WINDOW_BYTES=1 keeps the
// byte-lane rounds above for A/B). Same windows, look-back and cluster scans
// as k_fnv_window; only the per-thread arithmetic of a round changes: the
// thread's 64 bytes are held as two groups of eight 32-bit bit planes (bit i
// of plane j = bit j of byte i), and round K evaluates the column-K bits of
// the bit-sliced product x * 0xB3 (x = s ^ b) from the lower planes with
// carry-save full adders (one known bit per column, so each new plane adds
// one AND / majority), then an XOR prefix inside each 32-bit word -- ~40
// integer ops per round for 64 bytes instead of ~240. The low bytes go back
// to byte lanes once, for the final sum.
// ===========================================================================
__device__ __forceinline__ uint64_t sl_t8(uint64_t x) {  // 8x8 bit transpose: byte j bit b <-> byte b bit j
  uint64_t t = (x ^ (x >> 7)) & 0x00AA00AA00AA00AAull;
  x = x ^ t ^ (t << 7);
  t = (x ^ (x >> 14)) & 0x0000CCCC0000CCCCull;
  x = x ^ t ^ (t << 14);
  t = (x ^ (x >> 28)) & 0x00000000F0F0F0F0ull;
  return x ^ t ^ (t << 28);
}
__device__ __forceinline__ void sl_bt4(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {  // 4x4 byte transpose
  const uint32_t ab_lo = __byte_perm(a, b, 0x5140), ab_hi = __byte_perm(a, b, 0x7362);
  const uint32_t cd_lo = __byte_perm(c, d, 0x5140), cd_hi = __byte_perm(c, d, 0x7362);
  a = __byte_perm(ab_lo, cd_lo, 0x5410);
  b = __byte_perm(ab_lo, cd_lo, 0x7632);
  c = __byte_perm(ab_hi, cd_hi, 0x5410);
  d = __byte_perm(ab_hi, cd_hi, 0x7632);
}
// 32 bytes (w[i] byte k = byte 4i + k) <-> 8 planes (plane j bit i = bit j of byte i).
__device__ __forceinline__ void sl_to_planes(uint32_t (&w)[8]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t x = sl_t8(static_cast<uint64_t>(w[2 * k]) | (static_cast<uint64_t>(w[2 * k + 1]) << 32));
    w[2 * k] = static_cast<uint32_t>(x);
    w[2 * k + 1] = static_cast<uint32_t>(x >> 32);
  }
  uint32_t a = w[0], b = w[2], c = w[4], d = w[6], e = w[1], f = w[3], g = w[5], h = w[7];
  sl_bt4(a, b, c, d);
  sl_bt4(e, f, g, h);
  w[0] = a; w[1] = b; w[2] = c; w[3] = d; w[4] = e; w[5] = f; w[6] = g; w[7] = h;
}
__device__ __forceinline__ void sl_from_planes(uint32_t (&w)[8]) {
  uint32_t a = w[0], b = w[1], c = w[2], d = w[3], e = w[4], f = w[5], g = w[6], h = w[7];
  sl_bt4(a, b, c, d);
  sl_bt4(e, f, g, h);
  const uint32_t lo[4] = {a, b, c, d}, hi[4] = {e, f, g, h};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint64_t x = sl_t8(static_cast<uint64_t>(lo[k]) | (static_cast<uint64_t>(hi[k]) << 32));
    w[2 * k] = static_cast<uint32_t>(x);
    w[2 * k + 1] = static_cast<uint32_t>(x >> 32);
  }
}
__device__ __forceinline__ uint32_t sl_prefix32(uint32_t x) {  // inclusive prefix XOR along the bits
  x ^= x << 1;
  x ^= x << 2;
  x ^= x << 4;
  x ^= x << 8;
  x ^= x << 16;
  return x;
}
__device__ __forceinline__ uint32_t sl_maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

// One 32-byte group: its planes, the x planes solved so far and the
// carry-save state of the column sums of x * 0xB3 = x + 2x + 16x + 32x + 128x.
struct SlCol {
  uint32_t B[8], X[8];
  uint32_t c12, c23, c34, s4, c45a, c45b, s5, c56a, c56b, c56c, s6, c67a, c67b, c67c, c67d;
  uint32_t s5a_;  // column 5's known part (two-bit rounds)
  template <int K>
  __device__ __forceinline__ uint32_t g() {  // column K bits other than x_K (known bits pre-reduced)
    if constexpr (K == 0) return 0u;
    else if constexpr (K == 1) return X[0];
    else if constexpr (K == 2) return X[1] ^ c12;
    else if constexpr (K == 3) return X[2] ^ c23;
    else if constexpr (K == 4) {
      s4 = X[3] ^ X[0] ^ c34;
      c45a = sl_maj(X[3], X[0], c34);
      return s4;
    } else if constexpr (K == 5) {
      const uint32_t s5a = X[1] ^ X[0] ^ c45a;
      c56a = sl_maj(X[1], X[0], c45a);
      s5 = s5a ^ X[4] ^ c45b;
      c56b = sl_maj(s5a, X[4], c45b);
      return s5;
    } else if constexpr (K == 6) {
      const uint32_t s6a = X[2] ^ X[1] ^ c56a;
      c67a = sl_maj(X[2], X[1], c56a);
      const uint32_t s6b = s6a ^ c56b ^ c56c;
      c67b = sl_maj(s6a, c56b, c56c);
      s6 = s6b ^ X[5];
      c67c = s6b & X[5];
      return s6;
    } else {
      return X[6] ^ X[3] ^ X[2] ^ X[0] ^ c67a ^ c67b ^ c67c ^ c67d;  // only the parity of column 7
    }
  }
  template <int K>
  __device__ __forceinline__ void after() {  // carries out of column K once x_K is known
    if constexpr (K == 1) c12 = X[1] & X[0];
    else if constexpr (K == 2) c23 = sl_maj(X[2], X[1], c12);
    else if constexpr (K == 3) c34 = sl_maj(X[3], X[2], c23);
    else if constexpr (K == 4) c45b = X[4] & s4;
    else if constexpr (K == 5) c56c = X[5] & s5;
    else if constexpr (K == 6) c67d = X[6] & s6;
  }
};

struct WinSharedSl {
  uint64_t pw[kWT];                  // P^(64 t)
  uint32_t wpar[8][kWCS];            // [round][cluster rank]: bit x = parity of warp x of that CTA
  uint32_t gw;                       // window index, written by rank 0
  unsigned long long wsum[kWT / 32];
  uint64_t pblk;
};

// OR a u32 into the same smem variable of CTA `rank` of this cluster.
__device__ __forceinline__ void or_cluster_u32(uint32_t* local, uint32_t rank, uint32_t v) {
  uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(local)), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
  asm volatile("red.shared::cluster.or.b32 [%0], %1;" ::"r"(ra), "r"(v) : "memory");
}

// One round with ONE barrier: every warp ORs its parity bit into its CTA's
// word of this round in every CTA of the cluster, one cluster barrier, then
// each thread derives its carry from the 8 words; every warp walks the
// look-back itself (rank 0 / warp 0 publishes), and each round has its own
// slots, so no barrier separates the rounds.
template <int K>
__device__ __forceinline__ void win_round_sl(WinSharedSl& sh, uint32_t* flags, uint32_t gw, uint32_t w, uint32_t nc,
                                             uint64_t h0, uint32_t rank, SlCol (&G)[2], uint32_t& flag_word) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t inc0 = sl_prefix32(G[0].B[K] ^ G[0].template g<K>());
  const uint32_t inc1 = sl_prefix32(G[1].B[K] ^ G[1].template g<K>());
  const uint32_t par0 = inc0 >> 31;
  const uint32_t par = par0 ^ (inc1 >> 31);
  const uint32_t bal = __ballot_sync(0xFFFFFFFFu, par);
  uint32_t carry = __popc(bal & ((1u << lane) - 1u)) & 1u;
  if ((__popc(bal) & 1u) && lane < kWCS) or_cluster_u32(&sh.wpar[K][rank], static_cast<uint32_t>(lane), 1u << warp);
  cluster_sync_all();
  uint32_t win_tot = 0;
#pragma unroll
  for (int r = 0; r < kWCS; ++r) {
    const uint32_t t = __popc(sh.wpar[K][r]) & 1u;
    if (static_cast<uint32_t>(r) < rank) carry ^= t;
    win_tot ^= t;
  }
  carry ^= __popc(sh.wpar[K][rank] & ((1u << warp) - 1u)) & 1u;
  if (rank == 0 && warp == 0 && lane == 0) {
    flag_word |= (win_tot << K) | (1u << (16 + K));
    st_release_u32(flags + gw, flag_word);
  }
  const uint32_t entry = w == 0 ? static_cast<uint32_t>(h0 >> K) & 1u : lookback_entry<K>(flags, gw, w, nc, h0);
  if (rank == 0 && warp == 0 && lane == 0) {
    flag_word |= ((entry ^ win_tot) << (8 + K)) | (1u << (24 + K));
    st_release_u32(flags + gw, flag_word);
  }
  carry ^= entry;
  const uint32_t L0 = (inc0 << 1) ^ (0u - carry), L1 = (inc1 << 1) ^ (0u - (carry ^ par0));
  G[0].X[K] = L0 ^ G[0].B[K];
  G[1].X[K] = L1 ^ G[1].B[K];
  G[0].template after<K>();
  G[1].template after<K>();
}

__global__ void __cluster_dims__(kWCS, 1, 1) __launch_bounds__(kWT, 2)
    k_fnv_window_sl(const FnvJob j, uint64_t h0, const uint64_t* __restrict__ h0s, uint32_t nc, uint32_t total_windows,
                    uint32_t* counter, uint32_t* flags, unsigned long long* __restrict__ out) {
  __shared__ WinSharedSl sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  sh.pw[tid] = pow64(kFnvP, static_cast<uint64_t>(kFPer) * tid);
  cluster_sync_all();  // every CTA of the cluster has started before rank 0 writes into their smem
  for (;;) {
    if (tid < 8 * kWCS) (&sh.wpar[0][0])[tid] = 0;  // this window's parity words (no remote OR before the barrier)
    if (rank == 0 && tid == 0) {
      const uint32_t g = atomicAdd(counter, 1u);
      for (int r = 0; r < kWCS; ++r) st_cluster_u32(&sh.gw, static_cast<uint32_t>(r), g);
    }
    cluster_sync_all();
    const uint32_t gw = sh.gw;
    if (gw >= total_windows) break;
    const uint32_t w = gw / nc, c = gw - w * nc;
    const uint64_t hc = h0s ? h0s[c] : h0;
    const uint64_t cta0 = static_cast<uint64_t>(w) * kWin + static_cast<uint64_t>(rank) * kWB;
    const uint64_t pos0 = cta0 + static_cast<uint64_t>(tid) * kFPer;
    SlCol G[2];
    {
      uint4 d[4];
      load_groups(j, c, pos0, d);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t wv[8] = {d[2 * q].x, d[2 * q].y, d[2 * q].z, d[2 * q].w,
                          d[2 * q + 1].x, d[2 * q + 1].y, d[2 * q + 1].z, d[2 * q + 1].w};
        sl_to_planes(wv);
#pragma unroll
        for (int b = 0; b < 8; ++b) G[q].B[b] = wv[b];
      }
    }
    uint32_t fw = 0;
    win_round_sl<0>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<1>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<2>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<3>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<4>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<5>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<6>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_round_sl<7>(sh, flags, gw, w, nc, hc, rank, G, fw);
    // low bytes s = x ^ b back to byte lanes; the data re-read (cache-resident)
    uint4 s[4], d[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t wv[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) wv[b] = G[q].X[b] ^ G[q].B[b];
      sl_from_planes(wv);
      s[2 * q] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      s[2 * q + 1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
    }
    const int nvalid = load_groups(j, c, pos0, d);
    // sum over the thread's bytes of d_i P^(tend - i), four 16-byte Horner chains
    uint64_t accq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < nvalid) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const uint32_t sw = wd(s[q], x), xw = sw ^ wd(d[q], x);
#pragma unroll
          for (int by = 0; by < 4; ++by) {
            const int64_t di = static_cast<int64_t>((xw >> (8 * by)) & 0xFFu) -
                               static_cast<int64_t>((sw >> (8 * by)) & 0xFFu);
            accq[q] = (accq[q] + static_cast<uint64_t>(di)) * kFnvP;
          }
        }
      }
    }
    constexpr uint64_t kP16 = [] {
      uint64_t r = 1;
      for (int i = 0; i < 16; ++i) r *= kFnvP;
      return r;
    }();
    uint64_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nvalid) acc = acc * kP16 + accq[q];
    const uint64_t cend = cta0 + kWB;
    if (tid == 0) sh.pblk = cend <= j.n ? pow64(kFnvP, j.n - cend) : 0;
    __syncthreads();
    uint64_t contrib = 0;
    if (nvalid > 0) {
      const uint64_t tend = pos0 + 16u * nvalid;
      contrib = acc * (cend <= j.n ? sh.pblk * sh.pw[kWT - 1 - tid] : pow64(kFnvP, j.n - tend));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
    if (lane == 0) sh.wsum[warp] = contrib;
    __syncthreads();
    if (tid == 0) {
      uint64_t sum = 0;
#pragma unroll
      for (int x = 0; x < kWT / 32; ++x) sum += sh.wsum[x];
      atomicAdd(out + c, static_cast<unsigned long long>(sum));
    }
  }
}

// ---------------------------------------------------------------------------
// Two bits per round (k_fnv_window_sl2, the default; GS_FNV_PAIRS=0 keeps one
// bit per round). Bit K+1 depends on x_K, i.e. on the carry of bit K into the
// thread, which the window-level scan only knows later -- so bit K+1 is
// evaluated for BOTH values of that carry. A thread is then a two-state
// transducer (f = its bit-K parity, o_s = its bit-(K+1) parity when its
// incoming bit-K carry is s); transducers compose associatively,
//   (a then b) = (a.f ^ b.f, o_s = a.o_s ^ b.o_{s ^ a.f}),
// and a level of items (lanes / warps / CTAs / predecessor windows) composes
// with bit masks: P = exclusive prefix XOR of the f bits, then the item
// outputs for start state 0 / 1 are (o0 & ~P) | (o1 & P) / (o1 & ~P) | (o0 & P).
// A window's transducer does not depend on its entry bits, so it is
// published at once and the look-back composes predecessors' transducers up
// to one with published exit bits. One cluster barrier and one look-back per
// PAIR of bits: four per window instead of eight.
// ---------------------------------------------------------------------------
struct Tx {
  uint32_t f, o0, o1;
};
__device__ __forceinline__ Tx tx_then(Tx a, Tx b) {  // a, then b
  return Tx{a.f ^ b.f, a.o0 ^ (a.f ? b.o1 : b.o0), a.o1 ^ (a.f ? b.o0 : b.o1)};
}
__device__ __forceinline__ uint32_t excl_prefix_bits(uint32_t m) {  // bit i = XOR of bits < i
  return sl_prefix32(m) << 1;
}
// Compose the items of a level given as bit masks (bit i = item i, in chain
// order), restricted to `sel`: the composition of the selected items.
__device__ __forceinline__ Tx tx_masks(uint32_t fm, uint32_t o0m, uint32_t o1m, uint32_t sel) {
  fm &= sel;
  o0m &= sel;
  o1m &= sel;
  const uint32_t p = excl_prefix_bits(fm);
  const uint32_t a0 = (o0m & ~p) | (o1m & p), a1 = (o1m & ~p) | (o0m & p);
  return Tx{static_cast<uint32_t>(__popc(fm) & 1), static_cast<uint32_t>(__popc(a0) & 1),
            static_cast<uint32_t>(__popc(a1) & 1)};
}

// Per pair, the carry-save variables that depend on x_K (hypothesis state).
template <int K>
struct SlHyp {
  uint32_t c23, c45b, s5, c56b, c67d;
};
// g_{K+1} for a given x_K plane (and the x_K-dependent carry-save values).
template <int K>
__device__ __forceinline__ uint32_t sl_next(SlCol& c, uint32_t xk, SlHyp<K>& h) {
  if constexpr (K == 0) {
    return xk;  // column 1 = {x1, x0}
  } else if constexpr (K == 2) {
    h.c23 = sl_maj(xk, c.X[1], c.c12);
    return xk ^ h.c23;  // column 3 = {x3, x2, c23}
  } else if constexpr (K == 4) {
    h.c45b = xk & c.s4;
    h.s5 = c.s5a_ ^ xk ^ h.c45b;
    h.c56b = sl_maj(c.s5a_, xk, h.c45b);
    return h.s5;
  } else {
    h.c67d = xk & c.s6;
    return xk ^ c.X[3] ^ c.X[2] ^ c.X[0] ^ c.c67a ^ c.c67b ^ c.c67c ^ h.c67d;
  }
}
// x_K-independent pre-reduction of columns K and K+1 (before the pair).
template <int K>
__device__ __forceinline__ uint32_t sl_pre(SlCol& c) {  // returns G_K
  if constexpr (K == 0) {
    return 0u;
  } else if constexpr (K == 2) {
    return c.X[1] ^ c.c12;
  } else if constexpr (K == 4) {
    c.s4 = c.X[3] ^ c.X[0] ^ c.c34;
    c.c45a = sl_maj(c.X[3], c.X[0], c.c34);
    c.s5a_ = c.X[1] ^ c.X[0] ^ c.c45a;
    c.c56a = sl_maj(c.X[1], c.X[0], c.c45a);
    return c.s4;
  } else {
    const uint32_t s6a = c.X[2] ^ c.X[1] ^ c.c56a;
    c.c67a = sl_maj(c.X[2], c.X[1], c.c56a);
    const uint32_t s6b = s6a ^ c.c56b ^ c.c56c;
    c.c67b = sl_maj(s6a, c.c56b, c.c56c);
    c.s6 = s6b ^ c.X[5];
    c.c67c = s6b & c.X[5];
    return c.s6;
  }
}
// Commit the chosen hypothesis and the carries out of column K+1.
template <int K>
__device__ __forceinline__ void sl_commit(SlCol& c, uint32_t xk, uint32_t xk1, const SlHyp<K>& h) {
  c.X[K] = xk;
  c.X[K + 1] = xk1;
  if constexpr (K == 0) {
    c.c12 = xk1 & xk;
  } else if constexpr (K == 2) {
    c.c23 = h.c23;
    c.c34 = sl_maj(xk1, xk, h.c23);
  } else if constexpr (K == 4) {
    c.c45b = h.c45b;
    c.s5 = h.s5;
    c.c56b = h.c56b;
    c.c56c = xk1 & h.s5;
  } else {
    c.c67d = h.c67d;
  }
}

struct WinSharedPair {
  uint64_t pw[kWT];                  // P^(64 t)
  uint32_t wm[4][3][kWCS];           // [pair][f, o0, o1][cluster rank]: bit x = warp x of that CTA
  uint32_t gw;
  unsigned long long wsum[kWT / 32];
  uint64_t pblk;
};

// Window flag word, 7 bits per pair P at 7P: transducer f, o0, o1, valid;
// exit bits K, K+1, valid.
template <int P>
__device__ __forceinline__ void lookback_pair(const uint32_t* flags, uint32_t gw, uint32_t w, uint32_t nc,
                                              uint64_t h0, uint32_t& eK, uint32_t& eK1) {
  constexpr int K = 2 * P, B = 7 * P;
  const int lane = threadIdx.x & 31;
  Tx acc{0, 0, 0};  // composition of the windows between the search front and w (chain order)
  uint32_t back = 0;
  for (;;) {
    const uint32_t dist = back + lane + 1;  // lane l: predecessor w - dist (nearest first)
    const bool exists = dist <= w;
    uint32_t v = 0;
    if (exists) v = ld_acquire_u32(flags + (gw - dist * nc));
    const bool have_t = exists && ((v >> (B + 3)) & 1u);
    const bool have_x = exists && ((v >> (B + 6)) & 1u);
    const bool start = !exists && dist == w + 1;
    const uint32_t stop_bal = __ballot_sync(0xFFFFFFFFu, have_x || start);
    const int first = stop_bal ? __ffs(stop_bal) - 1 : 32;
    const uint32_t need = first >= 32 ? 0xFFFFFFFFu : ((1u << first) - 1u);
    const uint32_t ok = __ballot_sync(0xFFFFFFFFu, have_t);
    if ((ok & need) != need) continue;  // a nearer transducer is not published yet: spin
    // lanes < first, in chain order (farthest first): bit-reverse the lane masks
    const uint32_t fm = __brev(__ballot_sync(0xFFFFFFFFu, (v >> B) & 1u) & need);
    const uint32_t o0m = __brev(__ballot_sync(0xFFFFFFFFu, (v >> (B + 1)) & 1u) & need);
    const uint32_t o1m = __brev(__ballot_sync(0xFFFFFFFFu, (v >> (B + 2)) & 1u) & need);
    const Tx blk = tx_masks(fm, o0m, o1m, 0xFFFFFFFFu);
    acc = tx_then(blk, acc);  // this block is farther in the chain than what acc holds
    if (first < 32) {
      const uint32_t ax = __shfl_sync(0xFFFFFFFFu, start ? static_cast<uint32_t>(h0 >> K) : (v >> (B + 4)), first) & 1u;
      const uint32_t ax1 =
          __shfl_sync(0xFFFFFFFFu, start ? static_cast<uint32_t>(h0 >> (K + 1)) : (v >> (B + 5)), first) & 1u;
      eK = ax ^ acc.f;
      eK1 = ax1 ^ (ax ? acc.o1 : acc.o0);
      return;
    }
    back += 32;
  }
}

template <int P>
__device__ __forceinline__ void win_pair_sl(WinSharedPair& sh, uint32_t* flags, uint32_t gw, uint32_t w, uint32_t nc,
                                            uint64_t h0, uint32_t rank, SlCol (&G)[2], uint32_t& flag_word) {
  constexpr int K = 2 * P, B = 7 * P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // bit K (independent of the entry bits)
  uint32_t incK[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) incK[q] = sl_prefix32(G[q].B[K] ^ sl_pre<K>(G[q]));
  const uint32_t pK0 = incK[0] >> 31, fT = pK0 ^ (incK[1] >> 31);
  const uint32_t relK0 = incK[0] << 1, relK1 = (incK[1] << 1) ^ (0u - pK0);
  // bit K+1 under both values h of the thread's incoming bit-K carry
  SlHyp<K> hy[2][2] = {};
  uint32_t incH[2][2], oT[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const uint32_t xk = (q == 0 ? relK0 : relK1) ^ (0u - static_cast<uint32_t>(h)) ^ G[q].B[K];
      incH[h][q] = sl_prefix32(G[q].B[K + 1] ^ sl_next<K>(G[q], xk, hy[h][q]));
    }
    oT[h] = (incH[h][0] >> 31) ^ (incH[h][1] >> 31);
  }
  // lanes
  const uint32_t fm = __ballot_sync(0xFFFFFFFFu, fT);
  const uint32_t o0m = __ballot_sync(0xFFFFFFFFu, oT[0]);
  const uint32_t o1m = __ballot_sync(0xFFFFFFFFu, oT[1]);
  const Tx t_lanes = tx_masks(fm, o0m, o1m, (1u << lane) - 1u);
  const Tx t_warp = tx_masks(fm, o0m, o1m, 0xFFFFFFFFu);
  if (lane < kWCS) {
    if (t_warp.f) or_cluster_u32(&sh.wm[P][0][rank], static_cast<uint32_t>(lane), 1u << warp);
    if (t_warp.o0) or_cluster_u32(&sh.wm[P][1][rank], static_cast<uint32_t>(lane), 1u << warp);
    if (t_warp.o1) or_cluster_u32(&sh.wm[P][2][rank], static_cast<uint32_t>(lane), 1u << warp);
  }
  cluster_sync_all();
  // warps of this CTA before mine, and the CTAs' totals
  const Tx t_warps = tx_masks(sh.wm[P][0][rank], sh.wm[P][1][rank], sh.wm[P][2][rank], (1u << warp) - 1u);
  // CTA r's total computed by lane r of every warp, gathered as masks
  Tx tc{0, 0, 0};
  if (lane < kWCS) tc = tx_masks(sh.wm[P][0][lane], sh.wm[P][1][lane], sh.wm[P][2][lane], 0xFFFFFFFFu);
  const uint32_t cf = __ballot_sync(0xFFFFFFFFu, tc.f) & ((1u << kWCS) - 1u);
  const uint32_t co0 = __ballot_sync(0xFFFFFFFFu, tc.o0) & ((1u << kWCS) - 1u);
  const uint32_t co1 = __ballot_sync(0xFFFFFFFFu, tc.o1) & ((1u << kWCS) - 1u);
  const Tx t_ctas = tx_masks(cf, co0, co1, (1u << rank) - 1u);
  const Tx t_win = tx_masks(cf, co0, co1, 0xFFFFFFFFu);
  if (rank == 0 && warp == 0 && lane == 0) {
    flag_word |= ((t_win.f | (t_win.o0 << 1) | (t_win.o1 << 2)) << B) | (1u << (B + 3));
    st_release_u32(flags + gw, flag_word);
  }
  uint32_t eK, eK1;
  if (w == 0) {
    eK = static_cast<uint32_t>(h0 >> K) & 1u;
    eK1 = static_cast<uint32_t>(h0 >> (K + 1)) & 1u;
  } else {
    lookback_pair<P>(flags, gw, w, nc, h0, eK, eK1);
  }
  if (rank == 0 && warp == 0 && lane == 0) {
    const uint32_t xK = eK ^ t_win.f, xK1 = eK1 ^ (eK ? t_win.o1 : t_win.o0);
    flag_word |= ((xK | (xK1 << 1)) << (B + 4)) | (1u << (B + 6));
    st_release_u32(flags + gw, flag_word);
  }
  // this thread's incoming carries
  const Tx before = tx_then(tx_then(t_ctas, t_warps), t_lanes);
  const uint32_t cK = before.f ^ eK;
  const uint32_t cK1 = (eK ? before.o1 : before.o0) ^ eK1;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const uint32_t xk = (q == 0 ? relK0 : relK1) ^ (0u - cK) ^ G[q].B[K];
    const uint32_t inc = cK ? incH[1][q] : incH[0][q];
    const uint32_t pre = q == 0 ? 0u : ((cK ? incH[1][0] : incH[0][0]) >> 31);
    const uint32_t l1 = (inc << 1) ^ (0u - (pre ^ cK1));
    const uint32_t xk1 = l1 ^ G[q].B[K + 1];
    SlHyp<K> hs;  // the chosen hypothesis, field by field (no dynamic indexing: registers, not stack)
    hs.c23 = cK ? hy[1][q].c23 : hy[0][q].c23;
    hs.c45b = cK ? hy[1][q].c45b : hy[0][q].c45b;
    hs.s5 = cK ? hy[1][q].s5 : hy[0][q].s5;
    hs.c56b = cK ? hy[1][q].c56b : hy[0][q].c56b;
    hs.c67d = cK ? hy[1][q].c67d : hy[0][q].c67d;
    sl_commit<K>(G[q], xk, xk1, hs);
  }
}

__global__ void __cluster_dims__(kWCS, 1, 1) __launch_bounds__(kWT, 2)
    k_fnv_window_sl2(const FnvJob j, uint64_t h0, const uint64_t* __restrict__ h0s, uint32_t nc, uint32_t total_windows,
                    uint32_t* counter, uint32_t* flags, unsigned long long* __restrict__ out) {
  __shared__ WinSharedPair sh;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  sh.pw[tid] = pow64(kFnvP, static_cast<uint64_t>(kFPer) * tid);
  cluster_sync_all();  // every CTA of the cluster has started before rank 0 writes into their smem
  for (;;) {
    if (tid < 4 * 3 * kWCS) (&sh.wm[0][0][0])[tid] = 0;  // this window's transducer words
    if (rank == 0 && tid == 0) {
      const uint32_t g = atomicAdd(counter, 1u);
      for (int r = 0; r < kWCS; ++r) st_cluster_u32(&sh.gw, static_cast<uint32_t>(r), g);
    }
    cluster_sync_all();
    const uint32_t gw = sh.gw;
    if (gw >= total_windows) break;
    const uint32_t w = gw / nc, c = gw - w * nc;
    const uint64_t hc = h0s ? h0s[c] : h0;
    const uint64_t cta0 = static_cast<uint64_t>(w) * kWin + static_cast<uint64_t>(rank) * kWB;
    const uint64_t pos0 = cta0 + static_cast<uint64_t>(tid) * kFPer;
    SlCol G[2];
    {
      uint4 d[4];
      load_groups(j, c, pos0, d);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint32_t wv[8] = {d[2 * q].x, d[2 * q].y, d[2 * q].z, d[2 * q].w,
                          d[2 * q + 1].x, d[2 * q + 1].y, d[2 * q + 1].z, d[2 * q + 1].w};
        sl_to_planes(wv);
#pragma unroll
        for (int b = 0; b < 8; ++b) G[q].B[b] = wv[b];
      }
    }
    uint32_t fw = 0;
    win_pair_sl<0>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_pair_sl<1>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_pair_sl<2>(sh, flags, gw, w, nc, hc, rank, G, fw);
    win_pair_sl<3>(sh, flags, gw, w, nc, hc, rank, G, fw);
    // low bytes s = x ^ b back to byte lanes; the data re-read (cache-resident)
    uint4 s[4], d[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      uint32_t wv[8];
#pragma unroll
      for (int b = 0; b < 8; ++b) wv[b] = G[q].X[b] ^ G[q].B[b];
      sl_from_planes(wv);
      s[2 * q] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
      s[2 * q + 1] = make_uint4(wv[4], wv[5], wv[6], wv[7]);
    }
    const int nvalid = load_groups(j, c, pos0, d);
    // sum over the thread's bytes of d_i P^(tend - i), four 16-byte Horner chains
    uint64_t accq[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (q < nvalid) {
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          const uint32_t sw = wd(s[q], x), xw = sw ^ wd(d[q], x);
#pragma unroll
          for (int by = 0; by < 4; ++by) {
            const int64_t di = static_cast<int64_t>((xw >> (8 * by)) & 0xFFu) -
                               static_cast<int64_t>((sw >> (8 * by)) & 0xFFu);
            accq[q] = (accq[q] + static_cast<uint64_t>(di)) * kFnvP;
          }
        }
      }
    }
    constexpr uint64_t kP16 = [] {
      uint64_t r = 1;
      for (int i = 0; i < 16; ++i) r *= kFnvP;
      return r;
    }();
    uint64_t acc = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q < nvalid) acc = acc * kP16 + accq[q];
    const uint64_t cend = cta0 + kWB;
    if (tid == 0) sh.pblk = cend <= j.n ? pow64(kFnvP, j.n - cend) : 0;
    __syncthreads();
    uint64_t contrib = 0;
    if (nvalid > 0) {
      const uint64_t tend = pos0 + 16u * nvalid;
      contrib = acc * (cend <= j.n ? sh.pblk * sh.pw[kWT - 1 - tid] : pow64(kFnvP, j.n - tend));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) contrib += __shfl_xor_sync(0xFFFFFFFFu, contrib, o);
    if (lane == 0) sh.wsum[warp] = contrib;
    __syncthreads();
    if (tid == 0) {
      uint64_t sum = 0;
#pragma unroll
      for (int x = 0; x < kWT / 32; ++x) sum += sh.wsum[x];
      atomicAdd(out + c, static_cast<unsigned long long>(sum));
    }
  }
}

const bool g_fnv_legacy = [] {
  const char* e = std::getenv("GS_FNV_LEGACY");
  return e && std::atoi(e) != 0;
}();
const bool g_fnv_bytes = [] {  // the byte-lane window rounds instead of the bit-sliced ones (A/B)
  const char* e = std::getenv("GS_FNV_WINDOW_BYTES");
  return e && std::atoi(e) != 0;
}();
const bool g_fnv_pairs = [] {  // bit-sliced rounds two bits at a time (GS_FNV_PAIRS=0: one bit, A/B)
  const char* e = std::getenv("GS_FNV_PAIRS");
  return !(e && std::atoi(e) == 0);
}();
int g_win_clusters = 0;

int g_sms = 0;
std::mutex g_pool_mu;
std::set<int> g_pool_tuned;

// Keep the device's stream-ordered allocations mapped between calls (the
// scratch of the FNV kernels and the verification buffers are reused at
// every call), and cache the SM count.
void tune_pool(int dev) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  if (!g_sms) cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
  if (!g_pool_tuned.count(dev)) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    g_pool_tuned.insert(dev);
  }
}

}  // namespace

static int fnv_device(const void* const* bufs, int n_chains, int k, uint64_t len, uint64_t h0, const uint64_t* d_h0,
                      uint64_t* d_out, void* stream);

extern "C" int gs_fnv1a64_device(const void* const* bufs, int n_chains, int k, uint64_t len, uint64_t h0,
                                 uint64_t* d_out, void* stream) {
  return fnv_device(bufs, n_chains, k, len, h0, nullptr, d_out, stream);
}

extern "C" int gs_fnv1a64_device_seeded(const void* const* bufs, int n_chains, int k, uint64_t len,
                                        const uint64_t* d_h0, uint64_t* d_out, void* stream) {
  if (!d_h0 || d_h0 == d_out) return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device_seeded: seeds NULL or aliasing out");
  return fnv_device(bufs, n_chains, k, len, 0, d_h0, d_out, stream);
}

static int fnv_device(const void* const* bufs, int n_chains, int k, uint64_t len, uint64_t h0, const uint64_t* d_h0,
                      uint64_t* d_out, void* stream) {
  if (n_chains < 0 || k < 1 || k > kFCap || (n_chains > 0 && (!bufs || !d_out)))
    return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device: bad arguments");
  if (len % 16) return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device: buffer length must be a multiple of 16");
  for (int i = 0; i < n_chains * k; ++i)
    if (!bufs[i] || (reinterpret_cast<uintptr_t>(bufs[i]) & 15u))
      return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device: buffer %d is NULL or not 16-B aligned", i);
  if (reinterpret_cast<uintptr_t>(d_out) & 7u)
    return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device: output must be 8-B aligned");
  if (n_chains == 0) return GS_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return ffail(GS_CUDA_ERROR, "fnv1a64_device: %s", cudaGetErrorString(e));
  tune_pool(dev);
  const uint64_t n = static_cast<uint64_t>(k) * len;
  if (!g_fnv_legacy || d_h0) {
    k_fnv_init<<<(n_chains + 255) / 256, 256, 0, st>>>(d_out, n_chains, h0, n, d_h0);
    if ((e = cudaGetLastError()) != cudaSuccess) return ffail(GS_CUDA_ERROR, "fnv init: %s", cudaGetErrorString(e));
    if (n == 0) return GS_OK;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      if (!g_win_clusters) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kWCS, 1, 1);
        cfg.blockDim = dim3(kWT, 1, 1);
        int nc = 0;
        if (cudaOccupancyMaxActiveClusters(&nc, reinterpret_cast<void*>(k_fnv_window), &cfg) != cudaSuccess || nc < 1)
          nc = 1;
        cudaGetLastError();
        g_win_clusters = nc;
      }
    }
    const uint64_t nw64 = (n + kWin - 1) / kWin;
    const int per_job = std::max(1, std::min(kFCap / k, n_chains));
    const uint64_t max_total = nw64 * static_cast<uint64_t>(per_job);
    if (max_total > 0xFFFFFFF0ull) return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device: chain too long");
    uint32_t* ctl = nullptr;  // [counter, flags[total windows]]
    const size_t ctl_bytes = sizeof(uint32_t) * (1 + max_total);
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&ctl), ctl_bytes, st)) != cudaSuccess)
      return ffail(GS_CUDA_ERROR, "fnv window flags: %s", cudaGetErrorString(e));
    int status = GS_OK;
    for (int c0 = 0; c0 < n_chains && status == GS_OK; c0 += per_job) {
      const int cnt = std::min(per_job, n_chains - c0);
      FnvJob j{};
      for (int i = 0; i < cnt * k; ++i) j.p[i] = static_cast<const uint8_t*>(bufs[static_cast<size_t>(c0) * k + i]);
      j.k = k;
      j.len = len;
      j.n = n;
      const uint32_t total = static_cast<uint32_t>(nw64 * static_cast<uint64_t>(cnt));
      cudaError_t r = cudaMemsetAsync(ctl, 0, sizeof(uint32_t) * (1 + static_cast<size_t>(total)), st);
      const int clusters = static_cast<int>(std::min<uint64_t>(g_win_clusters, total));
      if (r == cudaSuccess) {
        if (g_fnv_bytes)
          k_fnv_window<<<clusters * kWCS, kWT, 0, st>>>(j, h0, d_h0 ? d_h0 + c0 : nullptr, static_cast<uint32_t>(cnt),
                                                       total, ctl, ctl + 1,
                                                       reinterpret_cast<unsigned long long*>(d_out) + c0);
        else if (g_fnv_pairs)
          k_fnv_window_sl2<<<clusters * kWCS, kWT, 0, st>>>(j, h0, d_h0 ? d_h0 + c0 : nullptr,
                                                           static_cast<uint32_t>(cnt), total, ctl, ctl + 1,
                                                           reinterpret_cast<unsigned long long*>(d_out) + c0);
        else
          k_fnv_window_sl<<<clusters * kWCS, kWT, 0, st>>>(j, h0, d_h0 ? d_h0 + c0 : nullptr,
                                                          static_cast<uint32_t>(cnt), total, ctl, ctl + 1,
                                                          reinterpret_cast<unsigned long long*>(d_out) + c0);
        r = cudaGetLastError();
      }
      if (r != cudaSuccess) status = ffail(GS_CUDA_ERROR, "fnv window kernel: %s", cudaGetErrorString(r));
    }
    cudaFreeAsync(ctl, st);
    return status;
  }
  const uint64_t bpc64 = (n + kFB - 1) / kFB;
  if (bpc64 > 0xFFFFFFFFull) return ffail(GS_INVALID_ARGUMENT, "fnv1a64_device: chain too long");
  const uint32_t bpc = static_cast<uint32_t>(bpc64);
  k_fnv_init<<<(n_chains + 255) / 256, 256, 0, st>>>(d_out, n_chains, h0, n, nullptr);
  if ((e = cudaGetLastError()) != cudaSuccess) return ffail(GS_CUDA_ERROR, "fnv init: %s", cudaGetErrorString(e));
  if (n == 0) return GS_OK;
  const uint64_t chain_scratch = bpc64 * kFB;
  int per_job = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(kScratchBudget / chain_scratch, kFCap / k)));
  per_job = std::min(per_job, n_chains);
  const size_t scratch_bytes = static_cast<size_t>(per_job) * chain_scratch;  // low bytes, then D planes (1/8)
  const size_t dplane_bytes = scratch_bytes / 8;
  const size_t meta = static_cast<size_t>(per_job) * bpc;
  uint8_t* mem = nullptr;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&mem), scratch_bytes + dplane_bytes + 2 * meta, st)) != cudaSuccess)
    return ffail(GS_CUDA_ERROR, "fnv scratch (%zu bytes): %s", scratch_bytes + dplane_bytes + 2 * meta,
                 cudaGetErrorString(e));
  uint64_t* dplane = reinterpret_cast<uint64_t*>(mem + scratch_bytes);
  uint8_t* agg = mem + scratch_bytes + dplane_bytes;
  uint8_t* entry = agg + meta;
  int status = GS_OK;
  for (int c0 = 0; c0 < n_chains && status == GS_OK; c0 += per_job) {
    const int cnt = std::min(per_job, n_chains - c0);
    FnvJob j{};
    for (int i = 0; i < cnt * k; ++i) j.p[i] = static_cast<const uint8_t*>(bufs[static_cast<size_t>(c0) * k + i]);
    j.k = k;
    j.len = len;
    j.n = n;
    j.bpc = bpc;
    j.nblocks = static_cast<uint32_t>(static_cast<uint64_t>(cnt) * bpc);
    const int grid = static_cast<int>(std::min<uint64_t>(j.nblocks, static_cast<uint64_t>(g_sms > 0 ? g_sms : 148) * 4));
    cudaError_t r = pair_and_scan<0>(j, grid, cnt, mem, dplane, agg, entry, h0, st);
    if (r == cudaSuccess) r = pair_and_scan<2>(j, grid, cnt, mem, dplane, agg, entry, h0, st);
    if (r == cudaSuccess) r = pair_and_scan<4>(j, grid, cnt, mem, dplane, agg, entry, h0, st);
    if (r == cudaSuccess) r = pair_and_scan<6>(j, grid, cnt, mem, dplane, agg, entry, h0, st);
    if (r == cudaSuccess) {
      k_fnv_final<<<grid, kFT, 0, st>>>(j, mem, dplane, entry, reinterpret_cast<unsigned long long*>(d_out) + c0);
      r = cudaGetLastError();
    }
    if (r != cudaSuccess) status = ffail(GS_CUDA_ERROR, "fnv kernels: %s", cudaGetErrorString(r));
  }
  cudaFreeAsync(mem, st);
  return status;
}

// Upload chunks' host parity rows into HBM on `copy` and checksum them on
// `compute` as they land (groups of kUpGroup chunks, one event per group), so
// the hashing of group g overlaps the upload of group g + 1.
extern "C" int gs_parity_upload_checksum(const void* const* h_parity, int n_chunks, int k, uint64_t len,
                                         void* const* d_parity, uint64_t* d_sums, void* compute, void* copy) {
  constexpr int kUpGroup = 4;
  constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
  if (n_chunks < 0 || k < 1 || (n_chunks > 0 && (!h_parity || !d_parity || !d_sums)))
    return ffail(GS_INVALID_ARGUMENT, "parity_upload_checksum: bad arguments");
  cudaStream_t cs = static_cast<cudaStream_t>(compute), ys = static_cast<cudaStream_t>(copy);
  for (int g0 = 0; g0 < n_chunks; g0 += kUpGroup) {
    const int cnt = std::min(kUpGroup, n_chunks - g0);
    for (int i = g0 * k; i < (g0 + cnt) * k; ++i) {
      if (!h_parity[i] || !d_parity[i]) return ffail(GS_INVALID_ARGUMENT, "parity_upload_checksum: NULL row %d", i);
      cudaError_t e = cudaMemcpyAsync(d_parity[i], h_parity[i], len, cudaMemcpyHostToDevice, ys);
      if (e != cudaSuccess) return ffail(GS_CUDA_ERROR, "parity upload: %s", cudaGetErrorString(e));
    }
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ev, ys);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev, 0);
    cudaEventDestroy(ev);  // released once the recorded work completes
    if (e != cudaSuccess) return ffail(GS_CUDA_ERROR, "parity upload event: %s", cudaGetErrorString(e));
    if (int s = gs_fnv1a64_device(d_parity + static_cast<size_t>(g0) * k, cnt, k, len, kOffset, d_sums + g0, cs))
      return s;
  }
  return GS_OK;
}

// K1's parity rows already in HBM (d_parity, written on `compute` before this
// call) -> pinned host rows on `copy`, and their chunk checksums computed on
// the GPU (`compute`) and copied to h_sums (pinned host or device) behind them: the seal of
// ParityChunk (parity_store.hpp:46-53) without a host FNV pass. Stream order:
// rows D2H after K1; sums D2H after the FNV; a store commit enqueued on `copy`
// after this call sees both.
extern "C" int gs_parity_offload_sealed(const void* const* d_parity, int n_chunks, int k, uint64_t len,
                                        void* const* h_parity, uint64_t* h_sums, void* compute, void* copy) {
  constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
  if (n_chunks < 0 || k < 1 || (n_chunks > 0 && (!d_parity || !h_parity || !h_sums)))
    return ffail(GS_INVALID_ARGUMENT, "parity_offload_sealed: bad arguments");
  if (n_chunks == 0) return GS_OK;
  cudaStream_t cs = static_cast<cudaStream_t>(compute), ys = static_cast<cudaStream_t>(copy);
  cudaEvent_t ev;
  cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(ev, cs);  // K1 done
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ys, ev, 0);
  for (int i = 0; e == cudaSuccess && i < n_chunks * k; ++i) {
    if (!d_parity[i] || !h_parity[i]) {
      cudaEventDestroy(ev);
      return ffail(GS_INVALID_ARGUMENT, "parity_offload_sealed: NULL row %d", i);
    }
  }
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    return ffail(GS_CUDA_ERROR, "parity offload: %s", cudaGetErrorString(e));
  }
  // rows of consecutive store entries merge into one copy (or one 2-D copy per row)
  if (int s = gsb::batch_copies(h_parity, d_parity, n_chunks * k, len, 1, ys)) {
    cudaEventDestroy(ev);
    return s;
  }
  uint64_t* d_sums = nullptr;
  e = cudaMallocAsync(reinterpret_cast<void**>(&d_sums), sizeof(uint64_t) * n_chunks, cs);
  if (e != cudaSuccess) {
    cudaEventDestroy(ev);
    return ffail(GS_CUDA_ERROR, "parity offload sums: %s", cudaGetErrorString(e));
  }
  int st = gs_fnv1a64_device(d_parity, n_chunks, k, len, kOffset, d_sums, cs);
  if (st == GS_OK) {
    // the few checksum bytes travel on the compute stream: a small copy queued
    // on `copy` between two blocks' parity rows costs the host link a DMA
    // round trip per call (C2 blocks: ~5% of the offload rate)
    e = cudaMemcpyAsync(h_sums, d_sums, sizeof(uint64_t) * n_chunks, cudaMemcpyDefault, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev, cs);  // checksums landed
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ys, ev, 0);
    if (e != cudaSuccess) st = ffail(GS_CUDA_ERROR, "parity offload sums: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(d_sums, cs);
  cudaEventDestroy(ev);
  return st;
}

// ---------------------------------------------------------------------------
// Recovery-side verification split between the GPU and host threads.
//
// Chunks [0, n_full) upload all k parity rows and are hashed entirely on the
// GPU. Chunks [n_full, n) upload only their first u rows (the rows K2 uses);
// the GPU hashes those rows, giving the chain state after row u-1, and host
// threads continue the serial chain over rows u..k-1 from the host copy. A
// host-verified chunk therefore costs one serial chain over (k-u) rows
// instead of k, and its u rows cross the link once (for the decode AND the
// hash). Host chunks go first on the copy stream so their threads start early.
// ---------------------------------------------------------------------------
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <thread>
#include <vector>

#include "gs_fnv.hpp"

struct gs_verify {
  int n = 0, n_full = 0, k = 0, u = 0;
  uint64_t len = 0;
  std::vector<const uint8_t*> host_rows;  // n * k
  uint64_t* pinned = nullptr;             // [0, n): GPU sums (full) / chain states after row u-1 (split)
  std::vector<cudaEvent_t> group_ev;      // per split group: its states are in `pinned`
  std::vector<int> group_of;              // chunk -> group index (split chunks)
  cudaEvent_t full_ev = nullptr;          // full chunks' sums are in `pinned`
  // dynamic mode (n_full < 0): the rows >= u of each chunk are hashed by
  // whichever side claims the chunk first -- host threads from the front (as
  // the chunks' GPU states arrive), a GPU feeder from the back (upload into a
  // ring + seeded GPU FNV continuing from the state)
  bool dynamic = false;
  int device = 0;
  cudaStream_t cs = nullptr, ys = nullptr;
  uint64_t* d_state = nullptr;            // [n] chain states after rows < u (device)
  uint64_t* d_sum = nullptr;              // [n] GPU-continued checksums (device)
  uint64_t* gsum = nullptr;               // [n] the same, pinned
  uint8_t* ring = nullptr;                // kRing slots x (k - u) rows x len
  std::vector<cudaEvent_t> slot_ev;       // slot's last hash + sum D2H done
  std::vector<cudaEvent_t> up_ev;         // slot's upload landed
  std::mutex mu;
  int lo = 0, hi = -1;                    // unclaimed chunks [lo, hi]
  std::vector<char> on_gpu;               // chunk claimed by the GPU feeder
  // claim pacing (gs_verify_set_rates): a host thread takes chunks only while
  // it would finish them before the GPU could finish everything unclaimed
  double link_bps = 0, host_chain_bps = 0;
  // hand-offs: a host thread that falls behind the GPU publishes its chain
  // state at a byte offset and the feeder finishes the chain on the GPU
  struct Handoff {
    int c;
    uint64_t off;
  };
  std::deque<Handoff> handoffs;
  uint64_t handoff_bytes = 0;             // queued for the GPU, not yet issued
  uint64_t* hseed = nullptr;              // [n] host chain states of handed-off chunks (pinned)
  uint64_t* d_seed = nullptr;             // [n] the same on the device
  void* host_block = nullptr;             // pinned, recycled: [pinned | gsum | hseed]
  size_t host_bytes = 0;
  uint8_t* dev_block = nullptr;           // stream-ordered on cs: [d_state | d_sum | d_seed | ring]
  int hosts_active = 0;
  std::condition_variable cv;
  // the feeder leaves unclaimed chunks to the host threads until this many
  // seconds into finish (its uploads queue behind the row-0 uploads anyway)
  double feeder_hold_s = 0;
  std::chrono::steady_clock::time_point t0;
  // gs_verify_hold / gs_verify_release: a caller still queueing work behind
  // the upload events (gs_verify_stream_wait) keeps finish from destroying them
  int holds = 0;
  std::mutex hold_mu;
  std::condition_variable hold_cv;
  void wait_unheld() {
    std::unique_lock<std::mutex> lk(hold_mu);
    hold_cv.wait(lk, [&] { return holds == 0; });
  }
};

namespace {
constexpr int kSplitGroup = 4;  // chunks per GPU hash launch / host lockstep group
constexpr int kRing = 4;        // dynamic mode: GPU-claimed chunks in flight
std::atomic<uint64_t> g_verify_handoffs{0};  // chains a host thread handed over to the GPU
// last dynamic verification: host threads done, feeder done, hash stream
// drained (s after finish started), chunks by host / GPU / handed off
std::mutex g_vstats_mu;
double g_vstats[6] = {0, 0, 0, 0, 0, 0};
}

extern "C" uint64_t gs_verify_handoffs(void) { return g_verify_handoffs.load(); }

namespace {
// Small pinned arrays of the dynamic verification, recycled across calls:
// cudaFreeHost synchronises the whole device (it would wait for every stream
// of the caller -- e.g. an unrelated decode -- at the end of a verification).
std::mutex g_pinned_mu;
std::vector<std::pair<size_t, void*>> g_pinned_free;

void* pinned_take(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    for (size_t i = 0; i < g_pinned_free.size(); ++i)
      if (g_pinned_free[i].first >= bytes) {
        void* p = g_pinned_free[i].second;
        g_pinned_free.erase(g_pinned_free.begin() + static_cast<long>(i));
        return p;
      }
  }
  void* p = nullptr;
  return cudaMallocHost(&p, std::max<size_t>(bytes, 4096)) == cudaSuccess ? p : nullptr;
}
void pinned_give(void* p, size_t bytes) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back({std::max<size_t>(bytes, 4096), p});
}
}  // namespace

extern "C" int gs_verify_last_stats(double* out6) {
  if (!out6) return ffail(GS_INVALID_ARGUMENT, "verify_last_stats: NULL output");
  std::lock_guard<std::mutex> lk(g_vstats_mu);
  for (int i = 0; i < 6; ++i) out6[i] = g_vstats[i];
  return GS_OK;
}

// Dynamic split (n_full < 0, the recovery default): rows 0..u-1 of EVERY
// chunk are uploaded (the decode needs them anyway) and hashed on the GPU in
// groups; the rest of each chain is claimed at run time -- host threads take
// chunks from the front as their GPU states land, a feeder thread takes them
// from the back and uploads their remaining rows behind the row-0 uploads,
// continuing the chain on the GPU from the device state. Whichever side is
// faster on this host takes more chunks; both finish together.
static int verify_enqueue_dynamic(const void* const* h_parity, int n_chunks, int k, uint64_t len, int u,
                                  void* const* d_parity, cudaStream_t cs, cudaStream_t ys, gs_verify** out) {
  constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
  auto* v = new gs_verify;
  v->dynamic = true;
  v->n = n_chunks;
  v->k = k;
  v->u = u;
  v->len = len;
  v->cs = cs;
  v->ys = ys;
  v->lo = 0;
  v->hi = n_chunks - 1;
  v->on_gpu.assign(n_chunks, 0);
  cudaGetDevice(&v->device);
  v->host_rows.resize(static_cast<size_t>(n_chunks) * k);
  for (size_t i = 0; i < v->host_rows.size(); ++i) v->host_rows[i] = static_cast<const uint8_t*>(h_parity[i]);
  v->group_of.assign(n_chunks, -1);
  auto bail = [&](int st) {
    cudaStreamSynchronize(cs);
    cudaStreamSynchronize(ys);
    for (auto e : v->group_ev) cudaEventDestroy(e);
    for (auto e : v->slot_ev) cudaEventDestroy(e);
    for (auto e : v->up_ev) cudaEventDestroy(e);
    pinned_give(v->host_block, v->host_bytes);
    if (v->dev_block) cudaFreeAsync(v->dev_block, cs);
    delete v;
    return st;
  };
  tune_pool(v->device);
  const size_t nb = sizeof(uint64_t) * std::max(1, n_chunks);
  v->host_bytes = 3 * nb;
  v->host_block = pinned_take(v->host_bytes);
  cudaError_t e = v->host_block ? cudaSuccess : cudaErrorMemoryAllocation;
  if (e == cudaSuccess) {
    v->pinned = static_cast<uint64_t*>(v->host_block);
    v->gsum = v->pinned + std::max(1, n_chunks);
    v->hseed = v->gsum + std::max(1, n_chunks);
    const size_t ring = k > u ? static_cast<size_t>(kRing) * (k - u) * len : 0;
    e = cudaMallocAsync(reinterpret_cast<void**>(&v->dev_block), 3 * nb + 256 + ring, cs);
  }
  if (e == cudaSuccess) {
    v->d_state = reinterpret_cast<uint64_t*>(v->dev_block);
    v->d_sum = v->d_state + std::max(1, n_chunks);
    v->d_seed = v->d_sum + std::max(1, n_chunks);
    if (k > u) v->ring = v->dev_block + (3 * nb + 255) / 256 * 256;
    cudaEvent_t ready;  // the copy stream's ring uploads come after the stream-ordered allocation
    e = cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventRecord(ready, cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ys, ready, 0);
    cudaEventDestroy(ready);
  }
  for (int r = 0; e == cudaSuccess && k > u && r < kRing; ++r) {
    cudaEvent_t a, b;
    e = cudaEventCreateWithFlags(&a, cudaEventDisableTiming | cudaEventBlockingSync);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&b, cudaEventDisableTiming);
    if (e == cudaSuccess) {
      v->slot_ev.push_back(a);
      v->up_ev.push_back(b);
    }
  }
  if (e != cudaSuccess) return bail(ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e)));
  cudaEvent_t up;
  if ((e = cudaEventCreateWithFlags(&up, cudaEventDisableTiming)) != cudaSuccess)
    return bail(ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e)));
  int st = GS_OK;
  for (int g0 = 0; g0 < n_chunks && st == GS_OK; g0 += kSplitGroup) {
    const int cnt = std::min(kSplitGroup, n_chunks - g0);
    for (int c = g0; c < g0 + cnt && e == cudaSuccess; ++c)
      for (int i = 0; i < u && e == cudaSuccess; ++i) {
        const size_t r = static_cast<size_t>(c) * k + i;
        e = (!h_parity[r] || !d_parity[r]) ? cudaErrorInvalidValue
                                           : cudaMemcpyAsync(d_parity[r], h_parity[r], len, cudaMemcpyHostToDevice, ys);
      }
    if (e == cudaSuccess) e = cudaEventRecord(up, ys);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, up, 0);
    if (e != cudaSuccess) {
      st = ffail(GS_CUDA_ERROR, "verify_enqueue upload: %s", cudaGetErrorString(e));
      break;
    }
    std::vector<const void*> rows(static_cast<size_t>(cnt) * u);
    for (int c = 0; c < cnt; ++c)
      for (int i = 0; i < u; ++i) rows[static_cast<size_t>(c) * u + i] = d_parity[static_cast<size_t>(g0 + c) * k + i];
    if ((st = gs_fnv1a64_device(rows.data(), cnt, u, len, kOffset, v->d_state + g0, cs)) != GS_OK) break;
    cudaEvent_t ge;
    e = cudaEventCreateWithFlags(&ge, cudaEventDisableTiming | cudaEventBlockingSync);
    if (e == cudaSuccess) {
      v->group_ev.push_back(ge);
      e = cudaMemcpyAsync(v->pinned + g0, v->d_state + g0, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost, cs);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ge, cs);
    if (e != cudaSuccess) st = ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e));
    for (int c = g0; c < g0 + cnt; ++c) v->group_of[c] = static_cast<int>(v->group_ev.size()) - 1;
  }
  cudaEventDestroy(up);
  if (st != GS_OK) return bail(st);
  *out = v;
  return GS_OK;
}

// End-game balancing of the dynamic split (GS_VERIFY_ENDGAME=0: off, for
// A/B): idle host threads keep claiming chunks until the row-0 uploads are
// over, and once the link is free a host thread hands the rest of its chain
// to the GPU feeder when the upload + GPU hash of that rest (queued behind
// the rows already handed over) would end sooner -- the chains' serial
// 80 MiB units otherwise leave the last few chunks to a thread or two while
// the rest idle (tools/c3_threads_trace.sh).
static bool v_endgame() {
  static const bool on = [] {
    const char* e = std::getenv("GS_VERIFY_ENDGAME");
    return !(e && e[0] == '0');
  }();
  return on;
}

// GS_VERIFY_TRACE=1: one stderr line per claim of the dynamic split (who,
// chunk, whole chain or continuation, claim / state-ready / done seconds), for
// reading where the verification's tail goes (tools/c3_probe.py).
static bool v_trace() {
  static const bool on = [] {
    const char* e = std::getenv("GS_VERIFY_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}
struct VTrace {
  int who, chunk, kind;  // who: host thread index, -1 = GPU feeder; kind: 0 continuation, 1 whole, 2 feeder, 3 handed over
  double claim, ready, done;
};
static std::mutex g_vtrace_mu;
static std::vector<VTrace> g_vtrace;
static void vtrace_push(const VTrace& t) {
  if (!v_trace()) return;
  std::lock_guard<std::mutex> lk(g_vtrace_mu);
  g_vtrace.push_back(t);
}

// The GPU feeder: hashes the remaining rows (u..k-1, one contiguous chain of
// (k-u)*len bytes per chunk) of (a) chunks handed off by host threads, from
// their byte offset and host state, and (b) unclaimed chunks, taken from the
// back, from their device state. Each goes through a ring slot: upload on the
// copy stream, seeded GPU FNV on the hash stream, checksum to pinned.
static int verify_feeder(gs_verify* v) {
  cudaSetDevice(v->device);
  int issued = 0, st = GS_OK;
  const uint64_t total = static_cast<uint64_t>(v->k - v->u) * v->len;
  for (;;) {
    const int r = issued % kRing;
    if (issued >= kRing && cudaEventSynchronize(v->slot_ev[r]) != cudaSuccess)  // slot free again
      return ffail(GS_CUDA_ERROR, "verify feeder: slot wait failed");
    int c = -1;
    uint64_t off = 0;
    {
      std::unique_lock<std::mutex> lk(v->mu);
      for (;;) {
        if (!v->handoffs.empty()) {
          c = v->handoffs.front().c;
          off = v->handoffs.front().off;
          v->handoffs.pop_front();
          v->handoff_bytes -= total - off;
          v->on_gpu[c] = 2;
          break;
        }
        const bool held = std::chrono::duration<double>(std::chrono::steady_clock::now() - v->t0).count() <
                          v->feeder_hold_s && v->hosts_active > 0;
        if (v->lo <= v->hi && !held) {
          c = v->hi--;
          v->on_gpu[c] = 1;
          break;
        }
        if (v->hosts_active == 0 && v->lo > v->hi) break;
        v->cv.wait_for(lk, std::chrono::microseconds(200));
      }
    }
    if (c < 0) break;
    if (v_trace()) {
      const double t = std::chrono::duration<double>(std::chrono::steady_clock::now() - v->t0).count();
      vtrace_push({-1, c, 2, t, t, t});
    }
    uint8_t* slot = v->ring + static_cast<size_t>(r) * total;
    cudaError_t e = cudaSuccess;
    for (uint64_t o = off; o < total && e == cudaSuccess;) {  // the chain's bytes [off, total), packed
      const uint64_t row = o / v->len, in = o - row * v->len, n = v->len - in;
      e = cudaMemcpyAsync(slot + (o - off), v->host_rows[static_cast<size_t>(c) * v->k + v->u + row] + in, n,
                          cudaMemcpyHostToDevice, v->ys);
      o += n;
    }
    if (e == cudaSuccess) e = cudaEventRecord(v->up_ev[r], v->ys);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(v->cs, v->up_ev[r], 0);
    const uint64_t* seed = v->d_state + c;
    if (e == cudaSuccess && off > 0) {
      e = cudaMemcpyAsync(v->d_seed + c, v->hseed + c, sizeof(uint64_t), cudaMemcpyHostToDevice, v->cs);
      seed = v->d_seed + c;
    }
    if (e != cudaSuccess) return ffail(GS_CUDA_ERROR, "verify feeder: %s", cudaGetErrorString(e));
    const void* ptr = slot;
    if ((st = gs_fnv1a64_device_seeded(&ptr, 1, 1, total - off, seed, v->d_sum + c, v->cs)) != GS_OK) return st;
    e = cudaMemcpyAsync(v->gsum + c, v->d_sum + c, sizeof(uint64_t), cudaMemcpyDeviceToHost, v->cs);
    if (e == cudaSuccess) e = cudaEventRecord(v->slot_ev[r], v->cs);
    if (e != cudaSuccess) return ffail(GS_CUDA_ERROR, "verify feeder: %s", cudaGetErrorString(e));
    ++issued;
  }
  return st;
}

// Chains a host thread claims at once and hashes in lockstep (FNV is one
// serial multiply chain per stream: two chains cost a core about the latency
// of one; C3 recovery, tools/c3_probe.py: 2 -> 157-165 ms, 3 -> 166 ms,
// 4 -> 184 ms). GS_VERIFY_CLAIM overrides (A/B).
static int v_claim_chains() {
  static const int n = [] {
    const char* e = std::getenv("GS_VERIFY_CLAIM");
    return e ? std::atoi(e) : 0;
  }();
  return n > 0 ? n : gsb::fnv_simd_available() ? 1 : 2;  // the SIMD chain needs no lockstep partner
}

// Whole chains on idle host threads (GS_VERIFY_HOST_FULL=0: off, for A/B):
// while the next front chunk's GPU state is still in flight, a host thread
// takes the LAST unclaimed chunk and hashes its whole chain from host memory
// (rows 0..k-1, twice the bytes of a continuation) -- the chunks that land
// last are then verified early, without the feeder re-uploading their other
// rows over the link the decode is bound by.
static bool v_host_full() {
  static const bool on = [] {
    const char* e = std::getenv("GS_VERIFY_HOST_FULL");
    return !(e && e[0] == '0');
  }();
  return on;
}

static int verify_finish_dynamic(gs_verify* v, int threads, uint64_t* sums, int* gpu_chunks) {
  using clk = std::chrono::steady_clock;
  constexpr uint64_t kSlice = 4ull << 20;  // host progress check / hand-off granularity (bytes per chain)
  constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
  int st = GS_OK;
  std::atomic<int> err{0};
  const uint64_t total = static_cast<uint64_t>(v->k - v->u) * v->len;
  const uint64_t head = static_cast<uint64_t>(v->u) * v->len;  // the rows the GPU hashes
  int fst = GS_OK;
  const auto t0 = clk::now();
  v->t0 = t0;
  auto secs = [&] { return std::chrono::duration<double>(clk::now() - t0).count(); };
  // pacing model: the GPU hashes the remaining rows once the row-0 uploads
  // (already queued) have landed, at the link rate; a host thread hashes its
  // claimed chains at host_chain_bps each (learned online)
  const double link = v->link_bps;
  const double t_rows0 = link > 0 ? static_cast<double>(v->n) * v->u * static_cast<double>(v->len) / link : 0;
  double chain_bps = v->host_chain_bps;
  auto gpu_queue_s = [&] {  // under v->mu: GPU work not yet issued
    return link > 0 ? (static_cast<double>(v->hi - v->lo + 1) * total + v->handoff_bytes) / link : 0;
  };
  const bool host_full = v_host_full() && link > 0 && chain_bps > 0;
  if (host_full) v->feeder_hold_s = std::max(0.0, t_rows0 - kRing * (total / link));
  v->hosts_active = total > 0 ? std::max(threads, 1) : 0;
  std::thread feeder;
  if (total > 0) feeder = std::thread([&] { fst = verify_feeder(v); });
  const int per = std::max(1, std::min(8, v_claim_chains()));
  std::atomic<int> next_tid{0};
  auto work = [&] {
    const int tid = next_tid.fetch_add(1);
    for (;;) {
      int c[8], m = 0;
      bool whole = false;
      const double t_claim = secs();
      {
        std::lock_guard<std::mutex> lk(v->mu);
        const double now = secs();
        bool idle = false;
        if (v->lo <= v->hi && host_full && now + (head + total) / chain_bps < t_rows0) {
          idle = cudaEventQuery(v->group_ev[v->group_of[v->lo]]) == cudaErrorNotReady;
          if (idle) cudaGetLastError();  // "not ready" is a status, not an error for later checks
        }
        if (idle) {
          c[m++] = v->hi--;  // idle until the next state lands: a whole chain from the back
          whole = true;
        } else {
          // the GPU would finish first: quit, but only once the row-0 uploads
          // are over -- before that a claim costs nothing the link could do
          // sooner, and the end-game hand-off below gives the GPU just the
          // chain's rest (GS_VERIFY_ENDGAME=0: the earlier rule, for A/B)
          if (link > 0 && chain_bps > 0 && (!v_endgame() || now >= t_rows0) &&
              now + total / chain_bps >= std::max(now, t_rows0) + gpu_queue_s())
            break;
          while (m < per && v->lo <= v->hi) c[m++] = v->lo++;
        }
      }
      if (m == 0) break;
      uint64_t h[8];
      if (whole) {
        h[0] = kOffset;
        for (int i = 0; i < v->u; ++i) {
          const uint8_t* p = v->host_rows[static_cast<size_t>(c[0]) * v->k + i];
          gsb::fnv1a64_chains(&p, 1, v->len, h);
        }
      } else {
        for (int q = 0; q < m; ++q) {
          if (cudaEventSynchronize(v->group_ev[v->group_of[c[q]]]) != cudaSuccess) {
            err = 1;
            break;
          }
          h[q] = v->pinned[c[q]];
        }
      }
      if (err) break;
      const double start = secs();
      bool handed = false;
      for (uint64_t o = 0; o < total;) {
        const uint64_t row = o / v->len, in = o - row * v->len;
        const uint64_t n = std::min<uint64_t>(kSlice, v->len - in);
        const uint8_t* ps[8];
        for (int q = 0; q < m; ++q) ps[q] = v->host_rows[static_cast<size_t>(c[q]) * v->k + v->u + row] + in;
        gsb::fnv1a64_chains(ps, m, n, h);
        o += n;
        if (o >= total || link <= 0) continue;
        std::lock_guard<std::mutex> lk(v->mu);
        const double now = secs(), rate = o / std::max(now - start, 1e-6);
        chain_bps = chain_bps > 0 ? 0.5 * chain_bps + 0.5 * rate : rate;
        const double host_left = (total - o) / rate;
        // the GPU's finish if it took the rest: behind the row-0 uploads, the
        // ring already in flight and the queue; hand over only when clearly
        // later on the host (a hand-over re-uploads the rest of the chain)
        const double gpu_done =
            std::max(now, t_rows0) + kRing * (total / link) + gpu_queue_s() + m * (total - o) / link;
        // a safety net for a host that stalls (not a balancing tool: the claim
        // pacing balances): at least a quarter of the chain done, and the host
        // would need over twice as long as the GPU for the rest
        // end game: the link is (about to be) free and the feeder's queue is
        // what the GPU still has to upload -- hand over the chain's rest when
        // the GPU would finish it clearly sooner than this thread
        const double gpu_end = std::max(now, t_rows0) + gpu_queue_s() + m * (total - o) / link + 1e-3;
        const bool endgame = v_endgame() && now >= t_rows0 - 2e-3 && host_left > gpu_end - now + 2e-3;
        if (endgame || (4 * o >= total && host_left > 2e-3 && host_left > 2.0 * (gpu_done - now))) {
          for (int q = 0; q < m; ++q) {
            v->hseed[c[q]] = h[q];
            v->handoffs.push_back({c[q], o});
            v->handoff_bytes += total - o;
          }
          handed = true;
          g_verify_handoffs.fetch_add(static_cast<uint64_t>(m));
          v->cv.notify_all();
          break;
        }
      }
      for (int q = 0; q < m; ++q) vtrace_push({tid, c[q], handed ? 3 : whole ? 1 : 0, t_claim, start, secs()});
      if (handed) break;
      for (int q = 0; q < m; ++q) sums[c[q]] = h[q];
    }
    {
      std::lock_guard<std::mutex> lk(v->mu);
      --v->hosts_active;
    }
    v->cv.notify_all();
  };
  if (total > 0) {
    std::vector<std::thread> pool;
    for (int t = 1; t < std::max(threads, 1); ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
  }
  const double t_hosts = secs();
  if (feeder.joinable()) feeder.join();
  if (v_trace()) {
    std::lock_guard<std::mutex> lk(g_vtrace_mu);
    std::fprintf(stderr, "VTRACE begin n=%d t_rows0=%.4f chain_bps=%.3g link=%.3g threads=%d\n", v->n, t_rows0,
                 v->host_chain_bps, link, threads);
    for (const auto& t : g_vtrace)
      std::fprintf(stderr, "VTRACE %d %d %d %.4f %.4f %.4f\n", t.who, t.chunk, t.kind, t.claim, t.ready, t.done);
    std::fprintf(stderr, "VTRACE end hosts=%.4f feeder=%.4f\n", t_hosts, secs());
    g_vtrace.clear();
  }
  const double t_feeder = secs();
  if (err) st = ffail(GS_CUDA_ERROR, "verify_finish: GPU chain state unavailable");
  if (st == GS_OK && fst != GS_OK) st = fst;
  // every D2H into pinned / gsum has landed before they are read or freed
  cudaSetDevice(v->device);
  if (cudaStreamSynchronize(v->cs) != cudaSuccess && st == GS_OK)
    st = ffail(GS_CUDA_ERROR, "verify_finish: hash stream failed");
  cudaStreamSynchronize(v->ys);
  int on = 0;
  if (st == GS_OK) {
    for (int c = 0; c < v->n; ++c) {
      if (total == 0) {
        sums[c] = v->pinned[c];  // every row was uploaded: the state is the checksum
        ++on;
      } else if (v->on_gpu[c]) {
        sums[c] = v->gsum[c];
        on += v->on_gpu[c] == 1;
      }
    }
  }
  if (gpu_chunks) *gpu_chunks = on;
  {
    int handed = 0, by_host = 0;
    for (int c = 0; c < v->n; ++c) {
      handed += v->on_gpu[c] == 2;
      by_host += v->on_gpu[c] == 0;
    }
    std::lock_guard<std::mutex> lk(g_vstats_mu);
    const double vals[6] = {t_hosts, t_feeder, secs(), static_cast<double>(by_host), static_cast<double>(on),
                            static_cast<double>(handed)};
    for (int i = 0; i < 6; ++i) g_vstats[i] = vals[i];
  }
  v->wait_unheld();
  for (auto e : v->group_ev) cudaEventDestroy(e);
  for (auto e : v->slot_ev) cudaEventDestroy(e);
  for (auto e : v->up_ev) cudaEventDestroy(e);
  pinned_give(v->host_block, v->host_bytes);
  cudaFreeAsync(v->dev_block, v->cs);  // stream-ordered: no device-wide synchronisation
  delete v;
  return st;
}

extern "C" int gs_verify_enqueue(const void* const* h_parity, int n_chunks, int k, uint64_t len, int n_full, int u,
                                 void* const* d_parity, void* compute, void* copy, gs_verify** out) {
  constexpr uint64_t kOffset = 0xcbf29ce484222325ull;
  if (!out || n_chunks < 0 || k < 1 || u < 1 || u > k || n_full > n_chunks ||
      (n_chunks > 0 && (!h_parity || !d_parity)))
    return ffail(GS_INVALID_ARGUMENT, "verify_enqueue: bad arguments");
  *out = nullptr;
  cudaStream_t cs = static_cast<cudaStream_t>(compute), ys = static_cast<cudaStream_t>(copy);
  if (n_full < 0) return verify_enqueue_dynamic(h_parity, n_chunks, k, len, u, d_parity, cs, ys, out);
  auto* v = new gs_verify;
  v->n = n_chunks;
  v->n_full = n_full;
  v->k = k;
  v->u = u;
  v->len = len;
  v->host_rows.resize(static_cast<size_t>(n_chunks) * k);
  for (size_t i = 0; i < v->host_rows.size(); ++i) v->host_rows[i] = static_cast<const uint8_t*>(h_parity[i]);
  v->group_of.assign(n_chunks, -1);
  auto bail = [&](int st) {
    cudaStreamSynchronize(cs);  // nothing may still write `pinned`
    for (auto e : v->group_ev) cudaEventDestroy(e);
    if (v->full_ev) cudaEventDestroy(v->full_ev);
    if (v->pinned) cudaFreeHost(v->pinned);
    delete v;
    return st;
  };
  cudaError_t e = cudaMallocHost(reinterpret_cast<void**>(&v->pinned), sizeof(uint64_t) * std::max(1, n_chunks));
  uint64_t* d_state = nullptr;
  if (e == cudaSuccess) e = cudaMallocAsync(reinterpret_cast<void**>(&d_state), sizeof(uint64_t) * std::max(1, n_chunks), cs);
  if (e != cudaSuccess) return bail(ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e)));
  cudaEvent_t up;
  if ((e = cudaEventCreateWithFlags(&up, cudaEventDisableTiming)) != cudaSuccess)
    return bail(ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e)));
  auto upload_rows = [&](int c, int rows) -> cudaError_t {
    for (int i = 0; i < rows; ++i) {
      const size_t r = static_cast<size_t>(c) * k + i;
      if (!h_parity[r] || !d_parity[r]) return cudaErrorInvalidValue;
      cudaError_t x = cudaMemcpyAsync(d_parity[r], h_parity[r], len, cudaMemcpyHostToDevice, ys);
      if (x != cudaSuccess) return x;
    }
    return cudaSuccess;
  };
  int st = GS_OK;
  // split chunks first: rows 0..u-1, hashed per group, states D2H'd per group
  for (int g0 = n_full; g0 < n_chunks && st == GS_OK; g0 += kSplitGroup) {
    const int cnt = std::min(kSplitGroup, n_chunks - g0);
    for (int c = g0; c < g0 + cnt && e == cudaSuccess; ++c) e = upload_rows(c, u);
    if (e == cudaSuccess) e = cudaEventRecord(up, ys);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, up, 0);
    if (e != cudaSuccess) {
      st = ffail(GS_CUDA_ERROR, "verify_enqueue upload: %s", cudaGetErrorString(e));
      break;
    }
    std::vector<const void*> rows(static_cast<size_t>(cnt) * u);
    for (int c = 0; c < cnt; ++c)
      for (int i = 0; i < u; ++i) rows[static_cast<size_t>(c) * u + i] = d_parity[static_cast<size_t>(g0 + c) * k + i];
    if ((st = gs_fnv1a64_device(rows.data(), cnt, u, len, kOffset, d_state + g0, cs)) != GS_OK) break;
    cudaEvent_t ge;
    e = cudaEventCreateWithFlags(&ge, cudaEventDisableTiming | cudaEventBlockingSync);
    if (e == cudaSuccess) {
      v->group_ev.push_back(ge);
      e = cudaMemcpyAsync(v->pinned + g0, d_state + g0, sizeof(uint64_t) * cnt, cudaMemcpyDeviceToHost, cs);
    }
    if (e == cudaSuccess) e = cudaEventRecord(ge, cs);
    if (e != cudaSuccess) st = ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e));
    for (int c = g0; c < g0 + cnt; ++c) v->group_of[c] = static_cast<int>(v->group_ev.size()) - 1;
  }
  // full chunks: every row, hashed on the GPU as groups land
  for (int g0 = 0; g0 < n_full && st == GS_OK; g0 += kSplitGroup) {
    const int cnt = std::min(kSplitGroup, n_full - g0);
    for (int c = g0; c < g0 + cnt && e == cudaSuccess; ++c) e = upload_rows(c, k);
    if (e == cudaSuccess) e = cudaEventRecord(up, ys);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, up, 0);
    if (e != cudaSuccess) {
      st = ffail(GS_CUDA_ERROR, "verify_enqueue upload: %s", cudaGetErrorString(e));
      break;
    }
    st = gs_fnv1a64_device(d_parity + static_cast<size_t>(g0) * k, cnt, k, len, kOffset, d_state + g0, cs);
  }
  if (st == GS_OK && n_full > 0) {
    e = cudaEventCreateWithFlags(&v->full_ev, cudaEventDisableTiming | cudaEventBlockingSync);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(v->pinned, d_state, sizeof(uint64_t) * n_full, cudaMemcpyDeviceToHost, cs);
    if (e == cudaSuccess) e = cudaEventRecord(v->full_ev, cs);
    if (e != cudaSuccess) st = ffail(GS_CUDA_ERROR, "verify_enqueue: %s", cudaGetErrorString(e));
  }
  cudaEventDestroy(up);
  cudaFreeAsync(d_state, cs);
  if (st != GS_OK) return bail(st);
  *out = v;
  return GS_OK;
}

// Blocks: host threads continue the split chunks' chains over rows u..k-1 as
// their GPU states arrive; sums[c] = chunk c's checksum. Frees `v`.
extern "C" int gs_verify_finish_ex(gs_verify* v, int threads, uint64_t* sums, int* gpu_chunks);

extern "C" int gs_verify_hold(gs_verify* v) {
  if (!v) return ffail(GS_INVALID_ARGUMENT, "verify_hold: NULL handle");
  std::lock_guard<std::mutex> lk(v->hold_mu);
  ++v->holds;
  return GS_OK;
}

extern "C" int gs_verify_release(gs_verify* v) {
  if (!v) return ffail(GS_INVALID_ARGUMENT, "verify_release: NULL handle");
  {
    std::lock_guard<std::mutex> lk(v->hold_mu);
    if (v->holds == 0) return ffail(GS_LOGIC_ERROR, "verify_release: not held");
    --v->holds;
  }
  v->hold_cv.notify_all();
  return GS_OK;
}

extern "C" int gs_verify_stream_wait(gs_verify* v, int chunk, void* stream) {
  if (!v || chunk < 0 || chunk >= v->n) return ffail(GS_INVALID_ARGUMENT, "verify_stream_wait: bad arguments");
  cudaEvent_t ev = v->group_of[chunk] >= 0 ? v->group_ev[v->group_of[chunk]] : v->full_ev;
  if (!ev) return ffail(GS_INVALID_ARGUMENT, "verify_stream_wait: chunk %d has no upload event", chunk);
  const cudaError_t e = cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), ev, 0);
  return e == cudaSuccess ? GS_OK : ffail(GS_CUDA_ERROR, "verify_stream_wait: %s", cudaGetErrorString(e));
}

extern "C" int gs_verify_set_rates(gs_verify* v, double link_gbs, double host_chain_gbs) {
  if (!v || link_gbs < 0 || host_chain_gbs < 0) return ffail(GS_INVALID_ARGUMENT, "verify_set_rates: bad arguments");
  v->link_bps = link_gbs * 1e9;
  v->host_chain_bps = host_chain_gbs * 1e9;
  return GS_OK;
}

extern "C" int gs_verify_finish(gs_verify* v, int threads, uint64_t* sums) {
  return gs_verify_finish_ex(v, threads, sums, nullptr);
}

extern "C" int gs_verify_finish_ex(gs_verify* v, int threads, uint64_t* sums, int* gpu_chunks) {
  if (!v) return ffail(GS_INVALID_ARGUMENT, "verify_finish: NULL handle");
  if (v->dynamic) {
    if (v->n > 0 && !sums) {
      uint64_t* tmp = new uint64_t[v->n];  // still drain and free the handle
      verify_finish_dynamic(v, threads, tmp, gpu_chunks);
      delete[] tmp;
      return ffail(GS_INVALID_ARGUMENT, "verify_finish: NULL output");
    }
    return verify_finish_dynamic(v, threads, sums, gpu_chunks);
  }
  if (gpu_chunks) *gpu_chunks = v->n_full;
  int st = GS_OK;
  if (v->n > 0 && !sums) st = ffail(GS_INVALID_ARGUMENT, "verify_finish: NULL output");
  const int ns = v->n - v->n_full;
  if (st == GS_OK && ns > 0) {
    // one chain per claim with the SIMD chain (claims follow the upload order,
    // so a thread never waits on a late chunk while earlier ones are ready)
    const int per = gsb::fnv_simd_available()
                        ? 1
                        : std::max(1, std::min(8, (ns + std::max(threads, 1) - 1) / std::max(threads, 1)));
    const int groups = (ns + per - 1) / per;
    std::atomic<int> next{0};
    std::atomic<int> err{0};
    auto work = [&] {
      for (int g = next.fetch_add(1); g < groups; g = next.fetch_add(1)) {
        const int c0 = v->n_full + g * per, m = std::min(per, v->n - c0);
        for (int c = c0; c < c0 + m; ++c) {
          const int ge = v->group_of[c];
          if (ge < 0 || cudaEventSynchronize(v->group_ev[ge]) != cudaSuccess) err = 1;
        }
        if (err) return;
        uint64_t h[8];
        for (int q = 0; q < m; ++q) h[q] = v->pinned[c0 + q];
        for (int i = v->u; i < v->k; ++i) {
          const uint8_t* ps[8];
          for (int q = 0; q < m; ++q) ps[q] = v->host_rows[static_cast<size_t>(c0 + q) * v->k + i];
          gsb::fnv1a64_chains(ps, m, v->len, h);
        }
        for (int q = 0; q < m; ++q) sums[c0 + q] = h[q];
      }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < std::min(std::max(threads, 1), groups); ++t) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    if (err) st = ffail(GS_CUDA_ERROR, "verify_finish: GPU chain state unavailable");
  }
  if (st == GS_OK && v->n_full > 0) {
    if (cudaEventSynchronize(v->full_ev) != cudaSuccess)
      st = ffail(GS_CUDA_ERROR, "verify_finish: GPU checksums unavailable");
    else
      for (int c = 0; c < v->n_full; ++c) sums[c] = v->pinned[c];
  }
  v->wait_unheld();
  for (auto e : v->group_ev) {  // every D2H into `pinned` has landed before it is freed
    cudaEventSynchronize(e);
    cudaEventDestroy(e);
  }
  if (v->full_ev) {
    cudaEventSynchronize(v->full_ev);
    cudaEventDestroy(v->full_ev);
  }
  cudaFreeHost(v->pinned);
  delete v;
  return st;
}
